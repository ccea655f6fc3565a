// Host->device micro-batch streamer (the B200 re-design of engine.py:140-163).
//
// The reference materialises micro-batch k+1 on one prefetch worker thread
// while micro-batch k computes (two slots: one in flight, one in use) and
// guarantees bit-identical results with prefetch on or off.
// Here a slot is a page-locked host buffer plus the caller's device
// destination; a job is: wait until the slot's previous copy has drained,
// gather the micro-batch rows into the pinned slot with a native thread pool
// (or skip the gather when the source is already pinned and contiguous), then
// cudaMemcpyAsync every part on the copy stream — ordered after the compute
// stream released the slot's device buffers — and record the slot's ready
// event. Compute waits on that event only (never the host), so the H2D copy
// of micro-batch k+1 overlaps the forward/backward of micro-batch k exactly
// like the two-slot schedule of streaming.py:96-108.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <deque>
#include <functional>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include "mbs_common.h"

namespace mbs {

// Fixed pool of gather threads; parallel_for splits [0, n) into contiguous blocks.
class ThreadPool {
  public:
    explicit ThreadPool(int n) : n_(std::max(1, n)) {
        for (int i = 1; i < n_; ++i) workers_.emplace_back([this, i] { loop(i); });
    }
    ~ThreadPool() {
        {
            std::lock_guard<std::mutex> g(m_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : workers_) t.join();
    }
    int size() const { return n_; }
    void parallel_for(int64_t n, const std::function<void(int64_t, int64_t)>& fn) {
        if (n <= 0) return;
        if (n_ == 1 || n < 2) {
            fn(0, n);
            return;
        }
        {
            std::lock_guard<std::mutex> g(m_);
            fn_ = &fn;
            total_ = n;
            pending_ = n_ - 1;
            ++gen_;
        }
        cv_.notify_all();
        run_part(0, fn, n);
        std::unique_lock<std::mutex> lk(m_);
        done_cv_.wait(lk, [this] { return pending_ == 0; });
        fn_ = nullptr;
    }

  private:
    void run_part(int i, const std::function<void(int64_t, int64_t)>& fn, int64_t n) {
        const int64_t per = (n + n_ - 1) / n_;
        const int64_t lo = std::min<int64_t>(n, per * i), hi = std::min<int64_t>(n, lo + per);
        if (lo < hi) fn(lo, hi);
    }
    void loop(int i) {
        uint64_t seen = 0;
        for (;;) {
            const std::function<void(int64_t, int64_t)>* fn;
            int64_t n;
            {
                std::unique_lock<std::mutex> lk(m_);
                cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
                if (stop_) return;
                seen = gen_;
                fn = fn_;
                n = total_;
            }
            run_part(i, *fn, n);
            {
                std::lock_guard<std::mutex> g(m_);
                if (--pending_ == 0) done_cv_.notify_one();
            }
        }
    }
    int n_;
    std::vector<std::thread> workers_;
    std::mutex m_;
    std::condition_variable cv_, done_cv_;
    const std::function<void(int64_t, int64_t)>* fn_ = nullptr;
    int64_t total_ = 0;
    int pending_ = 0;
    uint64_t gen_ = 0;
    bool stop_ = false;
};

static void gather_rows(ThreadPool& pool, const uint8_t* src, int64_t row_bytes, const int64_t* rows, int64_t row0,
                        int64_t n_rows, uint8_t* dst) {
    // split by bytes so a few huge rows still use every thread
    const int64_t total = n_rows * row_bytes;
    const int64_t parts = std::max<int64_t>(1, std::min<int64_t>(pool.size() * 4, total / (256 << 10)));
    pool.parallel_for(parts, [&](int64_t lo, int64_t hi) {
        for (int64_t p = lo; p < hi; ++p) {
            int64_t b0 = total * p / parts, b1 = total * (p + 1) / parts;
            while (b0 < b1) {
                const int64_t r = b0 / row_bytes, off = b0 % row_bytes;
                const int64_t n = std::min(b1 - b0, row_bytes - off);
                const int64_t sr = rows ? rows[r] : row0 + r;
                memcpy(dst + b0, src + sr * row_bytes + off, (size_t)n);
                b0 += n;
            }
        }
    });
}

constexpr int MBS_STREAMER_RING = 256;

enum SlotState { kFree = 0, kPending = 1, kIssued = 2, kConsumed = 3 };

struct Job {
    int slot;
    int64_t seq;
    mbs_part_t parts[MBS_MAX_PARTS];
    int n_parts;
    std::vector<int64_t> rows;
    bool has_rows;
    int64_t row0, n_rows;
};

// Per-job timing record (a ring, so timings stay readable long after the slot is reused).
struct JobRec {
    cudaEvent_t start = nullptr, ready = nullptr, compute = nullptr;
    int64_t seq = -1;
    double gather_ms = 0.0;
    int64_t bytes = 0;
    bool compute_recorded = false;
};

}  // namespace mbs

using namespace mbs;

struct mbs_streamer {
    int n_slots = 0;
    int64_t slot_bytes = 0;
    cudaStream_t copy = nullptr;
    std::vector<uint8_t*> host;              // pinned slots
    std::vector<cudaEvent_t> ev_released;    // compute finished reading the slot's device buffers
    std::vector<int64_t> slot_job;           // seq of the slot's last job (-1 = none)
    // slot state machine: FREE -> (submit) PENDING -> (worker) ISSUED -> (wait) CONSUMED
    // -> (release) FREE. A slot is re-submitted only when FREE or ISSUED-but-unused,
    // so the next copy into its device buffers is always ordered after the release.
    std::vector<int> state;
    std::vector<int> pending;                // job submitted, not yet issued by the worker
    std::vector<int> released_recorded;
    std::vector<int> status;
    std::vector<JobRec> ring;
    int64_t next_seq = 0;
    int64_t issued_count = 0;                // jobs run FIFO on one worker: seq < issued_count => issued
    std::unique_ptr<ThreadPool> pool;
    std::thread worker;
    std::mutex m;
    std::condition_variable cv;
    std::deque<Job> q;
    bool stop = false;
    int device = 0;

    JobRec& rec(int64_t seq) { return ring[(size_t)(seq % (int64_t)ring.size())]; }

    void run() {
        cudaSetDevice(device);
        for (;;) {
            Job job;
            {
                std::unique_lock<std::mutex> lk(m);
                cv.wait(lk, [&] { return stop || !q.empty(); });
                if (stop && q.empty()) return;
                job = std::move(q.front());
                q.pop_front();
            }
            const int rc = execute(job);
            {
                std::lock_guard<std::mutex> g(m);
                status[job.slot] = rc;
                pending[job.slot] = 0;
                state[job.slot] = kIssued;
                issued_count = job.seq + 1;
            }
            cv.notify_all();
        }
    }

    int execute(Job& job) {
        const int s = job.slot;
        // the pinned slot may still feed the previous copy out of it
        const int64_t prev = slot_job[s];
        if (prev >= 0) {
            cudaError_t e = cudaEventSynchronize(rec(prev).ready);
            if (e != cudaSuccess) return cuda_status(e, "streamer: wait previous copy");
        }
        JobRec& r = rec(job.seq);
        r.seq = job.seq;
        r.compute_recorded = false;
        bool need_host = false;
        for (int p = 0; p < job.n_parts; ++p)
            if (job.has_rows || !job.parts[p].src_pinned) need_host = true;
        auto t0 = std::chrono::steady_clock::now();
        int64_t off = 0;
        const uint8_t* srcs[MBS_MAX_PARTS];
        for (int p = 0; p < job.n_parts; ++p) {
            const auto& part = job.parts[p];
            const int64_t nbytes = job.n_rows * part.row_bytes;
            if (job.has_rows || !part.src_pinned) {
                off = (off + 255) & ~int64_t(255);
                if (off + nbytes > slot_bytes) {
                    set_error("streamer: micro-batch does not fit the pinned slot");
                    return MBS_EINVAL;
                }
                gather_rows(*pool, static_cast<const uint8_t*>(part.src), part.row_bytes,
                            job.has_rows ? job.rows.data() : nullptr, job.row0, job.n_rows, host[s] + off);
                srcs[p] = host[s] + off;
                off += nbytes;
            } else {
                srcs[p] = static_cast<const uint8_t*>(part.src) + job.row0 * part.row_bytes;
            }
        }
        auto t1 = std::chrono::steady_clock::now();
        r.gather_ms = need_host ? std::chrono::duration<double, std::milli>(t1 - t0).count() : 0.0;
        // device buffers of this slot must have been released by compute first
        if (released_recorded[s]) {
            cudaError_t e = cudaStreamWaitEvent(copy, ev_released[s], 0);
            if (e != cudaSuccess) return cuda_status(e, "streamer: wait release");
        }
        MBS_CK(cudaEventRecord(r.start, copy));
        int64_t total = 0;
        for (int p = 0; p < job.n_parts; ++p) {
            const int64_t nbytes = job.n_rows * job.parts[p].row_bytes;
            MBS_CK(cudaMemcpyAsync(job.parts[p].dst, srcs[p], (size_t)nbytes, cudaMemcpyHostToDevice, copy));
            total += nbytes;
        }
        r.bytes = total;
        MBS_CK(cudaEventRecord(r.ready, copy));
        slot_job[s] = job.seq;
        return MBS_OK;
    }
};

extern "C" {

int mbs_streamer_create(int n_slots, int64_t slot_bytes, int n_threads, void* copy_stream, mbs_streamer_t* out) {
    if (!out || n_slots < 1 || n_slots > 64 || slot_bytes < 0 || !copy_stream)
        return invalid("mbs_streamer_create: bad arguments");
    auto* h = new mbs_streamer();
    h->n_slots = n_slots;
    h->slot_bytes = slot_bytes;
    h->copy = (cudaStream_t)copy_stream;
    cudaGetDevice(&h->device);
    h->host.assign(n_slots, nullptr);
    h->ev_released.assign(n_slots, nullptr);
    h->slot_job.assign(n_slots, -1);
    h->state.assign(n_slots, kFree);
    h->pending.assign(n_slots, 0);
    h->released_recorded.assign(n_slots, 0);
    h->status.assign(n_slots, 0);
    h->ring.resize((size_t)std::max(MBS_STREAMER_RING, 4 * n_slots));
    cudaError_t e = cudaSuccess;
    for (int s = 0; s < n_slots && e == cudaSuccess; ++s) {
        if (slot_bytes > 0) e = cudaHostAlloc((void**)&h->host[s], (size_t)slot_bytes, cudaHostAllocPortable);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_released[s], cudaEventDisableTiming);
    }
    for (auto& r : h->ring) {
        if (e == cudaSuccess) e = cudaEventCreate(&r.start);
        if (e == cudaSuccess) e = cudaEventCreate(&r.ready);
        if (e == cudaSuccess) e = cudaEventCreate(&r.compute);
    }
    if (e != cudaSuccess) {
        mbs_streamer_destroy(h);
        return cuda_status(e, "mbs_streamer_create");
    }
    h->pool.reset(new ThreadPool(n_threads < 1 ? 1 : n_threads));
    h->worker = std::thread([h] { h->run(); });
    *out = h;
    return MBS_OK;
}

int mbs_streamer_destroy(mbs_streamer_t h) {
    if (!h) return MBS_OK;
    if (h->worker.joinable()) {
        {
            std::lock_guard<std::mutex> g(h->m);
            h->stop = true;
        }
        h->cv.notify_all();
        h->worker.join();
    }
    for (auto& r : h->ring) {
        if (r.ready) cudaEventSynchronize(r.ready);
        if (r.start) cudaEventDestroy(r.start);
        if (r.ready) cudaEventDestroy(r.ready);
        if (r.compute) cudaEventDestroy(r.compute);
    }
    for (int s = 0; s < h->n_slots; ++s) {
        if (h->host[s]) cudaFreeHost(h->host[s]);
        if (h->ev_released[s]) cudaEventDestroy(h->ev_released[s]);
    }
    delete h;
    return MBS_OK;
}

int mbs_streamer_submit(mbs_streamer_t h, int slot, const mbs_part_t* parts, int n_parts, const int64_t* rows,
                        int64_t row0, int64_t n_rows, int64_t* job_out) {
    if (!h || slot < 0 || slot >= h->n_slots || !parts || n_parts < 1 || n_parts > MBS_MAX_PARTS || n_rows < 0 ||
        (!rows && row0 < 0))
        return invalid("mbs_streamer_submit: bad arguments");
    Job job;
    job.slot = slot;
    job.n_parts = n_parts;
    for (int p = 0; p < n_parts; ++p) {
        if (!parts[p].src || !parts[p].dst || parts[p].row_bytes < 1) return invalid("mbs_streamer_submit: bad part");
        job.parts[p] = parts[p];
    }
    job.has_rows = rows != nullptr;
    if (rows) job.rows.assign(rows, rows + n_rows);
    job.row0 = row0;
    job.n_rows = n_rows;
    {
        std::lock_guard<std::mutex> g(h->m);
        if (h->state[slot] != kFree && h->state[slot] != kIssued)
            return invalid("mbs_streamer_submit: slot is pending or consumed but not released");
        job.seq = h->next_seq++;
        h->pending[slot] = 1;
        h->state[slot] = kPending;
        h->q.push_back(std::move(job));
        if (job_out) *job_out = h->q.back().seq;
    }
    h->cv.notify_all();
    return MBS_OK;
}

int mbs_streamer_wait(mbs_streamer_t h, int slot, void* compute_stream) {
    if (!h || slot < 0 || slot >= h->n_slots) return invalid("mbs_streamer_wait: bad slot");
    int rc;
    int64_t seq;
    {
        std::unique_lock<std::mutex> lk(h->m);
        if (h->state[slot] == kFree) return invalid("mbs_streamer_wait: slot has no submitted job");
        h->cv.wait(lk, [&] { return !h->pending[slot]; });
        rc = h->status[slot];
        if (rc == MBS_OK) h->state[slot] = kConsumed;
        seq = h->slot_job[slot];
    }
    if (rc) return rc;
    auto cs = (cudaStream_t)compute_stream;
    JobRec& r = h->rec(seq);
    MBS_CK(cudaEventRecord(r.compute, cs));  // compute reached the wait point
    r.compute_recorded = true;
    MBS_CK(cudaStreamWaitEvent(cs, r.ready, 0));
    return MBS_OK;
}

int mbs_streamer_release(mbs_streamer_t h, int slot, void* compute_stream) {
    if (!h || slot < 0 || slot >= h->n_slots) return invalid("mbs_streamer_release: bad slot");
    MBS_CK(cudaEventRecord(h->ev_released[slot], (cudaStream_t)compute_stream));
    std::lock_guard<std::mutex> g(h->m);
    h->released_recorded[slot] = 1;
    if (h->state[slot] == kConsumed) h->state[slot] = kFree;
    return MBS_OK;
}

int mbs_streamer_timing(mbs_streamer_t h, int64_t job, double* gather_ms, double* copy_ms, double* blocked_ms,
                        int64_t* bytes) {
    if (!h || job < 0) return invalid("mbs_streamer_timing: bad job");
    {
        std::unique_lock<std::mutex> lk(h->m);
        if (job >= h->next_seq || job < h->next_seq - (int64_t)h->ring.size())
            return invalid("mbs_streamer_timing: job record no longer (or not yet) available");
        // wait until the worker issued it
        h->cv.wait(lk, [&] { return job < h->issued_count; });
    }
    JobRec& r = h->rec(job);
    MBS_CK(cudaEventSynchronize(r.ready));
    float c = 0.f, b = 0.f;
    MBS_CK(cudaEventElapsedTime(&c, r.start, r.ready));
    if (r.compute_recorded) {
        MBS_CK(cudaEventSynchronize(r.compute));
        MBS_CK(cudaEventElapsedTime(&b, r.compute, r.ready));
    }
    if (gather_ms) *gather_ms = r.gather_ms;
    if (copy_ms) *copy_ms = c;
    if (blocked_ms) *blocked_ms = std::max(0.f, b);
    if (bytes) *bytes = r.bytes;
    return MBS_OK;
}

int mbs_streamer_timeline(mbs_streamer_t h, int64_t job, void* origin_event, double* copy_start_ms,
                          double* copy_end_ms) {
    if (!h || job < 0 || !origin_event) return invalid("mbs_streamer_timeline: bad arguments");
    {
        std::unique_lock<std::mutex> lk(h->m);
        if (job >= h->next_seq || job < h->next_seq - (int64_t)h->ring.size())
            return invalid("mbs_streamer_timeline: job record no longer (or not yet) available");
        h->cv.wait(lk, [&] { return job < h->issued_count; });
    }
    JobRec& r = h->rec(job);
    auto origin = (cudaEvent_t)origin_event;
    MBS_CK(cudaEventSynchronize(r.ready));
    float a = 0.f, b = 0.f;
    MBS_CK(cudaEventElapsedTime(&a, origin, r.start));
    MBS_CK(cudaEventElapsedTime(&b, origin, r.ready));
    if (copy_start_ms) *copy_start_ms = a;
    if (copy_end_ms) *copy_end_ms = b;
    return MBS_OK;
}

int mbs_host_gather(const void* src, int64_t row_bytes, const int64_t* rows, int64_t n_rows, void* dst,
                    int n_threads) {
    if (!src || !dst || !rows || row_bytes < 1 || n_rows < 0) return invalid("mbs_host_gather: bad arguments");
    ThreadPool pool(n_threads < 1 ? 1 : n_threads);
    gather_rows(pool, static_cast<const uint8_t*>(src), row_bytes, rows, 0, n_rows, static_cast<uint8_t*>(dst));
    return MBS_OK;
}

}  // extern "C"
