// Fused last-micro-batch accumulate + all-reduce over peer memory (K1C).
//
// The data-parallel exchange step of SURVEY §8e — every rank's accumulated
// gradient (engine.py:206-216 summed across ranks) — as ONE kernel instead of
// K1 followed by an NCCL all-reduce. Each rank exports a symmetric exchange
// buffer X (the accumulator's layout) and a signal block S through CUDA IPC;
// peers map them (NVLink/NVSwitch P2P on a multi-GPU node; the same device for
// the single-GPU test). The kernel is persistent (grid = co-resident CTAs) and
// runs three phases separated by grid barriers and cross-rank flags:
//
//   1. local accumulate, the K1 math: X_self = acc (+)= s*g   (tile walk over segments)
//   2. reduce-scatter: rank r sums its 1/W slice over all X_q in rank order
//      (deterministic, identical on every rank) into X_self and acc
//   3. all-gather: rank r copies every peer's reduced slice from X_q into acc
//
// NVLink traffic per rank is 2(W-1)/W x 4P bytes (bandwidth-optimal, like a
// ring) with only two cross-rank synchronisation points, and phase 1 of one
// tile overlaps phase-1 stores of the others. Every spin-wait is bounded
// (timeout -> device error flag, the kernel drains instead of hanging).
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <vector>

#include "mbs_common.h"

namespace mbs {

constexpr int kPeerThreads = 256;
constexpr int kPeerMaxWorld = 16;
constexpr int kPeerMaxPtrs = 1024;

struct PeerSeg {
    int64_t off;
    int64_t num;
};

struct PeerGradPtrs {
    const float* p[kPeerMaxPtrs];
};

struct PeerPtrs {
    float* x[kPeerMaxWorld];
    unsigned* s[kPeerMaxWorld];
};

// signal block layout (uint32): [0, W) ready-1 flags, [W, 2W) ready-2 flags, [2W, 3W) done flags,
// [3W] error flag, [3W+1] grid-barrier counter (local only)
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Wait (thread 0 of the CTA) until flags[i*stride] >= want for i in [0, n); bounded by `budget` cycles.
__device__ bool wait_flags(const unsigned* flags, int n, unsigned want, long long budget, unsigned* err) {
    const long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        while (ld_acquire_sys(flags + i) < want) {
            if (ld_acquire_sys(err) != 0) return false;
            if (clock64() - t0 > budget) {
                atomicExch(err, 1u);
                return false;
            }
            __nanosleep(64);
        }
    }
    return true;
}

__device__ void grid_barrier(unsigned* bar, unsigned target, long long budget, unsigned* err) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        atomicAdd(bar, 1u);
        const long long t0 = clock64();
        while (ld_acquire_gpu(bar) < target) {
            if (clock64() - t0 > budget) {
                atomicExch(err, 1u);
                break;
            }
            __nanosleep(32);
        }
    }
    __syncthreads();
}

__device__ __forceinline__ float4 ldcg4(const float4* p) { return __ldcg(p); }

template <bool ASSIGN, bool HAVE>
__global__ void __launch_bounds__(kPeerThreads)
k_accum_allreduce(float* __restrict__ acc, const PeerSeg* __restrict__ segs, int nseg, int64_t tile, int64_t n_tiles,
                  int64_t total, int64_t slice, const __grid_constant__ PeerGradPtrs gp, float s,
                  const __grid_constant__ PeerPtrs peers, int rank, int world, unsigned epoch, unsigned bar_base,
                  long long budget, const float* __restrict__ loss, double* __restrict__ loss_slot,
                  double* __restrict__ factor_slot, double factor, double* __restrict__ weight_slot, double weight) {
    float* __restrict__ X = peers.x[rank];
    unsigned* S = peers.s[rank];
    unsigned* err = S + 3 * world;
    unsigned* bar = S + 3 * world + 1;

    // phase 0: every peer finished reading our X in the previous exchange
    if (threadIdx.x == 0 && epoch > 1) wait_flags(S + 2 * world, world, epoch - 1, budget, err);
    __syncthreads();

    // phase 1: X = (ASSIGN ? 0 : acc) + s * g over the segments (padding of X stays zero)
    for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        const int64_t lo = t * tile, hi = min(lo + tile, total);
        int a = 0, b = nseg - 1;
        while (a < b) {
            const int m = (a + b + 1) >> 1;
            if (segs[m].off <= lo) a = m; else b = m - 1;
        }
        for (int si = a; si < nseg; ++si) {
            const PeerSeg sg = segs[si];
            if (sg.off >= hi) break;
            const int64_t p0 = max(lo, sg.off), p1 = min(hi, sg.off + sg.num);
            if (p1 <= p0) continue;
            const int n = (int)(p1 - p0);
            const float* g = HAVE ? gp.p[si] + (p0 - sg.off) : nullptr;
            const float* ac = acc + p0;
            float* xo = X + p0;
            const bool vec = !HAVE || (reinterpret_cast<uintptr_t>(g) & 15) == 0;
            int done = 0;
            if (vec) {
                const int n4 = n >> 2;
                for (int i = threadIdx.x; i < n4; i += kPeerThreads) {
                    float4 r = ASSIGN ? make_float4(0.f, 0.f, 0.f, 0.f) : reinterpret_cast<const float4*>(ac)[i];
                    if (HAVE) {
                        const float4 gv = __ldcs(reinterpret_cast<const float4*>(g) + i);
                        r.x = fmaf(s, gv.x, r.x); r.y = fmaf(s, gv.y, r.y);
                        r.z = fmaf(s, gv.z, r.z); r.w = fmaf(s, gv.w, r.w);
                    }
                    reinterpret_cast<float4*>(xo)[i] = r;
                }
                done = n4 << 2;
            }
            for (int i = done + threadIdx.x; i < n; i += kPeerThreads) {
                float r = ASSIGN ? 0.f : ac[i];
                if (HAVE) r = fmaf(s, g[i], r);
                xo[i] = r;
            }
        }
    }
    if (loss != nullptr && blockIdx.x == 0 && threadIdx.x == 0) {
        *loss_slot = (double)*loss;
        *factor_slot = factor;
        *weight_slot = weight;
    }
    grid_barrier(bar, bar_base + gridDim.x, budget, err);
    if (blockIdx.x == 0 && threadIdx.x == 0)
        for (int q = 0; q < world; ++q) st_release_sys(peers.s[q] + rank, epoch);
    if (threadIdx.x == 0) wait_flags(S, world, epoch, budget, err);
    __syncthreads();

    // phase 2: reduce my slice over all ranks in rank order -> X (for the peers) and acc
    const int64_t my0 = (int64_t)rank * slice, my1 = min(my0 + slice, total);
    for (int64_t i = (int64_t)blockIdx.x * kPeerThreads + threadIdx.x; my0 + 4 * i < my1;
         i += (int64_t)gridDim.x * kPeerThreads) {
        const int64_t e = my0 + 4 * i;
        float4 sum = ldcg4(reinterpret_cast<const float4*>(peers.x[0] + e));
        for (int q = 1; q < world; ++q) {
            const float4 v = ldcg4(reinterpret_cast<const float4*>(peers.x[q] + e));
            sum.x += v.x; sum.y += v.y; sum.z += v.z; sum.w += v.w;
        }
        reinterpret_cast<float4*>(X + e)[0] = sum;
        reinterpret_cast<float4*>(acc + e)[0] = sum;
    }
    grid_barrier(bar, bar_base + 2 * gridDim.x, budget, err);
    if (blockIdx.x == 0 && threadIdx.x == 0)
        for (int q = 0; q < world; ++q) st_release_sys(peers.s[q] + world + rank, epoch);
    if (threadIdx.x == 0) wait_flags(S + world, world, epoch, budget, err);
    __syncthreads();

    // phase 3: gather every peer's reduced slice
    for (int q = 0; q < world; ++q) {
        if (q == rank) continue;
        const int64_t q0 = (int64_t)q * slice, q1 = min(q0 + slice, total);
        for (int64_t i = (int64_t)blockIdx.x * kPeerThreads + threadIdx.x; q0 + 4 * i < q1;
             i += (int64_t)gridDim.x * kPeerThreads) {
            const int64_t e = q0 + 4 * i;
            reinterpret_cast<float4*>(acc + e)[0] = ldcg4(reinterpret_cast<const float4*>(peers.x[q] + e));
        }
    }
    grid_barrier(bar, bar_base + 3 * gridDim.x, budget, err);
    if (blockIdx.x == 0 && threadIdx.x == 0)
        for (int q = 0; q < world; ++q) st_release_sys(peers.s[q] + 2 * world + rank, epoch);
}

}  // namespace mbs

using namespace mbs;

struct mbs_peer {
    int rank = 0, world = 1;
    int64_t numel = 0;
    float* x = nullptr;         // own exchange buffer
    unsigned* sig = nullptr;    // own signal block
    PeerPtrs peers{};
    std::vector<void*> opened;  // IPC-mapped peer allocations to close
    unsigned epoch = 0;
    unsigned bar_base = 0;
    int grid = 0;
    bool open = false;
    std::vector<PeerSeg> segs;  // host copy of the segment table last uploaded
    PeerSeg* d_segs = nullptr;
};

extern "C" {

int mbs_peer_create(int rank, int world, int64_t numel, mbs_peer_t* out) {
    if (!out || world < 1 || world > kPeerMaxWorld || rank < 0 || rank >= world || numel <= 0 || numel % 4)
        return invalid("mbs_peer_create: bad arguments (world <= 16, numel a positive multiple of 4)");
    auto* h = new mbs_peer();
    h->rank = rank;
    h->world = world;
    h->numel = numel;
    cudaError_t e = cudaMalloc(&h->x, sizeof(float) * numel);
    if (e == cudaSuccess) e = cudaMemset(h->x, 0, sizeof(float) * numel);
    if (e == cudaSuccess) e = cudaMalloc(&h->sig, sizeof(unsigned) * (3 * world + 32));
    if (e == cudaSuccess) e = cudaMemset(h->sig, 0, sizeof(unsigned) * (3 * world + 32));
    if (e != cudaSuccess) {
        mbs_peer_destroy(h);
        return cuda_status(e, "mbs_peer_create");
    }
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_accum_allreduce<false, true>, kPeerThreads, 0);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // co-resident by construction (the grid barriers need every CTA resident); one CTA per SM leaves
    // room for a concurrently running backward kernel
    h->grid = std::max(1, std::min(per_sm, 2)) * sms;
    *out = h;
    return MBS_OK;
}

int mbs_peer_handle(mbs_peer_t h, void* out) {
    if (!h || !out) return invalid("mbs_peer_handle: bad arguments");
    cudaIpcMemHandle_t hx, hs;
    MBS_CK(cudaIpcGetMemHandle(&hx, h->x));
    MBS_CK(cudaIpcGetMemHandle(&hs, h->sig));
    memcpy(out, &hx, sizeof(hx));
    memcpy(static_cast<char*>(out) + 64, &hs, sizeof(hs));
    return MBS_OK;
}

int mbs_peer_open(mbs_peer_t h, const void* handles) {
    if (!h || !handles) return invalid("mbs_peer_open: bad arguments");
    if (h->open) return invalid("mbs_peer_open: already open");
    for (int q = 0; q < h->world; ++q) {
        if (q == h->rank) {
            h->peers.x[q] = h->x;
            h->peers.s[q] = h->sig;
            continue;
        }
        cudaIpcMemHandle_t hx, hs;
        memcpy(&hx, static_cast<const char*>(handles) + (size_t)q * MBS_PEER_HANDLE_BYTES, sizeof(hx));
        memcpy(&hs, static_cast<const char*>(handles) + (size_t)q * MBS_PEER_HANDLE_BYTES + 64, sizeof(hs));
        void *px = nullptr, *ps = nullptr;
        MBS_CK(cudaIpcOpenMemHandle(&px, hx, cudaIpcMemLazyEnablePeerAccess));
        h->opened.push_back(px);
        MBS_CK(cudaIpcOpenMemHandle(&ps, hs, cudaIpcMemLazyEnablePeerAccess));
        h->opened.push_back(ps);
        h->peers.x[q] = static_cast<float*>(px);
        h->peers.s[q] = static_cast<unsigned*>(ps);
    }
    h->open = true;
    return MBS_OK;
}

int mbs_peer_destroy(mbs_peer_t h) {
    if (!h) return MBS_OK;
    cudaDeviceSynchronize();
    for (void* p : h->opened) cudaIpcCloseMemHandle(p);
    if (h->x) cudaFree(h->x);
    if (h->sig) cudaFree(h->sig);
    if (h->d_segs) cudaFree(h->d_segs);
    delete h;
    return MBS_OK;
}

int mbs_peer_status(mbs_peer_t h, int* error_flag) {
    if (!h || !error_flag) return invalid("mbs_peer_status: bad arguments");
    unsigned v = 0;
    MBS_CK(cudaMemcpy(&v, h->sig + 3 * h->world, sizeof(v), cudaMemcpyDeviceToHost));
    *error_flag = (int)v;
    return MBS_OK;
}

int mbs_accum_add_allreduce(mbs_accum_t acc, mbs_peer_t h, const float* const* grads, double factor,
                            const float* loss_dev, double loss_factor, double loss_weight, double timeout_ms,
                            void* stream) {
    if (!acc || !h || !h->open) return invalid("mbs_accum_add_allreduce: null handle or peers not opened");
    AccumView v;
    int st = accum_view(acc, &v);
    if (st) return st;
    if (v.numel != h->numel) return invalid("mbs_accum_add_allreduce: accumulator and exchange sizes differ");
    const int nseg = (int)v.off->size();
    if (nseg > kPeerMaxPtrs) return invalid("mbs_accum_add_allreduce: more than 1024 parameter segments");
    if (*v.covered != 0) return invalid("mbs_accum_add_allreduce: a bucketed micro-batch is in progress");
    const bool have = grads != nullptr;
    if (have) {
        if (v.expected >= 0 && *v.seen >= v.expected) {
            set_error("already accumulated " + std::to_string(*v.seen) + " of " + std::to_string(v.expected) +
                      " micro-batches");
            return MBS_EOVERFLOW;
        }
        if (*v.seen >= v.max_micro) {
            set_error("micro-batch count exceeds the handle's max_micro");
            return MBS_EOVERFLOW;
        }
    }
    std::vector<PeerSeg> segs(nseg);
    for (int i = 0; i < nseg; ++i) segs[i] = PeerSeg{(*v.off)[i], (*v.num)[i]};
    auto cs = (cudaStream_t)stream;
    const bool same = segs.size() == h->segs.size() &&
                      std::equal(segs.begin(), segs.end(), h->segs.begin(),
                                 [](const PeerSeg& x, const PeerSeg& y) { return x.off == y.off && x.num == y.num; });
    if (!same) {  // first use (or a different accumulator): upload the segment table once
        if (h->d_segs) {
            MBS_CK(cudaStreamSynchronize(cs));
            cudaFree(h->d_segs);
            h->d_segs = nullptr;
        }
        MBS_CK(cudaMalloc(&h->d_segs, sizeof(PeerSeg) * nseg));
        MBS_CK(cudaMemcpy(h->d_segs, segs.data(), sizeof(PeerSeg) * nseg, cudaMemcpyHostToDevice));
        h->segs = segs;
    }
    PeerSeg* d_segs = h->d_segs;
    PeerGradPtrs gp;
    for (int i = 0; i < nseg; ++i) gp.p[i] = have ? grads[i] : nullptr;
    if (have)
        for (int i = 0; i < nseg; ++i)
            if (!grads[i] && (*v.num)[i] > 0) {
                set_error("missing gradient for segment " + std::to_string(i));
                return MBS_EKEY;
            }
    const int64_t tile = 8192;
    const int64_t n_tiles = (v.numel + tile - 1) / tile;
    const int64_t slice = ((v.numel / 4 + h->world - 1) / h->world) * 4;
    h->epoch += 1;
    const long long budget = (long long)(timeout_ms * 2.0e6);  // ~2 GHz SM clock
    const int64_t slot = *v.seen;
    const float* lp = have ? loss_dev : nullptr;
    const bool assign = *v.fresh;
#define MBS_AR(A, H)                                                                                        \
    k_accum_allreduce<A, H><<<h->grid, kPeerThreads, 0, cs>>>(                                              \
        v.acc, d_segs, nseg, tile, n_tiles, v.numel, slice, gp, (float)factor, h->peers, h->rank, h->world, \
        h->epoch, h->bar_base, budget, lp, v.d_losses + slot, v.d_factors + slot, loss_factor,            \
        v.d_weights + slot, loss_weight)
    if (assign && have) MBS_AR(true, true);
    else if (assign) MBS_AR(true, false);
    else if (have) MBS_AR(false, true);
    else MBS_AR(false, false);
#undef MBS_AR
    MBS_CK_LAUNCH("k_accum_allreduce");
    h->bar_base += 3u * (unsigned)h->grid;
    if (have) *v.seen += 1;
    *v.fresh = false;
    *v.n_partials = 0;  // the norm is of the reduced sum: finalize recomputes it
    return MBS_OK;
}

}  // extern "C"
