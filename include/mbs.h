/*
 * mbs.h — C-ABI of the B200 Micro-Batch Streaming hot path (libmbs_native.so).
 *
 * The reference (`/root/reference/pkg/src/mbstream`) is a pure-Python/NumPy
 * package with no FFI; its "interface" for this path is the functional API in
 * engine.py / optim.py / tensor.py. Each entry point below names the reference
 * symbol (file:line) whose semantics it implements. The Python host package
 * `paper_2110_12484_b200` binds these with ctypes (INTEGRATION.md shows the
 * binding a reference maintainer would add).
 *
 * ABI rules
 *  - every function is extern "C" and returns an int status (MBS_*); no C++
 *    exception crosses the boundary;
 *  - device pointers are BORROWED (owned by the caller, e.g. torch tensors);
 *    handles own only their scratch (chunk tables, norm partials, stats);
 *  - `stream` arguments are cudaStream_t passed as void*; every device call is
 *    stream-ordered and asynchronous unless documented otherwise;
 *  - one host thread per handle (the reference's threading rule).
 */
#ifndef MBS_H
#define MBS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (mapped to the reference exception types by the shim) ---- */
#define MBS_OK          0  /* success                                                   */
#define MBS_EINVAL      1  /* bad argument          -> ValueError                         */
#define MBS_EOVERFLOW   2  /* too many micro-batches -> AccumulatorOverflowError (engine.py:118-121) */
#define MBS_EKEY        3  /* key/shape mismatch    -> GradientKeyMismatchError (tensor.py:132-146) */
#define MBS_ECUDA       4  /* CUDA runtime error    -> RuntimeError                       */
#define MBS_ENONFINITE  5  /* non-finite gradient   -> NonFiniteError (errors.py:14-19)  */

/* normalization modes, engine.py:34 NORMALIZATION_MODES */
#define MBS_NORM_PAPER_FAITHFUL 0
#define MBS_NORM_EXACT_WEIGHTED 1
#define MBS_NORM_OFF            2

/* element types for staging */
#define MBS_U8   0
#define MBS_F32  1
#define MBS_BF16 2
#define MBS_F16  3
#define MBS_F64  4  /* source only (the reference's float64 arrays) */

/* layouts for staging */
#define MBS_NCHW 0
#define MBS_NHWC 1

const char* mbs_status_string(int status);
const char* mbs_last_error(void);         /* last CUDA / argument error text (process-wide) */
int mbs_version(void);

/* ---------------------------------------------------------------------------
 * Plan — engine.py:56-78 plan_split, engine.py:81-91 normalization_factor
 * ------------------------------------------------------------------------- */

/* Writes n_mu (after the n_b < n_mu clamp, engine.py:66-67), n_s_mu
 * (= ceil(n_b/n_mu), engine.py:68) and, if sizes_out != NULL, up to `cap`
 * micro-batch sizes (engine.py:69-71). Returns MBS_EINVAL for n_b<1 or n_mu<1
 * (engine.py:64-65) and when cap < n_s_mu with sizes_out != NULL. */
int mbs_plan_split(int64_t n_b, int64_t n_mu, int64_t* n_mu_out, int64_t* n_s_mu_out,
                   int64_t* sizes_out, int64_t cap);

/* engine.py:81-91. MBS_EINVAL for k outside [0, n_s_mu) or unknown mode. */
int mbs_normalization_factor(int64_t n_b, int64_t n_mu, int64_t k, int mode, double* out);

/* ---------------------------------------------------------------------------
 * Gradient accumulator — engine.py:100-131 GradientAccumulator (+ accumulate,
 * engine.py:134-137; the grad norm, tensor.py:126-130). K1.
 *
 * The accumulator is a flat fp32 device buffer (borrowed) holding n_segments
 * parameter segments; segment i lives at seg_offsets[i] (multiple of 4 floats)
 * with seg_numels[i] elements. begin() is lazy: the first add() after begin()
 * ASSIGNS acc = s*g (no zero pass, no acc read); later adds do acc += s*g.
 * ------------------------------------------------------------------------- */
typedef struct mbs_accum* mbs_accum_t;

int mbs_accum_create(float* acc_dev, int64_t acc_numel, int64_t n_segments,
                     const int64_t* seg_offsets, const int64_t* seg_numels,
                     int64_t max_micro, mbs_accum_t* out);
int mbs_accum_destroy(mbs_accum_t h);
/* engine.py:110-115 begin(expected); expected < 0 means "no limit". */
int mbs_accum_begin(mbs_accum_t h, int64_t expected);
/* Materialise the pending zero of begin() (only needed when the sums are read
 * before any add()). */
int mbs_accum_zero(mbs_accum_t h, void* stream);
/* engine.py:117-128 add(grads) with the normalisation factor fused (the
 * reference folds it into the backward seed, engine.py:214-215, which is the
 * same linear map). `grads[i]` is the device gradient of segment
 * seg_begin+i (dense, same element order as the parameter). `loss_dev`
 * (nullable) is this micro-batch's raw mean loss, recorded for the stats
 * (engine.py:217-218) with its normalisation factor `loss_factor` (which
 * equals `factor` unless the caller already applied it in the backward seed)
 * and `loss_weight` = its sample count size_k (the weight of engine.py:221). `last` != 0 additionally emits per-chunk
 * ||acc||^2 partials for the grad norm. Returns MBS_EOVERFLOW past
 * `expected`. */
int mbs_accum_add(mbs_accum_t h, const float* const* grads, int64_t seg_begin,
                  int64_t seg_count, double factor, const float* loss_dev,
                  double loss_factor, double loss_weight, int last, void* stream);
/* Same, with a per-segment gradient dtype: dtypes[i] is MBS_F32 or MBS_BF16 (NULL: all fp32). bf16
 * gradients (the weight gradients of a bf16 shadow-weight forward) are widened exactly in K1, so no
 * fp32 conversion pass is needed before accumulation. */
int mbs_accum_add_typed(mbs_accum_t h, const void* const* grads, const int* dtypes, int64_t seg_begin,
                        int64_t seg_count, double factor, const float* loss_dev, double loss_factor,
                        double loss_weight, int last, void* stream);
/* Same, over a flat gradient buffer laid out exactly like acc. */
int mbs_accum_add_flat(mbs_accum_t h, const float* g_flat, double factor,
                       const float* loss_dev, double loss_factor, double loss_weight, int last,
                       void* stream);
/* Recompute the ||acc||^2 partials over the whole buffer (used after an
 * all-reduce in data-parallel mode). */
int mbs_accum_norm(mbs_accum_t h, void* stream);
/* Reduce the partials and the loss record: writes to device `stats_dev`
 * (double[4 + 2*max_micro]): [0]=||acc||^2, [1]=mini-batch loss
 * sum_k size_k*loss_k/n_b (engine.py:221, sequential in plan order),
 * [2]=non-finite flag, [3]=#micro, [4..4+n)=raw losses,
 * [4+max_micro..)=normalised losses (raw*factor, engine.py:218).
 * Deterministic (fixed reduction order). */
int mbs_accum_finalize(mbs_accum_t h, int64_t n_b, double* stats_dev, void* stream);
int mbs_accum_seen(mbs_accum_t h, int64_t* seen, int64_t* expected);

/* ---------------------------------------------------------------------------
 * Optimizer step over flat buffers — optim.py:52-65 sgd_step, optim.py:68-93
 * adam_step (coupled weight decay). K3. `guard_dev` (nullable) points at a
 * double; when it is non-finite the step is skipped on device (params stay
 * intact, the host raises NonFiniteError when it reads the stats).
 * `velocity`/`m`/`v` are device fp32 buffers of `numel` elements, zero at
 * step 0 (the reference creates them lazily as zeros, optim.py:58-61,78-83).
 * `shadow_bf16` (nullable, 8-byte aligned, numel bf16 values) receives the
 * round-to-nearest-even bf16 copy of the updated weights in the same pass —
 * the weights the next mini-batch's bf16 forward reads (shadow-weight mode).
 * ------------------------------------------------------------------------- */
int mbs_sgd_step(float* w, const float* grad, float* velocity, int64_t numel, double lr,
                 double momentum, double weight_decay, const double* guard_dev, void* shadow_bf16,
                 void* stream);
int mbs_adam_step(float* w, const float* grad, float* m, float* v, int64_t numel, double lr,
                  double beta1, double beta2, double eps, double weight_decay,
                  int64_t step /* t = step_count + 1 */, const double* guard_dev, void* shadow_bf16,
                  void* stream);

/* ---------------------------------------------------------------------------
 * Staging — engine.py:310-311 (x[order[mini]]) + engine.py:149-151
 * (ascontiguousarray(x[lo:hi])) + tensor.py:20-22 (dtype coercion). K2.
 *
 * dst row r := cast(src row (rows ? rows[r] : row0 + r)); each row is a
 * C x H x W sample stored NCHW in `src`; dst is NCHW or NHWC in dst_dtype.
 * Casts are exact (u8->f32/bf16/f16) or IEEE round-to-nearest-even
 * (f32/f64->f32/bf16/f16), bit-identical to torch's .to(dtype) (f64->bf16
 * rounds through f32 exactly like torch does). `src` may be device
 * memory or pinned/registered host memory (zero-copy). `rows` is a DEVICE
 * array (nullable).
 * ------------------------------------------------------------------------- */
int mbs_stage(const void* src, int src_dtype, const int64_t* rows, int64_t row0, int64_t n_rows,
              int64_t C, int64_t H, int64_t W, void* dst, int dst_dtype, int dst_layout,
              void* stream);
/* Byte-exact row gather (targets, masks, labels): dst[r] = src[rows? rows[r] : row0+r]. */
int mbs_gather_rows(const void* src, const int64_t* rows, int64_t row0, int64_t n_rows,
                    int64_t row_bytes, void* dst, void* stream);

/* ---------------------------------------------------------------------------
 * Host->device micro-batch streamer — engine.py:140-163 _micro_batches
 * (prefetch worker, two slots) re-designed as a pinned ring of `n_slots`
 * slots, a native gather thread pool and cudaMemcpyAsync on a copy stream.
 *
 * A job gathers `n_rows` rows (rows[] host indices, or row0.. contiguous) of
 * up to MBS_MAX_PARTS host tensors into pinned slot `slot`, then copies each
 * part to its device destination on `copy_stream` and records the slot's
 * "ready" event. When a part's host source is already pinned and the rows are
 * contiguous, the gather is skipped and the copy reads the source directly.
 * mbs_streamer_wait() makes `compute_stream` wait for the slot (host blocks
 * only until the job has been issued, never for the copy itself);
 * mbs_streamer_release() records that compute finished reading the slot's
 * device buffers so the next copy into them is ordered after it.
 * ------------------------------------------------------------------------- */
#define MBS_MAX_PARTS 4
typedef struct mbs_streamer* mbs_streamer_t;
typedef struct {
    const void* src;        /* host base pointer of the dataset tensor        */
    int64_t row_bytes;      /* bytes per sample                                */
    void* dst;              /* device destination (n_rows * row_bytes)         */
    int src_pinned;         /* src is page-locked (skip gather when contiguous)*/
} mbs_part_t;

int mbs_streamer_create(int n_slots, int64_t slot_bytes, int n_threads, void* copy_stream,
                        mbs_streamer_t* out);
int mbs_streamer_destroy(mbs_streamer_t h);
/* `job_out` (nullable) receives the job's sequence number for mbs_streamer_timing. */
int mbs_streamer_submit(mbs_streamer_t h, int slot, const mbs_part_t* parts, int n_parts,
                        const int64_t* rows, int64_t row0, int64_t n_rows, int64_t* job_out);
int mbs_streamer_wait(mbs_streamer_t h, int slot, void* compute_stream);
int mbs_streamer_release(mbs_streamer_t h, int slot, void* compute_stream);
/* Timing of job `job` (ms): host gather time, device copy time (copy-stream
 * events) and the time compute was blocked waiting for it
 * (max(0, copy_end - compute_reached_wait)); bytes copied. Synchronises on the
 * job's events; records are kept for the last 256 jobs. */
int mbs_streamer_timing(mbs_streamer_t h, int64_t job, double* gather_ms, double* copy_ms,
                        double* blocked_ms, int64_t* bytes);
/* Absolute copy times of a job: copy start / end in ms after `origin_event` (a cudaEvent_t recorded with
 * timing, e.g. torch.cuda.Event(enable_timing=True).cuda_event) — the "transfer" StreamEvent of the
 * reference's schedule (streaming.py:41-46) measured on the copy stream. Blocks until the copy ended. */
int mbs_streamer_timeline(mbs_streamer_t h, int64_t job, void* origin_event, double* copy_start_ms,
                          double* copy_end_ms);
/* Multi-threaded host gather into a caller buffer (used by tests and the
 * epoch driver): dst[r] = src[rows[r]] for row_bytes-sized rows. */
int mbs_host_gather(const void* src, int64_t row_bytes, const int64_t* rows, int64_t n_rows,
                    void* dst, int n_threads);

/* ---------------------------------------------------------------------------
 * Fused last-micro-batch accumulate + all-reduce over peer memory (K1C) — the
 * data-parallel exchange of SURVEY §8e (no reference equivalent) as ONE
 * kernel: X_self = acc (+)= factor*g, reduce-scatter over the peers' X in rank
 * order, all-gather into acc. Exchange buffers are exported with CUDA IPC
 * (NVLink/NVSwitch P2P between the GPUs of a node).
 * ------------------------------------------------------------------------- */
#define MBS_PEER_HANDLE_BYTES 128
typedef struct mbs_peer* mbs_peer_t;

/* Allocate this rank's exchange buffer (numel floats, numel % 4 == 0) and signal block. */
int mbs_peer_create(int rank, int world, int64_t numel, mbs_peer_t* out);
/* Export this rank's IPC handles (MBS_PEER_HANDLE_BYTES bytes) for the other ranks. */
int mbs_peer_handle(mbs_peer_t h, void* out);
/* Map every peer's exchange buffer: `handles` holds world x MBS_PEER_HANDLE_BYTES bytes, rank order. */
int mbs_peer_open(mbs_peer_t h, const void* handles);
int mbs_peer_destroy(mbs_peer_t h);
/* Device error flag (1 = a peer did not arrive within the timeout); synchronous. */
int mbs_peer_status(mbs_peer_t h, int* error_flag);
/* The last micro-batch of this rank: acc := SUM_ranks(acc_r (+)= factor*g_r) on every rank, as
 * mbs_accum_add would (loss record, overflow guard) followed by an all-reduce. `grads` may be NULL
 * for a rank without a micro-batch in this mini-batch (it contributes its accumulator). Spin-waits
 * are bounded by timeout_ms; on timeout the device error flag is set and the kernel drains. */
int mbs_accum_add_allreduce(mbs_accum_t h, mbs_peer_t peer, const float* const* grads, double factor,
                            const float* loss_dev, double loss_factor, double loss_weight,
                            double timeout_ms, void* stream);

/* ---------------------------------------------------------------------------
 * Micro-batch BatchNorm (K5) — the model-side op of every micro-batch forward
 * in training mode: statistics over the MICRO-batch (reference nn.py:275-282
 * BatchNorm2d.forward, biased variance for the normalisation), one
 * running-statistics update per micro-batch (nn.py:329-332; torch's unbiased
 * running_var convention), fused with the ReLU that follows it and, for
 * residual blocks, the skip add before that ReLU: y = relu(bn(x) [+ residual]).
 *
 * x / residual / y / dy / dx / dresidual are channels-last activations:
 * `rows` (= N*H*W) x `C` row-major, dtype MBS_BF16 or MBS_F32. weight/bias
 * (may be NULL: 1 / 0), running stats (both NULL: not tracked), save_* and
 * dweight/dbias are fp32 [C]. `workspace` is device scratch of at least
 * mbs_bn_workspace_bytes() bytes, exclusively owned by the call until it has
 * executed on `stream`. A residual is only accepted together with relu=1.
 * Deterministic: fixed-order reductions, no atomics.
 * ------------------------------------------------------------------------- */
int mbs_bn_workspace_bytes(int64_t rows, int64_t C, int dtype, int64_t* bytes);
/* num_batches_tracked (nullable, device int64): incremented by one on the stream (torch's
 * BatchNorm2d.num_batches_tracked += 1), so no separate counter kernel runs per layer.
 * `relu` is a flag word: MBS_BN_RELU fuses the ReLU; MBS_BN_BIASED_RUNNING_VAR makes the running-variance
 * update take the biased micro-batch variance, as the reference does (nn.py:329-332), instead of torch's
 * unbiased one. */
#define MBS_BN_RELU 1
#define MBS_BN_BIASED_RUNNING_VAR 2
int mbs_bn_forward(const void* x, const void* residual, void* y, int dtype, int64_t rows, int64_t C,
                   const float* weight, const float* bias, float* running_mean, float* running_var,
                   int64_t* num_batches_tracked, double momentum, double eps, int relu, float* save_mean,
                   float* save_invstd, void* workspace, void* stream);
/* Gradients of mbs_bn_forward: dx, dresidual (iff residual), dweight/dbias (may be NULL).
 * The ReLU mask is recomputed from x (and residual) bit-identically to the forward.
 * dy2 (nullable): a second gradient of y (the output feeds both the next block's main path and its
 * skip), summed with dy inside the kernel and rounded to the activation dtype exactly like torch's add;
 * only with residual + relu, C/8 (bf16) or C/4 (fp32)
 * vectors <= 256 and every pointer 16-byte aligned — otherwise MBS_ERR_INVALID. */
int mbs_bn_backward(const void* x, const void* residual, const void* dy, const void* dy2, void* dx,
                    void* dresidual, int dtype, int64_t rows, int64_t C, const float* weight, const float* bias,
                    const float* save_mean, const float* save_invstd, int relu, float* dweight, float* dbias,
                    void* workspace, void* stream);

/* ---------------------------------------------------------------------------
 * Max-pool (K6) — the model's MaxPool2d in every micro-batch forward/backward,
 * channels-last. x [N,H,W,C], y / idx / dy [N,Ho,Wo,C] with Ho = (H+2p-k)/s+1;
 * idx holds the window-relative argmax (kh*k + kw, one byte). torch semantics
 * (first maximum wins, NaN propagates, padding never wins); the backward sums
 * the gradients of an input element in ascending window order in fp32, so both
 * directions are bit-identical to torch's max_pool2d. dilation 1, floor mode.
 * ------------------------------------------------------------------------- */
/* stash (nullable): also write x into channel columns [stash_c0, stash_c0+C) of a channels-last
 * tensor with stash_C channels (the U-Net skip lands in its concat buffer); needs k == s, p == 0,
 * k | H, k | W (every input element read exactly once). */
int mbs_maxpool_forward(const void* x, void* y, uint8_t* idx, int dtype, int64_t N, int64_t H, int64_t W, int64_t C,
                        int k, int s, int p, void* stash, int64_t stash_C, int64_t stash_c0, void* stream);
/* addend (nullable): dx += addend[..., add_c0:add_c0+C] (channels-last, add_C channels), summed in
 * fp32 before dx's single rounding (the skip-connection gradient, fused).
 * dy2 (nullable): a second gradient of y (y has two consumers), added to dy per window and rounded to the
 * activation dtype like torch's add. */
int mbs_maxpool_backward(const void* dy, const void* dy2, const uint8_t* idx, void* dx, int dtype, int64_t N,
                         int64_t H, int64_t W, int64_t C, int k, int s, int p, const void* addend, int64_t add_C,
                         int64_t add_c0, void* stream);
/* Channel-slice copy between channels-last tensors seen as [M, C_total] rows:
 * dst[m, dst_c0 + c] = src[m, src_c0 + c] (+ bias[c], fp32, nullable) for c < C (the U-Net skip join
 * and its backward). colsum (nullable): fp32 [colsum_rows][C] per-CTA column sums of the copied
 * values (the ConvTranspose bias gradient; sum the rows), grid = colsum_rows CTAs. */
int mbs_copy_channels(const void* src, int64_t src_C, int64_t src_c0, void* dst, int64_t dst_C, int64_t dst_c0,
                      int64_t M, int64_t C, const float* bias, float* colsum, int64_t colsum_rows, int dtype,
                      void* stream);

/* ---------------------------------------------------------------------------
 * Stem im2col (K7) — the model's first (3-channel) convolution as one library
 * GEMM: cols[N*Ho*Wo, Kp] with column (kh*k + kw)*C + c = x[n, oh*s-p+kh,
 * ow*s-p+kw, c] (0 outside the image), columns [k*k*C, Kp) zero. x channels-
 * last [N,H,W,C]; dtype MBS_BF16 or MBS_F32; Kp >= k*k*C.
 * ------------------------------------------------------------------------- */
int mbs_im2col(const void* x, void* cols, int dtype, int64_t N, int64_t H, int64_t W, int64_t C, int k, int s, int p,
               int64_t Kp, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MBS_H */
