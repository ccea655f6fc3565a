// K1 (fused normalise + accumulate + grad-norm partials), the loss-stat /
// grad-norm finalize, and K3 (fused SGD-momentum / Adam step) for sm_100a.
//
// Reference semantics:
//   GradientAccumulator.begin/add      engine.py:110-128 (sums[name] += grad, plan order)
//   factor folded into backward seed   engine.py:210-215, nn.py:596 (linear in the seed)
//   mini-batch loss / stats            engine.py:217-221
//   GradientSet.l2_norm                tensor.py:126-130
//   sgd_step / adam_step               optim.py:52-65 / optim.py:68-93
//
// All kernels are HBM-bound streaming passes: 128-bit loads/stores, a few
// independent float4s in flight per thread, one CTA per 8192-element chunk
// (the hardware block scheduler balances the tail), no atomics, and a fixed
// reduction order so the grad norm is bit-reproducible run to run.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdlib.h>
#include <stdint.h>

#include <algorithm>
#include <mutex>
#include <string>
#include <vector>

#include "mbs_common.h"

namespace mbs {

static std::mutex g_err_mu;
static std::string g_last_error;  // process-wide: the streamer's worker thread reports here too
void set_error(const std::string& msg) {
    std::lock_guard<std::mutex> g(g_err_mu);
    g_last_error = msg;
}

constexpr int kThreads = 256;
constexpr int64_t kMinPerBlock = 4096;   // elements: smallest CTA share (tiny buckets)
constexpr int64_t kDefaultTile = 8192;   // elements per K1 CTA (MBS_K1_TILE overrides; 0 = balanced)
constexpr int kMaxPtrs = 1024;     // gradient pointers per K1 launch (kernel-param table)
#ifndef MBS_K1_UNROLL
#define MBS_K1_UNROLL 4
#endif
#ifndef MBS_K1_MINBLOCKS
#define MBS_K1_MINBLOCKS 4
#endif
constexpr int kUnroll = MBS_K1_UNROLL;
// bf16-gradient (shadow-weight) path, A/B in the C2 pipeline (profiles/r01_k1_bf16_ab.txt): 8-byte
// bf16x4 loads with the 64-register cap (38.8 us/launch, 0.89 of the copy peak) beat 16-byte bf16x8
// loads at 3 CTAs/SM (46.2 us) or 2 CTAs/SM (42.9 us).
#ifndef MBS_K1_MIXED_MINBLOCKS
#define MBS_K1_MIXED_MINBLOCKS 4
#endif
#ifndef MBS_K1_U8
#define MBS_K1_U8 2
#endif
#ifndef MBS_K1_BF16_X4
#define MBS_K1_BF16_X4 1
#endif

struct Seg {
    int64_t off;   // element offset of the segment in acc (multiple of 4)
    int64_t num;   // elements of the segment (its gradient tensor's numel)
};

struct GradPtrs {
    const float* p[kMaxPtrs];
};

__device__ __forceinline__ float4 ld_stream(const float4* p) {
#if defined(MBS_K1_PLAIN_G)
    return __ldg(p);
#else
    float4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w) : "l"(p));
    return r;
#endif
}

// the accumulator is read then written by the same thread only: the non-coherent path is safe
__device__ __forceinline__ float4 ld_acc(const float4* p) {
#if defined(MBS_K1_NC_ACC)
    return __ldg(p);
#else
    return *p;
#endif
}

__device__ __forceinline__ double sq4(float4 a) {
    double x = a.x, y = a.y, z = a.z, w = a.w;
    return x * x + y * y + z * z + w * w;
}

// bf16 gradients (the shadow-weight path: cuDNN's weight gradients stay bf16, no conversion pass):
// 4 elements per 8-byte streaming load, widened exactly to fp32.
__device__ __forceinline__ float4 ld_stream_bf16x4(const uint2* p) {
    uint32_t a, b;
    asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(a), "=r"(b) : "l"(p));
    return make_float4(__uint_as_float(a << 16), __uint_as_float(a & 0xffff0000u), __uint_as_float(b << 16),
                       __uint_as_float(b & 0xffff0000u));
}

__device__ __forceinline__ float bf16_to_f32(const __nv_bfloat16 v) { return __bfloat162float(v); }

// round-to-nearest-even fp32 -> bf16 of 4 values packed for one 8-byte store (torch's .to(bfloat16))
__device__ __forceinline__ uint2 pack_bf16x4(const float4 v) {
    __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y), hi = __floats2bfloat162_rn(v.z, v.w);
    return make_uint2(*reinterpret_cast<uint32_t*>(&lo), *reinterpret_cast<uint32_t*>(&hi));
}

template <int NT>
__device__ __forceinline__ double block_sum(double v, double* smem) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) smem[warp] = v;
    __syncthreads();
    double r = 0.0;
    if (threadIdx.x == 0) {
#pragma unroll
        for (int i = 0; i < NT / 32; ++i) r += smem[i];
    }
    return r;  // valid in thread 0 only
}

// Last segment index in [s0, s1) whose offset is <= x (segments sorted, non-overlapping).
__device__ __forceinline__ int find_seg(const Seg* __restrict__ segs, int s0, int s1, int64_t x) {
    int a = s0, b = s1 - 1;
    while (a < b) {
        const int m = (a + b + 1) >> 1;
        if (segs[m].off <= x) a = m; else b = m - 1;
    }
    return a;
}

// One contiguous piece of one segment: acc[0..n) (+)= s * g[0..n). Pieces never exceed one CTA
// share (<= 2^31 elements), so the inner loops use 32-bit indices (keeps K1 at ~56 registers).
__device__ __forceinline__ void ld_stream_bf16x8(const uint4* p, float4& lo, float4& hi) {
    uint32_t a, b, c, d;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "l"(p));
    lo = make_float4(__uint_as_float(a << 16), __uint_as_float(a & 0xffff0000u), __uint_as_float(b << 16),
                     __uint_as_float(b & 0xffff0000u));
    hi = make_float4(__uint_as_float(c << 16), __uint_as_float(c & 0xffff0000u), __uint_as_float(d << 16),
                     __uint_as_float(d & 0xffff0000u));
}

template <bool ASSIGN>
__device__ __forceinline__ float4 axpy4(float s, float4 g, float4 a) {
    float4 r;
    if (ASSIGN) {
        r.x = s * g.x; r.y = s * g.y; r.z = s * g.z; r.w = s * g.w;
    } else {
        r.x = fmaf(s, g.x, a.x); r.y = fmaf(s, g.y, a.y); r.z = fmaf(s, g.z, a.z); r.w = fmaf(s, g.w, a.w);
    }
    return r;
}

template <bool ASSIGN, bool NORM, typename G>
__device__ __forceinline__ void accum_piece(float* __restrict__ a, const G* __restrict__ g, int n, float s,
                                            double& sq) {
    int done = 0;
    float4* a4 = reinterpret_cast<float4*>(a);
    if constexpr (sizeof(G) == 4) {
        if ((reinterpret_cast<uintptr_t>(g) & 15) == 0) {
            const int n4 = n >> 2;
            for (int base = threadIdx.x; base < n4; base += kThreads * kUnroll) {
                float4 gv[kUnroll], av[kUnroll];
#pragma unroll
                for (int u = 0; u < kUnroll; ++u) {
                    const int i = base + u * kThreads;
                    if (i < n4) {
                        gv[u] = ld_stream(reinterpret_cast<const float4*>(g) + i);
                        if (!ASSIGN) av[u] = ld_acc(a4 + i);
                    }
                }
#pragma unroll
                for (int u = 0; u < kUnroll; ++u) {
                    const int i = base + u * kThreads;
                    if (i < n4) {
                        const float4 r = axpy4<ASSIGN>(s, gv[u], av[u]);
                        a4[i] = r;
                        if (NORM) sq += sq4(r);
                    }
                }
            }
            done = n4 << 2;
        }
    } else {
        // bf16: 8 gradients per 16-byte load against two float4 of the accumulator, so a thread keeps as
        // many bytes in flight as the fp32 path
        constexpr int kU8 = MBS_K1_U8;   // only instantiated in the MIXED kernel
        if (!MBS_K1_BF16_X4 && (reinterpret_cast<uintptr_t>(g) & 15) == 0) {
            const int n8 = n >> 3;
            for (int base = threadIdx.x; base < n8; base += kThreads * kU8) {
                float4 gl[kU8], gh[kU8], al[kU8], ah[kU8];
#pragma unroll
                for (int u = 0; u < kU8; ++u) {
                    const int i = base + u * kThreads;
                    if (i < n8) {
                        ld_stream_bf16x8(reinterpret_cast<const uint4*>(g) + i, gl[u], gh[u]);
                        if (!ASSIGN) {
                            al[u] = ld_acc(a4 + 2 * i);
                            ah[u] = ld_acc(a4 + 2 * i + 1);
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < kU8; ++u) {
                    const int i = base + u * kThreads;
                    if (i < n8) {
                        const float4 rl = axpy4<ASSIGN>(s, gl[u], al[u]);
                        const float4 rh = axpy4<ASSIGN>(s, gh[u], ah[u]);
                        a4[2 * i] = rl;
                        a4[2 * i + 1] = rh;
                        if (NORM) sq += sq4(rl) + sq4(rh);
                    }
                }
            }
            done = n8 << 3;
        } else if ((reinterpret_cast<uintptr_t>(g) & 7) == 0) {
            const int n4 = n >> 2;
            for (int i = threadIdx.x; i < n4; i += kThreads) {
                const float4 gv = ld_stream_bf16x4(reinterpret_cast<const uint2*>(g) + i);
                const float4 r = axpy4<ASSIGN>(s, gv, ASSIGN ? gv : ld_acc(a4 + i));
                a4[i] = r;
                if (NORM) sq += sq4(r);
            }
            done = n4 << 2;
        }
    }
    for (int i = done + threadIdx.x; i < n; i += kThreads) {  // tail / unaligned gradient
        float gi;
        if constexpr (sizeof(G) == 4) gi = g[i]; else gi = bf16_to_f32(g[i]);
        const float r = ASSIGN ? s * gi : fmaf(s, gi, a[i]);
        a[i] = r;
        if (NORM) sq += (double)r * (double)r;
    }
}
// MIXED: the launch has bf16 segments (shadow-weight mode); compiled with a larger register budget
// (3 CTAs/SM) so the 8-wide bf16 path keeps a full unroll of 16-byte loads in flight without spills.
template <bool ASSIGN, bool NORM, bool MIXED>
__global__ void __launch_bounds__(kThreads, MIXED ? MBS_K1_MIXED_MINBLOCKS : MBS_K1_MINBLOCKS)
k_accum(float* __restrict__ acc, const Seg* __restrict__ segs, const int* __restrict__ tile_seg, int seg0, int seg1,
        int64_t lo0, int64_t hi0, int64_t per_block, const __grid_constant__ GradPtrs gp, float s,
        double* __restrict__ partials,
        const float* __restrict__ loss, double* __restrict__ loss_slot, double* __restrict__ factor_slot,
        double factor, double* __restrict__ weight_slot, double weight) {
    __shared__ double red[kThreads / 32];
    const int64_t lo = lo0 + (int64_t)blockIdx.x * per_block;
    const int64_t hi = min(lo + per_block, hi0);
    double sq = 0.0;
    if (lo < hi) {
        // full-range launches read their first segment from a precomputed table (one load instead of a
        // chain of dependent binary-search loads at every CTA start)
        const int first = tile_seg != nullptr ? tile_seg[blockIdx.x] : find_seg(segs, seg0, seg1, lo);
        for (int si = first; si < seg1; ++si) {
            const Seg sg = segs[si];
            if (sg.off >= hi) break;
            const int64_t p0 = max(lo, sg.off), p1 = min(hi, sg.off + sg.num);
            if (p1 <= p0) continue;
            // bit 0 of a gradient pointer tags bf16 data (bf16 is 2-byte aligned, fp32 4-byte)
            const uintptr_t raw = reinterpret_cast<uintptr_t>(gp.p[si - seg0]);
            if (MIXED && (raw & 1))
                accum_piece<ASSIGN, NORM>(acc + p0, reinterpret_cast<const __nv_bfloat16*>(raw & ~(uintptr_t)1) +
                                                        (p0 - sg.off), (int)(p1 - p0), s, sq);
            else
                accum_piece<ASSIGN, NORM>(acc + p0, reinterpret_cast<const float*>(raw) + (p0 - sg.off),
                                          (int)(p1 - p0), s, sq);
        }
    }
    if (NORM) {
        const double t = block_sum<kThreads>(sq, red);
        if (threadIdx.x == 0) partials[blockIdx.x] = t;
    }
    if (loss != nullptr && blockIdx.x == 0 && threadIdx.x == 0) {
        *loss_slot = (double)*loss;
        *factor_slot = factor;
        *weight_slot = weight;
    }
}

// ||acc||^2 partials over [0, n) (padding is zero), one balanced slice per CTA.
__global__ void __launch_bounds__(kThreads)
k_sumsq(const float* __restrict__ acc, int64_t n, int64_t per_block, double* __restrict__ partials) {
    __shared__ double red[kThreads / 32];
    const int64_t lo = (int64_t)blockIdx.x * per_block;
    const int64_t hi = min(lo + per_block, n);
    double sq = 0.0;
    if (lo < hi) {
        const float4* a4 = reinterpret_cast<const float4*>(acc + lo);
        const int64_t n4 = (hi - lo) >> 2;
        for (int64_t i = threadIdx.x; i < n4; i += kThreads) sq += sq4(ld_stream(a4 + i));
        for (int64_t i = lo + (n4 << 2) + threadIdx.x; i < hi; i += kThreads) sq += (double)acc[i] * (double)acc[i];
    }
    const double t = block_sum<kThreads>(sq, red);
    if (threadIdx.x == 0) partials[blockIdx.x] = t;
}

// Finalize: deterministic reduction of the norm partials + the loss record (engine.py:217-221).
__global__ void __launch_bounds__(1024)
k_finalize(const double* __restrict__ partials, int64_t n_partials,
           const double* __restrict__ losses, const double* __restrict__ factors,
           const double* __restrict__ weights, int64_t n_micro, int64_t max_micro, int64_t n_b,
           double* __restrict__ stats) {
    __shared__ double red[32];
    double v = 0.0;
    for (int64_t i = threadIdx.x; i < n_partials; i += blockDim.x) v += partials[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double norm2 = 0.0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) norm2 += red[i];
        // mini-batch loss: sequential sum over micro-batches in plan order (engine.py:221)
        double lsum = 0.0;
        for (int64_t j = 0; j < n_micro; ++j) lsum += weights[j] * losses[j];
        stats[0] = norm2;
        stats[1] = lsum / (double)n_b;
        stats[2] = isfinite(norm2) ? 0.0 : 1.0;
        stats[3] = (double)n_micro;
        for (int64_t j = 0; j < n_micro; ++j) {
            stats[4 + j] = losses[j];
            stats[4 + max_micro + j] = losses[j] * factors[j];
        }
    }
}

__device__ __forceinline__ bool guard_tripped(const double* guard) {
    return guard != nullptr && !isfinite(*guard);
}

// K3a: optim.py:52-65 — g' = g + wd*w; v = mu*v + g'; w -= lr*v. Two float4s per thread per
// iteration (6 independent 16-byte loads in flight).
template <bool READ_V, bool WD>
__device__ __forceinline__ void sgd4(float4& ww, float4& vv, const float4 gg, float lr, float mu, float wd) {
    const float gx = WD ? fmaf(wd, ww.x, gg.x) : gg.x;
    const float gy = WD ? fmaf(wd, ww.y, gg.y) : gg.y;
    const float gz = WD ? fmaf(wd, ww.z, gg.z) : gg.z;
    const float gw = WD ? fmaf(wd, ww.w, gg.w) : gg.w;
    if (!READ_V) vv = make_float4(0.f, 0.f, 0.f, 0.f);
    vv.x = fmaf(mu, vv.x, gx); vv.y = fmaf(mu, vv.y, gy);
    vv.z = fmaf(mu, vv.z, gz); vv.w = fmaf(mu, vv.w, gw);
    ww.x = fmaf(-lr, vv.x, ww.x); ww.y = fmaf(-lr, vv.y, ww.y);
    ww.z = fmaf(-lr, vv.z, ww.z); ww.w = fmaf(-lr, vv.w, ww.w);
}

#ifndef MBS_K3_UNROLL
#define MBS_K3_UNROLL 2
#endif
template <bool READ_V, bool WD>
__global__ void __launch_bounds__(kThreads)
k_sgd(float4* __restrict__ w, const float4* __restrict__ g, float4* __restrict__ v, int64_t n4,
      float lr, float mu, float wd, const double* __restrict__ guard, uint2* __restrict__ shadow) {
    if (guard_tripped(guard)) return;
    constexpr int U = MBS_K3_UNROLL;
    const int64_t stride = (int64_t)gridDim.x * kThreads;
    for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n4; i += U * stride) {
        float4 gg[U], ww[U], vv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t j = i + u * stride;
            if (j < n4) {
                gg[u] = ld_stream(g + j);
                ww[u] = w[j];
                vv[u] = READ_V ? v[j] : make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t j = i + u * stride;
            if (j < n4) {
                sgd4<READ_V, WD>(ww[u], vv[u], gg[u], lr, mu, wd);
                v[j] = vv[u];
                w[j] = ww[u];
                if (shadow) shadow[j] = pack_bf16x4(ww[u]);   // the bf16 weights the next forward reads
            }
        }
    }
}

__device__ __forceinline__ void adam1(float& w, float& m, float& v, float g, float lr, float b1,
                                      float omb1, float b2, float omb2, float c1, float c2,
                                      float eps, float wd) {
    if (wd != 0.f) g = fmaf(wd, w, g);
    m = fmaf(b1, m, omb1 * g);
    v = fmaf(b2, v, omb2 * g * g);
    const float mh = __fdiv_rn(m, c1);
    const float vh = __fsqrt_rn(__fdiv_rn(v, c2));
    w = w - __fdiv_rn(lr * mh, vh + eps);
}

// K3b: optim.py:68-93 — bias-corrected Adam, coupled weight decay; two float4s per iteration.
__device__ __forceinline__ void adam4(float4& ww, float4& mm, float4& vv, const float4 gg, float lr, float b1,
                                      float omb1, float b2, float omb2, float c1, float c2, float eps, float wd) {
    adam1(ww.x, mm.x, vv.x, gg.x, lr, b1, omb1, b2, omb2, c1, c2, eps, wd);
    adam1(ww.y, mm.y, vv.y, gg.y, lr, b1, omb1, b2, omb2, c1, c2, eps, wd);
    adam1(ww.z, mm.z, vv.z, gg.z, lr, b1, omb1, b2, omb2, c1, c2, eps, wd);
    adam1(ww.w, mm.w, vv.w, gg.w, lr, b1, omb1, b2, omb2, c1, c2, eps, wd);
}

__global__ void __launch_bounds__(kThreads)
k_adam(float4* __restrict__ w, const float4* __restrict__ g, float4* __restrict__ m,
       float4* __restrict__ v, int64_t n4, float lr, float b1, float b2, float omb1, float omb2, float c1, float c2,
       float eps, float wd, const double* __restrict__ guard, uint2* __restrict__ shadow) {
    // omb = 1 - beta is formed in double on the host: 1.f - 0.999f carries a 1.3e-5 relative error
    if (guard_tripped(guard)) return;
    const int64_t stride = (int64_t)gridDim.x * kThreads;
    for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n4; i += 2 * stride) {
        const int64_t i2 = i + stride;
        const bool two = i2 < n4;
        const float4 g0 = ld_stream(g + i);
        float4 w0 = w[i], m0 = m[i], v0 = v[i];
        float4 g1, w1, m1, v1;
        if (two) {
            g1 = ld_stream(g + i2);
            w1 = w[i2]; m1 = m[i2]; v1 = v[i2];
        }
        adam4(w0, m0, v0, g0, lr, b1, omb1, b2, omb2, c1, c2, eps, wd);
        w[i] = w0; m[i] = m0; v[i] = v0;
        if (shadow) shadow[i] = pack_bf16x4(w0);
        if (two) {
            adam4(w1, m1, v1, g1, lr, b1, omb1, b2, omb2, c1, c2, eps, wd);
            w[i2] = w1; m[i2] = m1; v[i2] = v1;
            if (shadow) shadow[i2] = pack_bf16x4(w1);
        }
    }
}

static int sm_count() {
    static int n = 0;
    if (n == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    }
    return n;
}

static int stream_grid(int64_t n4) {
    const int64_t want = (n4 + kThreads - 1) / kThreads;
    const int64_t cap = (int64_t)sm_count() * (2048 / kThreads) * 2;  // two full waves, grid-stride
    return (int)std::max<int64_t>(1, std::min(want, cap));
}

}  // namespace mbs

using namespace mbs;

struct mbs_accum {
    float* acc = nullptr;
    int64_t numel = 0;
    std::vector<int64_t> off, num;
    Seg* d_segs = nullptr;             // device copy of (off, num) per segment
    int grid = 0;                      // CTAs of a full-range launch (resident CTAs on the device)
    double* d_partials = nullptr;      // [grid] ||acc||^2 partials, one per CTA of the last NORM launch
    int n_partials = 0;                // valid partials (0 = stale: finalize recomputes the norm)
    int64_t tile = kDefaultTile;       // elements per CTA (0 = balanced over resident CTAs)
    int* d_tile_seg = nullptr;         // first segment of every full-range tile (tile > 0)
    int64_t max_partials = 0;
    double* d_losses = nullptr;        // [max_micro] raw loss per local micro-batch
    double* d_factors = nullptr;       // [max_micro]
    double* d_weights = nullptr;       // [max_micro] sample count of each micro-batch
    int64_t max_micro = 0;
    int64_t expected = -1;
    int64_t seen = 0;
    bool fresh = true;                 // begin() pending: next add assigns
    int64_t covered = 0;               // segments added so far for the current micro-batch
};

namespace mbs {
int accum_view(mbs_accum_t h, AccumView* v) {
    if (!h || !v) return invalid("null accumulator");
    v->acc = h->acc;
    v->numel = h->numel;
    v->off = &h->off;
    v->num = &h->num;
    v->d_losses = h->d_losses;
    v->d_factors = h->d_factors;
    v->d_weights = h->d_weights;
    v->seen = &h->seen;
    v->covered = &h->covered;
    v->expected = h->expected;
    v->max_micro = h->max_micro;
    v->fresh = &h->fresh;
    v->n_partials = &h->n_partials;
    return MBS_OK;
}
}  // namespace mbs

extern "C" {

const char* mbs_status_string(int s) {
    switch (s) {
        case MBS_OK: return "ok";
        case MBS_EINVAL: return "invalid argument";
        case MBS_EOVERFLOW: return "accumulator overflow";
        case MBS_EKEY: return "gradient key/shape mismatch";
        case MBS_ECUDA: return "CUDA error";
        case MBS_ENONFINITE: return "non-finite values";
        default: return "unknown status";
    }
}

const char* mbs_last_error(void) {
    static thread_local std::string copy;
    std::lock_guard<std::mutex> g(g_err_mu);
    copy = g_last_error;
    return copy.c_str();
}

int mbs_version(void) { return 1; }

int mbs_plan_split(int64_t n_b, int64_t n_mu, int64_t* n_mu_out, int64_t* n_s_mu_out,
                   int64_t* sizes_out, int64_t cap) {
    if (n_b < 1 || n_mu < 1)
        return invalid("batch sizes must be positive, got n_b=" + std::to_string(n_b) +
                       ", n_mu=" + std::to_string(n_mu));
    if (n_b < n_mu) n_mu = n_b;                       // engine.py:66-67
    const int64_t q = n_b / n_mu, r = n_b % n_mu;
    const int64_t n_s_mu = q + (r ? 1 : 0);           // ceil, engine.py:68
    if (n_mu_out) *n_mu_out = n_mu;
    if (n_s_mu_out) *n_s_mu_out = n_s_mu;
    if (sizes_out) {
        if (cap < n_s_mu) return invalid("sizes_out capacity smaller than n_s_mu");
        for (int64_t i = 0; i < q; ++i) sizes_out[i] = n_mu;   // engine.py:69
        if (r) sizes_out[q] = r;                               // engine.py:70-71
    }
    return MBS_OK;
}

int mbs_normalization_factor(int64_t n_b, int64_t n_mu, int64_t k, int mode, double* out) {
    int64_t nm = 0, ns = 0;
    int st = mbs_plan_split(n_b, n_mu, &nm, &ns, nullptr, 0);
    if (st) return st;
    if (k < 0 || k >= ns)
        return invalid("micro-batch index " + std::to_string(k) + " outside plan of " + std::to_string(ns));
    const int64_t size_k = (k == ns - 1 && n_b % nm) ? n_b % nm : nm;
    switch (mode) {
        case MBS_NORM_PAPER_FAITHFUL: *out = 1.0 / (double)ns; return MBS_OK;          // engine.py:85-86
        case MBS_NORM_EXACT_WEIGHTED: *out = (double)size_k / (double)n_b; return MBS_OK;  // 87-88
        case MBS_NORM_OFF: *out = 1.0; return MBS_OK;                                   // 89-90
        default: return invalid("unknown normalization mode " + std::to_string(mode));
    }
}

int mbs_accum_create(float* acc_dev, int64_t acc_numel, int64_t n_segments,
                     const int64_t* seg_offsets, const int64_t* seg_numels, int64_t max_micro,
                     mbs_accum_t* out) {
    if (!out || !acc_dev || acc_numel <= 0 || n_segments <= 0 || !seg_offsets || !seg_numels || max_micro < 1)
        return invalid("mbs_accum_create: bad arguments");
    if ((reinterpret_cast<uintptr_t>(acc_dev) & 15) != 0) return invalid("accumulator must be 16-byte aligned");
    auto* h = new mbs_accum();
    h->acc = acc_dev;
    h->numel = acc_numel;
    h->max_micro = max_micro;
    std::vector<Seg> segs;
    int64_t prev_end = 0;
    for (int64_t i = 0; i < n_segments; ++i) {
        const int64_t o = seg_offsets[i], n = seg_numels[i];
        if (o % 4 != 0 || n < 0 || o < prev_end || o + n > acc_numel) {
            delete h;
            return invalid("segment " + std::to_string(i) + " misaligned, overlapping or out of range");
        }
        prev_end = o + n;
        h->off.push_back(o);
        h->num.push_back(n);
        segs.push_back(Seg{o, n});
    }
    // one full-range launch = exactly the resident CTAs of the device: every CTA gets the same
    // share of elements, so there is no tail wave
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_accum<false, true, false>, kThreads, 0);
    h->grid = std::max(1, per_sm) * sm_count();
    if (const char* t = getenv("MBS_K1_TILE")) h->tile = atoll(t);
    if (h->tile > 0 && h->tile < 1024) h->tile = 1024;
    h->max_partials = std::max<int64_t>(h->grid, (acc_numel + 1023) / 1024);
    std::vector<int> tile_seg;
    if (h->tile > 0) {
        const int64_t lo = h->off[0], hi = h->off.back() + h->num.back();
        const int64_t per = (h->tile + 31) / 32 * 32;
        size_t si = 0;
        for (int64_t t = lo; t < hi; t += per) {
            while (si + 1 < segs.size() && segs[si + 1].off <= t) ++si;   // last segment with off <= t
            tile_seg.push_back((int)si);
        }
    }
    cudaError_t e = cudaMalloc(&h->d_segs, sizeof(Seg) * segs.size());
    if (e == cudaSuccess && !tile_seg.empty()) e = cudaMalloc(&h->d_tile_seg, sizeof(int) * tile_seg.size());
    if (e == cudaSuccess && !tile_seg.empty())
        e = cudaMemcpy(h->d_tile_seg, tile_seg.data(), sizeof(int) * tile_seg.size(), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(h->d_segs, segs.data(), sizeof(Seg) * segs.size(), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMalloc(&h->d_partials, sizeof(double) * h->max_partials);
    if (e == cudaSuccess) e = cudaMemset(h->d_partials, 0, sizeof(double) * h->max_partials);
    if (e == cudaSuccess) e = cudaMalloc(&h->d_losses, sizeof(double) * max_micro * 3);
    if (e == cudaSuccess) e = cudaMemset(h->d_losses, 0, sizeof(double) * max_micro * 3);
    if (e != cudaSuccess) {
        mbs_accum_destroy(h);
        return cuda_status(e, "mbs_accum_create");
    }
    h->d_factors = h->d_losses + max_micro;
    h->d_weights = h->d_losses + 2 * max_micro;
    *out = h;
    return MBS_OK;
}

int mbs_accum_destroy(mbs_accum_t h) {
    if (!h) return MBS_OK;
    if (h->d_segs) cudaFree(h->d_segs);
    if (h->d_tile_seg) cudaFree(h->d_tile_seg);
    if (h->d_partials) cudaFree(h->d_partials);
    if (h->d_losses) cudaFree(h->d_losses);
    delete h;
    return MBS_OK;
}

int mbs_accum_begin(mbs_accum_t h, int64_t expected) {
    if (!h) return invalid("null accumulator");
    if (expected > h->max_micro) return invalid("expected micro-batches exceed the handle's max_micro");
    h->expected = expected;
    h->seen = 0;
    h->covered = 0;
    h->fresh = true;
    return MBS_OK;
}

int mbs_accum_zero(mbs_accum_t h, void* stream) {
    if (!h) return invalid("null accumulator");
    MBS_CK(cudaMemsetAsync(h->acc, 0, sizeof(float) * h->numel, (cudaStream_t)stream));
    h->fresh = false;
    h->n_partials = 0;
    return MBS_OK;
}

int mbs_accum_seen(mbs_accum_t h, int64_t* seen, int64_t* expected) {
    if (!h) return invalid("null accumulator");
    if (seen) *seen = h->seen;
    if (expected) *expected = h->expected;
    return MBS_OK;
}

// Elements per CTA for a launch over `range` elements: a balanced share for `grid` CTAs,
// rounded to 128 bytes so every CTA boundary is float4-aligned inside a segment.
static int64_t share(int64_t range, int grid, int64_t tile) {
    if (tile > 0) return (tile + 31) / 32 * 32;  // fixed tiles, one CTA each (hardware-balanced)
    int64_t per = (range + grid - 1) / grid;     // balanced: exactly `grid` CTAs
    per = std::max<int64_t>(per, kMinPerBlock);
    return (per + 31) / 32 * 32;
}

static int launch_accum(mbs_accum_t h, const void* const* grads, const int* dtypes, int64_t seg_begin,
                        int64_t seg_count, float s, const float* loss_dev, double factor, double weight, bool assign,
                        bool norm, cudaStream_t st) {
    const int64_t slot = h->seen;
    const int64_t nseg = (int64_t)h->off.size();
    // the norm partials are only meaningful for a launch covering every segment
    norm = norm && seg_begin == 0 && seg_count == nseg && seg_count <= kMaxPtrs;
    for (int64_t b = 0; b < seg_count; b += kMaxPtrs) {
        const int64_t cnt = std::min<int64_t>(kMaxPtrs, seg_count - b);
        GradPtrs gp;
        bool mixed = false;
        for (int64_t i = 0; i < cnt; ++i) {
            const bool bf = dtypes != nullptr && dtypes[b + i] == MBS_BF16;
            mixed |= bf;
            gp.p[i] = reinterpret_cast<const float*>(reinterpret_cast<uintptr_t>(grads[b + i]) | (bf ? 1u : 0u));
        }
        const int s0 = (int)(seg_begin + b), s1 = (int)(seg_begin + b + cnt);
        const int64_t lo = h->off[s0], hi = h->off[s1 - 1] + h->num[s1 - 1];
        if (hi <= lo) continue;
        const int64_t per = share(hi - lo, h->grid, h->tile);
        const unsigned grid = (unsigned)((hi - lo + per - 1) / per);
        const float* lp = (b == 0) ? loss_dev : nullptr;
        const int* ts = (h->d_tile_seg != nullptr && s0 == 0 && s1 == (int)nseg) ? h->d_tile_seg : nullptr;
        double* ls = h->d_losses + slot;
        double* fs = h->d_factors + slot;
        double* ws = h->d_weights + slot;
#define MBS_K1_LAUNCH(A, NM, MX)                                                                          \
    k_accum<A, NM, MX><<<grid, kThreads, 0, st>>>(h->acc, h->d_segs, ts, s0, s1, lo, hi, per, gp, s, h->d_partials, \
                                                  lp, ls, fs, factor, ws, weight)
        if (mixed) {
            if (assign && norm) MBS_K1_LAUNCH(true, true, true);
            else if (assign) MBS_K1_LAUNCH(true, false, true);
            else if (norm) MBS_K1_LAUNCH(false, true, true);
            else MBS_K1_LAUNCH(false, false, true);
        } else {
            if (assign && norm) MBS_K1_LAUNCH(true, true, false);
            else if (assign) MBS_K1_LAUNCH(true, false, false);
            else if (norm) MBS_K1_LAUNCH(false, true, false);
            else MBS_K1_LAUNCH(false, false, false);
        }
#undef MBS_K1_LAUNCH
        MBS_CK_LAUNCH("k_accum");
        h->n_partials = norm ? (int)grid : 0;
    }
    return MBS_OK;
}

int mbs_accum_add_typed(mbs_accum_t h, const void* const* grads, const int* dtypes, int64_t seg_begin,
                        int64_t seg_count, double factor, const float* loss_dev, double loss_factor,
                        double loss_weight, int last, void* stream) {
    if (!h || !grads) return invalid("null accumulator or gradient table");
    if (dtypes)
        for (int64_t i = 0; i < seg_count; ++i) {
            if (dtypes[i] != MBS_F32 && dtypes[i] != MBS_BF16) return invalid("gradient dtype must be f32 or bf16");
            if (dtypes[i] == MBS_BF16 && (reinterpret_cast<uintptr_t>(grads[i]) & 1))
                return invalid("bf16 gradient pointer not 2-byte aligned");
        }
    const int64_t nseg = (int64_t)h->off.size();
    if (seg_begin < 0 || seg_count < 1 || seg_begin + seg_count > nseg)
        return invalid("segment range out of bounds");
    // A micro-batch may arrive as several calls (gradient buckets issued during
    // the last backward, any order); it is complete once every segment has been
    // added. The overflow guard (engine.py:118-121) runs on its first call.
    if (h->covered == 0) {
        if (h->expected >= 0 && h->seen >= h->expected) {
            set_error("already accumulated " + std::to_string(h->seen) + " of " +
                      std::to_string(h->expected) + " micro-batches");
            return MBS_EOVERFLOW;
        }
        if (h->seen >= h->max_micro) {
            set_error("micro-batch count exceeds the handle's max_micro");
            return MBS_EOVERFLOW;
        }
    }
    if (h->covered + seg_count > nseg) {
        set_error("gradient segments exceed the accumulator's parameter set");
        return MBS_EKEY;
    }
    for (int64_t i = 0; i < seg_count; ++i)
        if (!grads[i] && h->num[seg_begin + i] > 0) {
            set_error("missing gradient for segment " + std::to_string(seg_begin + i));
            return MBS_EKEY;
        }
    int st = launch_accum(h, grads, dtypes, seg_begin, seg_count, (float)factor, loss_dev, loss_factor, loss_weight,
                          h->fresh, last != 0, (cudaStream_t)stream);
    if (st) return st;
    h->covered += seg_count;
    if (h->covered == nseg) {
        h->covered = 0;
        h->seen += 1;
        h->fresh = false;
    }
    return MBS_OK;
}

int mbs_accum_add(mbs_accum_t h, const float* const* grads, int64_t seg_begin, int64_t seg_count,
                  double factor, const float* loss_dev, double loss_factor, double loss_weight, int last,
                  void* stream) {
    return mbs_accum_add_typed(h, reinterpret_cast<const void* const*>(grads), nullptr, seg_begin, seg_count, factor,
                               loss_dev, loss_factor, loss_weight, last, stream);
}

int mbs_accum_add_flat(mbs_accum_t h, const float* g_flat, double factor, const float* loss_dev,
                       double loss_factor, double loss_weight, int last, void* stream) {
    if (!h || !g_flat) return invalid("null accumulator or gradient");
    std::vector<const float*> ptrs(h->off.size());
    for (size_t i = 0; i < ptrs.size(); ++i) ptrs[i] = g_flat + h->off[i];
    return mbs_accum_add(h, ptrs.data(), 0, (int64_t)ptrs.size(), factor, loss_dev, loss_factor, loss_weight, last,
                         stream);
}

int mbs_accum_norm(mbs_accum_t h, void* stream) {
    if (!h) return invalid("null accumulator");
    const int64_t per = share(h->numel, h->grid, 0);
    const unsigned grid = (unsigned)((h->numel + per - 1) / per);
    k_sumsq<<<grid, kThreads, 0, (cudaStream_t)stream>>>(h->acc, h->numel, per, h->d_partials);
    MBS_CK_LAUNCH("k_sumsq");
    h->n_partials = (int)grid;
    return MBS_OK;
}

int mbs_accum_finalize(mbs_accum_t h, int64_t n_b, double* stats_dev, void* stream) {
    if (!h || !stats_dev || n_b < 1) return invalid("mbs_accum_finalize: null handle/stats or n_b < 1");
    if (h->n_partials == 0) {  // no fused norm since the last change of acc: compute it now
        int st = mbs_accum_norm(h, stream);
        if (st) return st;
    }
    k_finalize<<<1, 1024, 0, (cudaStream_t)stream>>>(h->d_partials, h->n_partials, h->d_losses, h->d_factors,
                                                    h->d_weights, h->seen, h->max_micro, n_b, stats_dev);
    MBS_CK_LAUNCH("k_finalize");
    return MBS_OK;
}

int mbs_sgd_step(float* w, const float* grad, float* velocity, int64_t numel, double lr, double momentum,
                 double weight_decay, const double* guard_dev, void* shadow_bf16, void* stream) {
    if (shadow_bf16 && ((uintptr_t)shadow_bf16 & 7)) return invalid("mbs_sgd_step: shadow must be 8-byte aligned");
    auto SH = reinterpret_cast<uint2*>(shadow_bf16);
    if (!w || !grad || !velocity || numel <= 0 || numel % 4)
        return invalid("mbs_sgd_step: null buffer or numel not a positive multiple of 4");
    if (((uintptr_t)w | (uintptr_t)grad | (uintptr_t)velocity) & 15) return invalid("mbs_sgd_step: buffers must be 16-byte aligned");
    const int64_t n4 = numel / 4;
    const int grid = stream_grid(n4);
    auto st = (cudaStream_t)stream;
    auto W = reinterpret_cast<float4*>(w);
    auto G = reinterpret_cast<const float4*>(grad);
    auto V = reinterpret_cast<float4*>(velocity);
    const bool rv = momentum != 0.0, wd = weight_decay != 0.0;
    if (rv && wd) k_sgd<true, true><<<grid, kThreads, 0, st>>>(W, G, V, n4, (float)lr, (float)momentum, (float)weight_decay, guard_dev, SH);
    else if (rv) k_sgd<true, false><<<grid, kThreads, 0, st>>>(W, G, V, n4, (float)lr, (float)momentum, 0.f, guard_dev, SH);
    else if (wd) k_sgd<false, true><<<grid, kThreads, 0, st>>>(W, G, V, n4, (float)lr, 0.f, (float)weight_decay, guard_dev, SH);
    else k_sgd<false, false><<<grid, kThreads, 0, st>>>(W, G, V, n4, (float)lr, 0.f, 0.f, guard_dev, SH);
    MBS_CK_LAUNCH("k_sgd");
    return MBS_OK;
}

int mbs_adam_step(float* w, const float* grad, float* m, float* v, int64_t numel, double lr, double beta1,
                  double beta2, double eps, double weight_decay, int64_t step, const double* guard_dev,
                  void* shadow_bf16, void* stream) {
    if (shadow_bf16 && ((uintptr_t)shadow_bf16 & 7)) return invalid("mbs_adam_step: shadow must be 8-byte aligned");
    if (!w || !grad || !m || !v || numel <= 0 || numel % 4 || step < 1)
        return invalid("mbs_adam_step: null buffer, numel not a positive multiple of 4, or step < 1");
    if (((uintptr_t)w | (uintptr_t)grad | (uintptr_t)m | (uintptr_t)v) & 15) return invalid("mbs_adam_step: buffers must be 16-byte aligned");
    const double c1 = 1.0 - pow(beta1, (double)step), c2 = 1.0 - pow(beta2, (double)step);  // optim.py:73-74
    const int64_t n4 = numel / 4;
    k_adam<<<stream_grid(n4), kThreads, 0, (cudaStream_t)stream>>>(
        reinterpret_cast<float4*>(w), reinterpret_cast<const float4*>(grad), reinterpret_cast<float4*>(m),
        reinterpret_cast<float4*>(v), n4, (float)lr, (float)beta1, (float)beta2, (float)(1.0 - beta1),
        (float)(1.0 - beta2), (float)c1, (float)c2, (float)eps,
        (float)weight_decay, guard_dev, reinterpret_cast<uint2*>(shadow_bf16));
    MBS_CK_LAUNCH("k_adam");
    return MBS_OK;
}

}  // extern "C"
