// K5: training-mode BatchNorm over a channels-last activation with MICRO-BATCH
// statistics, fused with the ReLU (and the residual add) that follows it.
//
// Every micro-batch forward of the benchmark models runs BatchNorm in training
// mode: statistics over the micro-batch only (reference nn.py:275-282
// BatchNorm2d.forward, the reason MBS keeps micro-batch membership intact) and
// one running-statistics update per micro-batch (nn.py:329-332; torch's
// convention here: running_var takes the UNBIASED batch variance, momentum
// 0.1). On B200 torch's own channels-last BN kernels were 60 % of the
// ResNet-50 micro-batch step at ~7 % of HBM bandwidth (profiles/r01_c2_launches.md),
// so the model's normalisation runs here; convolutions stay on cuDNN.
//
// Layout: x is NHWC = `rows` x `C` row-major (rows = N*H*W), dtype bf16 or fp32.
// Thread mapping for every kernel: a CTA owns a channel group (<= 256 16-byte
// vectors of channels) and a chunk of rows; thread t handles channel vector
// t % gv of rows t / gv, t / gv + RP, ... (RP = 256 / gv rows per pass), so
// per-channel coefficients live in registers and a warp reads contiguous
// 16-byte vectors. Algorithmic bytes (E = rows*C elements, s = sizeof(T)):
//   forward : stats E*s (read x)  + apply 2*E*s (+E*s residual)
//   backward: reduce 2*E*s (x, dy; +2*E*s residual: read r, write d_r = g) + elemt 3*E*s (x, dy or g, dx)
// Reductions: per-thread fp32 partial sums of (x - K) and (x - K)^2 with a
// per-channel shift K = x[0, c] (no catastrophic cancellation when |mean| >>
// std), per-CTA partials in a fixed order, then a warp per channel merges the
// CTA partials in fp64 in a fixed order — bit-reproducible, atomic-free.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <stdlib.h>

#include <algorithm>
#include <map>
#include <mutex>

#include "mbs_common.h"
#include "mbs_tma.h"

#include <cooperative_groups.h>
namespace cg = cooperative_groups;

namespace mbs {

constexpr int kBnThreads = 256;

template <typename T, int V> struct BnIO;

template <> struct BnIO<float, 4> {
    static __device__ __forceinline__ void load(const float* p, float (&f)[4]) {
        float4 v = *reinterpret_cast<const float4*>(p);
        f[0] = v.x; f[1] = v.y; f[2] = v.z; f[3] = v.w;
    }
    static __device__ __forceinline__ void store(float* p, const float (&f)[4]) {
        *reinterpret_cast<float4*>(p) = make_float4(f[0], f[1], f[2], f[3]);
    }
    static constexpr float kMaskThreshold = 0.f;
};
template <> struct BnIO<float, 1> {
    static __device__ __forceinline__ void load(const float* p, float (&f)[1]) { f[0] = *p; }
    static __device__ __forceinline__ void store(float* p, const float (&f)[1]) { *p = f[0]; }
    static constexpr float kMaskThreshold = 0.f;
};
template <> struct BnIO<__nv_bfloat16, 8> {
    static __device__ __forceinline__ void load(const __nv_bfloat16* p, float (&f)[8]) {
        uint4 v = *reinterpret_cast<const uint4*>(p);
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            f[2 * i] = __uint_as_float(w[i] << 16);
            f[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
        }
    }
    static __device__ __forceinline__ void store(__nv_bfloat16* p, const float (&f)[8]) {
        uint32_t w[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            __nv_bfloat162 h = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
            w[i] = *reinterpret_cast<uint32_t*>(&h);
        }
        *reinterpret_cast<uint4*>(p) = make_uint4(w[0], w[1], w[2], w[3]);
    }
    // ReLU mask on the STORED value: bf16(z) <= 0  <=>  z <= 2^-134 (RNE: larger positives round up to the
    // smallest bf16 subnormal 2^-133, 2^-134 ties to even = 0), so the mask needs no conversion
    static constexpr float kMaskThreshold = 0x1p-134f;
};
template <> struct BnIO<__nv_bfloat16, 1> {
    static __device__ __forceinline__ void load(const __nv_bfloat16* p, float (&f)[1]) { f[0] = __bfloat162float(*p); }
    static __device__ __forceinline__ void store(__nv_bfloat16* p, const float (&f)[1]) { *p = __float2bfloat16_rn(f[0]); }
    static constexpr float kMaskThreshold = 0x1p-134f;
};

struct BnGeom {
    int64_t rows, C;
    int gv;            // vectors per channel group (<= 256)
    int rp;            // rows per pass = 256 / gv
    int64_t chunk;     // rows per CTA
    int P;             // CTAs along rows (= partials per channel for the reductions)
    long long* nbt = nullptr;   // num_batches_tracked, incremented once by the statistics finalize (nullable)
    bool biased_rv = false;     // running_var takes the biased variance (the reference, nn.py:329-332)
};

// Per-channel affine of the forward (shared by forward apply and the backward mask
// recomputation so both see bit-identical values): y = x*scale + shift.
// Per-channel affine of the normalisation, z = (x - mu) * scale + beta. Centring BEFORE the scale (not
// x*scale + (beta - mu*scale)) keeps x_hat exact when |mean| >> std (e.g. a stem fed raw 0..255 pixels,
// where the folded form cancels ~log2(|mean|/std) bits) and makes x == mean give exactly beta (a
// one-value channel, then meets a following ReLU at exactly 0 like the reference).
__device__ __forceinline__ void bn_affine(const float* w, const float* b, const float* mean, const float* invstd,
                                          int64_t c, float& scale, float& mu, float& beta) {
    const float g = w ? w[c] : 1.f;
    beta = b ? b[c] : 0.f;
    scale = g * invstd[c];
    mu = mean[c];
}

__device__ __forceinline__ float bn_z(float x, float scale, float mu, float beta) {
    return fmaf(x - mu, scale, beta);
}

// torch's relu (clamp_min) propagates NaN; fmaxf would not
__device__ __forceinline__ float relu_nan(float z) { return z < 0.f ? 0.f : z; }

// threshold_backward on the stored output y = T(relu(z)): the gradient is zeroed where y <= 0
// (NaN passes, as in torch); y <= 0 is decided on z without a conversion (kMaskThreshold).
template <typename T, int V, bool RES>
__device__ __forceinline__ float relu_mask(float x, float sc, float mu, float be, float r, float d) {
    const float z = bn_z(x, sc, mu, be) + (RES ? r : 0.f);
    return z <= BnIO<T, V>::kMaskThreshold ? 0.f : d;
}

// MODE 0: statistics — partial (sum(x-K), sum((x-K)^2)).
// MODE 1: backward reduce — partial (sum g, sum g*(x-mean)), g = dy * relu-mask.
template <typename T, int V, int MODE, bool RELU, bool RES>
__device__ __forceinline__ void bn_reduce_body(const T* __restrict__ x, const T* __restrict__ dy,
                                                          const T* __restrict__ res, const float* __restrict__ w,
                                                          const float* __restrict__ b,
                                                          const float* __restrict__ mean,
                                                          const float* __restrict__ invstd, float2* __restrict__ part,
                                                          BnGeom g, int bx, int by){
    __shared__ float red[2][kBnThreads * V];
    const int tid = threadIdx.x;
    const int lane = tid % g.gv, rph = tid / g.gv;
    const int64_t c0 = ((int64_t)by * g.gv + lane) * V;
    const bool active = rph < g.rp && c0 < g.C;
    float s1[V], s2[V], k[V], sc[V], sh[V];
#pragma unroll
    for (int i = 0; i < V; ++i) { s1[i] = 0.f; s2[i] = 0.f; k[i] = 0.f; sc[i] = 0.f; sh[i] = 0.f; }
    if (active) {
        if (MODE == 0) {
            BnIO<T, V>::load(x + c0, k);  // shift K = x[0, c]
        } else {
#pragma unroll
            for (int i = 0; i < V; ++i) {
                if (RELU) bn_affine(w, b, mean, invstd, c0 + i, sc[i], k[i], sh[i]);
                else k[i] = mean[c0 + i];
            }
        }
        const int64_t r0 = (int64_t)bx * g.chunk;
        const int64_t r1 = min(g.rows, r0 + g.chunk);
        constexpr int U = MODE == 0 ? 8 : 4;  // statistics: one stream, more loads in flight per thread
        int64_t r = r0 + rph;
        for (; r + (U - 1) * g.rp < r1; r += U * g.rp) {
            float xv[U][V], dv[U][V], rv[U][V];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int64_t o = (r + u * g.rp) * g.C + c0;
                BnIO<T, V>::load(x + o, xv[u]);
                if (MODE == 1) BnIO<T, V>::load(dy + o, dv[u]);
                if (MODE == 1 && RELU && RES) BnIO<T, V>::load(res + o, rv[u]);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (MODE == 1 && RELU) {
#pragma unroll
                    for (int i = 0; i < V; ++i)
                        dv[u][i] = relu_mask<T, V, RES>(xv[u][i], sc[i], k[i], sh[i], rv[u][i], dv[u][i]);
                }
#pragma unroll
                for (int i = 0; i < V; ++i) {
                    const float d = xv[u][i] - k[i];
                    if (MODE == 0) {
                        s1[i] += d;
                        s2[i] = fmaf(d, d, s2[i]);
                    } else {
                        s1[i] += dv[u][i];
                        s2[i] = fmaf(dv[u][i], d, s2[i]);
                    }
                }
            }
        }
        for (; r < r1; r += g.rp) {
            float xv[V], dv[V], rv[V];
            const int64_t o = r * g.C + c0;
            BnIO<T, V>::load(x + o, xv);
            if (MODE == 1) BnIO<T, V>::load(dy + o, dv);
            if (MODE == 1 && RELU && RES) BnIO<T, V>::load(res + o, rv);
            if (MODE == 1 && RELU) {
#pragma unroll
                for (int i = 0; i < V; ++i) dv[i] = relu_mask<T, V, RES>(xv[i], sc[i], k[i], sh[i], rv[i], dv[i]);
            }
#pragma unroll
            for (int i = 0; i < V; ++i) {
                const float d = xv[i] - k[i];
                if (MODE == 0) {
                    s1[i] += d;
                    s2[i] = fmaf(d, d, s2[i]);
                } else {
                    s1[i] += dv[i];
                    s2[i] = fmaf(dv[i], d, s2[i]);
                }
            }
        }
    }
    // CTA reduction over the row phases, fixed order
#pragma unroll
    for (int i = 0; i < V; ++i) {
        red[0][rph * g.gv * V + lane * V + i] = s1[i];
        red[1][rph * g.gv * V + lane * V + i] = s2[i];
    }
    __syncthreads();
    const int gc = g.gv * V;  // channels in this group
    for (int j = tid; j < gc; j += kBnThreads) {
        const int64_t c = (int64_t)by * gc + j;
        if (c >= g.C) break;
        float a = 0.f, q = 0.f;
        for (int p = 0; p < g.rp; ++p) {
            a += red[0][p * gc + j];
            q += red[1][p * gc + j];
        }
        part[c * g.P + bx] = make_float2(a, q);
    }
}

template <typename T, int V, int MODE, bool RELU, bool RES>
__global__ void __launch_bounds__(kBnThreads) k_bn_reduce(const T* __restrict__ x, const T* __restrict__ dy,
                                                          const T* __restrict__ res, const float* __restrict__ w,
                                                          const float* __restrict__ b,
                                                          const float* __restrict__ mean,
                                                          const float* __restrict__ invstd, float2* __restrict__ part,
                                                          BnGeom g) {
    cudaGridDependencySynchronize();  // PDL: inputs come from the preceding kernel
    bn_reduce_body<T, V, MODE, RELU, RES>(x, dy, res, w, b, mean, invstd, part, g, blockIdx.x, blockIdx.y);
}

// TPC threads per channel (power of two, 32..256) merge the P CTA partials in fp64: thread j
// sums partials j, j+TPC, ... in order, then a fixed xor tree within the warp and a fixed-order
// sum over the channel's warps. Returns true on the thread that owns the channel's result.
template <int TPC>
__device__ __forceinline__ bool group_merge(const float2* part, int P, bool valid, double& a, double& q) {
    __shared__ double red[2][kBnThreads / 32];
    const int t = threadIdx.x % TPC;
    a = 0.0;
    q = 0.0;
    if (valid) {
#pragma unroll 4
        for (int p = t; p < P; p += TPC) {
            const float2 v = part[p];
            a += (double)v.x;
            q += (double)v.y;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        q += __shfl_xor_sync(0xffffffffu, q, o);
    }
    if (TPC > 32) {
        const int warp = threadIdx.x / 32;
        if (threadIdx.x % 32 == 0) {
            red[0][warp] = a;
            red[1][warp] = q;
        }
        __syncthreads();
        if (t == 0) {
            a = 0.0;
            q = 0.0;
            for (int k = 0; k < TPC / 32; ++k) {
                a += red[0][warp + k];
                q += red[1][warp + k];
            }
        }
    }
    return valid && t == 0;
}

template <typename T>
__device__ __forceinline__ void bn_stats_write(const T* __restrict__ x, const BnGeom& g, const float* __restrict__ w,
                                               const float* __restrict__ b, float* running_mean, float* running_var,
                                               double momentum, double eps, float* __restrict__ save_mean,
                                               float* __restrict__ save_invstd, float* __restrict__ coef, int64_t c,
                                               double s1, double s2) {
    const double m = (double)g.rows;
    const double K = (double)static_cast<float>(x[c]);
    const double dm = s1 / m;
    const double var = fmax(s2 / m - dm * dm, 0.0);  // biased: normalisation uses it (nn.py:278)
    const double mean = K + dm;
    save_mean[c] = (float)mean;
    save_invstd[c] = (float)(1.0 / sqrt(var + eps));
    if (running_mean) {
        running_mean[c] = (float)((1.0 - momentum) * (double)running_mean[c] + momentum * mean);
        const double unbiased = (g.rows > 1 && !g.biased_rv) ? var * m / (m - 1.0) : var;
        running_var[c] = (float)((1.0 - momentum) * (double)running_var[c] + momentum * unbiased);
    }
    float sc, mu, be;
    bn_affine(w, b, save_mean, save_invstd, c, sc, mu, be);
    coef[3 * c] = sc;
    coef[3 * c + 1] = mu;
    coef[3 * c + 2] = be;
}

template <typename T, int TPC>
__global__ void __launch_bounds__(kBnThreads) k_bn_stats_finalize(
        const T* __restrict__ x, const float2* __restrict__ part, BnGeom g, const float* __restrict__ w,
        const float* __restrict__ b, float* running_mean, float* running_var, double momentum, double eps,
        float* __restrict__ save_mean, float* __restrict__ save_invstd, float* __restrict__ coef) {
    const int64_t c = (int64_t)blockIdx.x * (kBnThreads / TPC) + threadIdx.x / TPC;
    cudaGridDependencySynchronize();  // PDL: partials come from the statistics kernel
    if (g.nbt && blockIdx.x == 0 && threadIdx.x == 0) *g.nbt += 1;   // torch's num_batches_tracked += 1
    double s1, s2;
    if (group_merge<TPC>(part + c * g.P, g.P, c < g.C, s1, s2))
        bn_stats_write(x, g, w, b, running_mean, running_var, momentum, eps, save_mean, save_invstd, coef, c, s1, s2);
}

// backward finalize: dgamma = invstd * sum g(x-mean), dbeta = sum g; dx coefficients
// dx = k1*g + A*(x-mean) + B with k1 = gamma*invstd, A = -k1*invstd*dgamma/M, B = -k1*dbeta/M
// (stored: A, B, B - A*mean).
__device__ __forceinline__ void bn_bwd_write(const BnGeom& g, const float* __restrict__ w,
                                             const float* __restrict__ mean, const float* __restrict__ invstd,
                                             float* __restrict__ dweight, float* __restrict__ dbias,
                                             float* __restrict__ coef, int64_t c, double sg, double sgx) {
    const double is = (double)invstd[c];
    const double dgam = sgx * is;
    if (dweight) dweight[c] = (float)dgam;
    if (dbias) dbias[c] = (float)sg;
    const double m = (double)g.rows;
    const double k1 = (w ? (double)w[c] : 1.0) * is;
    const double A = -k1 * is * dgam / m, B = -k1 * sg / m;
    coef[3 * c] = (float)A;
    coef[3 * c + 1] = (float)B;
    coef[3 * c + 2] = (float)(B - A * (double)mean[c]);
}

template <int TPC>
__global__ void __launch_bounds__(kBnThreads) k_bn_bwd_finalize(
        const float2* __restrict__ part, BnGeom g, const float* __restrict__ w, const float* __restrict__ mean,
        const float* __restrict__ invstd, float* __restrict__ dweight, float* __restrict__ dbias,
        float* __restrict__ coef) {
    const int64_t c = (int64_t)blockIdx.x * (kBnThreads / TPC) + threadIdx.x / TPC;
    cudaGridDependencySynchronize();  // PDL: partials come from the backward reduce kernel
    double sg, sgx;
    if (group_merge<TPC>(part + c * g.P, g.P, c < g.C, sg, sgx))
        bn_bwd_write(g, w, mean, invstd, dweight, dbias, coef, c, sg, sgx);
}

template <typename T, int V, bool RELU, bool RES>
__device__ __forceinline__ void bn_apply_body(const T* __restrict__ x, const T* __restrict__ res,
                                                         T* __restrict__ y, const float* __restrict__ coef, BnGeom g, int bx, int by){
    const int tid = threadIdx.x;
    const int lane = tid % g.gv, rph = tid / g.gv;
    const int64_t c0 = ((int64_t)by * g.gv + lane) * V;
    if (rph >= g.rp || c0 >= g.C) return;
    float sc[V], mu[V], be[V];
#pragma unroll
    for (int i = 0; i < V; ++i) {
        sc[i] = coef[3 * (c0 + i)];
        mu[i] = coef[3 * (c0 + i) + 1];
        be[i] = coef[3 * (c0 + i) + 2];
    }
    const int64_t r0 = (int64_t)bx * g.chunk;
    const int64_t r1 = min(g.rows, r0 + g.chunk);
    constexpr int U = 4;
    int64_t r = r0 + rph;
    for (; r + (U - 1) * g.rp < r1; r += U * g.rp) {
        float xv[U][V], rv[U][V];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t o = (r + u * g.rp) * g.C + c0;
            BnIO<T, V>::load(x + o, xv[u]);
            if (RES) BnIO<T, V>::load(res + o, rv[u]);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
#pragma unroll
            for (int i = 0; i < V; ++i) {
                float z = bn_z(xv[u][i], sc[i], mu[i], be[i]) + (RES ? rv[u][i] : 0.f);
                xv[u][i] = RELU ? relu_nan(z) : z;
            }
            BnIO<T, V>::store(y + (r + u * g.rp) * g.C + c0, xv[u]);
        }
    }
    for (; r < r1; r += g.rp) {
        float xv[V], rv[V];
        const int64_t o = r * g.C + c0;
        BnIO<T, V>::load(x + o, xv);
        if (RES) BnIO<T, V>::load(res + o, rv);
#pragma unroll
        for (int i = 0; i < V; ++i) {
            float z = bn_z(xv[i], sc[i], mu[i], be[i]) + (RES ? rv[i] : 0.f);
            xv[i] = RELU ? relu_nan(z) : z;
        }
        BnIO<T, V>::store(y + o, xv);
    }
}

template <typename T, int V, bool RELU, bool RES>
__global__ void __launch_bounds__(kBnThreads) k_bn_apply(const T* __restrict__ x, const T* __restrict__ res,
                                                         T* __restrict__ y, const float* __restrict__ coef, BnGeom g) {
    cudaGridDependencySynchronize();  // PDL: inputs come from the preceding kernel
    bn_apply_body<T, V, RELU, RES>(x, res, y, coef, g, blockIdx.x, blockIdx.y);
}

// dx = k1*g + A*(x-mean) + B, g = dy * mask; with a residual, dres = g. k1 = gamma*invstd is
// bit-identical to the forward scale (a float product; the fp64 product of two floats rounds to
// the same value). bf16 activations use the folded dx = k1*g + (A*x + (B - A*mean)): the fp32
// rounding of A*x (~6e-8 |A*mean|) is far below the bf16 output ulp, and it frees V registers.
template <typename T, int V, bool RELU, bool RES>
__device__ __forceinline__ void bn_elemt_body(const T* __restrict__ x, const T* __restrict__ dy,
                                                             const T* __restrict__ res, T* __restrict__ dx,
                                                             T* __restrict__ dres, const float* __restrict__ w,
                                                             const float* __restrict__ b,
                                                             const float* __restrict__ mean,
                                                             const float* __restrict__ invstd,
                                                             const float* __restrict__ coef, BnGeom g, int bx, int by){
    constexpr bool kFold = sizeof(T) == 2;
    const int tid = threadIdx.x;
    const int lane = tid % g.gv, rph = tid / g.gv;
    const int64_t c0 = ((int64_t)by * g.gv + lane) * V;
    if (rph >= g.rp || c0 >= g.C) return;
    float A[V], B[V], mu[V], sc[V], sh[V];
#pragma unroll
    for (int i = 0; i < V; ++i) {
        A[i] = coef[3 * (c0 + i)];
        B[i] = coef[3 * (c0 + i) + (kFold ? 2 : 1)];
        bn_affine(w, b, mean, invstd, c0 + i, sc[i], mu[i], sh[i]);
    }
    const int64_t r0 = (int64_t)bx * g.chunk;
    const int64_t r1 = min(g.rows, r0 + g.chunk);
    constexpr int U = 2;
    int64_t r = r0 + rph;
    auto body = [&](float (&xv)[V], float (&dv)[V], float (&rv)[V], int64_t o) {
        if (RELU) {
#pragma unroll
            for (int i = 0; i < V; ++i) dv[i] = relu_mask<T, V, RES>(xv[i], sc[i], mu[i], sh[i], rv[i], dv[i]);
        }
        if (RES) BnIO<T, V>::store(dres + o, dv);
#pragma unroll
        for (int i = 0; i < V; ++i) xv[i] = fmaf(sc[i], dv[i], fmaf(A[i], kFold ? xv[i] : xv[i] - mu[i], B[i]));
        BnIO<T, V>::store(dx + o, xv);
    };
    for (; r + (U - 1) * g.rp < r1; r += U * g.rp) {
        float xv[U][V], dv[U][V], rv[U][V];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t o = (r + u * g.rp) * g.C + c0;
            BnIO<T, V>::load(x + o, xv[u]);
            BnIO<T, V>::load(dy + o, dv[u]);
            if (RELU && RES) BnIO<T, V>::load(res + o, rv[u]);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) body(xv[u], dv[u], rv[u], (r + u * g.rp) * g.C + c0);
    }
    for (; r < r1; r += g.rp) {
        float xv[V], dv[V], rv[V];
        const int64_t o = r * g.C + c0;
        BnIO<T, V>::load(x + o, xv);
        BnIO<T, V>::load(dy + o, dv);
        if (RELU && RES) BnIO<T, V>::load(res + o, rv);
        body(xv, dv, rv, o);
    }
}

template <typename T, int V, bool RELU, bool RES>
__global__ void __launch_bounds__(kBnThreads) k_bn_bwd_elemt(const T* __restrict__ x, const T* __restrict__ dy,
                                                             const T* __restrict__ res, T* __restrict__ dx,
                                                             T* __restrict__ dres, const float* __restrict__ w,
                                                             const float* __restrict__ b,
                                                             const float* __restrict__ mean,
                                                             const float* __restrict__ invstd,
                                                             const float* __restrict__ coef, BnGeom g) {
    cudaGridDependencySynchronize();  // PDL: inputs come from the preceding kernel
    bn_elemt_body<T, V, RELU, RES>(x, dy, res, dx, dres, w, b, mean, invstd, coef, g, blockIdx.x, blockIdx.y);
}

// ---------------------------------------------------------------------------------------------
// Cooperative single-kernel path for the smallest BatchNorm layers: reduce -> grid barrier ->
// per-channel finalize (a warp per channel, grid-strided) -> grid barrier -> apply / elemt over the
// CTA's own rows, which it read moments ago (L2 hits). Removes two kernel boundaries and the
// separate finalize launch per direction. Measured (profiles/r01_k5_fused_ab.txt, ResNet-50 step):
// with PDL already hiding most launch gaps, limits of 0 / 8 / 16 MB are within 0.4 % of each other
// and 32 / 64 MB are slower (the grid barriers and the register-path apply cost more than the
// saved launches on mid-size layers), so it is off by default (MBS_K5_FUSED_MB enables it; the parity test forces it). Same arithmetic as the
// three-kernel path; the partial grouping (grid size) may differ, so agreement is to fp32 noise.
// ---------------------------------------------------------------------------------------------
template <typename T, int V, bool RELU, bool RES>
__global__ void __launch_bounds__(kBnThreads) k_bn_fused_fwd(
        const T* __restrict__ x, const T* __restrict__ res, T* __restrict__ y, const float* __restrict__ w,
        const float* __restrict__ b, float* running_mean, float* running_var, double momentum, double eps,
        float* __restrict__ save_mean, float* __restrict__ save_invstd, float* __restrict__ coef,
        float2* __restrict__ part, BnGeom g) {
    cg::grid_group grid = cg::this_grid();
    cudaGridDependencySynchronize();
    if (g.nbt && blockIdx.x == 0 && threadIdx.x == 0) *g.nbt += 1;
    bn_reduce_body<T, V, 0, false, false>(x, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, part, g,
                                          blockIdx.x, 0);
    grid.sync();
    const int warp = threadIdx.x / 32, wpb = kBnThreads / 32;
    for (int64_t c = (int64_t)blockIdx.x * wpb + warp; c < g.C; c += (int64_t)gridDim.x * wpb) {
        double s1, s2;
        if (group_merge<32>(part + c * g.P, g.P, true, s1, s2))
            bn_stats_write(x, g, w, b, running_mean, running_var, momentum, eps, save_mean, save_invstd, coef, c, s1,
                           s2);
    }
    grid.sync();
    bn_apply_body<T, V, RELU, RES>(x, res, y, coef, g, blockIdx.x, 0);
}

template <typename T, int V, bool RELU, bool RES>
__global__ void __launch_bounds__(kBnThreads) k_bn_fused_bwd(
        const T* __restrict__ x, const T* __restrict__ dy, const T* __restrict__ res, T* __restrict__ dx,
        T* __restrict__ dres, const float* __restrict__ w, const float* __restrict__ b, const float* __restrict__ mean,
        const float* __restrict__ invstd, float* __restrict__ dweight, float* __restrict__ dbias,
        float* __restrict__ coef, float2* __restrict__ part, BnGeom g) {
    cg::grid_group grid = cg::this_grid();
    cudaGridDependencySynchronize();
    bn_reduce_body<T, V, 1, RELU, RES>(x, dy, res, w, b, mean, invstd, part, g, blockIdx.x, 0);
    grid.sync();
    const int warp = threadIdx.x / 32, wpb = kBnThreads / 32;
    for (int64_t c = (int64_t)blockIdx.x * wpb + warp; c < g.C; c += (int64_t)gridDim.x * wpb) {
        double sg, sgx;
        if (group_merge<32>(part + c * g.P, g.P, true, sg, sgx))
            bn_bwd_write(g, w, mean, invstd, dweight, dbias, coef, c, sg, sgx);
    }
    grid.sync();
    bn_elemt_body<T, V, RELU, RES>(x, dy, res, dx, dres, w, b, mean, invstd, coef, g, blockIdx.x, 0);
}

// ---------------------------------------------------------------------------------------------
// Bulk-async (TMA) streaming path — used whenever one CTA covers every channel (C <= 256 vectors)
// and the tensors are 16-byte aligned, i.e. for every BatchNorm of the benchmark models.
//
// A CTA owns a contiguous run of rows, which in NHWC is one contiguous byte range per tensor.
// One elected thread keeps kTmaStages tiles (tile_rows rows of every input tensor) in flight
// with cp.async.bulk into a smem ring, completion counted in bytes on the stage's mbarrier; the
// 256 threads consume a landed stage (thread = channel vector x row phase, 16-byte conflict-free
// smem reads), then the stage is refilled. So memory-level parallelism comes from the copy engine
// (up to 4 x 24 KB per CTA, 2 CTAs per SM), not from per-thread registers. Outputs leave with
// coalesced 16-byte stores. KIND: 0 statistics, 1 backward reduce, 2 apply, 3 backward elemt.
// ---------------------------------------------------------------------------------------------
constexpr int kTmaStages = 4;        // ring depth (A/B on B200: deeper rings of 6-12 stages were slower)
constexpr int kTmaTileBytes = 8192;  // per input tensor per stage
constexpr int kMaxTmaCtas = 4 * 148; // bounds the TMA path's partials (workspace)

template <int KIND, bool RES, bool DY2 = false>
__host__ __device__ constexpr int tma_inputs() {
    return 1 + ((KIND == 1 || KIND == 3) ? 1 : 0) + (RES ? 1 : 0) + (DY2 ? 1 : 0);
}

// four input tensors: 3 stages, so two CTAs (2 x 96 KB) still fit on an SM
__host__ __device__ constexpr int tma_stages(int nin) { return nin >= 4 ? 3 : kTmaStages; }


// DY2 (KIND 1 only): the output gradient arrives as two tensors (the residual block's two consumers,
// bn.py dual outputs) and is summed in fp32 on the fly — autograd's separate add pass disappears.
template <typename T, int V, int KIND, bool RELU, bool RES, bool DY2 = false>
__global__ void __launch_bounds__(kBnThreads, 2) k_bn_tma(
        const T* __restrict__ x, const T* __restrict__ dy, const T* __restrict__ res, T* __restrict__ out,
        T* __restrict__ dres, const float* __restrict__ w, const float* __restrict__ b,
        const float* __restrict__ mean, const float* __restrict__ invstd, const float* __restrict__ coef,
        float2* __restrict__ part, BnGeom g, int tile_rows, const T* __restrict__ dy2) {
    static_assert(!DY2 || KIND == 1, "a second output gradient is only read by the backward reduce");
    constexpr int NIN = tma_inputs<KIND, RES, DY2>();
    constexpr int STG = tma_stages(NIN);
    constexpr bool kFold = sizeof(T) == 2;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t full[STG];
    const int tid = threadIdx.x;
    const int lane = tid % g.gv, rph = tid / g.gv;
    const int64_t c0 = (int64_t)lane * V;
    const bool active = rph < g.rp;
    const int64_t r0 = (int64_t)blockIdx.x * g.chunk;
    const int64_t r1 = min(g.rows, r0 + g.chunk);
    const int n_tiles = (int)((r1 - r0 + tile_rows - 1) / tile_rows);

    cudaGridDependencySynchronize();  // PDL: inputs / coefficients come from the preceding kernel

    auto issue = [&](int i) {
        const int64_t rs = r0 + (int64_t)i * tile_rows;
        const uint32_t bytes = (uint32_t)(min((int64_t)tile_rows, r1 - rs) * g.C * (int64_t)sizeof(T));
        const int st = i % STG;
        unsigned char* slot = smem + (size_t)st * NIN * kTmaTileBytes;
        mbar_expect_tx(&full[st], bytes * NIN);
        bulk_load(slot, x + rs * g.C, bytes, &full[st]);
        int k = 1;
        if (KIND == 1 || KIND == 3) bulk_load(slot + (k++) * kTmaTileBytes, dy + rs * g.C, bytes, &full[st]);
        if (DY2) bulk_load(slot + (k++) * kTmaTileBytes, dy2 + rs * g.C, bytes, &full[st]);
        if (RES) bulk_load(slot + k * kTmaTileBytes, res + rs * g.C, bytes, &full[st]);
    };
    if (tid == 0) {
        for (int st = 0; st < STG; ++st) mbar_init(&full[st], 1);
        mbar_init_fence();
        for (int i = 0; i < min(STG, n_tiles); ++i) issue(i);
    }

    // per-channel state in registers
    float s1[V], s2[V], kk[V], sc[V], sh[V], A[V], B[V];
#pragma unroll
    for (int i = 0; i < V; ++i) {
        s1[i] = s2[i] = kk[i] = sc[i] = sh[i] = A[i] = B[i] = 0.f;
    }
    if (active) {
        if (KIND == 0) BnIO<T, V>::load(x + c0, kk);  // shift K = x[0, c]
#pragma unroll
        for (int i = 0; i < V; ++i) {
            // KIND 1 / 3: kk = the channel mean (centring for the reduce / dx, and the ReLU mask's mu)
            if (KIND == 1 || KIND == 3) bn_affine(w, b, mean, invstd, c0 + i, sc[i], kk[i], sh[i]);
            if (KIND == 2) {
                sc[i] = coef[3 * (c0 + i)];
                kk[i] = coef[3 * (c0 + i) + 1];
                sh[i] = coef[3 * (c0 + i) + 2];
            }
            if (KIND == 3) {
                A[i] = coef[3 * (c0 + i)];
                B[i] = coef[3 * (c0 + i) + (kFold ? 2 : 1)];
            }
        }
    }
    __syncthreads();  // barriers initialised

    for (int i = 0; i < n_tiles; ++i) {
        const int st = i % STG;
        const int64_t rs = r0 + (int64_t)i * tile_rows;
        const int nr = (int)min((int64_t)tile_rows, r1 - rs);
        mbar_wait(&full[st], (uint32_t)((i / STG) & 1));
        const T* xs = reinterpret_cast<const T*>(smem + (size_t)st * NIN * kTmaTileBytes);
        const T* ds = reinterpret_cast<const T*>(smem + ((size_t)st * NIN + 1) * kTmaTileBytes);
        const T* rsm = reinterpret_cast<const T*>(smem + ((size_t)st * NIN + NIN - 1) * kTmaTileBytes);
        if (active) {
#pragma unroll 2
            for (int j = rph; j < nr; j += g.rp) {
                const int64_t o = (int64_t)j * g.C + c0;
                float xv[V], dv[V], rv[V];
                BnIO<T, V>::load(xs + o, xv);
                if (KIND == 1 || KIND == 3) BnIO<T, V>::load(ds + o, dv);
                if (DY2) {
                    float d2[V];
                    BnIO<T, V>::load(ds + (size_t)kTmaTileBytes / sizeof(T) + o, d2);
#pragma unroll
                    for (int e = 0; e < V; ++e) {
                        dv[e] += d2[e];
                        // bf16: the sum is rounded like torch's bf16 add, so the statistics and the stored
                        // d_residual (read back by the elemt pass) see the same g
                        if constexpr (sizeof(T) == 2) dv[e] = __bfloat162float(__float2bfloat16(dv[e]));
                    }
                }
                if (RES) BnIO<T, V>::load(rsm + o, rv);
                if ((KIND == 1 || KIND == 3) && RELU) {
#pragma unroll
                    for (int e = 0; e < V; ++e) dv[e] = relu_mask<T, V, RES>(xv[e], sc[e], kk[e], sh[e], rv[e], dv[e]);
                }
                if (KIND == 0) {
#pragma unroll
                    for (int e = 0; e < V; ++e) {
                        const float d = xv[e] - kk[e];
                        s1[e] += d;
                        s2[e] = fmaf(d, d, s2[e]);
                    }
                } else if (KIND == 1) {
#pragma unroll
                    for (int e = 0; e < V; ++e) {
                        s1[e] += dv[e];
                        s2[e] = fmaf(dv[e], xv[e] - kk[e], s2[e]);
                    }
                    // residual layers: the masked gradient g IS d_residual — written here, so the elemt pass
                    // reads (x, g) instead of (x, dy, residual): 7 instead of 8 passes over the tensor
                    if (RES) BnIO<T, V>::store(dres + (rs + j) * g.C + c0, dv);
                } else if (KIND == 2) {
#pragma unroll
                    for (int e = 0; e < V; ++e) {
                        const float z = bn_z(xv[e], sc[e], kk[e], sh[e]) + (RES ? rv[e] : 0.f);
                        xv[e] = RELU ? relu_nan(z) : z;
                    }
                    BnIO<T, V>::store(out + (rs + j) * g.C + c0, xv);
                } else {
                    if (RES) BnIO<T, V>::store(dres + (rs + j) * g.C + c0, dv);
#pragma unroll
                    for (int e = 0; e < V; ++e)
                        xv[e] = fmaf(sc[e], dv[e], fmaf(A[e], kFold ? xv[e] : xv[e] - kk[e], B[e]));
                    BnIO<T, V>::store(out + (rs + j) * g.C + c0, xv);
                }
            }
        }
        __syncthreads();  // stage st consumed by every thread
        if (tid == 0 && i + STG < n_tiles) issue(i + STG);
    }

    if (KIND == 0 || KIND == 1) {
        // CTA reduction over the row phases (fixed order) into this CTA's partial; the ring is free now
        float* red0 = reinterpret_cast<float*>(smem);
        float* red1 = red0 + kBnThreads * V;
#pragma unroll
        for (int e = 0; e < V; ++e) {
            red0[e * kBnThreads + tid] = s1[e];
            red1[e * kBnThreads + tid] = s2[e];
        }
        __syncthreads();
        const int gc = g.gv * V;
        for (int j = tid; j < gc; j += kBnThreads) {
            const int ln = j / V, e = j % V;
            float a = 0.f, q = 0.f;
            for (int p = 0; p < g.rp; ++p) {
                a += red0[e * kBnThreads + p * g.gv + ln];
                q += red1[e * kBnThreads + p * g.gv + ln];
            }
            part[(int64_t)j * g.P + blockIdx.x] = make_float2(a, q);
        }
    }
}

constexpr int kMaxReduceCtas = 2048;  // bounds the partials (workspace) per BatchNorm call

static BnGeom bn_geom(int64_t rows, int64_t C, int V, int64_t min_rows_per_thread, int target_ctas,
                      int max_gv = kBnThreads) {
    BnGeom g;
    g.rows = rows;
    g.C = C;
    const int64_t cv = C / V;
    g.gv = (int)std::min<int64_t>(cv, max_gv);
    g.rp = kBnThreads / g.gv;
    const int64_t groups = (cv + g.gv - 1) / g.gv;
    const int64_t per_group = std::max<int64_t>(1, target_ctas / groups);
    const int64_t min_chunk = (int64_t)g.rp * min_rows_per_thread;
    int64_t P = std::min<int64_t>((rows + min_chunk - 1) / min_chunk, per_group);
    P = std::max<int64_t>(P, 1);
    g.chunk = (rows + P - 1) / P;
    g.P = (int)((rows + g.chunk - 1) / g.chunk);
    return g;
}

static int bn_vec(int dtype, int64_t C, const void* const* ptrs, int n) {
    const int V = dtype == MBS_BF16 ? 8 : 4;
    if (C % V) return 1;
    for (int i = 0; i < n; ++i)
        if (ptrs[i] && (reinterpret_cast<uintptr_t>(ptrs[i]) & 15)) return 1;
    return V;
}

static int stats_max_gv() {  // A/B: MBS_K5_STATS_GV
    const char* e = getenv("MBS_K5_STATS_GV");
    return e ? std::max(1, atoi(e)) : 32;
}

static int64_t bn_groups(const BnGeom& g, int V) { return (g.C / V + g.gv - 1) / g.gv; }

static int sm_count() {
    static int n = 0;
    if (n <= 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    }
    return n;
}

// One full wave of the kernel: resident CTAs per SM (registers / smem limited) x SMs.
template <typename K>
static int wave_ctas(K kernel) {
    static std::mutex mu;
    static std::map<const void*, int> cache;
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find((const void*)kernel);
    if (it != cache.end()) return it->second;
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kBnThreads, 0) != cudaSuccess || per_sm < 1)
        per_sm = 1;
    const int n = per_sm * sm_count();
    cache[(const void*)kernel] = n;
    return n;
}

// Every K5 kernel is launched with programmatic stream serialization (PDL): its launch and
// prologue overlap the previous kernel's tail; griddepcontrol.wait (cudaGridDependencySynchronize)
// at the top of each kernel orders its reads after the producer's writes.
template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(kBnThreads);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

static int tpc_for(int P) {
    int t = 32;
    while (t < 256 && 2 * t < P) t *= 2;
    return t;
}

template <typename T, int V, int MODE, bool RELU, bool RES>
static cudaError_t launch_reduce(const T* X, const T* DY, const T* R, const float* w, const float* b,
                                 const float* mean, const float* invstd, float2* part, BnGeom& g, cudaStream_t s) {
    auto k = k_bn_reduce<T, V, MODE, RELU, RES>;
    // statistics: at most 32 channel vectors per CTA (A/B: profiles/r01_k5_stats_gv_ab.txt), so wide layers (C = 1024 / 2048 on few rows) are
    // split into channel groups instead of into hundreds of row chunks — their per-CTA partials
    // (8 B per channel) were ~25 % of the input bytes
    const bool biased_rv = g.biased_rv;      // the geometry is recomputed; the update convention is kept
    g = bn_geom(g.rows, g.C, V, MODE == 0 ? 16 : 32, std::min(wave_ctas(k), kMaxReduceCtas),
                MODE == 0 ? stats_max_gv() : kBnThreads);
    g.biased_rv = biased_rv;
    return launch_pdl(k, dim3(g.P, (unsigned)bn_groups(g, V)), s, X, DY, R, w, b, mean, invstd, part, g);
}

template <typename T, int TPC>
static cudaError_t launch_stats_finalize(const T* X, const float2* part, const BnGeom& g, const float* w,
                                         const float* b, float* rm, float* rv, double momentum, double eps,
                                         float* smean, float* sinv, float* coef, cudaStream_t s) {
    const unsigned grid = (unsigned)((g.C + kBnThreads / TPC - 1) / (kBnThreads / TPC));
    return launch_pdl(k_bn_stats_finalize<T, TPC>, dim3(grid), s, X, part, g, w, b, rm, rv, momentum, eps, smean,
                      sinv, coef);
}

template <int TPC>
static cudaError_t launch_bwd_finalize(const float2* part, const BnGeom& g, const float* w, const float* mean,
                                       const float* invstd, float* dw, float* db, float* coef, cudaStream_t s) {
    const unsigned grid = (unsigned)((g.C + kBnThreads / TPC - 1) / (kBnThreads / TPC));
    return launch_pdl(k_bn_bwd_finalize<TPC>, dim3(grid), s, part, g, w, mean, invstd, dw, db, coef);
}

template <typename T, int V, bool RELU, bool RES>
static cudaError_t launch_apply(const T* X, const T* R, T* Y, const float* coef, int64_t rows, int64_t C,
                                cudaStream_t s) {
    auto k = k_bn_apply<T, V, RELU, RES>;
    BnGeom g = bn_geom(rows, C, V, 4, wave_ctas(k));
    return launch_pdl(k, dim3(g.P, (unsigned)bn_groups(g, V)), s, X, R, Y, coef, g);
}

template <typename T, int V, bool RELU, bool RES>
static cudaError_t launch_elemt(const T* X, const T* DY, const T* R, T* DX, T* DR, const float* w, const float* b,
                                const float* mean, const float* invstd, const float* coef, int64_t rows, int64_t C,
                                cudaStream_t s) {
    auto k = k_bn_bwd_elemt<T, V, RELU, RES>;
    BnGeom g = bn_geom(rows, C, V, 4, wave_ctas(k));
    return launch_pdl(k, dim3(g.P, (unsigned)bn_groups(g, V)), s, X, DY, R, DX, DR, w, b, mean, invstd, coef, g);
}

static int tma_tile_rows(const BnGeom& g, int elem_bytes) {
    int64_t rows = kTmaTileBytes / (g.C * elem_bytes);
    rows = rows / g.rp * g.rp;
    return (int)std::max<int64_t>(rows, g.rp);
}

// Geometry of the TMA path: one channel group, CTAs = min(resident CTAs, tiles), each CTA a
// contiguous run of whole tiles.
template <typename T, int V, int KIND, bool RELU, bool RES, bool DY2 = false>
static cudaError_t launch_tma(const T* X, const T* DY, const T* R, T* OUT, T* DR, const float* w, const float* b,
                              const float* mean, const float* invstd, const float* coef, float2* part,
                              BnGeom& g, cudaStream_t s, const T* DY2p = nullptr) {
  if constexpr (V == 1) {
    return cudaErrorInvalidValue;  // never taken: tma_ok() requires 16-byte vectors
  } else {
    auto k = k_bn_tma<T, V, KIND, RELU, RES, DY2>;
    constexpr int NIN = tma_inputs<KIND, RES, DY2>();
    const size_t smem = (size_t)tma_stages(NIN) * NIN * kTmaTileBytes;
    static int per_sm = 0;  // one static per template instance
    if (per_sm == 0) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kBnThreads, smem) != cudaSuccess || per_sm < 1)
            per_sm = 1;
    }
    g = bn_geom(g.rows, g.C, V, 1, 1);  // gv / rp for one group
    const int tr = tma_tile_rows(g, (int)sizeof(T));
    const int64_t tiles = (g.rows + tr - 1) / tr;
    int64_t ctas = std::min<int64_t>(std::min(per_sm * sm_count(), kMaxTmaCtas), tiles);
    ctas = std::max<int64_t>(ctas, 1);
    const int64_t tiles_per_cta = (tiles + ctas - 1) / ctas;
    g.chunk = tiles_per_cta * tr;
    g.P = (int)((g.rows + g.chunk - 1) / g.chunk);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(g.P);
    cfg.blockDim = dim3(kBnThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k, X, DY, R, OUT, DR, w, b, mean, invstd, coef, part, g, tr, DY2p);
  }
}

static bool tma_ok(int64_t C, int V) { return V > 1 && C / V <= kBnThreads; }

constexpr int64_t kFusedMaxBytes = 0;  // off by default: A/B 0 / 8 / 16 MB within 0.4 %, larger limits slower

static int64_t fused_max_bytes() {  // A/B: MBS_K5_FUSED_MB overrides the size limit of the cooperative path
    const char* e = getenv("MBS_K5_FUSED_MB");
    return e ? (int64_t)atoll(e) << 20 : kFusedMaxBytes;
}

static int fused_mode() {  // A/B and tests: MBS_K5_FUSED=0 selects the three-kernel path
    const char* e = getenv("MBS_K5_FUSED");
    return e ? atoi(e) : 1;
}

// Cooperative launch (every CTA resident: grid <= occupancy x SMs), with PDL when the driver accepts
// the combination (checked once per kernel). coop_geometry() sizes the grid first (the geometry is
// a kernel argument), coop_launch() launches it.
struct CoopInfo {
    int resident;
    int pdl;
};
static std::mutex g_coop_mu;
static std::map<const void*, CoopInfo> g_coop;

template <typename K>
static CoopInfo coop_info(K kernel) {
    std::lock_guard<std::mutex> lock(g_coop_mu);
    auto it = g_coop.find((const void*)kernel);
    if (it == g_coop.end()) {
        int per_sm = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kBnThreads, 0) != cudaSuccess) per_sm = 0;
        it = g_coop.emplace((const void*)kernel, CoopInfo{per_sm * sm_count(), 1}).first;
    }
    return it->second;
}

template <typename K>
static bool coop_geometry(K kernel, BnGeom& g, int V) {
    const CoopInfo info = coop_info(kernel);
    if (info.resident < 1) return false;
    const bool biased_rv = g.biased_rv;      // the geometry is recomputed; the update convention is kept
    g = bn_geom(g.rows, g.C, V, 16, std::min(info.resident, kMaxReduceCtas));
    g.biased_rv = biased_rv;
    return true;
}

template <typename... KArgs, typename... Args>
static cudaError_t coop_launch(void (*kernel)(KArgs...), int grid, cudaStream_t s, Args... args) {
    const CoopInfo info = coop_info(kernel);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kBnThreads);
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = info.pdl ? 2 : 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
    if (e != cudaSuccess && info.pdl) {  // PDL + cooperative refused: remember, retry cooperative only
        cudaGetLastError();
        {
            std::lock_guard<std::mutex> lock(g_coop_mu);
            g_coop[(const void*)kernel].pdl = 0;
        }
        cfg.numAttrs = 1;
        e = cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
    }
    return e;
}

template <typename T, int V, bool RELU, bool RES>
static cudaError_t fused_fwd(const T* X, const T* R, T* Y, const float* w, const float* b, float* rm, float* rv,
                             double momentum, double eps, float* smean, float* sinv, float* coef, float2* part,
                             BnGeom g, cudaStream_t s, long long* nbt) {
    auto k = k_bn_fused_fwd<T, V, RELU, RES>;
    if (!coop_geometry(k, g, V)) return cudaErrorCooperativeLaunchTooLarge;
    g.nbt = nbt;
    return coop_launch(k, g.P, s, X, R, Y, w, b, rm, rv, momentum, eps, smean, sinv, coef, part, g);
}

template <typename T, int V, bool RELU, bool RES>
static cudaError_t fused_bwd(const T* X, const T* DY, const T* R, T* DX, T* DR, const float* w, const float* b,
                             const float* smean, const float* sinv, float* dw, float* db, float* coef, float2* part,
                             BnGeom g, cudaStream_t s) {
    auto k = k_bn_fused_bwd<T, V, RELU, RES>;
    if (!coop_geometry(k, g, V)) return cudaErrorCooperativeLaunchTooLarge;
    return coop_launch(k, g.P, s, X, DY, R, DX, DR, w, b, smean, sinv, dw, db, coef, part, g);
}

template <typename T, int V>
static int bn_forward_t(const void* x, const void* res, void* y, int64_t rows, int64_t C, const float* w,
                        const float* b, float* rm, float* rv, long long* nbt, double momentum, double eps, int relu,
                        float* smean, float* sinv, void* ws, cudaStream_t s, bool biased_rv) {
    const T* X = static_cast<const T*>(x);
    const T* R = static_cast<const T*>(res);
    T* Y = static_cast<T*>(y);
    float* coef = static_cast<float*>(ws);
    float2* part = reinterpret_cast<float2*>(coef + 3 * ((C + 3) / 4 * 4));
    BnGeom g;
    g.rows = rows;
    g.C = C;
    g.biased_rv = biased_rv;
    const bool tma = tma_ok(C, V);
    if (tma && fused_mode() && rows * C * (int64_t)sizeof(T) <= fused_max_bytes()) {
        cudaError_t e;
        if (relu && res)
            e = fused_fwd<T, V, true, true>(X, R, Y, w, b, rm, rv, momentum, eps, smean, sinv, coef, part, g, s,
                                        nbt);
        else if (relu)
            e = fused_fwd<T, V, true, false>(X, R, Y, w, b, rm, rv, momentum, eps, smean, sinv, coef, part, g, s,
                                        nbt);
        else
            e = fused_fwd<T, V, false, false>(X, R, Y, w, b, rm, rv, momentum, eps, smean, sinv, coef, part, g, s,
                                        nbt);
        MBS_CK(e);
        return MBS_OK;
    }
    // statistics: the register-pipelined kernel (ncu A/B on B200: 40 us vs 48 us through the bulk-async
    // ring for a 205 MB single read-only stream); apply / backward use the ring.
    MBS_CK((launch_reduce<T, V, 0, false, false>(X, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, part, g,
                                                  s)));
    const int tpc = tpc_for(g.P);
    g.nbt = nbt;
    cudaError_t e;
    if (tpc == 32) e = launch_stats_finalize<T, 32>(X, part, g, w, b, rm, rv, momentum, eps, smean, sinv, coef, s);
    else if (tpc == 64) e = launch_stats_finalize<T, 64>(X, part, g, w, b, rm, rv, momentum, eps, smean, sinv, coef, s);
    else if (tpc == 128) e = launch_stats_finalize<T, 128>(X, part, g, w, b, rm, rv, momentum, eps, smean, sinv, coef, s);
    else e = launch_stats_finalize<T, 256>(X, part, g, w, b, rm, rv, momentum, eps, smean, sinv, coef, s);
    MBS_CK(e);
    BnGeom ga = g;
    if (tma && relu && res)
        e = launch_tma<T, V, 2, true, true>(X, nullptr, R, Y, nullptr, w, b, smean, sinv, coef, nullptr, ga, s);
    else if (tma && relu)
        e = launch_tma<T, V, 2, true, false>(X, nullptr, R, Y, nullptr, w, b, smean, sinv, coef, nullptr, ga, s);
    else if (tma)
        e = launch_tma<T, V, 2, false, false>(X, nullptr, R, Y, nullptr, w, b, smean, sinv, coef, nullptr, ga, s);
    else if (relu && res) e = launch_apply<T, V, true, true>(X, R, Y, coef, rows, C, s);
    else if (relu) e = launch_apply<T, V, true, false>(X, R, Y, coef, rows, C, s);
    else e = launch_apply<T, V, false, false>(X, R, Y, coef, rows, C, s);
    MBS_CK(e);
    return MBS_OK;
}

template <typename T, int V>
static int bn_backward_t(const void* x, const void* res, const void* dy, const void* dy2, void* dx, void* dres,
                         int64_t rows, int64_t C,
                         const float* w, const float* b, const float* smean, const float* sinv, int relu, float* dw,
                         float* db, void* ws, cudaStream_t s) {
    const T* X = static_cast<const T*>(x);
    const T* R = static_cast<const T*>(res);
    const T* DY = static_cast<const T*>(dy);
    float* coef = static_cast<float*>(ws);
    float2* part = reinterpret_cast<float2*>(coef + 3 * ((C + 3) / 4 * 4));
    BnGeom g;
    g.rows = rows;
    g.C = C;
    cudaError_t e;
    const bool tma = tma_ok(C, V);
    T* DX = static_cast<T*>(dx);
    T* DR = static_cast<T*>(dres);
    if (!dy2 && tma && fused_mode() && rows * C * (int64_t)sizeof(T) * (2 + (res ? 1 : 0)) <= fused_max_bytes()) {
        if (relu && res)
            e = fused_bwd<T, V, true, true>(X, DY, R, DX, DR, w, b, smean, sinv, dw, db, coef, part, g, s);
        else if (relu)
            e = fused_bwd<T, V, true, false>(X, DY, R, DX, DR, w, b, smean, sinv, dw, db, coef, part, g, s);
        else
            e = fused_bwd<T, V, false, false>(X, DY, R, DX, DR, w, b, smean, sinv, dw, db, coef, part, g, s);
        MBS_CK(e);
        return MBS_OK;
    }
    if (dy2 && !(tma && relu && res)) return invalid("mbs_bn_backward: dy2 needs the fused residual TMA path");
    if (dy2)
        e = launch_tma<T, V, 1, true, true, true>(X, DY, R, nullptr, static_cast<T*>(dres), w, b, smean, sinv,
                                                  nullptr, part, g, s, static_cast<const T*>(dy2));
    else if (tma && relu && res)
        e = launch_tma<T, V, 1, true, true>(X, DY, R, nullptr, static_cast<T*>(dres), w, b, smean, sinv, nullptr,
                                            part, g, s);   // also writes g = d_residual
    else if (tma && relu)
        e = launch_tma<T, V, 1, true, false>(X, DY, R, nullptr, nullptr, w, b, smean, sinv, nullptr, part, g, s);
    else if (tma)
        e = launch_tma<T, V, 1, false, false>(X, DY, R, nullptr, nullptr, w, b, smean, sinv, nullptr, part, g, s);
    else if (relu && res) e = launch_reduce<T, V, 1, true, true>(X, DY, R, w, b, smean, sinv, part, g, s);
    else if (relu) e = launch_reduce<T, V, 1, true, false>(X, DY, R, w, b, smean, sinv, part, g, s);
    else e = launch_reduce<T, V, 1, false, false>(X, DY, R, w, b, smean, sinv, part, g, s);
    MBS_CK(e);
    const int tpc = tpc_for(g.P);
    if (tpc == 32) e = launch_bwd_finalize<32>(part, g, w, smean, sinv, dw, db, coef, s);
    else if (tpc == 64) e = launch_bwd_finalize<64>(part, g, w, smean, sinv, dw, db, coef, s);
    else if (tpc == 128) e = launch_bwd_finalize<128>(part, g, w, smean, sinv, dw, db, coef, s);
    else e = launch_bwd_finalize<256>(part, g, w, smean, sinv, dw, db, coef, s);
    MBS_CK(e);
    BnGeom ge = g;
    if (tma && relu && res)
        e = launch_tma<T, V, 3, false, false>(X, DR, nullptr, DX, nullptr, w, b, smean, sinv, coef, nullptr, ge,
                                              s);            // dx from (x, g): no mask, no residual read
    else if (tma && relu)
        e = launch_tma<T, V, 3, true, false>(X, DY, R, DX, DR, w, b, smean, sinv, coef, nullptr, ge, s);
    else if (tma)
        e = launch_tma<T, V, 3, false, false>(X, DY, R, DX, DR, w, b, smean, sinv, coef, nullptr, ge, s);
    else if (relu && res) e = launch_elemt<T, V, true, true>(X, DY, R, DX, DR, w, b, smean, sinv, coef, rows, C, s);
    else if (relu) e = launch_elemt<T, V, true, false>(X, DY, R, DX, DR, w, b, smean, sinv, coef, rows, C, s);
    else e = launch_elemt<T, V, false, false>(X, DY, R, DX, DR, w, b, smean, sinv, coef, rows, C, s);
    MBS_CK(e);
    return MBS_OK;
}

}  // namespace mbs

using namespace mbs;

extern "C" {

int mbs_bn_workspace_bytes(int64_t rows, int64_t C, int dtype, int64_t* bytes) {
    if (rows < 1 || C < 1 || !bytes) return invalid("mbs_bn_workspace_bytes: rows and C must be >= 1");
    if (dtype != MBS_BF16 && dtype != MBS_F32) return invalid("mbs_bn: dtype must be MBS_BF16 or MBS_F32");
    int64_t worst = 0;
    for (int V : {1, dtype == MBS_BF16 ? 8 : 4}) {
        if (C % V) continue;
        BnGeom g = bn_geom(rows, C, V, 16, kMaxReduceCtas);  // generic path (statistics: 16 rows/thread): P bound
        int64_t P = g.P;
        if (tma_ok(C, V)) {                                     // TMA path: min(resident CTAs, tiles)
            const int tr = tma_tile_rows(g, dtype == MBS_BF16 ? 2 : 4);
            P = std::max<int64_t>(P, std::min<int64_t>(kMaxTmaCtas, (rows + tr - 1) / tr));
        }
        worst = std::max<int64_t>(worst, P * C * 8);
    }
    *bytes = 3 * 4 * ((C + 3) / 4 * 4) + worst;
    return MBS_OK;
}

int mbs_bn_forward(const void* x, const void* residual, void* y, int dtype, int64_t rows, int64_t C,
                   const float* weight, const float* bias, float* running_mean, float* running_var,
                   int64_t* num_batches_tracked, double momentum, double eps, int relu, float* save_mean,
                   float* save_invstd, void* workspace, void* stream) {
    if (!x || !y || !save_mean || !save_invstd || !workspace) return invalid("mbs_bn_forward: null pointer");
    if (rows < 1 || C < 1) return invalid("mbs_bn_forward: rows and C must be >= 1");
    if (relu & ~(MBS_BN_RELU | MBS_BN_BIASED_RUNNING_VAR)) return invalid("mbs_bn_forward: unknown flag bits");
    const bool biased_rv = (relu & MBS_BN_BIASED_RUNNING_VAR) != 0;
    relu &= MBS_BN_RELU;
    if (!!running_mean != !!running_var) return invalid("mbs_bn_forward: running_mean/running_var must both be set");
    if (residual && !relu) return invalid("mbs_bn_forward: a residual is only fused together with the ReLU");
    if (!(eps > 0.0)) return invalid("mbs_bn_forward: eps must be > 0");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    long long* nbt = reinterpret_cast<long long*>(num_batches_tracked);
    const void* ptrs[3] = {x, residual, y};
    const int V = dtype == MBS_BF16 || dtype == MBS_F32 ? bn_vec(dtype, C, ptrs, 3) : 0;
    if (dtype == MBS_BF16)
        return V == 8 ? bn_forward_t<__nv_bfloat16, 8>(x, residual, y, rows, C, weight, bias, running_mean, running_var,
                                                       nbt, momentum, eps, relu, save_mean, save_invstd, workspace, s, biased_rv)
                      : bn_forward_t<__nv_bfloat16, 1>(x, residual, y, rows, C, weight, bias, running_mean, running_var,
                                                       nbt, momentum, eps, relu, save_mean, save_invstd, workspace, s, biased_rv);
    if (dtype == MBS_F32)
        return V == 4 ? bn_forward_t<float, 4>(x, residual, y, rows, C, weight, bias, running_mean, running_var,
                                               nbt, momentum, eps, relu, save_mean, save_invstd, workspace, s, biased_rv)
                      : bn_forward_t<float, 1>(x, residual, y, rows, C, weight, bias, running_mean, running_var,
                                               nbt, momentum, eps, relu, save_mean, save_invstd, workspace, s, biased_rv);
    return invalid("mbs_bn_forward: dtype must be MBS_BF16 or MBS_F32");
}

int mbs_bn_backward(const void* x, const void* residual, const void* dy, const void* dy2, void* dx, void* dresidual,
                    int dtype, int64_t rows, int64_t C, const float* weight, const float* bias,
                    const float* save_mean, const float* save_invstd, int relu, float* dweight, float* dbias,
                    void* workspace, void* stream) {
    if (!x || !dy || !dx || !save_mean || !save_invstd || !workspace) return invalid("mbs_bn_backward: null pointer");
    if (rows < 1 || C < 1) return invalid("mbs_bn_backward: rows and C must be >= 1");
    if (!!residual != !!dresidual) return invalid("mbs_bn_backward: residual and dresidual go together");
    if (residual && !relu) return invalid("mbs_bn_backward: a residual is only fused together with the ReLU");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const void* ptrs[6] = {x, residual, dy, dx, dresidual, dy2};
    const int V = dtype == MBS_BF16 || dtype == MBS_F32 ? bn_vec(dtype, C, ptrs, 6) : 0;
    if (dtype == MBS_BF16)
        return V == 8 ? bn_backward_t<__nv_bfloat16, 8>(x, residual, dy, dy2, dx, dresidual, rows, C, weight, bias,
                                                        save_mean, save_invstd, relu, dweight, dbias, workspace, s)
                      : bn_backward_t<__nv_bfloat16, 1>(x, residual, dy, dy2, dx, dresidual, rows, C, weight, bias,
                                                        save_mean, save_invstd, relu, dweight, dbias, workspace, s);
    if (dtype == MBS_F32)
        return V == 4 ? bn_backward_t<float, 4>(x, residual, dy, dy2, dx, dresidual, rows, C, weight, bias, save_mean,
                                                save_invstd, relu, dweight, dbias, workspace, s)
                      : bn_backward_t<float, 1>(x, residual, dy, dy2, dx, dresidual, rows, C, weight, bias, save_mean,
                                                save_invstd, relu, dweight, dbias, workspace, s);
    return invalid("mbs_bn_backward: dtype must be MBS_BF16 or MBS_F32");
}

}  // extern "C"
