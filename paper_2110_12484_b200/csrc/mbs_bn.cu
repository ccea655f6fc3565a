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
//   backward: reduce 2*E*s (x, dy; +E*s residual) + elemt 3*E*s (+2*E*s residual)
// Reductions: per-thread fp32 partial sums of (x - K) and (x - K)^2 with a
// per-channel shift K = x[0, c] (no catastrophic cancellation when |mean| >>
// std), per-CTA partials in a fixed order, then a warp per channel merges the
// CTA partials in fp64 in a fixed order — bit-reproducible, atomic-free.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "mbs_common.h"

namespace mbs {

constexpr int kBnThreads = 256;
constexpr int kBnTargetCtas = 4 * 148;

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
};

// Per-channel affine of the forward (shared by forward apply and the backward mask
// recomputation so both see bit-identical values): y = x*scale + shift.
__device__ __forceinline__ void bn_affine(const float* w, const float* b, const float* mean, const float* invstd,
                                          int64_t c, float& scale, float& shift) {
    const float g = w ? w[c] : 1.f;
    const float be = b ? b[c] : 0.f;
    scale = g * invstd[c];
    shift = fmaf(-mean[c], scale, be);
}

// torch's relu (clamp_min) propagates NaN; fmaxf would not
__device__ __forceinline__ float relu_nan(float z) { return z < 0.f ? 0.f : z; }

// threshold_backward on the stored output y = T(relu(z)): the gradient is zeroed where y <= 0
// (NaN passes, as in torch); y <= 0 is decided on z without a conversion (kMaskThreshold).
template <typename T, int V, bool RES>
__device__ __forceinline__ float relu_mask(float x, float sc, float sh, float r, float d) {
    const float z = fmaf(x, sc, sh) + (RES ? r : 0.f);
    return z <= BnIO<T, V>::kMaskThreshold ? 0.f : d;
}

// MODE 0: statistics — partial (sum(x-K), sum((x-K)^2)).
// MODE 1: backward reduce — partial (sum g, sum g*(x-mean)), g = dy * relu-mask.
template <typename T, int V, int MODE, bool RELU, bool RES>
__global__ void __launch_bounds__(kBnThreads) k_bn_reduce(const T* __restrict__ x, const T* __restrict__ dy,
                                                          const T* __restrict__ res, const float* __restrict__ w,
                                                          const float* __restrict__ b,
                                                          const float* __restrict__ mean,
                                                          const float* __restrict__ invstd, float2* __restrict__ part,
                                                          BnGeom g) {
    __shared__ float red[2][kBnThreads * V];
    const int tid = threadIdx.x;
    const int lane = tid % g.gv, rph = tid / g.gv;
    const int64_t c0 = ((int64_t)blockIdx.y * g.gv + lane) * V;
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
                k[i] = mean[c0 + i];
                if (RELU) bn_affine(w, b, mean, invstd, c0 + i, sc[i], sh[i]);
            }
        }
        const int64_t r0 = (int64_t)blockIdx.x * g.chunk;
        const int64_t r1 = min(g.rows, r0 + g.chunk);
        constexpr int U = 4;
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
                        dv[u][i] = relu_mask<T, V, RES>(xv[u][i], sc[i], sh[i], rv[u][i], dv[u][i]);
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
                for (int i = 0; i < V; ++i) dv[i] = relu_mask<T, V, RES>(xv[i], sc[i], sh[i], rv[i], dv[i]);
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
        const int64_t c = (int64_t)blockIdx.y * gc + j;
        if (c >= g.C) break;
        float a = 0.f, q = 0.f;
        for (int p = 0; p < g.rp; ++p) {
            a += red[0][p * gc + j];
            q += red[1][p * gc + j];
        }
        part[c * g.P + blockIdx.x] = make_float2(a, q);
    }
}

// One warp per channel: merge the P CTA partials in fp64 (lane l takes partials
// l, l+32, ... in order, then a fixed xor-tree) and derive the per-channel values.
__device__ __forceinline__ void warp_merge(const float2* part, int P, int lane, double& a, double& q) {
    a = 0.0;
    q = 0.0;
    for (int p = lane; p < P; p += 32) {
        const float2 v = part[p];
        a += (double)v.x;
        q += (double)v.y;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        q += __shfl_xor_sync(0xffffffffu, q, o);
    }
}

template <typename T>
__global__ void k_bn_stats_finalize(const T* __restrict__ x, const float2* __restrict__ part, BnGeom g,
                                    const float* __restrict__ w, const float* __restrict__ b, float* running_mean,
                                    float* running_var, double momentum, double eps, float* __restrict__ save_mean,
                                    float* __restrict__ save_invstd, float* __restrict__ coef) {
    const int64_t c = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    if (c >= g.C) return;
    double s1, s2;
    warp_merge(part + c * g.P, g.P, lane, s1, s2);
    if (lane == 0) {
        const double m = (double)g.rows;
        const double K = (double)static_cast<float>(x[c]);
        const double dm = s1 / m;
        const double var = fmax(s2 / m - dm * dm, 0.0);  // biased: normalisation uses it (nn.py:278)
        const double mean = K + dm;
        save_mean[c] = (float)mean;
        save_invstd[c] = (float)(1.0 / sqrt(var + eps));
        if (running_mean) {
            running_mean[c] = (float)((1.0 - momentum) * (double)running_mean[c] + momentum * mean);
            const double unbiased = g.rows > 1 ? var * m / (m - 1.0) : var;
            running_var[c] = (float)((1.0 - momentum) * (double)running_var[c] + momentum * unbiased);
        }
        float sc, sh;
        bn_affine(w, b, save_mean, save_invstd, c, sc, sh);
        coef[2 * c] = sc;
        coef[2 * c + 1] = sh;
    }
}

// backward finalize: dgamma = invstd * sum g(x-mean), dbeta = sum g; dx coefficients
// dx = k1*g + A*(x-mean) + B with k1 = gamma*invstd, A = -k1*invstd*dgamma/M, B = -k1*dbeta/M.
__global__ void k_bn_bwd_finalize(const float2* __restrict__ part, BnGeom g, const float* __restrict__ w,
                                  const float* __restrict__ b, const float* __restrict__ mean,
                                  const float* __restrict__ invstd, float* __restrict__ dweight,
                                  float* __restrict__ dbias, float* __restrict__ coef) {
    const int64_t c = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x % 32;
    if (c >= g.C) return;
    double sg, sgx;
    warp_merge(part + c * g.P, g.P, lane, sg, sgx);
    if (lane == 0) {
        const double is = (double)invstd[c];
        const double dgam = sgx * is;
        if (dweight) dweight[c] = (float)dgam;
        if (dbias) dbias[c] = (float)sg;
        const double m = (double)g.rows;
        const double k1 = (w ? (double)w[c] : 1.0) * is;
        coef[3 * c] = (float)k1;
        coef[3 * c + 1] = (float)(-k1 * is * dgam / m);
        coef[3 * c + 2] = (float)(-k1 * sg / m);
    }
}

template <typename T, int V, bool RELU, bool RES>
__global__ void __launch_bounds__(kBnThreads) k_bn_apply(const T* __restrict__ x, const T* __restrict__ res,
                                                         T* __restrict__ y, const float* __restrict__ coef, BnGeom g) {
    const int tid = threadIdx.x;
    const int lane = tid % g.gv, rph = tid / g.gv;
    const int64_t c0 = ((int64_t)blockIdx.y * g.gv + lane) * V;
    if (rph >= g.rp || c0 >= g.C) return;
    float sc[V], sh[V];
#pragma unroll
    for (int i = 0; i < V; ++i) {
        sc[i] = coef[2 * (c0 + i)];
        sh[i] = coef[2 * (c0 + i) + 1];
    }
    const int64_t r0 = (int64_t)blockIdx.x * g.chunk;
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
                float z = fmaf(xv[u][i], sc[i], sh[i]) + (RES ? rv[u][i] : 0.f);
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
            float z = fmaf(xv[i], sc[i], sh[i]) + (RES ? rv[i] : 0.f);
            xv[i] = RELU ? relu_nan(z) : z;
        }
        BnIO<T, V>::store(y + o, xv);
    }
}

// dx = k1*g + A*(x-mean) + B, g = dy * mask; with a residual, dres = g.
template <typename T, int V, bool RELU, bool RES>
__global__ void __launch_bounds__(kBnThreads) k_bn_bwd_elemt(const T* __restrict__ x, const T* __restrict__ dy,
                                                             const T* __restrict__ res, T* __restrict__ dx,
                                                             T* __restrict__ dres, const float* __restrict__ w,
                                                             const float* __restrict__ b,
                                                             const float* __restrict__ mean,
                                                             const float* __restrict__ invstd,
                                                             const float* __restrict__ coef, BnGeom g) {
    const int tid = threadIdx.x;
    const int lane = tid % g.gv, rph = tid / g.gv;
    const int64_t c0 = ((int64_t)blockIdx.y * g.gv + lane) * V;
    if (rph >= g.rp || c0 >= g.C) return;
    float k1[V], A[V], B[V], mu[V], sc[V], sh[V];
#pragma unroll
    for (int i = 0; i < V; ++i) {
        k1[i] = coef[3 * (c0 + i)];
        A[i] = coef[3 * (c0 + i) + 1];
        B[i] = coef[3 * (c0 + i) + 2];
        mu[i] = mean[c0 + i];
        sc[i] = 0.f;
        sh[i] = 0.f;
        if (RELU) bn_affine(w, b, mean, invstd, c0 + i, sc[i], sh[i]);
    }
    const int64_t r0 = (int64_t)blockIdx.x * g.chunk;
    const int64_t r1 = min(g.rows, r0 + g.chunk);
    constexpr int U = 2;
    int64_t r = r0 + rph;
    auto body = [&](float (&xv)[V], float (&dv)[V], float (&rv)[V], int64_t o) {
        if (RELU) {
#pragma unroll
            for (int i = 0; i < V; ++i) dv[i] = relu_mask<T, V, RES>(xv[i], sc[i], sh[i], rv[i], dv[i]);
        }
        if (RES) BnIO<T, V>::store(dres + o, dv);
#pragma unroll
        for (int i = 0; i < V; ++i) xv[i] = fmaf(k1[i], dv[i], fmaf(A[i], xv[i] - mu[i], B[i]));
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

static BnGeom bn_geom(int64_t rows, int64_t C, int V, int64_t min_rows_per_thread, int target_ctas) {
    BnGeom g;
    g.rows = rows;
    g.C = C;
    const int64_t cv = C / V;
    g.gv = (int)std::min<int64_t>(cv, kBnThreads);
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

static int64_t bn_groups(const BnGeom& g, int V) { return (g.C / V + g.gv - 1) / g.gv; }

template <typename T, int V>
static int bn_forward_t(const void* x, const void* res, void* y, int64_t rows, int64_t C, const float* w,
                        const float* b, float* rm, float* rv, double momentum, double eps, int relu, float* smean,
                        float* sinv, void* ws, cudaStream_t s) {
    const T* X = static_cast<const T*>(x);
    const T* R = static_cast<const T*>(res);
    T* Y = static_cast<T*>(y);
    BnGeom gr = bn_geom(rows, C, V, 32, kBnTargetCtas);
    float* coef = static_cast<float*>(ws);
    float2* part = reinterpret_cast<float2*>(coef + 2 * ((C + 3) / 4 * 4));
    dim3 grid(gr.P, (unsigned)bn_groups(gr, V));
    k_bn_reduce<T, V, 0, false, false><<<grid, kBnThreads, 0, s>>>(X, nullptr, nullptr, nullptr, nullptr, nullptr,
                                                                   nullptr, part, gr);
    MBS_CK_LAUNCH("k_bn_reduce(stats)");
    k_bn_stats_finalize<T><<<(unsigned)((C + 7) / 8), 256, 0, s>>>(X, part, gr, w, b, rm, rv, momentum, eps, smean,
                                                                   sinv, coef);
    MBS_CK_LAUNCH("k_bn_stats_finalize");
    BnGeom ga = bn_geom(rows, C, V, 8, 8 * 148);
    dim3 ga_grid(ga.P, (unsigned)bn_groups(ga, V));
    if (relu && res) k_bn_apply<T, V, true, true><<<ga_grid, kBnThreads, 0, s>>>(X, R, Y, coef, ga);
    else if (relu) k_bn_apply<T, V, true, false><<<ga_grid, kBnThreads, 0, s>>>(X, R, Y, coef, ga);
    else if (res) k_bn_apply<T, V, false, true><<<ga_grid, kBnThreads, 0, s>>>(X, R, Y, coef, ga);
    else k_bn_apply<T, V, false, false><<<ga_grid, kBnThreads, 0, s>>>(X, R, Y, coef, ga);
    MBS_CK_LAUNCH("k_bn_apply");
    return MBS_OK;
}

template <typename T, int V>
static int bn_backward_t(const void* x, const void* res, const void* dy, void* dx, void* dres, int64_t rows, int64_t C,
                         const float* w, const float* b, const float* smean, const float* sinv, int relu, float* dw,
                         float* db, void* ws, cudaStream_t s) {
    const T* X = static_cast<const T*>(x);
    const T* R = static_cast<const T*>(res);
    const T* DY = static_cast<const T*>(dy);
    BnGeom gr = bn_geom(rows, C, V, 32, kBnTargetCtas);
    float* coef = static_cast<float*>(ws);
    float2* part = reinterpret_cast<float2*>(coef + 3 * ((C + 3) / 4 * 4));
    dim3 grid(gr.P, (unsigned)bn_groups(gr, V));
    if (relu && res)
        k_bn_reduce<T, V, 1, true, true><<<grid, kBnThreads, 0, s>>>(X, DY, R, w, b, smean, sinv, part, gr);
    else if (relu)
        k_bn_reduce<T, V, 1, true, false><<<grid, kBnThreads, 0, s>>>(X, DY, R, w, b, smean, sinv, part, gr);
    else
        k_bn_reduce<T, V, 1, false, false><<<grid, kBnThreads, 0, s>>>(X, DY, R, w, b, smean, sinv, part, gr);
    MBS_CK_LAUNCH("k_bn_reduce(backward)");
    k_bn_bwd_finalize<<<(unsigned)((C + 7) / 8), 256, 0, s>>>(part, gr, w, b, smean, sinv, dw, db, coef);
    MBS_CK_LAUNCH("k_bn_bwd_finalize");
    BnGeom ge = bn_geom(rows, C, V, 8, 8 * 148);
    dim3 ge_grid(ge.P, (unsigned)bn_groups(ge, V));
    T* DX = static_cast<T*>(dx);
    T* DR = static_cast<T*>(dres);
    if (relu && res)
        k_bn_bwd_elemt<T, V, true, true><<<ge_grid, kBnThreads, 0, s>>>(X, DY, R, DX, DR, w, b, smean, sinv, coef, ge);
    else if (relu)
        k_bn_bwd_elemt<T, V, true, false><<<ge_grid, kBnThreads, 0, s>>>(X, DY, R, DX, DR, w, b, smean, sinv, coef,
                                                                         ge);
    else
        k_bn_bwd_elemt<T, V, false, false><<<ge_grid, kBnThreads, 0, s>>>(X, DY, R, DX, DR, w, b, smean, sinv, coef,
                                                                          ge);
    MBS_CK_LAUNCH("k_bn_bwd_elemt");
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
        BnGeom g = bn_geom(rows, C, V, 32, kBnTargetCtas);
        worst = std::max<int64_t>(worst, (int64_t)g.P * C * 8);
    }
    *bytes = 3 * 4 * ((C + 3) / 4 * 4) + worst;
    return MBS_OK;
}

int mbs_bn_forward(const void* x, const void* residual, void* y, int dtype, int64_t rows, int64_t C,
                   const float* weight, const float* bias, float* running_mean, float* running_var, double momentum,
                   double eps, int relu, float* save_mean, float* save_invstd, void* workspace, void* stream) {
    if (!x || !y || !save_mean || !save_invstd || !workspace) return invalid("mbs_bn_forward: null pointer");
    if (rows < 1 || C < 1) return invalid("mbs_bn_forward: rows and C must be >= 1");
    if (!!running_mean != !!running_var) return invalid("mbs_bn_forward: running_mean/running_var must both be set");
    if (residual && !relu) return invalid("mbs_bn_forward: a residual is only fused together with the ReLU");
    if (!(eps > 0.0)) return invalid("mbs_bn_forward: eps must be > 0");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const void* ptrs[3] = {x, residual, y};
    const int V = dtype == MBS_BF16 || dtype == MBS_F32 ? bn_vec(dtype, C, ptrs, 3) : 0;
    if (dtype == MBS_BF16)
        return V == 8 ? bn_forward_t<__nv_bfloat16, 8>(x, residual, y, rows, C, weight, bias, running_mean, running_var,
                                                       momentum, eps, relu, save_mean, save_invstd, workspace, s)
                      : bn_forward_t<__nv_bfloat16, 1>(x, residual, y, rows, C, weight, bias, running_mean, running_var,
                                                       momentum, eps, relu, save_mean, save_invstd, workspace, s);
    if (dtype == MBS_F32)
        return V == 4 ? bn_forward_t<float, 4>(x, residual, y, rows, C, weight, bias, running_mean, running_var,
                                               momentum, eps, relu, save_mean, save_invstd, workspace, s)
                      : bn_forward_t<float, 1>(x, residual, y, rows, C, weight, bias, running_mean, running_var,
                                               momentum, eps, relu, save_mean, save_invstd, workspace, s);
    return invalid("mbs_bn_forward: dtype must be MBS_BF16 or MBS_F32");
}

int mbs_bn_backward(const void* x, const void* residual, const void* dy, void* dx, void* dresidual, int dtype,
                    int64_t rows, int64_t C, const float* weight, const float* bias, const float* save_mean,
                    const float* save_invstd, int relu, float* dweight, float* dbias, void* workspace, void* stream) {
    if (!x || !dy || !dx || !save_mean || !save_invstd || !workspace) return invalid("mbs_bn_backward: null pointer");
    if (rows < 1 || C < 1) return invalid("mbs_bn_backward: rows and C must be >= 1");
    if (!!residual != !!dresidual) return invalid("mbs_bn_backward: residual and dresidual go together");
    if (residual && !relu) return invalid("mbs_bn_backward: a residual is only fused together with the ReLU");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const void* ptrs[5] = {x, residual, dy, dx, dresidual};
    const int V = dtype == MBS_BF16 || dtype == MBS_F32 ? bn_vec(dtype, C, ptrs, 5) : 0;
    if (dtype == MBS_BF16)
        return V == 8 ? bn_backward_t<__nv_bfloat16, 8>(x, residual, dy, dx, dresidual, rows, C, weight, bias,
                                                        save_mean, save_invstd, relu, dweight, dbias, workspace, s)
                      : bn_backward_t<__nv_bfloat16, 1>(x, residual, dy, dx, dresidual, rows, C, weight, bias,
                                                        save_mean, save_invstd, relu, dweight, dbias, workspace, s);
    if (dtype == MBS_F32)
        return V == 4 ? bn_backward_t<float, 4>(x, residual, dy, dx, dresidual, rows, C, weight, bias, save_mean,
                                                save_invstd, relu, dweight, dbias, workspace, s)
                      : bn_backward_t<float, 1>(x, residual, dy, dx, dresidual, rows, C, weight, bias, save_mean,
                                                save_invstd, relu, dweight, dbias, workspace, s);
    return invalid("mbs_bn_backward: dtype must be MBS_BF16 or MBS_F32");
}

}  // extern "C"
