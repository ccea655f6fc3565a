// K6: channels-last max-pool (the model's MaxPool2d of every micro-batch forward), forward with a
// one-byte window-relative argmax, backward as a deterministic gather.
//
// torch's NHWC max-pool kernels keep an int64 index per output element (8 B) and were 8.5 % of
// the ResNet-50 micro-batch step on B200 (profiles/r01_c2_v3_launches.md: 0.86 ms backward +
// 0.38 ms forward for the 128x64x112x112 stem). Semantics are torch's (max_pool_forward_nhwc /
// max_pool_backward_nhwc): windows scanned h-major then w, a value replaces the running max if
// it is larger or NaN (first maximum wins, NaN propagates), padding never wins; the backward of
// an input element sums, in ascending (oh, ow) order and in fp32, dy of every window whose argmax
// is that element — so forward AND backward are bit-identical to torch's.
//
// Layout: x [N, H, W, C] (channels-last), y / idx / dy [N, Ho, Wo, C]; one thread per 16-byte
// channel vector of one output (forward) or input (backward) pixel: a warp reads contiguous
// 16-byte vectors of neighbouring pixels, window re-reads hit L1/L2.
// Algorithmic bytes: forward read x + write y + idx (C*(s*H*W + (s+1)*Ho*Wo) with s = elem size);
// backward read dy + idx, write dx.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "mbs_common.h"

namespace mbs {

constexpr int kPoolThreads = 256;

template <typename T, int V> struct PoolIO;
template <> struct PoolIO<__nv_bfloat16, 8> {
    static __device__ __forceinline__ void load(const __nv_bfloat16* p, float (&f)[8]) {
        const uint4 v = *reinterpret_cast<const uint4*>(p);
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
};
template <> struct PoolIO<float, 4> {
    static __device__ __forceinline__ void load(const float* p, float (&f)[4]) {
        const float4 v = *reinterpret_cast<const float4*>(p);
        f[0] = v.x; f[1] = v.y; f[2] = v.z; f[3] = v.w;
    }
    static __device__ __forceinline__ void store(float* p, const float (&f)[4]) {
        *reinterpret_cast<float4*>(p) = make_float4(f[0], f[1], f[2], f[3]);
    }
};
template <typename T> struct PoolIO<T, 1> {
    static __device__ __forceinline__ void load(const T* p, float (&f)[1]) { f[0] = static_cast<float>(*p); }
    static __device__ __forceinline__ void store(T* p, const float (&f)[1]) { *p = static_cast<T>(f[0]); }
};

struct PoolGeom {
    int64_t N, H, W, C, Ho, Wo;
    int k, s, p;
};

template <int V>
__device__ __forceinline__ void store_idx(uint8_t* p, const uint8_t (&v)[V]) {
    if constexpr (V == 8) {
        uint2 u;
        u.x = v[0] | (v[1] << 8) | (v[2] << 16) | ((uint32_t)v[3] << 24);
        u.y = v[4] | (v[5] << 8) | (v[6] << 16) | ((uint32_t)v[7] << 24);
        *reinterpret_cast<uint2*>(p) = u;
    } else if constexpr (V == 4) {
        *reinterpret_cast<uint32_t*>(p) = v[0] | (v[1] << 8) | (v[2] << 16) | ((uint32_t)v[3] << 24);
    } else {
        *p = v[0];
    }
}

template <int V>
__device__ __forceinline__ void load_idx(const uint8_t* p, uint8_t (&v)[V]) {
    if constexpr (V == 8) {
        const uint2 u = *reinterpret_cast<const uint2*>(p);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            v[i] = (u.x >> (8 * i)) & 0xff;
            v[4 + i] = (u.y >> (8 * i)) & 0xff;
        }
    } else if constexpr (V == 4) {
        const uint32_t u = *reinterpret_cast<const uint32_t*>(p);
#pragma unroll
        for (int i = 0; i < 4; ++i) v[i] = (u >> (8 * i)) & 0xff;
    } else {
        v[0] = *p;
    }
}

// Optional side copy ("stash"): with non-overlapping windows covering the input (k == s, p == 0,
// k | H, k | W) every input element is read exactly once, so the kernel also writes it into channel
// columns [sc0, sc0 + C) of a wider channels-last tensor with row stride sC — the U-Net skip
// connection lands in its concat buffer without a separate torch.cat pass.
template <typename T, int V>
__global__ void __launch_bounds__(kPoolThreads) k_maxpool_fwd(const T* __restrict__ x, T* __restrict__ y,
                                                              uint8_t* __restrict__ idx, PoolGeom g,
                                                              T* __restrict__ stash, int64_t sC, int64_t sc0) {
    cudaGridDependencySynchronize();
    const int64_t cv = g.C / V;
    const int64_t total = g.N * g.Ho * g.Wo * cv;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c0 = (t % cv) * V;
        int64_t q = t / cv;
        const int64_t ow = q % g.Wo;
        q /= g.Wo;
        const int64_t oh = q % g.Ho;
        const int64_t n = q / g.Ho;
        const int64_t h0 = oh * g.s - g.p, w0 = ow * g.s - g.p;
        float m[V];
        uint8_t a[V];
#pragma unroll
        for (int i = 0; i < V; ++i) {
            m[i] = -INFINITY;
            a[i] = 0;
        }
        for (int kh = 0; kh < g.k; ++kh) {
            const int64_t ih = h0 + kh;
            if (ih < 0 || ih >= g.H) continue;
            for (int kw = 0; kw < g.k; ++kw) {
                const int64_t iw = w0 + kw;
                if (iw < 0 || iw >= g.W) continue;
                float v[V];
                const int64_t pix = (n * g.H + ih) * g.W + iw;
                PoolIO<T, V>::load(x + pix * g.C + c0, v);
                if (stash) PoolIO<T, V>::store(stash + pix * sC + sc0 + c0, v);
                const uint8_t pos = (uint8_t)(kh * g.k + kw);
#pragma unroll
                for (int i = 0; i < V; ++i) {
                    if (v[i] > m[i] || isnan(v[i])) {
                        m[i] = v[i];
                        a[i] = pos;
                    }
                }
            }
        }
        const int64_t o = ((n * g.Ho + oh) * g.Wo + ow) * g.C + c0;
        PoolIO<T, V>::store(y + o, m);
        store_idx<V>(idx + o, a);
    }
}

// Optional addend: dx += add[pixel, ac0 + c] (row stride aC) in fp32 before the single rounding —
// the gradient that reached the same tensor through the U-Net skip connection, fused instead of
// autograd's separate add pass.
template <typename T, int V>
__global__ void __launch_bounds__(kPoolThreads) k_maxpool_bwd(const T* __restrict__ dy,
                                                              const uint8_t* __restrict__ idx, T* __restrict__ dx,
                                                              PoolGeom g, const T* __restrict__ add, int64_t aC,
                                                              int64_t ac0) {
    cudaGridDependencySynchronize();
    const int64_t cv = g.C / V;
    const int64_t total = g.N * g.H * g.W * cv;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c0 = (t % cv) * V;
        int64_t q = t / cv;
        const int64_t iw = q % g.W;
        q /= g.W;
        const int64_t ih = q % g.H;
        const int64_t n = q / g.H;
        // windows containing (ih, iw): oh*s - p <= ih <= oh*s - p + k - 1
        const int64_t ohs = max((int64_t)0, (ih + g.p - g.k + g.s) / g.s);
        const int64_t ohe = min(g.Ho, (ih + g.p) / g.s + 1);
        const int64_t ows = max((int64_t)0, (iw + g.p - g.k + g.s) / g.s);
        const int64_t owe = min(g.Wo, (iw + g.p) / g.s + 1);
        float acc[V];
#pragma unroll
        for (int i = 0; i < V; ++i) acc[i] = 0.f;
        for (int64_t oh = ohs; oh < ohe; ++oh) {
            const int kh = (int)(ih - (oh * g.s - g.p));
            if (kh < 0 || kh >= g.k) continue;
            for (int64_t ow = ows; ow < owe; ++ow) {
                const int kw = (int)(iw - (ow * g.s - g.p));
                if (kw < 0 || kw >= g.k) continue;
                const uint8_t pos = (uint8_t)(kh * g.k + kw);
                const int64_t o = ((n * g.Ho + oh) * g.Wo + ow) * g.C + c0;
                uint8_t a[V];
                load_idx<V>(idx + o, a);
                bool any = false;
#pragma unroll
                for (int i = 0; i < V; ++i) any |= a[i] == pos;
                if (!any) continue;
                float d[V];
                PoolIO<T, V>::load(dy + o, d);
#pragma unroll
                for (int i = 0; i < V; ++i)
                    if (a[i] == pos) acc[i] += d[i];
            }
        }
        const int64_t pix = (n * g.H + ih) * g.W + iw;
        if (add) {
            float a2[V];
            PoolIO<T, V>::load(add + pix * aC + ac0 + c0, a2);
#pragma unroll
            for (int i = 0; i < V; ++i) acc[i] += a2[i];
        }
        PoolIO<T, V>::store(dx + pix * g.C + c0, acc);
    }
}

// Channel-slice copy between channels-last tensors viewed as [M, C_total] rows:
// dst[m, dc0 + c] = src[m, sc0 + c] (+ bias[c]) — the U-Net skip join (the upsampled half lands in
// the concat buffer with its ConvTranspose bias added on the way) and its backward (the slice made
// dense for the ConvTranspose backward). One thread per 16-byte vector; consecutive threads walk
// consecutive channels, then rows.
template <typename T, int V>
__global__ void __launch_bounds__(kPoolThreads) k_copy_channels(const T* __restrict__ src, int64_t sC, int64_t sc0,
                                                                T* __restrict__ dst, int64_t dC, int64_t dc0,
                                                                int64_t M, int64_t C, const float* __restrict__ bias) {
    cudaGridDependencySynchronize();
    const int64_t cv = C / V;
    const int64_t total = M * cv;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c0 = (t % cv) * V;
        const int64_t m = t / cv;
        float v[V];
        PoolIO<T, V>::load(src + m * sC + sc0 + c0, v);
        if (bias) {
#pragma unroll
            for (int i = 0; i < V; ++i) v[i] += bias[c0 + i];
        }
        PoolIO<T, V>::store(dst + m * dC + dc0 + c0, v);
    }
}

static int pool_sms() {
    static int n = 0;
    if (n <= 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    }
    return n;
}

template <typename... KArgs, typename... Args>
static cudaError_t pool_launch(void (*kernel)(KArgs...), int64_t work, cudaStream_t s, Args... args) {
    // grid-stride: at most 8 resident 256-thread CTAs per SM, fewer when the work is small
    const int64_t want = (work + kPoolThreads - 1) / kPoolThreads;
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(want, 8LL * pool_sms()));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(kPoolThreads);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

static int pool_check(int dtype, int64_t N, int64_t H, int64_t W, int64_t C, int k, int s, int p, PoolGeom* g) {
    if (dtype != MBS_BF16 && dtype != MBS_F32) return invalid("mbs_maxpool: dtype must be MBS_BF16 or MBS_F32");
    if (N < 1 || H < 1 || W < 1 || C < 1) return invalid("mbs_maxpool: N, H, W, C must be >= 1");
    if (k < 1 || s < 1 || p < 0 || 2 * p > k || k * k > 255)
        return invalid("mbs_maxpool: need k >= 1, s >= 1, 0 <= p <= k/2, k*k <= 255");
    const int64_t Ho = (H + 2 * p - k) / s + 1, Wo = (W + 2 * p - k) / s + 1;
    if (H + 2 * p < k || W + 2 * p < k || Ho < 1 || Wo < 1) return invalid("mbs_maxpool: window larger than input");
    *g = PoolGeom{N, H, W, C, Ho, Wo, k, s, p};
    return MBS_OK;
}

static bool aligned16(const void* a, const void* b, const void* c) {
    return !((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b) | reinterpret_cast<uintptr_t>(c)) & 15);
}

}  // namespace mbs

using namespace mbs;

extern "C" {

int mbs_maxpool_forward(const void* x, void* y, uint8_t* idx, int dtype, int64_t N, int64_t H, int64_t W, int64_t C,
                        int k, int s, int p, void* stash, int64_t stash_C, int64_t stash_c0, void* stream) {
    if (!x || !y || !idx) return invalid("mbs_maxpool_forward: null pointer");
    PoolGeom g;
    int st = pool_check(dtype, N, H, W, C, k, s, p, &g);
    if (st) return st;
    if (stash && !(k == s && p == 0 && H % k == 0 && W % k == 0))
        return invalid("mbs_maxpool_forward: a stash needs non-overlapping windows tiling the input (k == s, p == 0)");
    if (stash && (stash_c0 < 0 || stash_c0 + C > stash_C)) return invalid("mbs_maxpool_forward: stash columns");
    cudaStream_t cs = static_cast<cudaStream_t>(stream);
    const int64_t outs = g.N * g.Ho * g.Wo;
    const int es = dtype == MBS_BF16 ? 2 : 4;
    const bool stash_vec = !stash || (!(reinterpret_cast<uintptr_t>(stash) & 15) && (stash_C * es) % 16 == 0 &&
                                      (stash_c0 * es) % 16 == 0);
    cudaError_t e;
    if (dtype == MBS_BF16) {
        using T = __nv_bfloat16;
        if (C % 8 == 0 && aligned16(x, y, nullptr) && !(reinterpret_cast<uintptr_t>(idx) & 7) && stash_vec)
            e = pool_launch(k_maxpool_fwd<T, 8>, outs * (C / 8), cs, (const T*)x, (T*)y, idx, g, (T*)stash, stash_C,
                            stash_c0);
        else
            e = pool_launch(k_maxpool_fwd<T, 1>, outs * C, cs, (const T*)x, (T*)y, idx, g, (T*)stash, stash_C, stash_c0);
    } else {
        if (C % 4 == 0 && aligned16(x, y, nullptr) && !(reinterpret_cast<uintptr_t>(idx) & 3) && stash_vec)
            e = pool_launch(k_maxpool_fwd<float, 4>, outs * (C / 4), cs, (const float*)x, (float*)y, idx, g,
                            (float*)stash, stash_C, stash_c0);
        else
            e = pool_launch(k_maxpool_fwd<float, 1>, outs * C, cs, (const float*)x, (float*)y, idx, g, (float*)stash,
                            stash_C, stash_c0);
    }
    MBS_CK(e);
    return MBS_OK;
}

int mbs_maxpool_backward(const void* dy, const uint8_t* idx, void* dx, int dtype, int64_t N, int64_t H, int64_t W,
                         int64_t C, int k, int s, int p, const void* addend, int64_t add_C, int64_t add_c0,
                         void* stream) {
    if (!dy || !idx || !dx) return invalid("mbs_maxpool_backward: null pointer");
    PoolGeom g;
    int st = pool_check(dtype, N, H, W, C, k, s, p, &g);
    if (st) return st;
    if (addend && (add_c0 < 0 || add_c0 + C > add_C)) return invalid("mbs_maxpool_backward: addend columns");
    cudaStream_t cs = static_cast<cudaStream_t>(stream);
    const int64_t ins = g.N * g.H * g.W;
    const int es = dtype == MBS_BF16 ? 2 : 4;
    const bool add_vec = !addend || (!(reinterpret_cast<uintptr_t>(addend) & 15) && (add_C * es) % 16 == 0 &&
                                     (add_c0 * es) % 16 == 0);
    cudaError_t e;
    if (dtype == MBS_BF16) {
        using T = __nv_bfloat16;
        if (C % 8 == 0 && aligned16(dy, dx, nullptr) && !(reinterpret_cast<uintptr_t>(idx) & 7) && add_vec)
            e = pool_launch(k_maxpool_bwd<T, 8>, ins * (C / 8), cs, (const T*)dy, idx, (T*)dx, g, (const T*)addend,
                            add_C, add_c0);
        else
            e = pool_launch(k_maxpool_bwd<T, 1>, ins * C, cs, (const T*)dy, idx, (T*)dx, g, (const T*)addend, add_C,
                            add_c0);
    } else {
        if (C % 4 == 0 && aligned16(dy, dx, nullptr) && !(reinterpret_cast<uintptr_t>(idx) & 3) && add_vec)
            e = pool_launch(k_maxpool_bwd<float, 4>, ins * (C / 4), cs, (const float*)dy, idx, (float*)dx, g,
                            (const float*)addend, add_C, add_c0);
        else
            e = pool_launch(k_maxpool_bwd<float, 1>, ins * C, cs, (const float*)dy, idx, (float*)dx, g,
                            (const float*)addend, add_C, add_c0);
    }
    MBS_CK(e);
    return MBS_OK;
}

int mbs_copy_channels(const void* src, int64_t src_C, int64_t src_c0, void* dst, int64_t dst_C, int64_t dst_c0,
                      int64_t M, int64_t C, const float* bias, int dtype, void* stream) {
    if (!src || !dst) return invalid("mbs_copy_channels: null pointer");
    if (dtype != MBS_BF16 && dtype != MBS_F32) return invalid("mbs_copy_channels: dtype must be MBS_BF16 or MBS_F32");
    if (M < 0 || C < 1 || src_c0 < 0 || dst_c0 < 0 || src_c0 + C > src_C || dst_c0 + C > dst_C)
        return invalid("mbs_copy_channels: bad geometry");
    if (M == 0) return MBS_OK;
    cudaStream_t cs = static_cast<cudaStream_t>(stream);
    const int es = dtype == MBS_BF16 ? 2 : 4;
    const int V = 16 / es;
    const bool vec = C % V == 0 && src_C % V == 0 && dst_C % V == 0 && src_c0 % V == 0 && dst_c0 % V == 0 &&
                     aligned16(src, dst, nullptr);
    cudaError_t e;
    if (dtype == MBS_BF16) {
        using T = __nv_bfloat16;
        e = vec ? pool_launch(k_copy_channels<T, 8>, M * (C / 8), cs, (const T*)src, src_C, src_c0, (T*)dst, dst_C, dst_c0,
                              M, C, bias)
                : pool_launch(k_copy_channels<T, 1>, M * C, cs, (const T*)src, src_C, src_c0, (T*)dst, dst_C, dst_c0, M,
                              C, bias);
    } else {
        e = vec ? pool_launch(k_copy_channels<float, 4>, M * (C / 4), cs, (const float*)src, src_C, src_c0, (float*)dst,
                              dst_C, dst_c0, M, C, bias)
                : pool_launch(k_copy_channels<float, 1>, M * C, cs, (const float*)src, src_C, src_c0, (float*)dst, dst_C,
                              dst_c0, M, C, bias);
    }
    MBS_CK(e);
    return MBS_OK;
}

}  // extern "C"
