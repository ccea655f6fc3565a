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
#include <stdlib.h>

#include <algorithm>
#include <type_traits>

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

// Index math runs in 32 bits whenever every element offset fits (the 64-bit divisions of the
// grid-stride decomposition dominated these memory-bound kernels: ncu, tools/k6_ncu.py).
// Division by a runtime-constant divisor: with 32-bit indices (every dividend < 2^31) a multiply-high
// and a shift, m = ceil(2^(31+l) / d), l = ceil(log2 d) — the pixel decomposition's five divisions
// were most of the instructions of these instruction-bound kernels (ncu, tools/k6_ncu.py).
template <typename I>
struct Div {
    I d;
    uint32_t m;
    int sh;
    __device__ __forceinline__ I div(I n) const {
        if constexpr (sizeof(I) == 4) return d == 1 ? n : (I)(__umulhi((uint32_t)n, m) >> sh);
        else return n / d;
    }
};

template <typename I>
static Div<I> make_div(int64_t d) {
    Div<I> r{(I)d, 0u, 0};
    if (sizeof(I) == 4 && d > 1) {
        int l = 0;
        while ((1LL << l) < d) ++l;
        r.m = (uint32_t)(((1ULL << (31 + l)) + (uint64_t)d - 1) / (uint64_t)d);
        r.sh = l - 1;
    }
    return r;
}

template <typename I>
struct PoolGeomT {
    I N, H, W, C, Ho, Wo;
    int k, s, p;
    Div<I> cv, dW, dH, dWo, dHo;   // C / V (the vector width of the launched kernel), W, H, Wo, Ho
};

template <typename I>
static PoolGeomT<I> narrow(const PoolGeom& g, int V) {
    return PoolGeomT<I>{(I)g.N, (I)g.H, (I)g.W, (I)g.C, (I)g.Ho, (I)g.Wo, g.k, g.s, g.p, make_div<I>(g.C / V),
                        make_div<I>(g.W), make_div<I>(g.H), make_div<I>(g.Wo), make_div<I>(g.Ho)};
}

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
// K > 0: the window size is a compile-time constant (the ResNet stem's 3x3, the U-Net's 2x2): the
// window loops unroll and all k*k loads are in flight at once instead of one per loop trip.
template <typename T, int V, typename I, int K = 0>
__global__ void __launch_bounds__(kPoolThreads) k_maxpool_fwd(const T* __restrict__ x, T* __restrict__ y,
                                                              uint8_t* __restrict__ idx, PoolGeomT<I> g,
                                                              T* __restrict__ stash, I sC, I sc0) {
    const int kk = K > 0 ? K : g.k;
    cudaGridDependencySynchronize();
    const I cv = g.C / V;
    const I total = g.N * g.Ho * g.Wo * cv;
    for (I t = (I)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (I)gridDim.x * blockDim.x) {
        I q = g.cv.div(t);
        const I c0 = (t - q * cv) * V;
        I q2 = g.dWo.div(q);
        const I ow = q - q2 * g.Wo;
        q = g.dHo.div(q2);
        const I oh = q2 - q * g.Ho;
        const I n = q;
        const I h0 = oh * g.s - g.p, w0 = ow * g.s - g.p;
        float m[V];
        uint8_t a[V];
#pragma unroll
        for (int i = 0; i < V; ++i) {
            m[i] = -INFINITY;
            a[i] = 0;
        }
        if constexpr (K > 0) {
            // every in-bounds window element loaded first (k*k loads in flight), then the scan in
            // torch's order
            // raw 16-byte words (unpacked only in the scan), out-of-bounds elements load a valid
            // address unconditionally and are skipped by the scan
            static_assert(sizeof(T) * V == 16, "the compile-time-window variant takes 16-byte channel vectors");
            uint4 raw[K * K];
            bool ok[K * K];
#pragma unroll
            for (int q2 = 0; q2 < K * K; ++q2) {
                const I ih = h0 + q2 / K, iw = w0 + q2 % K;
                ok[q2] = ih >= 0 && ih < g.H && iw >= 0 && iw < g.W;
                const I pix = ok[q2] ? (n * g.H + ih) * g.W + iw : (I)0;
                raw[q2] = __ldg(reinterpret_cast<const uint4*>(x + pix * g.C + c0));
            }
            if (stash) {   // after every load is issued
#pragma unroll
                for (int q2 = 0; q2 < K * K; ++q2) {
                    const I ih = h0 + q2 / K, iw = w0 + q2 % K;
                    if (ok[q2])
                        *reinterpret_cast<uint4*>(stash + ((n * g.H + ih) * g.W + iw) * sC + sc0 + c0) = raw[q2];
                }
            }
            if constexpr (sizeof(T) == 2) {
                // bf16: the scan on packed bf16x2 lanes — lane masks from the same ordered ">" and NaN
                // tests (bf16 -> fp32 is exact, so the decisions are the fp32 scan's), m and the 16-bit
                // argmax lanes blended under the mask: ~half the instructions of the per-element scan
                uint32_t mw[4] = {0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u, 0xFF80FF80u};   // -inf
                uint32_t aw[4] = {0u, 0u, 0u, 0u};
#pragma unroll
                for (int q2 = 0; q2 < K * K; ++q2) {
                    if (!ok[q2]) continue;
                    const uint32_t vw[4] = {raw[q2].x, raw[q2].y, raw[q2].z, raw[q2].w};
                    const uint32_t pw = (uint32_t)q2 | ((uint32_t)q2 << 16);
#pragma unroll
                    for (int w = 0; w < 4; ++w) {
                        const __nv_bfloat162 v2 = *reinterpret_cast<const __nv_bfloat162*>(&vw[w]);
                        const __nv_bfloat162 m2 = *reinterpret_cast<const __nv_bfloat162*>(&mw[w]);
                        const uint32_t msk = __hgt2_mask(v2, m2) | __hneu2_mask(v2, v2);
                        mw[w] = (mw[w] & ~msk) | (vw[w] & msk);
                        aw[w] = (aw[w] & ~msk) | (pw & msk);
                    }
                }
                const I o = ((n * g.Ho + oh) * g.Wo + ow) * g.C + c0;
                *reinterpret_cast<uint4*>(y + o) = make_uint4(mw[0], mw[1], mw[2], mw[3]);
                uint2 ib;
                ib.x = __byte_perm(aw[0], aw[1], 0x6420);
                ib.y = __byte_perm(aw[2], aw[3], 0x6420);
                *reinterpret_cast<uint2*>(idx + o) = ib;
                continue;
            }
#pragma unroll
            for (int q2 = 0; q2 < K * K; ++q2) {
                if (!ok[q2]) continue;
                float v[V];
                PoolIO<T, V>::load(reinterpret_cast<const T*>(&raw[q2]), v);
#pragma unroll
                for (int i = 0; i < V; ++i) {
                    if (v[i] > m[i] || isnan(v[i])) {
                        m[i] = v[i];
                        a[i] = (uint8_t)q2;
                    }
                }
            }
        } else
        for (int kh = 0; kh < kk; ++kh) {
            const I ih = h0 + kh;
            if (ih < 0 || ih >= g.H) continue;
            for (int kw = 0; kw < kk; ++kw) {
                const I iw = w0 + kw;
                if (iw < 0 || iw >= g.W) continue;
                float v[V];
                const I pix = (n * g.H + ih) * g.W + iw;
                PoolIO<T, V>::load(x + pix * g.C + c0, v);
                if (K == 0 && stash) PoolIO<T, V>::store(stash + pix * sC + sc0 + c0, v);
                const uint8_t pos = (uint8_t)(kh * kk + kw);
#pragma unroll
                for (int i = 0; i < V; ++i) {
                    if (v[i] > m[i] || isnan(v[i])) {
                        m[i] = v[i];
                        a[i] = pos;
                    }
                }
            }
        }
        const I o = ((n * g.Ho + oh) * g.Wo + ow) * g.C + c0;
        PoolIO<T, V>::store(y + o, m);
        store_idx<V>(idx + o, a);
    }
}

// Optional addend: dx += add[pixel, ac0 + c] (row stride aC) in fp32 before the single rounding —
// the gradient that reached the same tensor through the U-Net skip connection, fused instead of
// autograd's separate add pass.
// W2 = 1: non-overlapping windows tiling the input (the U-Net 2x2/s2 pools) — no window search.
// W2 = 2: 3x3 windows, stride 2 (the ResNet stem): at most 2x2 candidate windows, unrolled and
// predicated so their index/gradient loads are all in flight at once.
// dy2 (nullable): a second gradient of y (the pooled activation has two consumers), added to dy per
// window and rounded to T before the gather sum — exactly torch's (dy1 + dy2) in T, then gather.
template <typename T>
__device__ __forceinline__ float round_to(float v) {
    if constexpr (sizeof(T) == 2) return __bfloat162float(__float2bfloat16(v));
    else return v;
}

template <typename T, int V, typename I, int W2>
__global__ void __launch_bounds__(kPoolThreads) k_maxpool_bwd(const T* __restrict__ dy,
                                                              const uint8_t* __restrict__ idx, T* __restrict__ dx,
                                                              PoolGeomT<I> g, const T* __restrict__ add, I aC,
                                                              I ac0, const T* __restrict__ dy2) {
    cudaGridDependencySynchronize();
    const I cv = g.C / V;
    const I total = g.N * g.H * g.W * cv;
    for (I t = (I)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (I)gridDim.x * blockDim.x) {
        I q = g.cv.div(t);
        const I c0 = (t - q * cv) * V;
        I q2 = g.dW.div(q);
        const I iw = q - q2 * g.W;
        q = g.dH.div(q2);
        const I ih = q2 - q * g.H;
        const I n = q;
        const I pix = (n * g.H + ih) * g.W + iw;
        float a2[V];
        if (add) PoolIO<T, V>::load(add + pix * aC + ac0 + c0, a2);   // independent of the windows: issue first
        // windows containing (ih, iw): oh*s - p <= ih <= oh*s - p + k - 1
        const int sk = W2 == 2 ? 2 : g.s, kk = W2 == 2 ? 3 : g.k;   // 3x3/s2: constant divisions
        const I ohs = max((I)0, (ih + g.p - kk + sk) / sk);
        const I ohe = min(g.Ho, (ih + g.p) / sk + 1);
        const I ows = max((I)0, (iw + g.p - kk + sk) / sk);
        const I owe = min(g.Wo, (iw + g.p) / sk + 1);
        float acc[V];
#pragma unroll
        for (int i = 0; i < V; ++i) acc[i] = 0.f;
        if constexpr (W2 == 2 && sizeof(T) * V == 16) {
            // all four candidate windows' idx / dy loaded first (out-of-range ones from a valid
            // address, skipped below), then summed in ascending (oh, ow) order
            using IRaw = typename std::conditional<V == 8, uint2, uint32_t>::type;
            uint4 draw[4], draw2[4];
            IRaw iraw[4];
            bool ok[4];
            uint8_t pos[4];
#pragma unroll
            for (int q2 = 0; q2 < 4; ++q2) {
                const I oh = ohs + q2 / 2, ow = ows + q2 % 2;
                const int kh = (int)(ih - (oh * 2 - g.p)), kw = (int)(iw - (ow * 2 - g.p));
                ok[q2] = oh < ohe && ow < owe && kh >= 0 && kh < 3 && kw >= 0 && kw < 3;
                pos[q2] = (uint8_t)(kh * 3 + kw);
                const I o = ok[q2] ? ((n * g.Ho + oh) * g.Wo + ow) * g.C + c0 : (I)0;
                iraw[q2] = __ldg(reinterpret_cast<const IRaw*>(idx + o));
                draw[q2] = __ldg(reinterpret_cast<const uint4*>(dy + o));
                if (dy2) draw2[q2] = __ldg(reinterpret_cast<const uint4*>(dy2 + o));
            }
#pragma unroll
            for (int q2 = 0; q2 < 4; ++q2) {
                if (!ok[q2]) continue;
                uint8_t a[V];
                float d[V];
                load_idx<V>(reinterpret_cast<const uint8_t*>(&iraw[q2]), a);
                PoolIO<T, V>::load(reinterpret_cast<const T*>(&draw[q2]), d);
                if (dy2) {
                    float d2[V];
                    PoolIO<T, V>::load(reinterpret_cast<const T*>(&draw2[q2]), d2);
#pragma unroll
                    for (int i = 0; i < V; ++i) d[i] = round_to<T>(d[i] + d2[i]);
                }
#pragma unroll
                for (int i = 0; i < V; ++i)
                    if (a[i] == pos[q2]) acc[i] += d[i];
            }
        } else if constexpr (W2 == 1) {
            // non-overlapping windows (k == s, p == 0): exactly one window per input element
            const I oh = ih / g.s, ow = iw / g.s;
            const uint8_t pos = (uint8_t)((ih - oh * g.s) * g.k + (iw - ow * g.s));
            const I o = ((n * g.Ho + oh) * g.Wo + ow) * g.C + c0;
            uint8_t a[V];
            float d[V];
            load_idx<V>(idx + o, a);
            PoolIO<T, V>::load(dy + o, d);
            if (dy2) {
                float d2[V];
                PoolIO<T, V>::load(dy2 + o, d2);
#pragma unroll
                for (int i = 0; i < V; ++i) d[i] = round_to<T>(d[i] + d2[i]);
            }
#pragma unroll
            for (int i = 0; i < V; ++i)
                if (a[i] == pos) acc[i] = d[i];
        } else {
            for (I oh = ohs; oh < ohe; ++oh) {
                const int kh = (int)(ih - (oh * g.s - g.p));
                if (kh < 0 || kh >= g.k) continue;
                for (I ow = ows; ow < owe; ++ow) {
                    const int kw = (int)(iw - (ow * g.s - g.p));
                    if (kw < 0 || kw >= g.k) continue;
                    const uint8_t pos = (uint8_t)(kh * g.k + kw);
                    const I o = ((n * g.Ho + oh) * g.Wo + ow) * g.C + c0;
                    uint8_t a[V];
                    float d[V];
                    load_idx<V>(idx + o, a);
                    PoolIO<T, V>::load(dy + o, d);
                    if (dy2) {
                        float d2[V];
                        PoolIO<T, V>::load(dy2 + o, d2);
#pragma unroll
                        for (int i = 0; i < V; ++i) d[i] = round_to<T>(d[i] + d2[i]);
                    }
#pragma unroll
                    for (int i = 0; i < V; ++i)
                        if (a[i] == pos) acc[i] += d[i];
                }
            }
        }
        if (add) {
#pragma unroll
            for (int i = 0; i < V; ++i) acc[i] += a2[i];
        }
        PoolIO<T, V>::store(dx + pix * g.C + c0, acc);
    }
}

// 3x3 / stride 2 / pad 1 (the ResNet stem) backward on 2x2 input blocks: input rows 2a, 2a+1 and
// columns 2b, 2b+1 lie in windows oh in {a, a+1}, ow in {b, b+1} only, so one thread loads those 4
// windows' idx/dy once (all in flight) and serves 4 input pixels with the 9 (pixel, window) pairs
// that exist — the per-pixel kernel evaluated 16 candidate slots for every 4 pixels.
// Each pixel sums its windows in ascending (oh, ow) order in fp32: bit-identical to torch.
template <typename T, int V>
__global__ void __launch_bounds__(kPoolThreads) k_maxpool_bwd_blk(const T* __restrict__ dy,
                                                                  const uint8_t* __restrict__ idx,
                                                                  T* __restrict__ dx, PoolGeomT<int32_t> g,
                                                                  const T* __restrict__ dy2) {
    static_assert(sizeof(T) * V == 16, "16-byte channel vectors");
    using IRaw = typename std::conditional<V == 8, uint2, uint32_t>::type;
    cudaGridDependencySynchronize();
    const int cv = g.C / V;
    const int total = g.N * g.Ho * g.Wo * cv;   // blocks: Hb = Ho, Wb = Wo for k3/s2/p1
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
        int q = g.cv.div(t);
        const int c0 = (t - q * cv) * V;
        int q2 = g.dWo.div(q);
        const int b = q - q2 * g.Wo;
        const int n = g.dHo.div(q2);
        const int a = q2 - n * g.Ho;
        uint4 dr[4], dr2[4];
        IRaw ir[4];
        bool ok[4];
#pragma unroll
        for (int w = 0; w < 4; ++w) {
            const int oh = a + w / 2, ow = b + w % 2;
            ok[w] = oh < g.Ho && ow < g.Wo;
            const int o = ok[w] ? ((n * g.Ho + oh) * g.Wo + ow) * g.C + c0 : 0;
            ir[w] = __ldg(reinterpret_cast<const IRaw*>(idx + o));
            dr[w] = __ldg(reinterpret_cast<const uint4*>(dy + o));
            if (dy2) dr2[w] = __ldg(reinterpret_cast<const uint4*>(dy2 + o));
        }
        float d[4][V];
        uint8_t ai[4][V];
#pragma unroll
        for (int w = 0; w < 4; ++w) {
            PoolIO<T, V>::load(reinterpret_cast<const T*>(&dr[w]), d[w]);
            load_idx<V>(reinterpret_cast<const uint8_t*>(&ir[w]), ai[w]);
            if (dy2) {
                float d2[V];
                PoolIO<T, V>::load(reinterpret_cast<const T*>(&dr2[w]), d2);
#pragma unroll
                for (int i = 0; i < V; ++i) d[w][i] = round_to<T>(d[w][i] + d2[i]);
            }
        }
#pragma unroll
        for (int dh = 0; dh < 2; ++dh) {
#pragma unroll
            for (int dw = 0; dw < 2; ++dw) {
                const int ih = 2 * a + dh, iw = 2 * b + dw;
                if (ih >= g.H || iw >= g.W) continue;
                float acc[V];
#pragma unroll
                for (int i = 0; i < V; ++i) acc[i] = 0.f;
#pragma unroll
                for (int wh = 0; wh < 2; ++wh) {
#pragma unroll
                    for (int ww = 0; ww < 2; ++ww) {
                        if ((wh == 1 && dh == 0) || (ww == 1 && dw == 0)) continue;   // not in that window
                        const int w = wh * 2 + ww;
                        const uint8_t pos = (uint8_t)((dh + 1 - 2 * wh) * 3 + (dw + 1 - 2 * ww));
                        if (!ok[w]) continue;
#pragma unroll
                        for (int i = 0; i < V; ++i)
                            if (ai[w][i] == pos) acc[i] += d[w][i];
                    }
                }
                PoolIO<T, V>::store(dx + ((n * g.H + ih) * g.W + iw) * g.C + c0, acc);
            }
        }
    }
}

// Channel-slice copy between channels-last tensors viewed as [M, C_total] rows:
// dst[m, dc0 + c] = src[m, sc0 + c] (+ bias[c]) — the U-Net skip join (the upsampled half lands in
// the concat buffer with its ConvTranspose bias added on the way) and its backward (the slice made
// dense for the ConvTranspose backward). One thread per 16-byte vector; consecutive threads walk
// consecutive channels, then rows.
template <typename T, int V, typename I>
__global__ void __launch_bounds__(kPoolThreads) k_copy_channels(const T* __restrict__ src, I sC, I sc0,
                                                                T* __restrict__ dst, I dC, I dc0,
                                                                I M, I C, const float* __restrict__ bias,
                                                                float* __restrict__ colsum) {
    // colsum (nullable): per-CTA fp32 column sums of the copied values, [gridDim.x][C] — the ConvTranspose
    // bias gradient of the U-Net join backward, summed in fixed order without another pass. Needs the
    // grid-stride step to be a multiple of C / V, so a thread keeps one channel vector (host-checked).
    __shared__ float red[kPoolThreads * (V > 4 ? 8 : V)];
    cudaGridDependencySynchronize();
    const I cv = C / V;
    const I total = M * cv;
    float cs[V];
#pragma unroll
    for (int i = 0; i < V; ++i) cs[i] = 0.f;
    for (I t = (I)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (I)gridDim.x * blockDim.x) {
        const I c0 = (t % cv) * V;
        const I m = t / cv;
        float v[V];
        PoolIO<T, V>::load(src + m * sC + sc0 + c0, v);
        if (bias) {
#pragma unroll
            for (int i = 0; i < V; ++i) v[i] += bias[c0 + i];
        }
        PoolIO<T, V>::store(dst + m * dC + dc0 + c0, v);
        if (colsum) {
#pragma unroll
            for (int i = 0; i < V; ++i) cs[i] += v[i];
        }
    }
    if (colsum) {
#pragma unroll
        for (int i = 0; i < V; ++i) red[i * kPoolThreads + threadIdx.x] = cs[i];
        __syncthreads();
        // threads t, t + cv, t + 2 cv, ... of this CTA hold the same channel vector
        if ((I)threadIdx.x < cv) {
            for (int i = 0; i < V; ++i) {
                float a = 0.f;
                for (int j = threadIdx.x; j < kPoolThreads; j += (int)cv) a += red[i * kPoolThreads + j];
                colsum[(size_t)blockIdx.x * C + threadIdx.x * V + i] = a;
            }
        }
    }
}


template <typename... KArgs, typename... Args>
static cudaError_t pool_launch(void (*kernel)(KArgs...), int64_t work, cudaStream_t s, Args... args) {
    // grid-stride: at most 8 resident 256-thread CTAs per SM, fewer when the work is small
    static int sms = 0;
    if (sms <= 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) sms = 148;
    }
    // one full wave: resident CTAs per SM from the occupancy calculator (a 2nd partial wave of a
    // grid-stride loop costs a whole CTA lifetime)
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kPoolThreads, 0) != cudaSuccess || per_sm < 1)
        per_sm = 1;
    const int64_t want = (work + kPoolThreads - 1) / kPoolThreads;
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)std::min(per_sm, 8) * sms));
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

static bool block_mode() {   // A/B: MBS_K6_BLOCK=0 keeps the per-pixel 3x3/s2 backward
    const char* e = getenv("MBS_K6_BLOCK");
    return !e || atoi(e) != 0;
}

static bool fits_i32(int64_t v) { return v < (int64_t)INT32_MAX - (1 << 22); }  // grid-stride headroom

template <typename I>
static int maxpool_fwd(const void* x, void* y, uint8_t* idx, int dtype, const PoolGeom& g0, void* stash, int64_t sC,
                       int64_t sc0, cudaStream_t cs) {
    const PoolGeomT<I> gv = narrow<I>(g0, dtype == MBS_BF16 ? 8 : 4), g1 = narrow<I>(g0, 1);
    const int64_t outs = g0.N * g0.Ho * g0.Wo;
    const int es = dtype == MBS_BF16 ? 2 : 4;
    const bool stash_vec = !stash || (!(reinterpret_cast<uintptr_t>(stash) & 15) && (sC * es) % 16 == 0 &&
                                      (sc0 * es) % 16 == 0);
    const I isC = (I)sC, isc0 = (I)sc0;
    cudaError_t e;
    if (dtype == MBS_BF16) {
        using T = __nv_bfloat16;
        if (g0.C % 8 == 0 && aligned16(x, y, nullptr) && !(reinterpret_cast<uintptr_t>(idx) & 7) && stash_vec)
            e = g0.k == 3 ? pool_launch(k_maxpool_fwd<T, 8, I, 3>, outs * (g0.C / 8), cs, (const T*)x, (T*)y, idx, gv,
                                        (T*)stash, isC, isc0)
              : g0.k == 2 ? pool_launch(k_maxpool_fwd<T, 8, I, 2>, outs * (g0.C / 8), cs, (const T*)x, (T*)y, idx, gv,
                                        (T*)stash, isC, isc0)
                          : pool_launch(k_maxpool_fwd<T, 8, I>, outs * (g0.C / 8), cs, (const T*)x, (T*)y, idx, gv,
                                        (T*)stash, isC, isc0);
        else
            e = pool_launch(k_maxpool_fwd<T, 1, I>, outs * g0.C, cs, (const T*)x, (T*)y, idx, g1, (T*)stash, isC, isc0);
    } else {
        if (g0.C % 4 == 0 && aligned16(x, y, nullptr) && !(reinterpret_cast<uintptr_t>(idx) & 3) && stash_vec)
            e = pool_launch(k_maxpool_fwd<float, 4, I>, outs * (g0.C / 4), cs, (const float*)x, (float*)y, idx, gv,
                            (float*)stash, isC, isc0);
        else
            e = pool_launch(k_maxpool_fwd<float, 1, I>, outs * g0.C, cs, (const float*)x, (float*)y, idx, g1,
                            (float*)stash, isC, isc0);
    }
    MBS_CK(e);
    return MBS_OK;
}

template <typename I, int W2>
static int maxpool_bwd(const void* dy, const void* dy2, const uint8_t* idx, void* dx, int dtype, const PoolGeom& g0,
                       const void* add, int64_t aC, int64_t ac0, cudaStream_t cs) {
    const PoolGeomT<I> gv = narrow<I>(g0, dtype == MBS_BF16 ? 8 : 4), g1 = narrow<I>(g0, 1);
    const int64_t ins = g0.N * g0.H * g0.W;
    const int es = dtype == MBS_BF16 ? 2 : 4;
    const bool add_vec = !add || (!(reinterpret_cast<uintptr_t>(add) & 15) && (aC * es) % 16 == 0 &&
                                  (ac0 * es) % 16 == 0);
    const I iaC = (I)aC, iac0 = (I)ac0;
    cudaError_t e;
    if (dtype == MBS_BF16) {
        using T = __nv_bfloat16;
        if (g0.C % 8 == 0 && aligned16(dy, dx, dy2) && !(reinterpret_cast<uintptr_t>(idx) & 7) && add_vec)
            e = pool_launch(k_maxpool_bwd<T, 8, I, W2>, ins * (g0.C / 8), cs, (const T*)dy, idx, (T*)dx, gv, (const T*)add,
                            iaC, iac0, (const T*)dy2);
        else
            e = pool_launch(k_maxpool_bwd<T, 1, I, W2>, ins * g0.C, cs, (const T*)dy, idx, (T*)dx, g1, (const T*)add, iaC,
                            iac0, (const T*)dy2);
    } else {
        if (g0.C % 4 == 0 && aligned16(dy, dx, dy2) && !(reinterpret_cast<uintptr_t>(idx) & 3) && add_vec)
            e = pool_launch(k_maxpool_bwd<float, 4, I, W2>, ins * (g0.C / 4), cs, (const float*)dy, idx, (float*)dx, gv,
                            (const float*)add, iaC, iac0, (const float*)dy2);
        else
            e = pool_launch(k_maxpool_bwd<float, 1, I, W2>, ins * g0.C, cs, (const float*)dy, idx, (float*)dx, g1,
                            (const float*)add, iaC, iac0, (const float*)dy2);
    }
    MBS_CK(e);
    return MBS_OK;
}

template <typename I>
static int copy_channels(const void* src, int64_t sC, int64_t sc0, void* dst, int64_t dC, int64_t dc0, int64_t M,
                         int64_t C, const float* bias, float* colsum, int dtype, cudaStream_t cs) {
    const int es = dtype == MBS_BF16 ? 2 : 4;
    const int V = 16 / es;
    const bool vec = C % V == 0 && sC % V == 0 && dC % V == 0 && sc0 % V == 0 && dc0 % V == 0 &&
                     aligned16(src, dst, nullptr);
    cudaError_t e;
    if (dtype == MBS_BF16) {
        using T = __nv_bfloat16;
        e = vec ? pool_launch(k_copy_channels<T, 8, I>, M * (C / 8), cs, (const T*)src, (I)sC, (I)sc0, (T*)dst, (I)dC,
                              (I)dc0, (I)M, (I)C, bias, colsum)
                : pool_launch(k_copy_channels<T, 1, I>, M * C, cs, (const T*)src, (I)sC, (I)sc0, (T*)dst, (I)dC, (I)dc0,
                              (I)M, (I)C, bias, colsum);
    } else {
        e = vec ? pool_launch(k_copy_channels<float, 4, I>, M * (C / 4), cs, (const float*)src, (I)sC, (I)sc0,
                              (float*)dst, (I)dC, (I)dc0, (I)M, (I)C, bias, colsum)
                : pool_launch(k_copy_channels<float, 1, I>, M * C, cs, (const float*)src, (I)sC, (I)sc0, (float*)dst,
                              (I)dC, (I)dc0, (I)M, (I)C, bias, colsum);
    }
    MBS_CK(e);
    return MBS_OK;
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
    const bool i32 = fits_i32(g.N * g.H * g.W * std::max<int64_t>(g.C, stash ? stash_C : 0)) &&
                     fits_i32(g.N * g.Ho * g.Wo * g.C);
    return i32 ? maxpool_fwd<int32_t>(x, y, idx, dtype, g, stash, stash_C, stash_c0, cs)
               : maxpool_fwd<int64_t>(x, y, idx, dtype, g, stash, stash_C, stash_c0, cs);
}

int mbs_maxpool_backward(const void* dy, const void* dy2, const uint8_t* idx, void* dx, int dtype, int64_t N,
                         int64_t H, int64_t W, int64_t C, int k, int s, int p, const void* addend, int64_t add_C,
                         int64_t add_c0, void* stream) {
    if (!dy || !idx || !dx) return invalid("mbs_maxpool_backward: null pointer");
    PoolGeom g;
    int st = pool_check(dtype, N, H, W, C, k, s, p, &g);
    if (st) return st;
    if (addend && (add_c0 < 0 || add_c0 + C > add_C)) return invalid("mbs_maxpool_backward: addend columns");
    cudaStream_t cs = static_cast<cudaStream_t>(stream);
    const bool i32 = fits_i32(g.N * g.H * g.W * std::max<int64_t>(g.C, addend ? add_C : 0)) &&
                     fits_i32(g.N * g.Ho * g.Wo * g.C);
    const bool w2 = g.k == g.s && g.p == 0 && g.H % g.k == 0 && g.W % g.k == 0;   // one window per element
    const bool k3s2 = g.k == 3 && g.s == 2 && g.C % (dtype == MBS_BF16 ? 8 : 4) == 0 && aligned16(dy, dx, dy2) &&
                      !(reinterpret_cast<uintptr_t>(idx) & (dtype == MBS_BF16 ? 7 : 3));
    if (k3s2 && g.p == 1 && i32 && !addend && block_mode()) {
        const int V = dtype == MBS_BF16 ? 8 : 4;
        const PoolGeomT<int32_t> gv = narrow<int32_t>(g, V);
        const int64_t work = g.N * g.Ho * g.Wo * (g.C / V);
        cudaError_t e = dtype == MBS_BF16
            ? pool_launch(k_maxpool_bwd_blk<__nv_bfloat16, 8>, work, cs, (const __nv_bfloat16*)dy, idx,
                          (__nv_bfloat16*)dx, gv, (const __nv_bfloat16*)dy2)
            : pool_launch(k_maxpool_bwd_blk<float, 4>, work, cs, (const float*)dy, idx, (float*)dx, gv,
                          (const float*)dy2);
        MBS_CK(e);
        return MBS_OK;
    }
    if (i32)
        return w2     ? maxpool_bwd<int32_t, 1>(dy, dy2, idx, dx, dtype, g, addend, add_C, add_c0, cs)
               : k3s2 ? maxpool_bwd<int32_t, 2>(dy, dy2, idx, dx, dtype, g, addend, add_C, add_c0, cs)
                      : maxpool_bwd<int32_t, 0>(dy, dy2, idx, dx, dtype, g, addend, add_C, add_c0, cs);
    return w2 ? maxpool_bwd<int64_t, 1>(dy, dy2, idx, dx, dtype, g, addend, add_C, add_c0, cs)
              : maxpool_bwd<int64_t, 0>(dy, dy2, idx, dx, dtype, g, addend, add_C, add_c0, cs);
}

int mbs_copy_channels(const void* src, int64_t src_C, int64_t src_c0, void* dst, int64_t dst_C, int64_t dst_c0,
                      int64_t M, int64_t C, const float* bias, float* colsum, int64_t colsum_rows, int dtype,
                      void* stream) {
    if (!src || !dst) return invalid("mbs_copy_channels: null pointer");
    if (dtype != MBS_BF16 && dtype != MBS_F32) return invalid("mbs_copy_channels: dtype must be MBS_BF16 or MBS_F32");
    if (M < 0 || C < 1 || src_c0 < 0 || dst_c0 < 0 || src_c0 + C > src_C || dst_c0 + C > dst_C)
        return invalid("mbs_copy_channels: bad geometry");
    if (M == 0) return MBS_OK;
    cudaStream_t cs = static_cast<cudaStream_t>(stream);
    const bool i32 = fits_i32(M * std::max(src_C, dst_C));
    if (colsum) {
        // one thread per channel vector for the whole grid-stride: C/V must divide the CTA size, the grid is
        // exactly colsum_rows CTAs (the caller sums the [colsum_rows][C] partials)
        const int V = dtype == MBS_BF16 ? 8 : 4;
        const int64_t cv = C / V;
        if (C % V || kPoolThreads % cv || colsum_rows < 1)
            return invalid("mbs_copy_channels: colsum needs C/V to divide 256 and colsum_rows >= 1");
        if (!aligned16(src, dst, nullptr) || src_C % V || dst_C % V || src_c0 % V || dst_c0 % V)
            return invalid("mbs_copy_channels: colsum needs the vector path (16-byte aligned columns)");
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)colsum_rows);
        cfg.blockDim = dim3(kPoolThreads);
        cfg.stream = cs;
        cudaError_t e;
        if (dtype == MBS_BF16) {
            using T = __nv_bfloat16;
            e = i32 ? cudaLaunchKernelEx(&cfg, k_copy_channels<T, 8, int32_t>, (const T*)src, (int32_t)src_C,
                                         (int32_t)src_c0, (T*)dst, (int32_t)dst_C, (int32_t)dst_c0, (int32_t)M,
                                         (int32_t)C, bias, colsum)
                    : cudaLaunchKernelEx(&cfg, k_copy_channels<T, 8, int64_t>, (const T*)src, src_C, src_c0, (T*)dst,
                                         dst_C, dst_c0, M, C, bias, colsum);
        } else {
            e = i32 ? cudaLaunchKernelEx(&cfg, k_copy_channels<float, 4, int32_t>, (const float*)src, (int32_t)src_C,
                                         (int32_t)src_c0, (float*)dst, (int32_t)dst_C, (int32_t)dst_c0, (int32_t)M,
                                         (int32_t)C, bias, colsum)
                    : cudaLaunchKernelEx(&cfg, k_copy_channels<float, 4, int64_t>, (const float*)src, src_C, src_c0,
                                         (float*)dst, dst_C, dst_c0, M, C, bias, colsum);
        }
        MBS_CK(e);
        return MBS_OK;
    }
    return i32 ? copy_channels<int32_t>(src, src_C, src_c0, dst, dst_C, dst_c0, M, C, bias, nullptr, dtype, cs)
               : copy_channels<int64_t>(src, src_C, src_c0, dst, dst_C, dst_c0, M, C, bias, nullptr, dtype, cs);
}

}  // extern "C"
