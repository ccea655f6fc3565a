// K2: micro-batch staging — row gather + dtype cast + NCHW/NHWC layout, and a
// byte-exact row gather for targets.
//
// Reference semantics: the epoch gather xb = x[order[start:start+M]]
// (engine.py:310-312), the contiguous micro slice ascontiguousarray(x[lo:hi])
// (engine.py:149-151) and the dtype coercion as_array (tensor.py:20-22). The
// staged bytes are bit-identical to torch's x[rows].to(dtype[, channels_last]):
// u8 -> f32/bf16/f16 is exact, f32 -> bf16/f16 use cvt.rn (round-to-nearest-even,
// canonical NaN), i.e. the conversions torch's CUDA kernels use.
//
// The source may be device memory or page-locked host memory (zero-copy over
// PCIe); 128-bit loads and stores whenever the row base is 16-byte aligned.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <stdlib.h>
#include <string.h>

#include <algorithm>

#include "mbs_common.h"
#include "mbs_tma.h"

namespace mbs {

constexpr int kStageThreads = 256;
constexpr int kPix = 16;  // pixels (NHWC) or elements (NCHW) per thread

template <typename T> struct Elem;
template <> struct Elem<uint8_t> { static __device__ __forceinline__ float f(uint8_t v) { return (float)v; } };
template <> struct Elem<float> { static __device__ __forceinline__ float f(float v) { return v; } };
template <> struct Elem<double> { static __device__ __forceinline__ float f(double v) { return __double2float_rn(v); } };

__device__ __forceinline__ uint16_t f32_to_bf16_rne(float f) {
    // cvt.rn.bf16.f32: round-to-nearest-even, canonical NaN 0x7FFF — exactly what
    // torch's CUDA .to(torch.bfloat16) produces
    return __bfloat16_as_ushort(__float2bfloat16_rn(f));
}

template <int OUT> struct Out;
template <> struct Out<MBS_F32> {
    using T = float;
    static __device__ __forceinline__ T cvt(float v) { return v; }
};
template <> struct Out<MBS_BF16> {
    using T = uint16_t;
    static __device__ __forceinline__ T cvt(float v) { return f32_to_bf16_rne(v); }
};
template <> struct Out<MBS_F16> {
    using T = uint16_t;
    static __device__ __forceinline__ T cvt(float v) { return __half_as_ushort(__float2half_rn(v)); }
};

__device__ __forceinline__ int64_t src_row(const int64_t* rows, int64_t row0, int64_t r) {
    return rows ? rows[r] : row0 + r;
}

// u8 -> float without the conversion pipe: PRMT places byte b of w under the exponent of 2^23
// (0x4B0000vv = 2^23 + v, exact) and one FADD removes 2^23. I2F / F2F issue at a fraction of the
// ALU rate on sm_100; on the staging kernels they were the binding resource (ncu: 1.5 conversion
// instructions per staged element, 0.37 IPC, DRAM at 20 %).
__device__ __forceinline__ float u8_lane_to_f32(uint32_t w, int b) {
    return __uint_as_float(__byte_perm(w, 0x4B000000u, 0x7440u | (uint32_t)b)) - 8388608.0f;
}

// 16 bytes of interleaved NHWC output = elements [v*per, (v+1)*per) of a thread's PX pixels x C
// channels, from its C planes of raw source bytes (w[c][px / 4], byte px % 4). Exact for every
// output type: u8 values are integers below 256, so the float is exact, its bf16 (8 significant
// bits) is its upper half word — one PRMT packs two — and its fp16 is exact as well.
template <int OUT, int C, int NW>
__device__ __forceinline__ uint4 u8_nhwc_vec16(const uint32_t (&w)[C][NW], int v) {
    uint32_t q[4];
    if constexpr (OUT == MBS_F32) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int k = v * 4 + j, px = k / C, c = k % C;
            q[j] = __float_as_uint(u8_lane_to_f32(w[c][px >> 2], px & 3));
        }
    } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int k0 = v * 8 + 2 * j, k1 = k0 + 1;
            const float f0 = u8_lane_to_f32(w[k0 % C][(k0 / C) >> 2], (k0 / C) & 3);
            const float f1 = u8_lane_to_f32(w[k1 % C][(k1 / C) >> 2], (k1 / C) & 3);
            if constexpr (OUT == MBS_BF16)
                q[j] = __byte_perm(__float_as_uint(f0), __float_as_uint(f1), 0x7632u);
            else
                q[j] = (uint32_t)Out<OUT>::cvt(f0) | ((uint32_t)Out<OUT>::cvt(f1) << 16);
        }
    }
    return make_uint4(q[0], q[1], q[2], q[3]);
}

// Load kPix consecutive source elements as floats (vector path when aligned).
template <typename TI>
__device__ __forceinline__ void load_pix(const TI* p, float* v, bool vec) {
    if (vec) {
        if constexpr (sizeof(TI) == 1) {
            const uint4 q = *reinterpret_cast<const uint4*>(p);
            const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] = u8_lane_to_f32(w[i >> 2], i & 3);
        } else if constexpr (sizeof(TI) == 8) {
#pragma unroll
            for (int j = 0; j < kPix / 2; ++j) {
                const double2 q = reinterpret_cast<const double2*>(p)[j];
                v[2 * j] = __double2float_rn(q.x); v[2 * j + 1] = __double2float_rn(q.y);
            }
        } else {
#pragma unroll
            for (int j = 0; j < kPix / 4; ++j) {
                const float4 q = reinterpret_cast<const float4*>(p)[j];
                v[4 * j] = q.x; v[4 * j + 1] = q.y; v[4 * j + 2] = q.z; v[4 * j + 3] = q.w;
            }
        }
    } else {
#pragma unroll
        for (int i = 0; i < kPix; ++i) v[i] = Elem<TI>::f(p[i]);
    }
}

template <typename TO>
__device__ __forceinline__ void store_vec(TO* dst, const TO* vals, int n, bool vec) {
    // n elements, 16-byte chunks when aligned
    if (vec) {
        constexpr int per = 16 / sizeof(TO);
        for (int j = 0; j < n / per; ++j) {
            uint4 q;
            memcpy(&q, vals + j * per, 16);
            reinterpret_cast<uint4*>(dst)[j] = q;
        }
    } else {
        for (int i = 0; i < n; ++i) dst[i] = vals[i];
    }
}

// NCHW -> NCHW (cast only): thread handles kPix consecutive elements of one row.
template <typename TI, int OUT>
__global__ void __launch_bounds__(kStageThreads)
k_stage_nchw(const TI* __restrict__ src, const int64_t* __restrict__ rows, int64_t row0, int64_t E,
             typename Out<OUT>::T* __restrict__ dst, bool vec_ok) {
    using TO = typename Out<OUT>::T;
    const int64_t r = blockIdx.y;
    const int64_t e0 = ((int64_t)blockIdx.x * kStageThreads + threadIdx.x) * kPix;
    if (e0 >= E) return;
    const TI* s = src + src_row(rows, row0, r) * E + e0;
    TO* d = dst + r * E + e0;
    if (vec_ok && e0 + kPix <= E) {
        float v[kPix];
        load_pix<TI>(s, v, true);
        TO o[kPix];
#pragma unroll
        for (int i = 0; i < kPix; ++i) o[i] = Out<OUT>::cvt(v[i]);
        store_vec<TO>(d, o, kPix, true);
    } else {
        const int64_t n = min((int64_t)kPix, E - e0);
        for (int64_t i = 0; i < n; ++i) d[i] = Out<OUT>::cvt(Elem<TI>::f(s[i]));
    }
}

// NCHW -> NHWC: thread handles kPix consecutive pixels x all C (C <= 4) channels.
template <typename TI, int OUT, int C>
__global__ void __launch_bounds__(kStageThreads)
k_stage_nhwc(const TI* __restrict__ src, const int64_t* __restrict__ rows, int64_t row0, int64_t HW,
             typename Out<OUT>::T* __restrict__ dst, bool vec_ok) {
    using TO = typename Out<OUT>::T;
    const int64_t r = blockIdx.y;
    const int64_t p0 = ((int64_t)blockIdx.x * kStageThreads + threadIdx.x) * kPix;
    if (p0 >= HW) return;
    const TI* s = src + src_row(rows, row0, r) * (int64_t)C * HW;
    TO* d = dst + (r * HW + p0) * C;
    if (vec_ok && p0 + kPix <= HW) {
        TO o[kPix * C];
#pragma unroll
        for (int c = 0; c < C; ++c) {
            float v[kPix];
            load_pix<TI>(s + c * HW + p0, v, true);
#pragma unroll
            for (int i = 0; i < kPix; ++i) o[i * C + c] = Out<OUT>::cvt(v[i]);
        }
        store_vec<TO>(d, o, kPix * C, true);
    } else {
        const int64_t n = min((int64_t)kPix, HW - p0);
        for (int64_t i = 0; i < n; ++i)
            for (int c = 0; c < C; ++c) d[i * C + c] = Out<OUT>::cvt(Elem<TI>::f(s[c * HW + p0 + i]));
    }
}

// Fully vectorised path (every row a whole number of kPix units, 16-byte aligned): a
// grid-stride loop over (row, unit) with two units in flight per thread, grid = resident CTAs.
// The loads are kept as raw 16-byte vectors (4 registers each) until the conversion at store
// time, so the kernel stays at ~40 registers and keeps all 8 CTAs/SM resident.
template <typename TI>
__device__ __forceinline__ float raw_elem(const uint4* raw, int i) {
    if constexpr (sizeof(TI) == 1) {
        return u8_lane_to_f32(reinterpret_cast<const uint32_t*>(raw)[i >> 2], i & 3);
    } else if constexpr (sizeof(TI) == 4) {
        return reinterpret_cast<const float*>(raw)[i];
    } else {
        return __double2float_rn(reinterpret_cast<const double*>(raw)[i]);
    }
}

template <typename TI, int OUT, int C, bool NHWC>
__global__ void __launch_bounds__(kStageThreads)
k_stage_vec(const TI* __restrict__ src, const int64_t* __restrict__ rows, int64_t row0, int64_t HW,
            int64_t upr, int64_t total, typename Out<OUT>::T* __restrict__ dst) {
    using TO = typename Out<OUT>::T;
    constexpr int NV = kPix * (int)sizeof(TI) / 16;   // 16-byte vectors per channel unit
    constexpr int UN = sizeof(TI) == 1 ? 2 : 1;        // units in flight per thread (register budget)
    const int64_t stride = (int64_t)gridDim.x * kStageThreads;
    for (int64_t u0 = (int64_t)blockIdx.x * kStageThreads + threadIdx.x; u0 < total; u0 += UN * stride) {
        uint4 raw[UN][C][NV];
        int64_t r[UN], p[UN];
        bool ok[UN];
#pragma unroll
        for (int j = 0; j < UN; ++j) {
            const int64_t u = u0 + j * stride;
            ok[j] = u < total;
            r[j] = ok[j] ? u / upr : 0;
            p[j] = ok[j] ? (u - r[j] * upr) * kPix : 0;
            if (ok[j]) {
                const TI* s = src + src_row(rows, row0, r[j]) * (int64_t)C * HW + p[j];
#pragma unroll
                for (int c = 0; c < C; ++c)
#pragma unroll
                    for (int v = 0; v < NV; ++v) raw[j][c][v] = reinterpret_cast<const uint4*>(s + c * HW)[v];
            }
        }
#pragma unroll
        for (int j = 0; j < UN; ++j) {
            if (!ok[j]) continue;
            if (NHWC) {
                TO* d = dst + (r[j] * HW + p[j]) * C;
                constexpr int per = 16 / (int)sizeof(TO);          // outputs per 16-byte store
#pragma unroll
                for (int q = 0; q < kPix * C / per; ++q) {
                    TO o[per];
#pragma unroll
                    for (int e = 0; e < per; ++e) {
                        const int k = q * per + e;                 // interleaved index: pixel k / C, channel k % C
                        o[e] = Out<OUT>::cvt(raw_elem<TI>(raw[j][k % C], k / C));
                    }
                    uint4 w;
                    memcpy(&w, o, 16);
                    reinterpret_cast<uint4*>(d)[q] = w;
                }
            } else {
#pragma unroll
                for (int c = 0; c < C; ++c) {
                    TO* d = dst + (r[j] * C + c) * HW + p[j];
                    constexpr int per = 16 / (int)sizeof(TO);
#pragma unroll
                    for (int q = 0; q < kPix / per; ++q) {
                        TO o[per];
#pragma unroll
                        for (int e = 0; e < per; ++e) o[e] = Out<OUT>::cvt(raw_elem<TI>(raw[j][c], q * per + e));
                        uint4 w;
                        memcpy(&w, o, 16);
                        reinterpret_cast<uint4*>(d)[q] = w;
                    }
                }
            }
        }
    }
}

// NCHW -> NHWC through shared memory: a CTA converts a tile of kTilePx pixels x C channels
// (coalesced 16-byte plane loads), writes it NHWC-interleaved into smem, then the whole tile
// leaves with fully coalesced 16-byte stores (lane i writes bytes [16i, 16i+16) of the tile).
constexpr int kTilePx = kStageThreads * kPix;   // 4096 pixels per CTA tile

template <typename TI, int OUT, int C>
__global__ void __launch_bounds__(kStageThreads)
k_stage_nhwc_smem(const TI* __restrict__ src, const int64_t* __restrict__ rows, int64_t row0, int64_t HW,
                  int64_t tiles_per_row, int64_t total_tiles, typename Out<OUT>::T* __restrict__ dst) {
    using TO = typename Out<OUT>::T;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    TO* tile = reinterpret_cast<TO*>(smem_raw);
    for (int64_t t = blockIdx.x; t < total_tiles; t += gridDim.x) {
        const int64_t r = t / tiles_per_row;
        const int64_t p0 = (t - r * tiles_per_row) * kTilePx;
        const int64_t npx = min((int64_t)kTilePx, HW - p0);
        const TI* s = src + src_row(rows, row0, r) * (int64_t)C * HW + p0;
        const int q0 = threadIdx.x * kPix;
        if (q0 + kPix <= npx) {
            float v[C][kPix];
#pragma unroll
            for (int c = 0; c < C; ++c) load_pix<TI>(s + c * HW + q0, v[c], true);
            TO o[kPix * C];
#pragma unroll
            for (int i = 0; i < kPix; ++i)
#pragma unroll
                for (int c = 0; c < C; ++c) o[i * C + c] = Out<OUT>::cvt(v[c][i]);
            store_vec<TO>(tile + (int64_t)q0 * C, o, kPix * C, true);
        } else {
            for (int q = q0; q < npx; ++q)
                for (int c = 0; c < C; ++c) tile[q * C + c] = Out<OUT>::cvt(Elem<TI>::f(s[c * HW + q]));
        }
        __syncthreads();
        const int64_t nbytes = npx * C * (int64_t)sizeof(TO);
        uint4* d16 = reinterpret_cast<uint4*>(dst + (r * HW + p0) * C);
        const uint4* s16 = reinterpret_cast<const uint4*>(tile);
        for (int64_t j = threadIdx.x; j < nbytes / 16; j += kStageThreads) d16[j] = s16[j];
        for (int64_t b = (nbytes / 16) * 16 + threadIdx.x; b < nbytes; b += kStageThreads)
            reinterpret_cast<unsigned char*>(d16)[b] = smem_raw[b];
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------------------------
// NCHW u8 -> NHWC through the bulk-async copy engine (TMA, cp.async.bulk), persistent CTAs.
//
// Each CTA walks tiles t = blockIdx.x, +grid, ... of TP pixels of one row. One elected thread
// keeps S tiles of source planes in flight (one 1-D bulk copy per channel plane into a ring of
// S smem stages, completion counted in bytes on the stage's mbarrier). All threads convert a
// landed stage to the interleaved NHWC tile in one of two smem output buffers, and the elected
// thread sends it with ONE bulk store (smem -> global, bulk_group). So a CTA always has loads of
// the next tiles and the store of the previous tile outstanding while it converts the current
// one, without per-thread register staging; grid = resident CTAs (a multiple of the SM count).
// ---------------------------------------------------------------------------------------------
// (bulk-async PTX helpers: mbs_tma.h)

constexpr int kBulkStages = 3;

template <int TP, int C, typename TO>
constexpr size_t bulk_smem_bytes() {
    return (size_t)kBulkStages * C * TP + 2 * (size_t)TP * C * sizeof(TO);
}

template <int OUT, int C, int TP>
__global__ void __launch_bounds__(kStageThreads)
k_stage_nhwc_bulk(const uint8_t* __restrict__ src, const int64_t* __restrict__ rows, int64_t row0, int64_t HW,
                  int64_t tiles_per_row, int64_t total_tiles, typename Out<OUT>::T* __restrict__ dst) {
    using TO = typename Out<OUT>::T;
    constexpr int PX = TP / kStageThreads;                // pixels per thread in the conversion
    static_assert(PX == 8 || PX == 16, "tile must give 8 or 16 pixels per thread");
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t full[kBulkStages];
    uint8_t* in = smem_raw;                                             // [S][C][TP] source planes
    TO* out = reinterpret_cast<TO*>(smem_raw + (size_t)kBulkStages * C * TP);   // [2][TP*C] NHWC tiles
    const int tid = threadIdx.x;
    const int64_t G = gridDim.x;
    const int64_t n_mine = total_tiles > (int64_t)blockIdx.x ? (total_tiles - blockIdx.x + G - 1) / G : 0;

    auto tile_of = [&](int64_t i, int64_t& r, int64_t& p0, int& npx) {
        const int64_t t = blockIdx.x + i * G;
        r = t / tiles_per_row;
        p0 = (t - r * tiles_per_row) * TP;
        npx = (int)min((int64_t)TP, HW - p0);
    };
    auto issue = [&](int64_t i) {                         // elected thread: tile i's planes -> stage i % S
        int64_t r, p0;
        int npx;
        tile_of(i, r, p0, npx);
        const int s = (int)(i % kBulkStages);
        const uint8_t* base = src + src_row(rows, row0, r) * (int64_t)C * HW + p0;
        mbar_expect_tx(&full[s], (uint32_t)(C * npx));
#pragma unroll
        for (int c = 0; c < C; ++c) bulk_load(in + ((size_t)s * C + c) * TP, base + c * HW, (uint32_t)npx, &full[s]);
    };

    if (tid == 0) {
        for (int s = 0; s < kBulkStages; ++s) mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int64_t i = 0; i < min((int64_t)kBulkStages, n_mine); ++i) issue(i);
    }
    __syncthreads();

    for (int64_t i = 0; i < n_mine; ++i) {
        int64_t r, p0;
        int npx;
        tile_of(i, r, p0, npx);
        const int s = (int)(i % kBulkStages);
        const int ob = (int)(i & 1);
        TO* o = out + (size_t)ob * TP * C;
        if (tid == 0) bulk_wait_read<1>();                // the store of tile i-2 has finished reading out[ob]
        mbar_wait(&full[s], (uint32_t)((i / kBulkStages) & 1));
        __syncthreads();
        const uint8_t* pl = in + (size_t)s * C * TP;
        const int q0 = tid * PX;
        if (q0 + PX <= npx) {
            uint32_t w[C][PX / 4];
#pragma unroll
            for (int c = 0; c < C; ++c) {
                if constexpr (PX == 16) {
                    const uint4 q = *reinterpret_cast<const uint4*>(pl + c * TP + q0);
                    w[c][0] = q.x; w[c][1] = q.y; w[c][2] = q.z; w[c][3] = q.w;
                } else {
                    const uint2 q = *reinterpret_cast<const uint2*>(pl + c * TP + q0);
                    w[c][0] = q.x; w[c][1] = q.y;
                }
            }
            constexpr int per = 16 / (int)sizeof(TO);     // outputs per 16-byte smem store
            uint4* d16 = reinterpret_cast<uint4*>(o + (size_t)q0 * C);
#pragma unroll
            for (int v = 0; v < PX * C / per; ++v) d16[v] = u8_nhwc_vec16<OUT, C, PX / 4>(w, v);
        } else {
            for (int q = q0; q < npx && q < q0 + PX; ++q)
                for (int c = 0; c < C; ++c) o[q * C + c] = Out<OUT>::cvt((float)pl[c * TP + q]);
        }
        fence_proxy_async_smem();                          // generic-proxy smem writes -> visible to the bulk store
        __syncthreads();                                   // stage s consumed, out[ob] complete
        if (tid == 0) {
            bulk_store(dst + (r * HW + p0) * C, o, (uint32_t)(npx * C * sizeof(TO)));
            if (i + kBulkStages < n_mine) issue(i + kBulkStages);
        }
    }
    if (tid == 0) bulk_wait_all();
}

// ---------------------------------------------------------------------------------------------
// NCHW u8 -> NHWC, bulk-async, over the FLATTENED pixel space of the micro-batch with a balanced split:
// CTA b owns the contiguous output pixels [b*per_cta, (b+1)*per_cta) (per_cta a multiple of 16 chosen so
// that grid = the resident CTAs), walked in tiles of TP pixels through a kFlatStages-deep ring. A tile's
// source planes may cross row boundaries (rows are gathered / strided in the source, contiguous in the
// NHWC destination), so each plane is fetched as one bulk copy per row segment. Compared with the per-row
// tiling of k_stage_nhwc_bulk there is no ragged last tile per row and no CTA doing one tile more than
// another (C2: 24.5 tiles per row, 4.3 tiles per CTA -> 18 % of the CTAs ran a fifth tile).
// ---------------------------------------------------------------------------------------------
constexpr int kFlatStages = 4;

template <int TP, int C, typename TO>
constexpr size_t flat_smem_bytes() {
    return (size_t)kFlatStages * C * TP + 2 * (size_t)TP * C * sizeof(TO);
}

template <int OUT, int C, int TP, int NT = kStageThreads>
__global__ void __launch_bounds__(NT)
k_stage_nhwc_flat(const uint8_t* __restrict__ src, const int64_t* __restrict__ rows, int64_t row0, int64_t HW,
                  int64_t total_px, int64_t per_cta, typename Out<OUT>::T* __restrict__ dst) {
    using TO = typename Out<OUT>::T;
    constexpr int PX = TP / NT;
    static_assert(PX == 8 || PX == 16, "tile must give 8 or 16 pixels per thread");
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t full[kFlatStages];
    uint8_t* in = smem_raw;                                                       // [S][C][TP] planes
    TO* out = reinterpret_cast<TO*>(smem_raw + (size_t)kFlatStages * C * TP);     // [2][TP*C] NHWC tiles
    const int tid = threadIdx.x;
    const int64_t begin = (int64_t)blockIdx.x * per_cta;
    const int64_t end = min(total_px, begin + per_cta);
    const int64_t n_mine = end > begin ? (end - begin + TP - 1) / TP : 0;

    auto issue = [&](int64_t i) {                         // elected thread: tile i's planes -> stage i % S
        const int64_t p0 = begin + i * TP;
        const int npx = (int)min((int64_t)TP, end - p0);
        const int s = (int)(i % kFlatStages);
        mbar_expect_tx(&full[s], (uint32_t)(C * npx));
        int done = 0;
        while (done < npx) {                              // one bulk copy per plane per row segment
            const int64_t p = p0 + done;
            const int64_t r = p / HW, off = p - r * HW;
            const int seg = (int)min((int64_t)(npx - done), HW - off);
            const uint8_t* base = src + src_row(rows, row0, r) * (int64_t)C * HW + off;
#pragma unroll
            for (int c = 0; c < C; ++c)
                bulk_load(in + ((size_t)s * C + c) * TP + done, base + c * HW, (uint32_t)seg, &full[s]);
            done += seg;
        }
    };

    if (tid == 0) {
        for (int s = 0; s < kFlatStages; ++s) mbar_init(&full[s], 1);
        mbar_init_fence();
        for (int64_t i = 0; i < min((int64_t)kFlatStages, n_mine); ++i) issue(i);
    }
    __syncthreads();

    for (int64_t i = 0; i < n_mine; ++i) {
        const int64_t p0 = begin + i * TP;
        const int npx = (int)min((int64_t)TP, end - p0);
        const int s = (int)(i % kFlatStages);
        TO* o = out + (size_t)(i & 1) * TP * C;
        if (tid == 0) bulk_wait_read<1>();                // the store of tile i-2 has finished reading out[i&1]
        mbar_wait(&full[s], (uint32_t)((i / kFlatStages) & 1));
        __syncthreads();
        const uint8_t* pl = in + (size_t)s * C * TP;
        const int q0 = tid * PX;
        if (q0 + PX <= npx) {
            uint32_t w[C][PX / 4];
#pragma unroll
            for (int c = 0; c < C; ++c) {
                if constexpr (PX == 16) {
                    const uint4 q = *reinterpret_cast<const uint4*>(pl + c * TP + q0);
                    w[c][0] = q.x; w[c][1] = q.y; w[c][2] = q.z; w[c][3] = q.w;
                } else {
                    const uint2 q = *reinterpret_cast<const uint2*>(pl + c * TP + q0);
                    w[c][0] = q.x; w[c][1] = q.y;
                }
            }
            constexpr int per = 16 / (int)sizeof(TO);     // outputs per 16-byte smem store
            uint4* d16 = reinterpret_cast<uint4*>(o + (size_t)q0 * C);
#pragma unroll
            for (int v = 0; v < PX * C / per; ++v) d16[v] = u8_nhwc_vec16<OUT, C, PX / 4>(w, v);
        } else {
            for (int q = q0; q < npx && q < q0 + PX; ++q)
                for (int c = 0; c < C; ++c) o[q * C + c] = Out<OUT>::cvt((float)pl[c * TP + q]);
        }
        fence_proxy_async_smem();
        __syncthreads();                                  // stage s consumed, out[i&1] complete
        if (tid == 0) {
            bulk_store(dst + p0 * C, o, (uint32_t)(npx * C * sizeof(TO)));
            if (i + kFlatStages < n_mine) issue(i + kFlatStages);
        }
    }
    if (tid == 0) bulk_wait_all();
}

// ---------------------------------------------------------------------------------------------
// Warp-specialised NCHW u8 -> NHWC (default). Same balanced split of the flattened pixel space as
// k_stage_nhwc_flat, but no CTA-wide barrier in the loop (ncu on the flat kernel: 41 % of the warp
// cycles stalled at __syncthreads behind the one thread that issued loads and the tile store, and
// 3.75 issued instructions per staged byte):
//   * warp NCW (the producer) — one lane walks the CTA's pixels with a running (row, offset), no
//     division per tile, and issues each tile's planes as 1-D bulk copies into a kWsStages-deep ring
//     (full[s]: transaction bytes; empty[s]: one arrival per consumer warp);
//   * warps 0..NCW-1 (consumers) — warp w owns the 32*PX-pixel slice w of every tile: it converts its
//     slice into its own double-buffered NHWC buffer, releases the stage, and its lane 0 sends the slice
//     out with its own bulk store. Warps run independently; only the ring couples them.
// u8 -> float is PRMT (byte under the exponent of 2^23, immediate selector, the magic in one register)
// + one packed FADD2 per two elements; bf16 keeps the upper half-words (one PRMT per two outputs).
// ---------------------------------------------------------------------------------------------
constexpr int kWsStages = 4;

template <uint32_t SEL>
__device__ __forceinline__ uint32_t prmt_sel(uint32_t a, uint32_t b) {
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "n"(SEL));
    return d;
}

__device__ __forceinline__ uint32_t u8_under_exp(uint32_t w, uint32_t magic, int b) {   // 0x4B0000vv
    switch (b & 3) {                                     // b is a compile-time constant after unrolling
        case 0: return prmt_sel<0x7440>(w, magic);
        case 1: return prmt_sel<0x7441>(w, magic);
        case 2: return prmt_sel<0x7442>(w, magic);
        default: return prmt_sel<0x7443>(w, magic);
    }
}

__device__ __forceinline__ void sub_2p23_x2(uint32_t& a, uint32_t& b) {   // (a, b) -= 2^23, exact, one FADD2
    uint64_t v;
    asm("mov.b64 %0, {%1, %2};" : "=l"(v) : "r"(a), "r"(b));
    asm("add.rn.f32x2 %0, %0, %1;" : "+l"(v) : "l"(0xCB000000CB000000ull));
    asm("mov.b64 {%0, %1}, %2;" : "=r"(a), "=r"(b) : "l"(v));
}

template <int C, typename TO>
constexpr size_t ws_smem_bytes(int px, int ncw) {
    return (size_t)kWsStages * C * ncw * 32 * px + (size_t)ncw * 2 * 32 * px * C * sizeof(TO);
}

template <int OUT, int C, int PX, int NCW>
__global__ void __launch_bounds__((NCW + 1) * 32)
k_stage_nhwc_ws(const uint8_t* __restrict__ src, const int64_t* __restrict__ rows, int64_t row0, int64_t HW,
                int64_t total_px, int64_t per_cta, typename Out<OUT>::T* __restrict__ dst) {
    using TO = typename Out<OUT>::T;
    constexpr int WP = 32 * PX, TP = NCW * WP, E = PX * C;   // px per warp slice, px per tile, outputs per lane
    static_assert(PX == 8 || PX == 16, "8 or 16 pixels per lane");
    static_assert(OUT != MBS_F16, "f16 output takes the flat kernel");
    extern __shared__ __align__(128) unsigned char smem_raw[];
    __shared__ __align__(8) uint64_t full[kWsStages], empty[kWsStages];
    uint8_t* in = smem_raw;                                                        // [S][C][TP]
    TO* out = reinterpret_cast<TO*>(smem_raw + (size_t)kWsStages * C * TP);       // [NCW][2][WP*C]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t begin = (int64_t)blockIdx.x * per_cta;
    const int64_t end = min(total_px, begin + per_cta);
    const int64_t n_mine = end > begin ? (end - begin + TP - 1) / TP : 0;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kWsStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NCW);
        }
        mbar_init_fence();
    }
    __syncthreads();

    if (warp == NCW) {                                    // producer
        if (lane != 0) return;
        int64_t r = begin / HW, off = begin - r * HW;
        int64_t srow = r < total_px / HW ? src_row(rows, row0, r) : 0;
        for (int64_t i = 0; i < n_mine; ++i) {
            const int s = (int)(i % kWsStages);
            if (i >= kWsStages) mbar_wait(&empty[s], (uint32_t)(((i / kWsStages) + 1) & 1));
            const int npx = (int)min((int64_t)TP, end - (begin + i * TP));
            mbar_expect_tx(&full[s], (uint32_t)(C * npx));
            for (int done = 0; done < npx;) {             // one bulk copy per plane per row segment
                const int seg = (int)min((int64_t)(npx - done), HW - off);
                const uint8_t* base = src + srow * (int64_t)C * HW + off;
#pragma unroll
                for (int c = 0; c < C; ++c)
                    bulk_load(in + ((size_t)s * C + c) * TP + done, base + c * HW, (uint32_t)seg, &full[s]);
                done += seg;
                off += seg;
                if (off == HW) {
                    off = 0;
                    ++r;
                    if (r * HW < end) srow = src_row(rows, row0, r);
                }
            }
        }
        return;
    }

    const uint32_t magic = 0x4B000000u;
    const int q0 = warp * WP + lane * PX;                 // this lane's first pixel within a tile
    for (int64_t i = 0; i < n_mine; ++i) {
        const int s = (int)(i % kWsStages);
        const int64_t p0 = begin + i * TP;
        const int npx = (int)min((int64_t)TP, end - p0);
        const int wn = min(WP, npx - warp * WP);          // pixels of this warp's slice (<= 0: none)
        TO* o = out + ((size_t)warp * 2 + (size_t)(i & 1)) * WP * C;
        if (lane == 0) bulk_wait_read<1>();               // this warp's store of tile i-2 has left o
        __syncwarp();
        mbar_wait(&full[s], (uint32_t)((i / kWsStages) & 1));
        const uint8_t* pl = in + (size_t)s * C * TP;
        const bool mine = q0 + PX <= npx;                 // npx is a multiple of 16: whole lanes only
        uint32_t w[C][PX / 4];
        if (mine) {
#pragma unroll
            for (int c = 0; c < C; ++c) {
                if constexpr (PX == 16) {
                    const uint4 q = *reinterpret_cast<const uint4*>(pl + c * TP + q0);
                    w[c][0] = q.x; w[c][1] = q.y; w[c][2] = q.z; w[c][3] = q.w;
                } else {
                    const uint2 q = *reinterpret_cast<const uint2*>(pl + c * TP + q0);
                    w[c][0] = q.x; w[c][1] = q.y;
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);            // this warp is done reading stage s
        if (mine) {
            uint32_t f[E];                                // NHWC order: element k = pixel k / C, channel k % C
#pragma unroll
            for (int k = 0; k < E; ++k) f[k] = u8_under_exp(w[k % C][(k / C) >> 2], magic, (k / C) & 3);
#pragma unroll
            for (int k = 0; k < E; k += 2) sub_2p23_x2(f[k], f[k + 1]);
            uint4* d16 = reinterpret_cast<uint4*>(o + (size_t)(lane * PX) * C);
            if constexpr (OUT == MBS_BF16) {
#pragma unroll
                for (int v = 0; v < E / 8; ++v)
                    d16[v] = make_uint4(prmt_sel<0x7632>(f[8 * v], f[8 * v + 1]), prmt_sel<0x7632>(f[8 * v + 2], f[8 * v + 3]),
                                        prmt_sel<0x7632>(f[8 * v + 4], f[8 * v + 5]), prmt_sel<0x7632>(f[8 * v + 6], f[8 * v + 7]));
            } else {
#pragma unroll
                for (int v = 0; v < E / 4; ++v) d16[v] = make_uint4(f[4 * v], f[4 * v + 1], f[4 * v + 2], f[4 * v + 3]);
            }
        }
        fence_proxy_async_smem();                         // generic-proxy smem writes -> the bulk store
        __syncwarp();
        if (lane == 0 && wn > 0) bulk_store(dst + (p0 + warp * WP) * C, o, (uint32_t)(wn * C * sizeof(TO)));
    }
    if (lane == 0) bulk_wait_all();
}

static int stage_path() {
    // A/B only: 0 = per-row, 1 = grid-stride vec, 2 = smem, 3 = bulk-async per row, 4 = bulk-async over the
    // flattened, evenly split pixel space (default), 5 = the same split, warp-specialised (measured slower:
    // 12.3 vs 11.7 us per C2 micro-batch, profiles/r02_k2_ws_ab.txt)
    const char* e = getenv("MBS_K2_PATH");
    return e ? atoi(e) : 4;
}

static int ws_px() {   // A/B only: MBS_K2_WS_PX=16 -> 16 pixels per lane (4096-pixel tiles)
    const char* e = getenv("MBS_K2_WS_PX");
    return (e && atoi(e) == 16) ? 16 : 8;
}

static bool flat_small() {   // A/B only: MBS_K2_FLAT=128 -> 128-thread CTAs on 1024-pixel tiles (more CTAs per SM)
    const char* e = getenv("MBS_K2_FLAT");
    return e && atoi(e) == 128;
}

static int bulk_tile() {
    const char* e = getenv("MBS_K2_TILE");   // A/B only: 2048 (default) or 4096 pixels per tile
    return (e && atoi(e) == 4096) ? 4096 : 2048;
}

static bool is_device_memory(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice;
}

static int sm_count() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) sms = 148;
    }
    return sms;
}

template <int OUT, int C, int TP>
static int launch_bulk(const uint8_t* s, const int64_t* rows, int64_t row0, int64_t n_rows, int64_t HW,
                       typename Out<OUT>::T* d, cudaStream_t st) {
    using TO = typename Out<OUT>::T;
    auto kern = k_stage_nhwc_bulk<OUT, C, TP>;
    constexpr size_t sm = bulk_smem_bytes<TP, C, TO>();
    static int per_sm = 0;                                 // resident CTAs per SM (per template instance)
    if (!per_sm) {
        MBS_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        MBS_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kStageThreads, sm));
        if (per_sm < 1) per_sm = 1;
    }
    const int64_t tpr = (HW + TP - 1) / TP, total = n_rows * tpr;
    const int grid = (int)std::min<int64_t>(total, (int64_t)sm_count() * per_sm);
    kern<<<grid, kStageThreads, sm, st>>>(s, rows, row0, HW, tpr, total, d);
    MBS_CK_LAUNCH("k_stage_nhwc_bulk");
    return MBS_OK;
}

template <int OUT, int C, int TP, int NT = kStageThreads>
static int launch_flat(const uint8_t* s, const int64_t* rows, int64_t row0, int64_t n_rows, int64_t HW,
                       typename Out<OUT>::T* d, cudaStream_t st) {
    using TO = typename Out<OUT>::T;
    auto kern = k_stage_nhwc_flat<OUT, C, TP, NT>;
    constexpr size_t sm = flat_smem_bytes<TP, C, TO>();
    static int per_sm = 0;
    if (!per_sm) {
        MBS_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        MBS_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, sm));
        if (per_sm < 1) per_sm = 1;
    }
    const int64_t total = n_rows * HW;
    static const int cap = getenv("MBS_K2_CTAS_PER_SM") ? atoi(getenv("MBS_K2_CTAS_PER_SM")) : 0;  // A/B only
    const int64_t resident = (int64_t)sm_count() * (cap > 0 ? std::min(cap, per_sm) : per_sm);
    int64_t per_cta = (total + resident - 1) / resident;
    per_cta = std::max<int64_t>(16, (per_cta + 15) / 16 * 16);   // 16-byte aligned bulk copies
    const int grid = (int)((total + per_cta - 1) / per_cta);
    kern<<<grid, NT, sm, st>>>(s, rows, row0, HW, total, per_cta, d);
    MBS_CK_LAUNCH("k_stage_nhwc_flat");
    return MBS_OK;
}

template <int OUT, int C, int PX, int NCW = 8>
static int launch_ws(const uint8_t* s, const int64_t* rows, int64_t row0, int64_t n_rows, int64_t HW,
                     typename Out<OUT>::T* d, cudaStream_t st) {
    using TO = typename Out<OUT>::T;
    auto kern = k_stage_nhwc_ws<OUT, C, PX, NCW>;
    constexpr int NT = (NCW + 1) * 32;
    constexpr size_t sm = ws_smem_bytes<C, TO>(PX, NCW);
    static int per_sm = 0;
    if (!per_sm) {
        MBS_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        MBS_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, sm));
        if (per_sm < 1) per_sm = 1;
    }
    const int64_t total = n_rows * HW;
    static const int cap = getenv("MBS_K2_CTAS_PER_SM") ? atoi(getenv("MBS_K2_CTAS_PER_SM")) : 0;  // A/B only
    const int64_t resident = (int64_t)sm_count() * (cap > 0 ? std::min(cap, per_sm) : per_sm);
    int64_t per_cta = (total + resident - 1) / resident;
    per_cta = std::max<int64_t>(16, (per_cta + 15) / 16 * 16);   // 16-byte aligned bulk copies
    const int grid = (int)((total + per_cta - 1) / per_cta);
    kern<<<grid, NT, sm, st>>>(s, rows, row0, HW, total, per_cta, d);
    MBS_CK_LAUNCH("k_stage_nhwc_ws");
    return MBS_OK;
}

static int resident_grid(int64_t units) {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) sms = 148;
    }
    const int64_t want = (units + kStageThreads - 1) / kStageThreads;
    return (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sms * (2048 / kStageThreads)));
}

// Generic NHWC for any C (scalar; one thread per output element).
template <typename TI, int OUT>
__global__ void __launch_bounds__(kStageThreads)
k_stage_nhwc_generic(const TI* __restrict__ src, const int64_t* __restrict__ rows, int64_t row0, int64_t C,
                     int64_t HW, typename Out<OUT>::T* __restrict__ dst) {
    const int64_t r = blockIdx.y;
    const int64_t e = (int64_t)blockIdx.x * kStageThreads + threadIdx.x;
    if (e >= C * HW) return;
    const int64_t p = e / C, c = e % C;
    dst[r * C * HW + e] = Out<OUT>::cvt(Elem<TI>::f(src[src_row(rows, row0, r) * C * HW + c * HW + p]));
}

template <typename V>
__global__ void __launch_bounds__(kStageThreads)
k_gather_rows(const V* __restrict__ src, const int64_t* __restrict__ rows, int64_t row0, int64_t nv,
              V* __restrict__ dst) {
    const int64_t r = blockIdx.y;
    const V* s = src + src_row(rows, row0, r) * nv;
    V* d = dst + r * nv;
    for (int64_t i = (int64_t)blockIdx.x * kStageThreads + threadIdx.x; i < nv; i += (int64_t)gridDim.x * kStageThreads)
        d[i] = s[i];
}

template <typename TI, int OUT>
static int stage_typed(const void* src, const int64_t* rows, int64_t row0, int64_t n_rows, int64_t C, int64_t H,
                       int64_t W, void* dst, int layout, cudaStream_t st) {
    using TO = typename Out<OUT>::T;
    const int64_t HW = H * W, E = C * HW;
    const auto* s = static_cast<const TI*>(src);
    auto* d = static_cast<TO*>(dst);
    const uintptr_t sa = reinterpret_cast<uintptr_t>(src), da = reinterpret_cast<uintptr_t>(dst);
    if (n_rows > 65535) return invalid("mbs_stage: at most 65535 rows per call");
    {
        // fully vectorised grid-stride path: whole kPix units per channel plane, 16-byte aligned
        const bool nhwc = layout == MBS_NHWC && C > 1;
        const bool plane_ok = (HW % kPix == 0) && ((HW * (int64_t)sizeof(TI)) % 16 == 0) && (sa % 16 == 0) &&
                              (da % 16 == 0) && ((kPix * sizeof(TO)) % 16 == 0);
        const int path = stage_path();
        if constexpr (sizeof(TI) == 1) {
            if (path == 5 && OUT != MBS_F16 && nhwc && C <= 4 && HW % 16 == 0 && sa % 16 == 0 && da % 16 == 0 &&
                is_device_memory(src)) {
                if constexpr (OUT != MBS_F16) {
                    const bool wide = ws_px() == 16;
                    switch (C) {
                        case 2: return wide ? launch_ws<OUT, 2, 16>(s, rows, row0, n_rows, HW, d, st)
                                            : launch_ws<OUT, 2, 8>(s, rows, row0, n_rows, HW, d, st);
                        case 3: return wide ? launch_ws<OUT, 3, 16>(s, rows, row0, n_rows, HW, d, st)
                                            : launch_ws<OUT, 3, 8>(s, rows, row0, n_rows, HW, d, st);
                        default: return wide ? launch_ws<OUT, 4, 16>(s, rows, row0, n_rows, HW, d, st)
                                             : launch_ws<OUT, 4, 8>(s, rows, row0, n_rows, HW, d, st);
                    }
                }
            }
            if ((path == 4 || path == 5) && nhwc && C <= 4 && HW % 16 == 0 && sa % 16 == 0 && da % 16 == 0 &&
                is_device_memory(src)) {
                switch (C) {
                    case 2: return launch_flat<OUT, 2, 2048>(s, rows, row0, n_rows, HW, d, st);
                    case 3: return flat_small() ? launch_flat<OUT, 3, 1024, 128>(s, rows, row0, n_rows, HW, d, st)
                                                : launch_flat<OUT, 3, 2048>(s, rows, row0, n_rows, HW, d, st);
                    default: return launch_flat<OUT, 4, 2048>(s, rows, row0, n_rows, HW, d, st);
                }
            }
            if (path == 3 && nhwc && C <= 4 && HW % 16 == 0 && sa % 16 == 0 && da % 16 == 0 &&
                is_device_memory(src)) {
                const bool small = OUT == MBS_F32 || bulk_tile() == 2048;   // f32 tiles: 2048 px keeps 2 CTAs/SM
                switch (C) {
                    case 2: return small ? launch_bulk<OUT, 2, 2048>(s, rows, row0, n_rows, HW, d, st)
                                         : launch_bulk<OUT, 2, 4096>(s, rows, row0, n_rows, HW, d, st);
                    case 3: return small ? launch_bulk<OUT, 3, 2048>(s, rows, row0, n_rows, HW, d, st)
                                         : launch_bulk<OUT, 3, 4096>(s, rows, row0, n_rows, HW, d, st);
                    default: return small ? launch_bulk<OUT, 4, 2048>(s, rows, row0, n_rows, HW, d, st)
                                          : launch_bulk<OUT, 4, 4096>(s, rows, row0, n_rows, HW, d, st);
                }
            }
        }
        if ((path >= 2 && path <= 5) && nhwc && C <= 4 && (HW * (int64_t)sizeof(TI)) % 16 == 0 && sa % 16 == 0 && da % 16 == 0 &&
            ((int64_t)kTilePx * C * sizeof(TO)) % 16 == 0 && (HW * C * (int64_t)sizeof(TO)) % 16 == 0) {
            const int64_t tpr = (HW + kTilePx - 1) / kTilePx, total = n_rows * tpr;
            const size_t sm = (size_t)kTilePx * C * sizeof(TO);
            // one CTA per tile (the block scheduler balances); MBS_K2_GRID=resident caps it at the resident CTAs
            static const bool cap = getenv("MBS_K2_GRID") && strcmp(getenv("MBS_K2_GRID"), "resident") == 0;
            const int grid = (int)std::min<int64_t>(total, cap ? resident_grid(total * kStageThreads) : 2147483647);
#define MBS_STAGE_SMEM(CC)                                                                                   \
    do {                                                                                                     \
        auto kern = k_stage_nhwc_smem<TI, OUT, CC>;                                                          \
        if (sm > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm); \
        kern<<<grid, kStageThreads, sm, st>>>(s, rows, row0, HW, tpr, total, d);                             \
    } while (0)
            switch (C) {
                case 2: MBS_STAGE_SMEM(2); break;
                case 3: MBS_STAGE_SMEM(3); break;
                default: MBS_STAGE_SMEM(4); break;
            }
#undef MBS_STAGE_SMEM
            MBS_CK_LAUNCH("k_stage_nhwc_smem");
            return MBS_OK;
        }
        if (path == 1 && plane_ok && (layout == MBS_NCHW || layout == MBS_NHWC) && C >= 1 && C <= 4) {
            const int64_t upr = HW / kPix, total = n_rows * upr;
            const int grid = resident_grid((total + 1) / 2);
#define MBS_STAGE_VEC(CC)                                                                                   \
    do {                                                                                                    \
        if (nhwc) k_stage_vec<TI, OUT, CC, true><<<grid, kStageThreads, 0, st>>>(s, rows, row0, HW, upr, total, d); \
        else k_stage_vec<TI, OUT, CC, false><<<grid, kStageThreads, 0, st>>>(s, rows, row0, HW, upr, total, d);     \
    } while (0)
            switch (C) {
                case 1: MBS_STAGE_VEC(1); break;
                case 2: MBS_STAGE_VEC(2); break;
                case 3: MBS_STAGE_VEC(3); break;
                default: MBS_STAGE_VEC(4); break;
            }
#undef MBS_STAGE_VEC
            MBS_CK_LAUNCH("k_stage_vec");
            return MBS_OK;
        }
    }
    if (layout == MBS_NCHW || C == 1) {
        // vector path needs 16-byte aligned rows in both src and dst
        const bool vec = (sa % 16 == 0) && (da % 16 == 0) && ((E * (int64_t)sizeof(TI)) % 16 == 0) &&
                         ((E * (int64_t)sizeof(TO)) % 16 == 0) && ((kPix * sizeof(TO)) % 16 == 0);
        dim3 grid((unsigned)((E + (int64_t)kStageThreads * kPix - 1) / ((int64_t)kStageThreads * kPix)), (unsigned)n_rows);
        k_stage_nchw<TI, OUT><<<grid, kStageThreads, 0, st>>>(s, rows, row0, E, d, vec);
    } else if (layout == MBS_NHWC && C <= 4) {
        const bool vec = (sa % 16 == 0) && (da % 16 == 0) && ((HW * (int64_t)sizeof(TI)) % 16 == 0) &&
                         ((kPix * C * sizeof(TO)) % 16 == 0) && ((E * (int64_t)sizeof(TO)) % 16 == 0);
        dim3 grid((unsigned)((HW + (int64_t)kStageThreads * kPix - 1) / ((int64_t)kStageThreads * kPix)), (unsigned)n_rows);
        switch (C) {
            case 2: k_stage_nhwc<TI, OUT, 2><<<grid, kStageThreads, 0, st>>>(s, rows, row0, HW, d, vec); break;
            case 3: k_stage_nhwc<TI, OUT, 3><<<grid, kStageThreads, 0, st>>>(s, rows, row0, HW, d, vec); break;
            default: k_stage_nhwc<TI, OUT, 4><<<grid, kStageThreads, 0, st>>>(s, rows, row0, HW, d, vec); break;
        }
    } else if (layout == MBS_NHWC) {
        dim3 grid((unsigned)((E + kStageThreads - 1) / kStageThreads), (unsigned)n_rows);
        k_stage_nhwc_generic<TI, OUT><<<grid, kStageThreads, 0, st>>>(s, rows, row0, C, HW, d);
    } else {
        return invalid("mbs_stage: unknown layout");
    }
    MBS_CK_LAUNCH("k_stage");
    return MBS_OK;
}

}  // namespace mbs

using namespace mbs;

extern "C" {

int mbs_stage(const void* src, int src_dtype, const int64_t* rows, int64_t row0, int64_t n_rows, int64_t C,
              int64_t H, int64_t W, void* dst, int dst_dtype, int dst_layout, void* stream) {
    if (!src || !dst || n_rows < 0 || C < 1 || H < 1 || W < 1 || (!rows && row0 < 0))
        return invalid("mbs_stage: bad arguments");
    if (n_rows == 0) return MBS_OK;
    auto st = (cudaStream_t)stream;
    if (src_dtype == MBS_U8) {
        if (dst_dtype == MBS_F32) return stage_typed<uint8_t, MBS_F32>(src, rows, row0, n_rows, C, H, W, dst, dst_layout, st);
        if (dst_dtype == MBS_BF16) return stage_typed<uint8_t, MBS_BF16>(src, rows, row0, n_rows, C, H, W, dst, dst_layout, st);
        if (dst_dtype == MBS_F16) return stage_typed<uint8_t, MBS_F16>(src, rows, row0, n_rows, C, H, W, dst, dst_layout, st);
    } else if (src_dtype == MBS_F32) {
        if (dst_dtype == MBS_F32) return stage_typed<float, MBS_F32>(src, rows, row0, n_rows, C, H, W, dst, dst_layout, st);
        if (dst_dtype == MBS_BF16) return stage_typed<float, MBS_BF16>(src, rows, row0, n_rows, C, H, W, dst, dst_layout, st);
        if (dst_dtype == MBS_F16) return stage_typed<float, MBS_F16>(src, rows, row0, n_rows, C, H, W, dst, dst_layout, st);
    } else if (src_dtype == MBS_F64) {
        if (dst_dtype == MBS_F32) return stage_typed<double, MBS_F32>(src, rows, row0, n_rows, C, H, W, dst, dst_layout, st);
        if (dst_dtype == MBS_BF16) return stage_typed<double, MBS_BF16>(src, rows, row0, n_rows, C, H, W, dst, dst_layout, st);
        if (dst_dtype == MBS_F16) return stage_typed<double, MBS_F16>(src, rows, row0, n_rows, C, H, W, dst, dst_layout, st);
    }
    return invalid("mbs_stage: unsupported dtype pair");
}

int mbs_gather_rows(const void* src, const int64_t* rows, int64_t row0, int64_t n_rows, int64_t row_bytes, void* dst,
                    void* stream) {
    if (!src || !dst || n_rows < 0 || row_bytes < 1 || (!rows && row0 < 0)) return invalid("mbs_gather_rows: bad arguments");
    if (n_rows == 0) return MBS_OK;
    if (n_rows > 65535) return invalid("mbs_gather_rows: at most 65535 rows per call");
    auto st = (cudaStream_t)stream;
    const uintptr_t a = reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst);
    auto grid_for = [&](int64_t nv) {
        return dim3((unsigned)std::min<int64_t>((nv + kStageThreads - 1) / kStageThreads, 1024), (unsigned)n_rows);
    };
    if (a % 16 == 0 && row_bytes % 16 == 0) {
        const int64_t nv = row_bytes / 16;
        k_gather_rows<uint4><<<grid_for(nv), kStageThreads, 0, st>>>((const uint4*)src, rows, row0, nv, (uint4*)dst);
    } else if (a % 8 == 0 && row_bytes % 8 == 0) {
        const int64_t nv = row_bytes / 8;
        k_gather_rows<uint2><<<grid_for(nv), kStageThreads, 0, st>>>((const uint2*)src, rows, row0, nv, (uint2*)dst);
    } else if (a % 4 == 0 && row_bytes % 4 == 0) {
        const int64_t nv = row_bytes / 4;
        k_gather_rows<uint32_t><<<grid_for(nv), kStageThreads, 0, st>>>((const uint32_t*)src, rows, row0, nv, (uint32_t*)dst);
    } else {
        k_gather_rows<uint8_t><<<grid_for(row_bytes), kStageThreads, 0, st>>>((const uint8_t*)src, rows, row0, row_bytes, (uint8_t*)dst);
    }
    MBS_CK_LAUNCH("k_gather_rows");
    return MBS_OK;
}

}  // extern "C"
