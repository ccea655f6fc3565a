// K7: im2col of the model's first convolution (3 input channels) so it runs as one cuBLAS GEMM.
//
// A 3-channel stem conv cannot use the sm_100 implicit-GEMM kernels (C_in is not a multiple of
// 8): cuDNN falls back to sm80 kernels at ~37 TFLOP/s — 0.76 ms forward + 0.37 ms weight-grad of
// the 14.6 ms ResNet-50 micro-batch step (profiles/r01_c2_v3_launches.md); zero-padding the input
// to 8 channels is slower still for the 7x7 stem (tools/probe_stem.py). The patch matrix
// cols[M = N*Ho*Wo, Kp] (K = kh*kw*C ordered (kh, kw, c), zero-padded to Kp, a multiple of 8) is
// written once per micro-batch; forward = cols @ W[Kp, O] (the output IS the channels-last
// activation), weight grad = cols^T @ dy; both are plain library GEMMs.
//
// Layout: x [N, H, W, C] channels-last; cols row-major [M, Kp]. Algorithmic bytes: read x (~once,
// window re-reads hit L1/L2) + write M*Kp elements.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string.h>

#include <algorithm>

#include "mbs_common.h"

namespace mbs {

struct ColGeom {
    int64_t N, H, W, C, Ho, Wo, Kp;
    int k, s, p;
};

constexpr int kColMaxKp = 512;
constexpr int kColTileBytes = 16384;

// A CTA builds TM consecutive rows of cols in shared memory, then stores them as one contiguous
// TM*Kp run with 16-byte coalesced stores. Filling: work item (kh, i) copies the k*C contiguous
// input elements of kernel row kh for output pixel m0+i (consecutive threads take consecutive
// pixels of the same kernel row, so their global reads are neighbours); padding columns are zeroed.
// 32-bit index math (the host checks every offset fits).
// KS, CS > 0: kernel size and channel count are compile-time (the ResNet stem's 7x7x3): a work item's
// k*C loads unroll and are all in flight at once (the runtime loop kept one load per thread in
// flight: 1.8 TB/s).
template <typename T, int KS = 0, int CS = 0>
__global__ void __launch_bounds__(256) k_im2col(const T* __restrict__ x, T* __restrict__ cols, ColGeom g0, int TM) {
    extern __shared__ __align__(16) unsigned char csm[];
    T* tile = reinterpret_cast<T*>(csm);
    const int H = (int)g0.H, W = (int)g0.W, Ho = (int)g0.Ho, Wo = (int)g0.Wo, Kp = (int)g0.Kp;
    const int C = CS > 0 ? CS : (int)g0.C;
    const int k = KS > 0 ? KS : g0.k;
    const int s = g0.s, p = g0.p;
    const int KC = k * C, K = k * KC;
    const int64_t M = g0.N * g0.Ho * g0.Wo;
    const int64_t n_tiles = (M + TM - 1) / TM;
    cudaGridDependencySynchronize();
    for (int64_t tt = blockIdx.x; tt < n_tiles; tt += gridDim.x) {
        const int64_t m0 = tt * TM;
        const int rows = (int)min((int64_t)TM, M - m0);
        for (int it = threadIdx.x; it < k * TM; it += blockDim.x) {
            const int kh = it / TM, i = it - kh * TM;
            if (i >= rows) continue;
            const int m = (int)(m0 + i);
            const int ow = m % Wo, q = m / Wo;
            const int oh = q % Ho, n = q / Ho;
            const int ih = oh * s - p + kh, iw0 = ow * s - p;
            T* d = tile + i * Kp + kh * KC;
            if (ih < 0 || ih >= H) {
#pragma unroll
                for (int j = 0; j < KC; ++j) d[j] = T(0.f);
            } else {
                const T* src = x + ((size_t)(n * H + ih) * W) * C;
                if constexpr (KS > 0 && CS > 0) {
                    T v[KS * CS];
#pragma unroll
                    for (int kw = 0; kw < KS; ++kw) {
                        const int iw = iw0 + kw;
                        const bool in = iw >= 0 && iw < W;
#pragma unroll
                        for (int c = 0; c < CS; ++c) v[kw * CS + c] = in ? src[iw * CS + c] : T(0.f);
                    }
#pragma unroll
                    for (int j = 0; j < KS * CS; ++j) d[j] = v[j];
                } else {
                    for (int kw = 0; kw < k; ++kw) {
                        const int iw = iw0 + kw;
                        const bool in = iw >= 0 && iw < W;
                        for (int c = 0; c < C; ++c) d[kw * C + c] = in ? src[iw * C + c] : T(0.f);
                    }
                }
            }
            if (kh == 0)
                for (int j = K; j < Kp; ++j) tile[i * Kp + j] = T(0.f);
        }
        __syncthreads();
        const int64_t n16 = (int64_t)rows * Kp * sizeof(T) / 16;   // Kp*sizeof(T) is a multiple of 16
        const uint4* s16 = reinterpret_cast<const uint4*>(tile);
        uint4* d16 = reinterpret_cast<uint4*>(cols + m0 * Kp);
        for (int64_t v = threadIdx.x; v < n16; v += blockDim.x) d16[v] = s16[v];
        __syncthreads();
    }
}

// Row variant (the ResNet stem and U-Net first conv: compile-time k, C, Kp): one CTA per output row
// (n, oh). Its k input rows are staged once in shared memory with 16-byte coalesced loads (zero
// columns for the padding), then each thread owns one fixed 16-byte chunk j of the Kp-wide patch
// row — the 8 (kh, kw, c) sources of that chunk are computed once — and walks the row's output
// pixels: 8 two-byte shared loads, one 16-byte coalesced global store per pixel. The tile variant
// above spent its time on 2-byte shared stores and barriers (ncu: L1 91 % busy, 2.1 TB/s).
template <typename T, int KS, int CS, int KP>
__global__ void __launch_bounds__(256) k_im2col_rows(const T* __restrict__ x, T* __restrict__ cols, ColGeom g0,
                                                     int LP, int RS) {
    constexpr int NCH = KP * (int)sizeof(T) / 16;   // 16-byte chunks per patch row
    constexpr int EPC = 16 / (int)sizeof(T);        // elements per chunk
    constexpr int KK = KS * KS * CS;                // real (unpadded) patch length
    constexpr int ISTEP = 256 / NCH;
    extern __shared__ __align__(16) unsigned char csm[];
    T* rows = reinterpret_cast<T*>(csm);
    const int H = (int)g0.H, W = (int)g0.W, Ho = (int)g0.Ho, Wo = (int)g0.Wo;
    const int s = g0.s, p = g0.p;
    const int tid = threadIdx.x;
    const int j = tid % NCH, i0 = tid / NCH;
    int off[EPC];
    bool live[EPC];
#pragma unroll
    for (int e = 0; e < EPC; ++e) {
        const int k = j * EPC + e;
        const int kh = k / (KS * CS), r = k - kh * (KS * CS);
        live[e] = k < KK;
        off[e] = live[e] ? kh * RS + LP - p * CS + r : 0;
    }
    const int WC = W * CS;
    const bool vec = (WC * (int)sizeof(T)) % 16 == 0 && (LP * (int)sizeof(T)) % 16 == 0;
    cudaGridDependencySynchronize();
    for (int64_t row = blockIdx.x; row < g0.N * Ho; row += gridDim.x) {
        const int n = (int)(row / Ho), oh = (int)(row - (int64_t)n * Ho);
        // stage: k input rows, zero padding columns / rows
        for (int kh = 0; kh < KS; ++kh) {
            const int ih = oh * s - p + kh;
            T* dst = rows + kh * RS;
            if (ih < 0 || ih >= H) {
                for (int q = tid; q < RS; q += blockDim.x) dst[q] = T(0.f);
                continue;
            }
            const T* src = x + ((int64_t)n * H + ih) * WC;
            for (int q = tid; q < LP; q += blockDim.x) dst[q] = T(0.f);
            for (int q = LP + WC + tid; q < RS; q += blockDim.x) dst[q] = T(0.f);
            if (vec) {
                const uint4* s16 = reinterpret_cast<const uint4*>(src);
                uint4* d16 = reinterpret_cast<uint4*>(dst + LP);
                for (int q = tid; q < WC * (int)sizeof(T) / 16; q += blockDim.x) d16[q] = __ldg(s16 + q);
            } else {
                for (int q = tid; q < WC; q += blockDim.x) dst[LP + q] = src[q];
            }
        }
        __syncthreads();
        if (i0 < ISTEP) {
            T* out = cols + row * Wo * KP + j * EPC;
            for (int i = i0; i < Wo; i += ISTEP) {
                const int base = i * s * CS;
                uint16_t v[EPC];
#pragma unroll
                for (int e = 0; e < EPC; ++e) {
                    const T t = live[e] ? rows[base + off[e]] : T(0.f);
                    v[e] = *reinterpret_cast<const uint16_t*>(&t);
                }
                uint4 u;
                if constexpr (sizeof(T) == 2) {
                    u.x = v[0] | ((uint32_t)v[1] << 16);
                    u.y = v[2] | ((uint32_t)v[3] << 16);
                    u.z = v[4] | ((uint32_t)v[5] << 16);
                    u.w = v[6] | ((uint32_t)v[7] << 16);
                }
                *reinterpret_cast<uint4*>(out + (int64_t)i * KP) = u;
            }
        }
        __syncthreads();
    }
}

static int im2col_sms() {
    static int n = 0;
    if (n <= 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    }
    return n;
}

}  // namespace mbs

using namespace mbs;

extern "C" {

int mbs_im2col(const void* x, void* cols, int dtype, int64_t N, int64_t H, int64_t W, int64_t C, int k, int s, int p,
               int64_t Kp, void* stream) {
    if (!x || !cols) return invalid("mbs_im2col: null pointer");
    if (dtype != MBS_BF16 && dtype != MBS_F32) return invalid("mbs_im2col: dtype must be MBS_BF16 or MBS_F32");
    if (N < 1 || H < 1 || W < 1 || C < 1 || k < 1 || s < 1 || p < 0) return invalid("mbs_im2col: bad geometry");
    if (Kp < (int64_t)k * k * C) return invalid("mbs_im2col: Kp < k*k*C");
    if (Kp > kColMaxKp) return invalid("mbs_im2col: Kp > 512");
    const int64_t Ho = (H + 2 * p - k) / s + 1, Wo = (W + 2 * p - k) / s + 1;
    if (Ho < 1 || Wo < 1) return invalid("mbs_im2col: window larger than input");
    ColGeom g{N, H, W, C, Ho, Wo, Kp, k, s, p};
    const int es = dtype == MBS_BF16 ? 2 : 4;
    if ((Kp * es) % 16 || (reinterpret_cast<uintptr_t>(cols) & 15))
        return invalid("mbs_im2col: Kp * sizeof(elem) must be a multiple of 16 and cols 16-byte aligned");
    if (N * H * W * C >= INT32_MAX || N * Ho * Wo >= INT32_MAX) return invalid("mbs_im2col: tensor too large");
    const int TM = (int)std::max<int64_t>(32, kColTileBytes / (Kp * es));
    const size_t smem = (size_t)TM * Kp * es;
    const int64_t tiles = (N * Ho * Wo + TM - 1) / TM;
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(tiles, 8LL * im2col_sms()));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = static_cast<cudaStream_t>(stream);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e;
    // row variant: bf16, (k, C, Kp) in {(7, 3, 152), (3, 3, 32)}, k input rows fit in shared memory
    void (*rowk)(const __nv_bfloat16*, __nv_bfloat16*, ColGeom, int, int) = nullptr;
    if (dtype == MBS_BF16 && C == 3 && k == 7 && Kp == 152) rowk = k_im2col_rows<__nv_bfloat16, 7, 3, 152>;
    if (dtype == MBS_BF16 && C == 3 && k == 3 && Kp == 32) rowk = k_im2col_rows<__nv_bfloat16, 3, 3, 32>;
    const int LP = (int)((p * C + 7) / 8 * 8);
    const int RS = (int)((LP + (W + p) * C + 7) / 8 * 8);
    const size_t rsmem = (size_t)k * RS * 2;
    if (rowk && rsmem <= 96 * 1024 && !(reinterpret_cast<uintptr_t>(x) & 15) && N * H * W * C < INT32_MAX / 2) {
        if (rsmem > 48 * 1024) cudaFuncSetAttribute(rowk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rsmem);
        int per_sm = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, rowk, 256, rsmem) != cudaSuccess || per_sm < 1)
            per_sm = 1;
        cfg.gridDim = dim3((unsigned)std::max<int64_t>(1, std::min<int64_t>(N * Ho, (int64_t)per_sm * im2col_sms())));
        cfg.dynamicSmemBytes = rsmem;
        e = cudaLaunchKernelEx(&cfg, rowk, (const __nv_bfloat16*)x, (__nv_bfloat16*)cols, g, LP, RS);
        MBS_CK(e);
        return MBS_OK;
    }
    if (dtype == MBS_BF16) {
        auto kern = (k == 7 && C == 3) ? k_im2col<__nv_bfloat16, 7, 3> : k_im2col<__nv_bfloat16>;
        if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        e = cudaLaunchKernelEx(&cfg, kern, (const __nv_bfloat16*)x, (__nv_bfloat16*)cols, g, TM);
    } else {
        if (smem > 48 * 1024) cudaFuncSetAttribute(k_im2col<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        e = cudaLaunchKernelEx(&cfg, k_im2col<float>, (const float*)x, (float*)cols, g, TM);
    }
    MBS_CK(e);
    return MBS_OK;
}

}  // extern "C"
