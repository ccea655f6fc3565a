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

// One thread per 16-byte chunk (VE elements) of a cols row: consecutive threads write consecutive
// chunks (fully coalesced stores); the (kh, kw, c) decomposition of each column comes from a
// per-CTA smem table; the gathered input elements are L1/L2 hits (neighbouring output pixels
// share most of their window).
template <typename T, int VE>
__global__ void __launch_bounds__(256) k_im2col(const T* __restrict__ x, T* __restrict__ cols, ColGeom g) {
    __shared__ int16_t tdh[kColMaxKp], tdw[kColMaxKp], tc[kColMaxKp];
    const int64_t K = (int64_t)g.k * g.k * g.C;
    for (int j = threadIdx.x; j < g.Kp; j += blockDim.x) {
        if (j < K) {
            tdh[j] = (int16_t)(j / (g.k * g.C));
            const int r = j % (g.k * (int)g.C);
            tdw[j] = (int16_t)(r / g.C);
            tc[j] = (int16_t)(r % g.C);
        } else {
            tdh[j] = -1;
            tdw[j] = 0;
            tc[j] = 0;
        }
    }
    __syncthreads();
    cudaGridDependencySynchronize();
    const int64_t chunks = g.Kp / VE;
    const int64_t total = g.N * g.Ho * g.Wo * chunks;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int j0 = (int)(t % chunks) * VE;
        const int64_t m = t / chunks;
        const int64_t ow = m % g.Wo;
        const int64_t q = m / g.Wo;
        const int64_t oh = q % g.Ho;
        const int64_t n = q / g.Ho;
        const int64_t h0 = oh * g.s - g.p, w0 = ow * g.s - g.p;
        const T* base = x + n * g.H * g.W * g.C;
        T v[VE];
#pragma unroll
        for (int e = 0; e < VE; ++e) {
            const int j = j0 + e;
            const int dh = tdh[j];
            const int64_t ih = h0 + dh, iw = w0 + tdw[j];
            v[e] = (dh >= 0 && ih >= 0 && ih < g.H && iw >= 0 && iw < g.W) ? base[(ih * g.W + iw) * g.C + tc[j]] : T(0.f);
        }
        if constexpr (sizeof(T) * VE == 16) {
            uint4 u;
            memcpy(&u, v, 16);
            *reinterpret_cast<uint4*>(cols + m * g.Kp + j0) = u;
        } else {
#pragma unroll
            for (int e = 0; e < VE; ++e) cols[m * g.Kp + j0 + e] = v[e];
        }
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
    const int ve = dtype == MBS_BF16 ? 8 : 4;
    const bool vec = Kp % ve == 0 && !(reinterpret_cast<uintptr_t>(cols) & 15);
    const int64_t work = N * Ho * Wo * (vec ? Kp / ve : Kp);
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((work + 255) / 256, 8LL * im2col_sms()));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(256);
    cfg.stream = static_cast<cudaStream_t>(stream);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e;
    if (dtype == MBS_BF16)
        e = vec ? cudaLaunchKernelEx(&cfg, k_im2col<__nv_bfloat16, 8>, (const __nv_bfloat16*)x, (__nv_bfloat16*)cols, g)
                : cudaLaunchKernelEx(&cfg, k_im2col<__nv_bfloat16, 1>, (const __nv_bfloat16*)x, (__nv_bfloat16*)cols, g);
    else
        e = vec ? cudaLaunchKernelEx(&cfg, k_im2col<float, 4>, (const float*)x, (float*)cols, g)
                : cudaLaunchKernelEx(&cfg, k_im2col<float, 1>, (const float*)x, (float*)cols, g);
    MBS_CK(e);
    return MBS_OK;
}

}  // extern "C"
