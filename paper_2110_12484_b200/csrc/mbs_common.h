// Shared internals of libmbs_native.so (not part of the C-ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <string>
#include <vector>

#include "../../include/mbs.h"

namespace mbs {

void set_error(const std::string& msg);

inline int cuda_status(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return MBS_OK;
    set_error(std::string(what) + ": " + cudaGetErrorString(e));
    return MBS_ECUDA;
}

inline int invalid(const std::string& msg) {
    set_error(msg);
    return MBS_EINVAL;
}

// Internal view of an accumulator handle (mbs_accum.cu) for the fused peer all-reduce (mbs_peer.cu).
struct AccumView {
    float* acc;
    int64_t numel;
    const std::vector<int64_t>* off;
    const std::vector<int64_t>* num;
    double* d_losses;
    double* d_factors;
    double* d_weights;
    int64_t* seen;
    int64_t* covered;
    int64_t expected;
    int64_t max_micro;
    bool* fresh;
    int* n_partials;
};
int accum_view(mbs_accum_t h, AccumView* v);

}  // namespace mbs

#define MBS_CK(call)                                                   \
    do {                                                               \
        cudaError_t _e = (call);                                       \
        if (_e != cudaSuccess) return mbs::cuda_status(_e, #call);     \
    } while (0)

#define MBS_CK_LAUNCH(what)                                            \
    do {                                                               \
        cudaError_t _e = cudaGetLastError();                           \
        if (_e != cudaSuccess) return mbs::cuda_status(_e, what);      \
    } while (0)
