// Shared helpers for the pmx B200 kernels: error reporting, dtype load/store,
// reference scalar semantics (pmx/interp.py:32-37, 379-436).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>
#include "pmx_b200.h"

#define PMX_SM_COUNT_DEFAULT 148

namespace pmx {

// ---------------------------------------------------------------- host errors
void set_last_error(const char* fmt, ...);
int sm_count();                                  // cached per device

#define PMX_CHECK_LAUNCH(name)                                              \
    do {                                                                    \
        cudaError_t e_ = cudaGetLastError();                                \
        if (e_ != cudaSuccess) {                                            \
            ::pmx::set_last_error("%s: %s", name, cudaGetErrorString(e_)); \
            return -2;                                                      \
        }                                                                   \
    } while (0)

#define PMX_REQUIRE(cond, ...)                                              \
    do {                                                                    \
        if (!(cond)) { ::pmx::set_last_error(__VA_ARGS__); return -1; }     \
    } while (0)

inline int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }

// log of a forward step's scale c_t (or a product of them) for the running
// log-likelihood of the HMM kernels.  c = 0 (an observation no state can emit,
// with log-space inputs of -inf) gives NaN, as the reference's log-space
// recursion does: its max-shifted log-sum-exp over all -inf terms is NaN.
__device__ __forceinline__ double log_scale(double c) {
    return c > 0.0 ? log(c) : __longlong_as_double(0x7ff8000000000000ll);
}

inline size_t dtype_size(int dt) {
    switch (dt) {
        case PMX_F32: case PMX_I32: return 4;
        case PMX_F64: case PMX_I64: return 8;
        case PMX_BOOL: return 1;
    }
    return 0;
}
inline bool dtype_is_float(int dt) { return dt == PMX_F32 || dt == PMX_F64; }

}  // namespace pmx

#include "device_common.cuh"
