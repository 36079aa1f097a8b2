// Shared helpers for the pmx B200 kernels: error reporting, dtype load/store,
// reference scalar semantics (pmx/interp.py:32-37, 379-436).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>
#include "../../include/pmx_b200.h"

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

inline size_t dtype_size(int dt) {
    switch (dt) {
        case PMX_F32: case PMX_I32: return 4;
        case PMX_F64: case PMX_I64: return 8;
        case PMX_BOOL: return 1;
    }
    return 0;
}
inline bool dtype_is_float(int dt) { return dt == PMX_F32 || dt == PMX_F64; }

// -------------------------------------------------------------- device errors
// err word = (index << 8) | code ; atomicMin keeps the first failing element
__device__ __forceinline__ void raise_err(uint64_t* err, int64_t idx, int code) {
    if (err) atomicMin((unsigned long long*)err,
                       ((unsigned long long)idx << 8) | (unsigned long long)code);
}

// ------------------------------------------------------- untyped 64-bit values
__device__ __forceinline__ double as_f(int64_t v) { return __longlong_as_double(v); }
__device__ __forceinline__ int64_t of_f(double d) { return __double_as_longlong(d); }

// Load element j of a buffer of dtype dt as a 64-bit register value: floats
// widen to fp64, integers to int64 (the reference's Float/Int).
__device__ __forceinline__ int64_t load_elem(const void* p, int dt, int64_t j) {
    switch (dt) {
        case PMX_F32: return of_f((double)((const float*)p)[j]);
        case PMX_F64: return ((const int64_t*)p)[j];
        case PMX_I64: return ((const int64_t*)p)[j];
        case PMX_I32: return (int64_t)((const int32_t*)p)[j];
        default:      return (int64_t)((const uint8_t*)p)[j];
    }
}

// Store a register value as dtype dt. Returns false when an fp64 value is not
// representable in f32 storage (finite -> inf).
__device__ __forceinline__ bool store_elem(void* p, int dt, int64_t j, int64_t v) {
    switch (dt) {
        case PMX_F32: {
            double d = as_f(v);
            float f = __double2float_rn(d);
            ((float*)p)[j] = f;
            return !(isinf(f) && !isinf(d));
        }
        case PMX_F64: ((int64_t*)p)[j] = v; return true;
        case PMX_I64: ((int64_t*)p)[j] = v; return true;
        case PMX_I32: ((int32_t*)p)[j] = (int32_t)v; return true;
        default:      ((uint8_t*)p)[j] = (uint8_t)(v != 0); return true;
    }
}

// --------------------------------------------- reference scalar semantics
// int64 wrap-around (interp.py:32-37): unsigned arithmetic.
__device__ __forceinline__ int64_t wadd(int64_t a, int64_t b) { return (int64_t)((uint64_t)a + (uint64_t)b); }
__device__ __forceinline__ int64_t wsub(int64_t a, int64_t b) { return (int64_t)((uint64_t)a - (uint64_t)b); }
__device__ __forceinline__ int64_t wmul(int64_t a, int64_t b) { return (int64_t)((uint64_t)a * (uint64_t)b); }
// divi/modi truncate toward zero (interp.py:386-397); INT_MIN / -1 wraps.
__device__ __forceinline__ int64_t divi(int64_t a, int64_t b) {
    if (b == -1) return wsub(0, a);
    return a / b;
}
__device__ __forceinline__ int64_t modi(int64_t a, int64_t b) {
    if (b == -1) return 0;
    return a % b;
}
// floor of a float with the reference's int64 wrap (interp.py:426-427).
__device__ __forceinline__ int64_t floor_wrap(double x) {
    double f = floor(x);
    if (f >= -9223372036854775808.0 && f < 9223372036854775808.0) return (int64_t)f;
    // |f| >= 2^63: integer-valued double = m * 2^e with e >= 11; keep low 64 bits
    uint64_t bits = (uint64_t)__double_as_longlong(f);
    int e = (int)((bits >> 52) & 0x7ff) - 1075;
    uint64_t m = (bits & 0xfffffffffffffull) | 0x10000000000000ull;
    uint64_t low = (e >= 64) ? 0ull : (m << e);
    return (f < 0) ? (int64_t)(0ull - low) : (int64_t)low;
}

}  // namespace pmx
