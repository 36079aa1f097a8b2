// Device helpers shared by the precompiled kernels (nvcc) and the kernels the
// library compiles at run time (NVRTC, jit.cu): error reporting, dtype
// load/store, the reference's scalar semantics (pmx/interp.py:32-37,
// 379-436). Must stay free of host-only headers (NVRTC has none).
#pragma once
#include "pmx_b200.h"

namespace pmx {

// -------------------------------------------------------------- device errors
// err word = (index << 8) | code ; atomicMin keeps the first failing element
__device__ __forceinline__ void raise_err(uint64_t* err, int64_t idx, int code) {
    if (err) atomicMin((unsigned long long*)err,
                       ((unsigned long long)idx << 8) | (unsigned long long)code);
}

// isinf without the host math headers (NVRTC)
__device__ __forceinline__ bool is_inf(double x) {
    return (__double_as_longlong(x) & 0x7fffffffffffffffll) == 0x7ff0000000000000ll;
}
__device__ __forceinline__ bool is_inf(float x) { return (__float_as_uint(x) & 0x7fffffffu) == 0x7f800000u; }

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
            return !(is_inf(f) && !is_inf(d));
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
