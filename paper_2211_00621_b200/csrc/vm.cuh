// Device interpreter for compiled scalar PMExpr lambdas (pmx_program).
//
// This is the generic path of the skeletons: any lambda the host compiler can
// lower (scalar arithmetic, comparisons, match, captured scalars, `get` on
// captured sequences, tensorGet/tensorSet on marshalled tensor views) runs
// here, one element per thread, with the reference's scalar semantics
// (pmx/interp.py:379-436) including its runtime errors, which are recorded in
// the device error word instead of raised. Recognised shapes (affine maps,
// sum/product/min/max reductions) bypass the interpreter; see skeletons.cu.
#pragma once
#include "common.cuh"

namespace pmx {

// 64-bit register value of an operand: register 0..31, constant 32..63.
__device__ __forceinline__ int64_t vm_opnd(const pmx_program& P, const int64_t* r, int o) {
    return o < 32 ? r[o] : P.consts[o - 32];
}

// Linear element index of a tensor access (runtime.py:63-75). Returns -1 and
// sets *code on an out-of-bounds index.
__device__ __forceinline__ int64_t vm_tensor_linear(const pmx_array& A, const int64_t* idx, int* code) {
    int64_t pos = A.offset, stride = 1;
    for (int d = A.rank - 1; d >= 0; --d) {
        int64_t k = idx[d];
        if (k < 0 || k >= A.shape[d]) { *code = PMX_E_TENSOR_OOB; return -1; }
        pos += k * stride;
        stride *= A.shape[d];
    }
    return pos;
}

// Run program P over registers r (inputs already in r[0..n_inputs)).
// Returns 0 on success or an error code; the result is vm_opnd(P, r, P.out).
__device__ int vm_run(const pmx_program& P, int64_t* r) {
    int pc = 0;
    const int n = P.n_insns;
    while (pc < n) {
        const pmx_insn I = P.insns[pc++];
        const int64_t a = (I.op == PMX_OP_JMP) ? 0 : vm_opnd(P, r, I.a);
        switch (I.op) {
            case PMX_OP_NOP: break;
            case PMX_OP_MOV: r[I.dst] = a; break;
            // ---- Int (wrap-around int64)
            case PMX_OP_ADDI: r[I.dst] = wadd(a, vm_opnd(P, r, I.b)); break;
            case PMX_OP_SUBI: r[I.dst] = wsub(a, vm_opnd(P, r, I.b)); break;
            case PMX_OP_MULI: r[I.dst] = wmul(a, vm_opnd(P, r, I.b)); break;
            case PMX_OP_DIVI: { int64_t b = vm_opnd(P, r, I.b); if (b == 0) return PMX_E_DIVI0; r[I.dst] = divi(a, b); } break;
            case PMX_OP_MODI: { int64_t b = vm_opnd(P, r, I.b); if (b == 0) return PMX_E_MODI0; r[I.dst] = modi(a, b); } break;
            case PMX_OP_NEGI: r[I.dst] = wsub(0, a); break;
            // ---- Float (fp64, no contraction: each op rounds, like CPython)
            case PMX_OP_ADDF: r[I.dst] = of_f(__dadd_rn(as_f(a), as_f(vm_opnd(P, r, I.b)))); break;
            case PMX_OP_SUBF: r[I.dst] = of_f(__dsub_rn(as_f(a), as_f(vm_opnd(P, r, I.b)))); break;
            case PMX_OP_MULF: r[I.dst] = of_f(__dmul_rn(as_f(a), as_f(vm_opnd(P, r, I.b)))); break;
            case PMX_OP_DIVF: { double b = as_f(vm_opnd(P, r, I.b)); if (b == 0.0) return PMX_E_DIVF0; r[I.dst] = of_f(__ddiv_rn(as_f(a), b)); } break;
            case PMX_OP_NEGF: r[I.dst] = of_f(-as_f(a)); break;
            // ---- comparisons (results are 0/1 in an int register)
            case PMX_OP_EQI: r[I.dst] = a == vm_opnd(P, r, I.b); break;
            case PMX_OP_NEQI: r[I.dst] = a != vm_opnd(P, r, I.b); break;
            case PMX_OP_LTI: r[I.dst] = a < vm_opnd(P, r, I.b); break;
            case PMX_OP_GTI: r[I.dst] = a > vm_opnd(P, r, I.b); break;
            case PMX_OP_LEQI: r[I.dst] = a <= vm_opnd(P, r, I.b); break;
            case PMX_OP_GEQI: r[I.dst] = a >= vm_opnd(P, r, I.b); break;
            case PMX_OP_EQF: r[I.dst] = as_f(a) == as_f(vm_opnd(P, r, I.b)); break;
            case PMX_OP_LTF: r[I.dst] = as_f(a) < as_f(vm_opnd(P, r, I.b)); break;
            case PMX_OP_GTF: r[I.dst] = as_f(a) > as_f(vm_opnd(P, r, I.b)); break;
            case PMX_OP_LEQF: r[I.dst] = as_f(a) <= as_f(vm_opnd(P, r, I.b)); break;
            case PMX_OP_GEQF: r[I.dst] = as_f(a) >= as_f(vm_opnd(P, r, I.b)); break;
            case PMX_OP_EQB: r[I.dst] = (a != 0) == (vm_opnd(P, r, I.b) != 0); break;
            case PMX_OP_NOT: r[I.dst] = a == 0; break;
            // ---- conversions and math (interp.py:424-436)
            case PMX_OP_INT2FLOAT: r[I.dst] = of_f(__ll2double_rn(a)); break;
            case PMX_OP_FLOOR: r[I.dst] = floor_wrap(as_f(a)); break;
            case PMX_OP_EXP: {
                double x = as_f(a), y = exp(x);
                if (isinf(y) && !isinf(x)) return PMX_E_EXP_RANGE;
                r[I.dst] = of_f(y);
            } break;
            case PMX_OP_LOG: {
                double x = as_f(a);
                if (x <= 0.0) return PMX_E_LOG_DOMAIN;
                r[I.dst] = of_f(log(x));
            } break;
            case PMX_OP_SIN: { double x = as_f(a); if (isinf(x)) return PMX_E_SIN_COS_INF; r[I.dst] = of_f(sin(x)); } break;
            case PMX_OP_COS: { double x = as_f(a); if (isinf(x)) return PMX_E_SIN_COS_INF; r[I.dst] = of_f(cos(x)); } break;
            case PMX_OP_SQRT: { double x = as_f(a); if (x < 0.0) return PMX_E_SQRT_NEG; r[I.dst] = of_f(sqrt(x)); } break;
            case PMX_OP_SELECT: r[I.dst] = a ? vm_opnd(P, r, I.b) : vm_opnd(P, r, I.c); break;
            // ---- captured sequences (get/length, interp.py:446-451)
            case PMX_OP_GET: {
                const pmx_array& A = P.arrays[I.c];
                if (a < 0 || a >= A.shape[0]) return PMX_E_OOB;
                r[I.dst] = load_elem(A.data, A.dtype, A.offset + a);
            } break;
            case PMX_OP_LEN: r[I.dst] = P.arrays[I.c].shape[0]; break;
            // ---- tensors (interp.py:468-474; runtime.py:63-75)
            case PMX_OP_TGET: {
                const pmx_array& A = P.arrays[I.c];
                int64_t idx[PMX_MAX_RANK];
                for (int d = 0; d < A.rank; ++d) idx[d] = r[I.a + d];
                int code = 0;
                int64_t pos = vm_tensor_linear(A, idx, &code);
                if (code) return code;
                r[I.dst] = load_elem(A.data, A.dtype, pos);
            } break;
            case PMX_OP_TSET: {
                const pmx_array& A = P.arrays[I.c];
                int64_t idx[PMX_MAX_RANK];
                for (int d = 0; d < A.rank; ++d) idx[d] = r[I.a + d];
                int code = 0;
                int64_t pos = vm_tensor_linear(A, idx, &code);
                if (code) return code;
                if (!store_elem(A.data, A.dtype, pos, vm_opnd(P, r, I.b))) return PMX_E_F32_RANGE;
            } break;
            case PMX_OP_NEVER: return PMX_E_NEVER;
            case PMX_OP_FAIL: return I.b;
            case PMX_OP_JZ: if (a == 0) pc = I.b | (I.c << 8); break;
            case PMX_OP_JMP: pc = I.b | (I.c << 8); break;
            default: return PMX_E_NEVER;
        }
    }
    return 0;
}

}  // namespace pmx
