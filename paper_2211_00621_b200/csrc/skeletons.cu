// Parallel skeletons of the accelerated-expression runtime on sm_100a.
//
// Reference functions replaced (pmx/interp.py):
//   eval_map     294-304  -> pmx_map          (grid-stride, 128-bit ld/st)
//   eval_map2    307-319  -> pmx_map2
//   eval_reduce  328-343  -> pmx_map_reduce   (warp shuffle -> smem -> last-CTA
//   _fold        322-325                        combine in CTA order)
//   foldl        461-463  -> pmx_fold         (sequential, or the parallel tree
//                                              when the operator is exactly
//                                              associative)
//   eval_loop    346-358  -> pmx_loop
//   FlattenE     161-166  -> pmx_scan_lengths (offsets; values stay in place)
//   recursion as a device loop (programs/rk4.pmx:38-40) -> pmx_seq_loop
//
// Each skeleton has two paths. A recognised lambda shape (affine map,
// sum/product/min/max operator) runs in a templated kernel with vectorised
// streaming loads; anything else the host compiler lowered runs in the
// bytecode interpreter (vm.cuh). Both report runtime errors through the
// error word.
#include <cooperative_groups.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>
#include "common.cuh"
#include "vm.cuh"
#include "peer.cuh"

namespace cg = cooperative_groups;

namespace pmx {

// ===================================================================== host
static thread_local char g_last_error[512] = "";

void set_last_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
    va_end(ap);
}

int sm_count() {
    static int cache[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (!cache[dev]) {
        int v = 0;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0)
            v = PMX_SM_COUNT_DEFAULT;
        cache[dev] = v;
    }
    return cache[dev];
}

// ------------------------------------------------------- program recognition
// Fast-path kinds returned by pmx_program_kind (role 0 = unary map function
// r0 = x, role 1 = binary reduce operator r0 = acc, r1 = x).
enum FastKind {
    K_VM = 0,
    K_IDENTITY = 1,
    K_AFFINE_F = 2,   // y = a*x + b (fp64 semantics; flags choose mul/add)
    K_AFFINE_I = 3,   // y = a*x + b (int64 wrap)
    K_ADD_F = 10, K_MUL_F = 11, K_MIN_F = 12, K_MAX_F = 13,
    K_ADD_I = 20, K_MUL_I = 21, K_MIN_I = 22, K_MAX_I = 23,
};

struct Affine {
    double af, bf;       // float coefficients
    int64_t ai, bi;      // int coefficients
    int has_mul, has_add;
};

static inline bool is_const(int o) { return o >= 32 && o < 64; }

// y = f(x) with r0 = x. Recognises   mulf c x | mulf x c | addf x c | addf c x
// | subf x c | addf (mulf c x) d  (and the int analogues). Recognition only
// accepts forms whose fast evaluation is bit-identical to the interpreter.
static int recognise_map_raw(const pmx_program* f, Affine* A);
static int recognise_map(const pmx_program* f, Affine* A) {
    int k = recognise_map_raw(f, A);
    if (!A->has_mul) { A->af = 1.0; A->ai = 1; }
    if (!A->has_add) { A->bf = -0.0; A->bi = 0; }
    return k;
}
static int recognise_map_raw(const pmx_program* f, Affine* A) {
    memset(A, 0, sizeof(*A));
    if (!f) return K_IDENTITY;
    if (f->n_arrays != 0) return K_VM;
    if (f->n_insns == 0 && f->out == 0) return K_IDENTITY;
    auto cf = [&](int o) { double d; memcpy(&d, &f->consts[o - 32], 8); return d; };
    auto ci = [&](int o) { return f->consts[o - 32]; };
    auto other = [](const pmx_insn& I, int reg, int* c) -> bool {
        if (I.a == reg && is_const(I.b)) { *c = I.b; return true; }
        if (I.b == reg && is_const(I.a)) { *c = I.a; return true; }
        return false;
    };
    if (f->n_insns == 1) {
        const pmx_insn& I = f->insns[0];
        if (f->out != I.dst) return K_VM;
        int c;
        switch (I.op) {
            case PMX_OP_MULF: if (other(I, 0, &c)) { A->af = cf(c); A->has_mul = 1; return K_AFFINE_F; } break;
            case PMX_OP_ADDF: if (other(I, 0, &c)) { A->bf = cf(c); A->has_add = 1; return K_AFFINE_F; } break;
            case PMX_OP_SUBF: if (I.a == 0 && is_const(I.b)) { A->bf = -cf(I.b); A->has_add = 1; return K_AFFINE_F; } break;
            case PMX_OP_MULI: if (other(I, 0, &c)) { A->ai = ci(c); A->has_mul = 1; return K_AFFINE_I; } break;
            case PMX_OP_ADDI: if (other(I, 0, &c)) { A->bi = ci(c); A->has_add = 1; return K_AFFINE_I; } break;
            case PMX_OP_SUBI: if (I.a == 0 && is_const(I.b)) { A->bi = (int64_t)(0ull - (uint64_t)ci(I.b)); A->has_add = 1; return K_AFFINE_I; } break;
        }
        return K_VM;
    }
    if (f->n_insns == 2) {
        const pmx_insn& M = f->insns[0];
        const pmx_insn& D = f->insns[1];
        if (f->out != D.dst || M.dst < f->n_inputs) return K_VM;
        int c, d;
        bool mf = M.op == PMX_OP_MULF && other(M, 0, &c);
        bool mi = M.op == PMX_OP_MULI && other(M, 0, &c);
        if (mf && D.op == PMX_OP_ADDF && other(D, M.dst, &d)) {
            A->af = cf(c); A->bf = cf(d); A->has_mul = A->has_add = 1; return K_AFFINE_F;
        }
        if (mi && D.op == PMX_OP_ADDI && other(D, M.dst, &d)) {
            A->ai = ci(c); A->bi = ci(d); A->has_mul = A->has_add = 1; return K_AFFINE_I;
        }
    }
    return K_VM;
}

// op(acc, x) with r0 = acc, r1 = x.
static int recognise_reduce(const pmx_program* op) {
    if (!op || op->n_arrays != 0) return K_VM;
    auto both = [](const pmx_insn& I) {
        return (I.a == 0 && I.b == 1) || (I.a == 1 && I.b == 0);
    };
    if (op->n_insns == 1) {
        const pmx_insn& I = op->insns[0];
        if (op->out != I.dst || !both(I)) return K_VM;
        switch (I.op) {
            case PMX_OP_ADDF: return K_ADD_F;
            case PMX_OP_MULF: return K_MUL_F;
            case PMX_OP_ADDI: return K_ADD_I;
            case PMX_OP_MULI: return K_MUL_I;
        }
        return K_VM;
    }
    if (op->n_insns == 2) {
        // match lt x y with true then x else y  ->  SELECT(lt(x,y), x, y)
        const pmx_insn& C = op->insns[0];
        const pmx_insn& S = op->insns[1];
        if (S.op != PMX_OP_SELECT || op->out != S.dst || S.a != C.dst || C.dst < 2) return K_VM;
        int lo = C.a, hi = C.b;                 // cmp(lo, hi)
        if (!((lo == 0 && hi == 1) || (lo == 1 && hi == 0))) return K_VM;
        bool picks_lhs = (S.b == lo && S.c == hi);   // cmp ? lo : hi
        if (!picks_lhs) return K_VM;
        switch (C.op) {   // (lo < hi ? lo : hi) = min ; (lo > hi ? lo : hi) = max
            case PMX_OP_LTF: return K_MIN_F;
            case PMX_OP_GTF: return K_MAX_F;
            case PMX_OP_LTI: return K_MIN_I;
            case PMX_OP_GTI: return K_MAX_I;
        }
    }
    return K_VM;
}

// ==================================================================== device
// Streaming 128-bit load (read-only path, no L1 allocation). `volatile` keeps
// the U loads of an unrolled iteration issued back to back before their use,
// so every thread has U x 16 B in flight.
__device__ __forceinline__ uint4 ldg_stream(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}
__device__ __forceinline__ void stg_stream(void* p, uint4 v) {
    asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};"
                 :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

// ---- element functors (storage type T, compute type C) --------------------
struct FIdentity {
    template <class T> __device__ __forceinline__ T operator()(T x) const { return x; }
};
// y = a*x + b with each operation rounded separately, as CPython evaluates
// `addf (mulf a x) b`.  `mulf a x` alone is a = a, b = -0.0 and `addf x b` is
// a = 1.0: both identities are exact in IEEE arithmetic (signed zeros, NaN
// and infinities included), so one branch-free functor covers all three.
template <class C>
struct FAffineF {
    C a, b;
    template <class T> __device__ __forceinline__ T operator()(T x) const {
        return (T)add_rn(mul_rn(a, (C)x), b);
    }
    __device__ __forceinline__ static float mul_rn(float a, float b) { return __fmul_rn(a, b); }
    __device__ __forceinline__ static float add_rn(float a, float b) { return __fadd_rn(a, b); }
    __device__ __forceinline__ static double mul_rn(double a, double b) { return __dmul_rn(a, b); }
    __device__ __forceinline__ static double add_rn(double a, double b) { return __dadd_rn(a, b); }
};
struct FAffineI {   // wrap-around a*x + b (a = 1 / b = 0 when absent: exact)
    int64_t a, b;
    __device__ __forceinline__ int64_t operator()(int64_t x) const { return wadd(wmul(a, x), b); }
};

// ---- reduce operators on the accumulator type ------------------------------
struct OAddF { typedef double A; __device__ static double id() { return 0.0; }
               __device__ static double f(double a, double b) { return __dadd_rn(a, b); } };
struct OMulF { typedef double A; __device__ static double id() { return 1.0; }
               __device__ static double f(double a, double b) { return __dmul_rn(a, b); } };
struct OMinF { typedef double A; __device__ static double id() { return __longlong_as_double(0x7ff0000000000000ll); }
               __device__ static double f(double a, double b) { return a < b ? a : b; } };
struct OMaxF { typedef double A; __device__ static double id() { return __longlong_as_double(0xfff0000000000000ll); }
               __device__ static double f(double a, double b) { return a > b ? a : b; } };
struct OAddI { typedef int64_t A; __device__ static int64_t id() { return 0; }
               __device__ static int64_t f(int64_t a, int64_t b) { return wadd(a, b); } };
struct OMulI { typedef int64_t A; __device__ static int64_t id() { return 1; }
               __device__ static int64_t f(int64_t a, int64_t b) { return wmul(a, b); } };
struct OMinI { typedef int64_t A; __device__ static int64_t id() { return INT64_MAX; }
               __device__ static int64_t f(int64_t a, int64_t b) { return a < b ? a : b; } };
struct OMaxI { typedef int64_t A; __device__ static int64_t id() { return INT64_MIN; }
               __device__ static int64_t f(int64_t a, int64_t b) { return a > b ? a : b; } };

template <class Op>
__device__ __forceinline__ typename Op::A warp_reduce(typename Op::A v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = Op::f(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Deterministic block reduction: XOR butterfly in each warp, then warp 0
// folds the warp totals in warp order.
template <class Op>
__device__ __forceinline__ typename Op::A block_reduce(typename Op::A v) {
    typedef typename Op::A A;
    __shared__ A s_w[32];
    v = warp_reduce<Op>(v);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) s_w[wid] = v;
    __syncthreads();
    const int nw = (blockDim.x + 31) >> 5;
    if (wid == 0) {
        v = lane < nw ? s_w[lane] : Op::id();
        v = warp_reduce<Op>(v);
    }
    __syncthreads();
    return v;   // valid in warp 0
}

// Last CTA to arrive folds the per-CTA partials in CTA order and applies init
// once. Resets the ticket so the workspace can be reused on the stream.
// With a peer group (pg.world > 0) the result is this rank's chunk partial;
// warp 0 then exchanges it with the other GPUs over peer memory and writes
// the rank-ordered fold of all chunk partials (peer.cuh).
template <class Op>
struct OpFold {
    __device__ __forceinline__ typename Op::A operator()(typename Op::A a, typename Op::A b) const {
        return Op::f(a, b);
    }
};

template <class Op>
__device__ __forceinline__ void grid_combine(typename Op::A block_total, typename Op::A* partials,
                                             unsigned* ticket, typename Op::A init,
                                             typename Op::A* out, const pmx_peer_group& pg,
                                             int has, uint64_t* err) {
    typedef typename Op::A A;
    __shared__ bool s_last;
    if (threadIdx.x == 0) {
        partials[blockIdx.x] = block_total;
        __threadfence();
        unsigned t = atomicAdd(ticket, 1u);
        s_last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    A v = Op::id();
    for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) v = Op::f(v, __ldcg(&partials[i]));
    v = block_reduce<Op>(v);
    if (pg.world == 0) {
        if (threadIdx.x == 0) {
            *out = Op::f(init, v);
            *ticket = 0u;
        }
        return;
    }
    if (threadIdx.x < 32) {     // warp 0 holds v in every lane
        bool ok;
        int any;
        A tot = peer_exchange<A>(pg, Op::f(init, v), has, OpFold<Op>(), Op::id(), err, &ok, &any);
        if (threadIdx.x == 0) {
            *out = any ? tot : init;
            *ticket = 0u;
        }
    }
}

// ---- vectorised fused map -> reduce (and plain map when Op is void) --------
// T: storage type, F: functor on T, Op: reduce operator or NoReduce.
struct NoReduce { typedef double A; __device__ static double id() { return 0.0; }
                  __device__ static double f(double a, double) { return a; } };

// Read-only streams (reductions) keep 128 B per thread in flight at 4 CTAs/SM
// (measured 102% of the copy peak); read+write streams do better with more
// resident warps and 64 B per thread (the stores add their own parallelism).
template <class T, class F, class Op, bool WRITE_Y, bool DO_REDUCE>
__global__ void __launch_bounds__(256, WRITE_Y ? 8 : 4)
k_map_reduce_vec(const T* __restrict__ x, T* __restrict__ y, int64_t n, F f,
                 typename Op::A* partials, unsigned* ticket, typename Op::A init,
                 typename Op::A* out, const __grid_constant__ pmx_peer_group pg, uint64_t* err) {
    typedef typename Op::A A;
    constexpr int V = 16 / sizeof(T);     // elements per 128-bit packet
    constexpr int U = (WRITE_Y ? 16 : 32) / V;   // packets in flight per thread
    union P { uint4 u; T e[V]; };
    const int64_t npk = n / V;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    A acc0 = Op::id(), acc1 = Op::id();   // two chains: halves the dependent-add depth
    for (; p + (U - 1) * stride < npk; p += U * stride) {
        P v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u].u = ldg_stream(x + (p + u * stride) * V);
        // Join point on every loaded packet: a (never taken) branch on a value
        // that depends on all U loads forces ptxas to issue all of them before
        // any consumer, so U x 16 B per thread are in flight at once (it
        // otherwise interleaves each load with the previous packet's use).
        if (!WRITE_Y) {
            unsigned j = 0;
#pragma unroll
            for (int u = 0; u < U; ++u) j += v[u].u.x;
            if (j == 0x7fc00001u && n == -1) __trap();
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            P w;
#pragma unroll
            for (int e = 0; e < V; ++e) {
                w.e[e] = f(v[u].e[e]);
                if (DO_REDUCE) {
                    if (e & 1) acc1 = Op::f(acc1, (A)w.e[e]);
                    else acc0 = Op::f(acc0, (A)w.e[e]);
                }
            }
            if (WRITE_Y) stg_stream(y + (p + u * stride) * V, w.u);
        }
    }
    for (; p < npk; p += stride) {
        P v, w;
        v.u = ldg_stream(x + p * V);
#pragma unroll
        for (int e = 0; e < V; ++e) {
            w.e[e] = f(v.e[e]);
            if (DO_REDUCE) acc0 = Op::f(acc0, (A)w.e[e]);
        }
        if (WRITE_Y) stg_stream(y + p * V, w.u);
    }
    // scalar tail
    for (int64_t j = npk * V + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride) {
        T w = f(x[j]);
        if (WRITE_Y) y[j] = w;
        if (DO_REDUCE) acc0 = Op::f(acc0, (A)w);
    }
    if (DO_REDUCE) {
        A bt = block_reduce<Op>(Op::f(acc0, acc1));
        grid_combine<Op>(bt, partials, ticket, init, out, pg, n > 0, err);
    }
}

// Scalar variant for misaligned views.
template <class T, class F, class Op, bool WRITE_Y, bool DO_REDUCE>
__global__ void __launch_bounds__(256)
k_map_reduce_scalar(const T* __restrict__ x, T* __restrict__ y, int64_t n, F f,
                    typename Op::A* partials, unsigned* ticket, typename Op::A init,
                    typename Op::A* out, const __grid_constant__ pmx_peer_group pg, uint64_t* err) {
    typedef typename Op::A A;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    A acc = Op::id();
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride) {
        T w = f(x[j]);
        if (WRITE_Y) y[j] = w;
        if (DO_REDUCE) acc = Op::f(acc, (A)w);
    }
    if (DO_REDUCE) {
        A bt = block_reduce<Op>(acc);
        grid_combine<Op>(bt, partials, ticket, init, out, pg, n > 0, err);
    }
}

// ---- interpreter paths ------------------------------------------------------
__global__ void k_map_vm(const __grid_constant__ pmx_program P, const void* x, int xt,
                         void* y, int yt, int64_t n, uint64_t* err) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride) {
        int64_t r[PMX_MAX_REGS];
        r[0] = load_elem(x, xt, j);
        r[1] = j;
        int code = vm_run(P, r);
        if (!code && !store_elem(y, yt, j, vm_opnd(P, r, P.out))) code = PMX_E_F32_RANGE;
        if (code) raise_err(err, j, code);
    }
}

__global__ void k_map2_vm(const __grid_constant__ pmx_program P, const void* x, int xt,
                          const void* y, int yt, void* z, int zt, int64_t n, uint64_t* err) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride) {
        int64_t r[PMX_MAX_REGS];
        r[0] = load_elem(x, xt, j);
        r[1] = load_elem(y, yt, j);
        r[2] = j;
        int code = vm_run(P, r);
        if (!code && !store_elem(z, zt, j, vm_opnd(P, r, P.out))) code = PMX_E_F32_RANGE;
        if (code) raise_err(err, j, code);
    }
}

// Generic reduce: each thread folds a CONTIGUOUS chunk in element order, then
// chunk partials are combined left-to-right (shuffle-down keeps the lower
// index on the left), so any associative operator — commutative or not —
// gives the sequential answer. Empty partials carry has=0.
struct VMPart { int64_t v; int has; };

__device__ __forceinline__ VMPart vm_combine(const pmx_program& OP, VMPart l, VMPart r, uint64_t* err, int64_t idx) {
    if (!l.has) return r;
    if (!r.has) return l;
    int64_t R[PMX_MAX_REGS];
    R[0] = l.v; R[1] = r.v;
    int code = vm_run(OP, R);
    if (code) raise_err(err, idx, code);
    VMPart o; o.v = vm_opnd(OP, R, OP.out); o.has = 1;
    return o;
}

__device__ __forceinline__ VMPart vm_block_combine(const pmx_program& OP, VMPart v, uint64_t* err) {
    __shared__ int64_t s_v[32];
    __shared__ int s_h[32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int o = 1; o < 32; o <<= 1) {
        VMPart r;
        r.v = __shfl_down_sync(0xffffffffu, v.v, o);
        r.has = __shfl_down_sync(0xffffffffu, v.has, o);
        if (lane + o < 32 && (lane & (2 * o - 1)) == 0) v = vm_combine(OP, v, r, err, 0);
    }
    if (lane == 0) { s_v[wid] = v.v; s_h[wid] = v.has; }
    __syncthreads();
    if (threadIdx.x == 0) {
        VMPart acc; acc.has = 0; acc.v = 0;
        const int nw = (blockDim.x + 31) >> 5;
        for (int w = 0; w < nw; ++w) { VMPart q; q.v = s_v[w]; q.has = s_h[w]; acc = vm_combine(OP, acc, q, err, 0); }
        v = acc;
    }
    __syncthreads();
    return v;
}

__global__ void k_map_reduce_vm(const __grid_constant__ pmx_program F, int has_f,
                                const __grid_constant__ pmx_program OP,
                                const void* x, int xt, int64_t n, int64_t init,
                                int64_t* out, void* y, int yt,
                                VMPart* partials, unsigned* ticket, uint64_t* err) {
    const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t chunk = (n + nthreads - 1) / nthreads;
    const int64_t lo = t * chunk;
    const int64_t hi = min(n, lo + chunk);
    VMPart acc; acc.has = 0; acc.v = 0;
    for (int64_t j = lo; j < hi; ++j) {
        int64_t r[PMX_MAX_REGS];
        int64_t v = load_elem(x, xt, j);
        if (has_f) {
            r[0] = v; r[1] = j;
            int code = vm_run(F, r);
            if (code) { raise_err(err, j, code); continue; }
            v = vm_opnd(F, r, F.out);
            if (y && !store_elem(y, yt, j, v)) raise_err(err, j, PMX_E_F32_RANGE);
        }
        if (!acc.has) { acc.v = v; acc.has = 1; continue; }
        r[0] = acc.v; r[1] = v;
        int code = vm_run(OP, r);
        if (code) { raise_err(err, j, code); continue; }
        acc.v = vm_opnd(OP, r, OP.out);
    }
    VMPart bt = vm_block_combine(OP, acc, err);
    __shared__ bool s_last;
    if (threadIdx.x == 0) {
        partials[blockIdx.x] = bt;
        __threadfence();
        s_last = (atomicAdd(ticket, 1u) == gridDim.x - 1);
    }
    __syncthreads();
    if (s_last && threadIdx.x == 0) {
        __threadfence();
        VMPart a; a.has = 1; a.v = init;          // init applied once, on the left
        for (int b = 0; b < (int)gridDim.x; ++b) {
            VMPart q;
            q.v = __ldcg(&partials[b].v);
            q.has = __ldcg(&partials[b].has);
            a = vm_combine(OP, a, q, err, n > 0 ? n - 1 : 0);
        }
        *out = a.v;
        *ticket = 0u;
    }
}

// Sequential left fold on one thread (foldl semantics, interp.py:322-325).
__global__ void k_fold_seq(const __grid_constant__ pmx_program OP, const void* x, int xt,
                           int64_t n, int64_t init, int64_t* out, uint64_t* err) {
    if (blockIdx.x != 0 || threadIdx.x != 0) return;
    int64_t acc = init;
    for (int64_t j = 0; j < n; ++j) {
        int64_t r[PMX_MAX_REGS];
        r[0] = acc;
        r[1] = load_elem(x, xt, j);
        int code = vm_run(OP, r);
        if (code) { raise_err(err, j, code); break; }
        acc = vm_opnd(OP, r, OP.out);
    }
    *out = acc;
}

__global__ void k_loop_vm(const __grid_constant__ pmx_program P, int64_t n, uint64_t* err) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        int64_t r[PMX_MAX_REGS];
        r[0] = i;
        int code = vm_run(P, r);
        if (code) raise_err(err, i, code);
    }
}

// Persistent seqLoop: `steps` iterations of a parallel map over the state,
// one grid-wide barrier per step (cooperative launch).
__global__ void k_seq_loop(pmx_program P, double* a, double* b, int64_t m, int64_t steps,
                           uint64_t* err) {
    cg::grid_group grid = cg::this_grid();
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t t = 0; t < steps; ++t) {
        double* cur = (t & 1) ? b : a;
        double* nxt = (t & 1) ? a : b;
        P.arrays[0].data = cur;   // previous state visible to GET through arrays[0]
        P.arrays[0].offset = 0;
        P.arrays[0].shape[0] = m;
        P.arrays[0].rank = 1;
        P.arrays[0].dtype = PMX_F64;
        for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < m; j += stride) {
            int64_t r[PMX_MAX_REGS];
            r[0] = __double_as_longlong(cur[j]);
            r[1] = j;
            r[2] = t;
            int code = vm_run(P, r);
            if (code) raise_err(err, j, code);
            int64_t v = vm_opnd(P, r, P.out);
            nxt[j] = P.out_is_float ? __longlong_as_double(v) : (double)v;
        }
        grid.sync();
    }
}

__global__ void k_copy_f64(const double* s, double* d, int64_t m) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < m; j += (int64_t)gridDim.x * blockDim.x)
        d[j] = s[j];
}

// Exclusive scan of lengths into n+1 offsets with one CTA: each thread scans
// a contiguous chunk, block scan of chunk totals, then write.
__global__ void k_scan_lengths(const int64_t* len, int64_t* off, int64_t n) {
    __shared__ int64_t s[1024];
    const int64_t chunk = (n + blockDim.x - 1) / blockDim.x;
    const int64_t lo = threadIdx.x * chunk, hi = min(n, lo + chunk);
    int64_t tot = 0;
    for (int64_t j = lo; j < hi; ++j) tot += len[j];
    s[threadIdx.x] = tot;
    __syncthreads();
    for (int o = 1; o < (int)blockDim.x; o <<= 1) {
        int64_t v = threadIdx.x >= (unsigned)o ? s[threadIdx.x - o] : 0;
        __syncthreads();
        s[threadIdx.x] += v;
        __syncthreads();
    }
    int64_t run = s[threadIdx.x] - tot;
    for (int64_t j = lo; j < hi; ++j) { off[j] = run; run += len[j]; }
    if (threadIdx.x == blockDim.x - 1) off[n] = s[threadIdx.x];
}

// ================================================================ launchers
static inline int grid_for(int64_t work_items, int threads, int per_sm) {
    int64_t want = (work_items + threads - 1) / threads;
    int64_t cap = (int64_t)sm_count() * per_sm;
    if (want > cap) want = cap;
    if (want < 1) want = 1;
    return (int)want;
}

// Workspace layout: [ticket u32 | pad to 256][partials: grid * 16 bytes]
static const int kReduceThreads = 256;
static const int kReduceBlocksPerSM = 8;


// One resident wave: grid = SMs x (CTAs per SM the kernel can hold), capped by
// the work (a partial second wave would leave SMs idle at the tail).
template <class K>
static int occupancy_grid(K kernel, int64_t work_items, int threads) {
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, 0) != cudaSuccess || per_sm < 1)
        per_sm = 1;
    if (per_sm > kReduceBlocksPerSM) per_sm = kReduceBlocksPerSM;
    return grid_for(work_items, threads, per_sm);
}

template <class T, class F, class Op, bool WY, bool RED>
static int launch_mr(const T* x, T* y, int64_t n, F f, void* ws, typename Op::A init,
                     typename Op::A* out, cudaStream_t st, const pmx_peer_group* pgp = nullptr,
                     uint64_t* err = nullptr) {
    pmx_peer_group pg;
    if (pgp) pg = *pgp; else memset(&pg, 0, sizeof(pg));
    const int V = 16 / sizeof(T);
    static int grid_cache[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!grid_cache[dev & 63])
        grid_cache[dev & 63] = occupancy_grid(k_map_reduce_vec<T, F, Op, WY, RED>, (int64_t)1 << 40, kReduceThreads);
    int64_t want = (n / V + kReduceThreads * 8 - 1) / (kReduceThreads * 8);   // >= 8 packets per thread
    int grid = (int)(want < grid_cache[dev & 63] ? (want < 1 ? 1 : want) : grid_cache[dev & 63]);
    unsigned* ticket = (unsigned*)ws;
    typename Op::A* partials = (typename Op::A*)((char*)ws + 256);
    bool aligned = ((uintptr_t)x % 16 == 0) && (!WY || (uintptr_t)y % 16 == 0);
    if (aligned)
        k_map_reduce_vec<T, F, Op, WY, RED><<<grid, kReduceThreads, 0, st>>>(x, y, n, f, partials, ticket, init, out, pg, err);
    else
        k_map_reduce_scalar<T, F, Op, WY, RED><<<grid, kReduceThreads, 0, st>>>(x, y, n, f, partials, ticket, init, out, pg, err);
    PMX_CHECK_LAUNCH("map_reduce");
    return 0;
}

// Dispatch on reduce operator for storage type T and functor F.
template <class T, class F>
static int dispatch_op(int okind, const T* x, T* y, int64_t n, F f, void* ws,
                       const void* init_host, void* out, cudaStream_t st,
                       const pmx_peer_group* pg = nullptr, uint64_t* err = nullptr) {
    const bool wy = y != nullptr;
#define PMX_MR(OP, ACC)                                                                        \
    {                                                                                          \
        ACC init; memcpy(&init, init_host, 8);                                                 \
        return wy ? launch_mr<T, F, OP, true, true>(x, y, n, f, ws, init, (ACC*)out, st, pg, err)  \
                  : launch_mr<T, F, OP, false, true>(x, y, n, f, ws, init, (ACC*)out, st, pg, err); \
    }
    switch (okind) {
        case K_ADD_F: PMX_MR(OAddF, double)
        case K_MUL_F: PMX_MR(OMulF, double)
        case K_MIN_F: PMX_MR(OMinF, double)
        case K_MAX_F: PMX_MR(OMaxF, double)
        case K_ADD_I: PMX_MR(OAddI, int64_t)
        case K_MUL_I: PMX_MR(OMulI, int64_t)
        case K_MIN_I: PMX_MR(OMinI, int64_t)
        case K_MAX_I: PMX_MR(OMaxI, int64_t)
    }
#undef PMX_MR
    return 1;   // not handled
}

template <class T, class F>
static int dispatch_map_only(const T* x, T* y, int64_t n, F f, cudaStream_t st) {
    return launch_mr<T, F, NoReduce, true, false>(x, y, n, f, nullptr, 0.0, nullptr, st);
}

static bool f32_exact(double v) { return (double)(float)v == v; }

// Templated (recognised) path of map -> reduce; returns 1 when the program
// pair has no templated kernel.
static int map_reduce_fast(const pmx_program* f, const pmx_program* op, const void* x, int32_t xt,
                           int64_t n, const void* init_host, int32_t acc_dtype, void* out,
                           void* y, int32_t yt, void* ws, cudaStream_t st,
                           const pmx_peer_group* pg, uint64_t* err) {
    Affine A;
    int fk = recognise_map(f, &A);
    int ok = recognise_reduce(op);
    const bool float_op = ok >= K_ADD_F && ok <= K_MAX_F;
    const bool int_op = ok >= K_ADD_I && ok <= K_MAX_I;
    const bool same_y = (y == nullptr) || (yt == xt);
    if (!(same_y && ((float_op && acc_dtype == PMX_F64) || (int_op && acc_dtype == PMX_I64)))) return 1;
    if (xt == PMX_F32 && float_op) {
        if (fk == K_IDENTITY)
            return dispatch_op<float>(ok, (const float*)x, (float*)y, n, FIdentity{}, ws, init_host, out, st, pg, err);
        if (fk == K_AFFINE_F && f32_exact(A.af) && f32_exact(A.bf))
            return dispatch_op<float>(ok, (const float*)x, (float*)y, n, FAffineF<float>{(float)A.af, (float)A.bf},
                                      ws, init_host, out, st, pg, err);
    } else if (xt == PMX_F64 && float_op) {
        if (fk == K_IDENTITY)
            return dispatch_op<double>(ok, (const double*)x, (double*)y, n, FIdentity{}, ws, init_host, out, st, pg, err);
        if (fk == K_AFFINE_F)
            return dispatch_op<double>(ok, (const double*)x, (double*)y, n, FAffineF<double>{A.af, A.bf},
                                       ws, init_host, out, st, pg, err);
    } else if (xt == PMX_I64 && int_op) {
        if (fk == K_IDENTITY)
            return dispatch_op<int64_t>(ok, (const int64_t*)x, (int64_t*)y, n, FIdentity{}, ws, init_host, out, st, pg, err);
        if (fk == K_AFFINE_I)
            return dispatch_op<int64_t>(ok, (const int64_t*)x, (int64_t*)y, n, FAffineI{A.ai, A.bi},
                                        ws, init_host, out, st, pg, err);
    }
    return 1;
}

}  // namespace pmx

// =================================================================== C ABI
using namespace pmx;

extern "C" {

int pmx_abi_version(void) { return PMX_ABI_VERSION; }
const char* pmx_last_error(void) { return g_last_error; }

int pmx_program_kind(const pmx_program* f, int32_t role) {
    Affine A;
    return role == 0 ? recognise_map(f, &A) : recognise_reduce(f);
}

int pmx_err_reset(uint64_t* err, void* stream) {
    if (!err) return 0;
    cudaError_t e = cudaMemsetAsync(err, 0xff, sizeof(uint64_t), (cudaStream_t)stream);
    if (e != cudaSuccess) { set_last_error("err_reset: %s", cudaGetErrorString(e)); return -2; }
    return 0;
}

size_t pmx_reduce_workspace_bytes(int64_t n) {
    (void)n;
    return 256 + (size_t)sm_count() * kReduceBlocksPerSM * 16 + 256;
}

int pmx_map(const pmx_program* f, const void* x, int32_t xt, void* y, int32_t yt,
            int64_t n, uint64_t* err, void* stream) {
    PMX_REQUIRE(n >= 0, "pmx_map: negative length");
    if (n == 0) return 0;
    PMX_REQUIRE(x && y, "pmx_map: null buffer");
    cudaStream_t st = (cudaStream_t)stream;
    Affine A;
    int kind = recognise_map(f, &A);
    if (xt == yt && (kind == K_IDENTITY || kind == K_AFFINE_F || kind == K_AFFINE_I)) {
        if (kind == K_IDENTITY) {
            cudaError_t e = cudaMemcpyAsync(y, x, n * dtype_size(xt), cudaMemcpyDeviceToDevice, st);
            if (e != cudaSuccess) { set_last_error("map copy: %s", cudaGetErrorString(e)); return -2; }
            return 0;
        }
        if (kind == K_AFFINE_F && xt == PMX_F32 && f32_exact(A.af) && f32_exact(A.bf))
            return dispatch_map_only<float>((const float*)x, (float*)y, n,
                                            FAffineF<float>{(float)A.af, (float)A.bf}, st);
        if (kind == K_AFFINE_F && xt == PMX_F64)
            return dispatch_map_only<double>((const double*)x, (double*)y, n,
                                             FAffineF<double>{A.af, A.bf}, st);
        if (kind == K_AFFINE_I && xt == PMX_I64)
            return dispatch_map_only<int64_t>((const int64_t*)x, (int64_t*)y, n,
                                              FAffineI{A.ai, A.bi}, st);
    }
    PMX_REQUIRE(f, "pmx_map: null program with differing dtypes");
    int grid = grid_for(n, 256, 8);
    k_map_vm<<<grid, 256, 0, st>>>(*f, x, xt, y, yt, n, err);
    PMX_CHECK_LAUNCH("map_vm");
    return 0;
}

int pmx_map2(const pmx_program* f, const void* x, int32_t xt, const void* y, int32_t yt,
             void* z, int32_t zt, int64_t n, uint64_t* err, void* stream) {
    PMX_REQUIRE(n >= 0, "pmx_map2: negative length");
    if (n == 0) return 0;
    PMX_REQUIRE(f && x && y && z, "pmx_map2: null argument");
    int grid = grid_for(n, 256, 8);
    k_map2_vm<<<grid, 256, 0, (cudaStream_t)stream>>>(*f, x, xt, y, yt, z, zt, n, err);
    PMX_CHECK_LAUNCH("map2_vm");
    return 0;
}

int pmx_map_reduce(const pmx_program* f, const pmx_program* op, const void* x, int32_t xt,
                   int64_t n, const void* init_host, int32_t acc_dtype, void* out,
                   void* y, int32_t yt, void* ws, size_t ws_bytes, uint64_t* err, void* stream) {
    PMX_REQUIRE(op && init_host && out, "pmx_map_reduce: null argument");
    PMX_REQUIRE(n >= 0, "pmx_map_reduce: negative length");
    PMX_REQUIRE(acc_dtype == PMX_F64 || acc_dtype == PMX_I64, "pmx_map_reduce: acc dtype must be f64 or i64");
    cudaStream_t st = (cudaStream_t)stream;
    if (n == 0) {   // reduce over [] returns init (interp.py:329-330)
        cudaError_t e = cudaMemcpyAsync(out, init_host, 8, cudaMemcpyHostToDevice, st);
        if (e != cudaSuccess) { set_last_error("reduce init: %s", cudaGetErrorString(e)); return -2; }
        return 0;
    }
    PMX_REQUIRE(ws && ws_bytes >= pmx_reduce_workspace_bytes(n), "pmx_map_reduce: workspace too small");
    int r = map_reduce_fast(f, op, x, xt, n, init_host, acc_dtype, out, y, yt, ws, st, nullptr, err);
    if (r <= 0) return r;
    // interpreter path
    int64_t init;
    memcpy(&init, init_host, 8);
    int grid = grid_for(n, 256, 4);
    unsigned* ticket = (unsigned*)ws;
    VMPart* partials = (VMPart*)((char*)ws + 256);
    pmx_program none;
    memset(&none, 0, sizeof(none));
    k_map_reduce_vm<<<grid, 256, 0, st>>>(f ? *f : none, f ? 1 : 0, *op, x, xt, n, init,
                                          (int64_t*)out, y, yt, partials, ticket, err);
    PMX_CHECK_LAUNCH("map_reduce_vm");
    return 0;
}

int pmx_map_reduce_peers(const pmx_program* f, const pmx_program* op, const void* x, int32_t xt,
                         int64_t n, const void* init_host, int32_t acc_dtype, void* out,
                         void* ws, size_t ws_bytes, const pmx_peer_group* g, uint64_t* err, void* stream) {
    PMX_REQUIRE(op && init_host && out && g, "pmx_map_reduce_peers: null argument");
    PMX_REQUIRE(n >= 0, "pmx_map_reduce_peers: negative length");
    PMX_REQUIRE(g->world >= 1 && g->world <= PMX_MAX_PEERS && g->rank >= 0 && g->rank < g->world,
                "pmx_map_reduce_peers: bad group (rank %d of %d)", g->rank, g->world);
    PMX_REQUIRE(g->epoch >= 1, "pmx_map_reduce_peers: epoch must start at 1");
    for (int r = 0; r < g->world; ++r) PMX_REQUIRE(g->mbox[r], "pmx_map_reduce_peers: mailbox %d not mapped", r);
    PMX_REQUIRE(ws && ws_bytes >= pmx_reduce_workspace_bytes(n), "pmx_map_reduce_peers: workspace too small");
    PMX_REQUIRE(n == 0 || x, "pmx_map_reduce_peers: null input");
    int r = map_reduce_fast(f, op, x, xt, n, init_host, acc_dtype, out, nullptr, xt, ws,
                            (cudaStream_t)stream, g, err);
    if (r == 1) {
        set_last_error("pmx_map_reduce_peers: operator has no fused peer kernel (use the collective path)");
        return -3;
    }
    return r;
}

int pmx_fold(const pmx_program* op, const void* x, int32_t xt, int64_t n,
             const void* init_host, int32_t acc_dtype, void* out,
             void* ws, size_t ws_bytes, uint64_t* err, void* stream) {
    PMX_REQUIRE(op && init_host && out, "pmx_fold: null argument");
    int ok = recognise_reduce(op);
    // Exactly associative operators (int add/mul/min/max, float min/max) give
    // the left fold's answer under any bracketing: use the parallel tree.
    bool exact = (ok >= K_ADD_I && ok <= K_MAX_I) || ok == K_MIN_F || ok == K_MAX_F;
    if (exact && n > 4096 && ws && ws_bytes >= pmx_reduce_workspace_bytes(n))
        return pmx_map_reduce(nullptr, op, x, xt, n, init_host, acc_dtype, out, nullptr, xt,
                              ws, ws_bytes, err, stream);
    int64_t init;
    memcpy(&init, init_host, 8);
    k_fold_seq<<<1, 32, 0, (cudaStream_t)stream>>>(*op, x, xt, n, init, (int64_t*)out, err);
    PMX_CHECK_LAUNCH("fold");
    return 0;
}

int pmx_loop(const pmx_program* body, int64_t n, uint64_t* err, void* stream) {
    PMX_REQUIRE(body, "pmx_loop: null body");
    if (n <= 0) return 0;    // interp.py:347-348
    int grid = grid_for(n, 256, 8);
    k_loop_vm<<<grid, 256, 0, (cudaStream_t)stream>>>(*body, n, err);
    PMX_CHECK_LAUNCH("loop_vm");
    return 0;
}

int pmx_seq_loop(const pmx_program* f, double* state, double* scratch, int64_t m, int64_t steps,
                 uint64_t* err, void* stream) {
    PMX_REQUIRE(f && state && scratch, "pmx_seq_loop: null argument");
    PMX_REQUIRE(f->n_arrays >= 1, "pmx_seq_loop: program must reserve arrays[0] for the state");
    if (m <= 0 || steps <= 0) return 0;
    cudaStream_t st = (cudaStream_t)stream;
    int dev = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_seq_loop, 256, 0);
    if (per_sm < 1) per_sm = 1;
    int grid = grid_for(m, 256, per_sm);
    pmx_program P = *f;
    void* args[] = {&P, &state, &scratch, &m, &steps, &err};
    cudaError_t e = cudaLaunchCooperativeKernel((void*)k_seq_loop, grid, 256, args, 0, st);
    if (e != cudaSuccess) { set_last_error("seq_loop: %s", cudaGetErrorString(e)); return -2; }
    if (steps & 1) {   // result landed in scratch: copy back so `state` holds it
        k_copy_f64<<<grid_for(m, 256, 4), 256, 0, st>>>(scratch, state, m);
        PMX_CHECK_LAUNCH("seq_loop copy");
    }
    return 0;
}

int pmx_scan_lengths(const int64_t* lengths, int64_t* offsets, int64_t n, void* stream) {
    PMX_REQUIRE(offsets, "pmx_scan_lengths: null offsets");
    PMX_REQUIRE(n >= 0, "pmx_scan_lengths: negative n");
    if (n == 0) {
        cudaError_t e = cudaMemsetAsync(offsets, 0, 8, (cudaStream_t)stream);
        if (e != cudaSuccess) { set_last_error("scan: %s", cudaGetErrorString(e)); return -2; }
        return 0;
    }
    k_scan_lengths<<<1, 1024, 0, (cudaStream_t)stream>>>(lengths, offsets, n);
    PMX_CHECK_LAUNCH("scan_lengths");
    return 0;
}

}  // extern "C"
