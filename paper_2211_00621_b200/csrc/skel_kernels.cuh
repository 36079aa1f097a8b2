// Streaming skeleton kernels: map, map2, fused map -> reduce, parallel loop.
//
// These templates are instantiated twice over: by nvcc in skeletons.cu for the
// lambda shapes the library recognises (identity, affine maps), and at run
// time by NVRTC (jit.cu) with an element functor generated from the lambda's
// bytecode — so every lambda the host compiler lowers runs in the same
// vectorised, HBM-bound kernel instead of the bytecode interpreter.
// Header must stay NVRTC-safe (no host headers).
//
// Element functor protocol (map / map->reduce):
//   typedef R;                     double (Float) or int64_t (Int/Char/Bool):
//                                  the reference's value in a register
//   template <int V, class TX>
//   void operator()(const TX (&x)[V], int64_t j0, R (&r)[V], int (&code)[V]) const
//       r[e] = f(x[e]) for element index j0 + e; code[e] != 0 is a runtime
//       error of that element (enum pmx_code; first error in program order).
// map2 functors take (a[V], b[V], j0, r, code); loop bodies (`U` lanes)
// take (i[U], code[U]) with code[u] != 0 marking a dead lane on entry.
#pragma once
#include "device_common.cuh"
#include "peer.cuh"

namespace pmx {

// ------------------------------------------------------------ memory access
// Streaming 128-bit load (read-only path, no L1 allocation). `volatile` keeps
// the loads of an unrolled iteration issued back to back before their use.
__device__ __forceinline__ uint4 ldg_stream(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}
__device__ __forceinline__ unsigned ldg_stream32(const void* p) {
    unsigned r;
    asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(p));
    return r;
}
__device__ __forceinline__ void stg_stream(void* p, uint4 v) {
    asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};"
                 :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

// A packet of V = 4 elements: 4 B (bool), 16 B (f32/i32) or 32 B (f64/i64).
template <class T>
union Pack4 {
    T e[4];
    unsigned w[sizeof(T)];          // 4 * sizeof(T) / 4 words
    uint4 q[sizeof(T) >= 4 ? sizeof(T) / 4 : 1];
};

template <class T>
__device__ __forceinline__ void load_pack(Pack4<T>& p, const T* src) {
    if (sizeof(T) >= 4) {
#pragma unroll
        for (int k = 0; k < (int)(sizeof(T) / 4); ++k) p.q[k] = ldg_stream((const uint4*)src + k);
    } else {
        p.w[0] = ldg_stream32(src);
    }
}
template <class T>
__device__ __forceinline__ void store_pack(T* dst, const Pack4<T>& p) {
    if (sizeof(T) >= 4) {
#pragma unroll
        for (int k = 0; k < (int)(sizeof(T) / 4); ++k) stg_stream((uint4*)dst + k, p.q[k]);
    } else {
        *(unsigned*)dst = p.w[0];
    }
}

// ------------------------------------------------- register <-> storage
// The reference's value of a stored element (load_elem semantics).
__device__ __forceinline__ double widen_f(float v) { return (double)v; }
__device__ __forceinline__ double widen_f(double v) { return v; }
__device__ __forceinline__ int64_t widen_i(int64_t v) { return v; }
__device__ __forceinline__ int64_t widen_i(int v) { return (int64_t)v; }
__device__ __forceinline__ int64_t widen_i(unsigned char v) { return (int64_t)v; }
__device__ __forceinline__ double widen(float v) { return (double)v; }
__device__ __forceinline__ double widen(double v) { return v; }
__device__ __forceinline__ int64_t widen(int64_t v) { return v; }
__device__ __forceinline__ int64_t widen(int v) { return (int64_t)v; }
__device__ __forceinline__ int64_t widen(unsigned char v) { return (int64_t)v; }
// ... as an untyped 64-bit register (the bytecode's view).
__device__ __forceinline__ int64_t to_reg(float v) { return of_f((double)v); }
__device__ __forceinline__ int64_t to_reg(double v) { return of_f(v); }
__device__ __forceinline__ int64_t to_reg(int64_t v) { return v; }
__device__ __forceinline__ int64_t to_reg(int v) { return (int64_t)v; }
__device__ __forceinline__ int64_t to_reg(unsigned char v) { return (int64_t)v; }

// Storage conversion of a result (store_elem semantics): f32 storage of a
// finite fp64 that overflows is PMX_E_F32_RANGE.
__device__ __forceinline__ void cvt_store(double v, float& o, int& code) {
    o = __double2float_rn(v);
    if (is_inf(o) && !is_inf(v)) code = PMX_E_F32_RANGE;
}
__device__ __forceinline__ void cvt_store(double v, double& o, int&) { o = v; }
__device__ __forceinline__ void cvt_store(int64_t v, int64_t& o, int&) { o = v; }
__device__ __forceinline__ void cvt_store(int64_t v, int& o, int&) { o = (int)v; }
__device__ __forceinline__ void cvt_store(int64_t v, unsigned char& o, int&) { o = (unsigned char)(v != 0); }

// --------------------------------------------------- recognised functors
template <class R>
struct FIdentity {
    typedef R Res;
    template <int V, class TX>
    __device__ __forceinline__ void operator()(const TX (&x)[V], int64_t, R (&r)[V], int (&)[V]) const {
#pragma unroll
        for (int e = 0; e < V; ++e) r[e] = (R)widen(x[e]);
    }
};

// y = a*x + b in fp64 with each operation rounded separately, as CPython
// evaluates `addf (mulf a x) b` on Floats. `mulf a x` alone is b = -0.0 and
// `addf x b` is a = 1.0: both identities are exact in IEEE arithmetic.
struct FAffineF {
    typedef double Res;
    double a, b;
    template <int V, class TX>
    __device__ __forceinline__ void operator()(const TX (&x)[V], int64_t, double (&r)[V], int (&)[V]) const {
#pragma unroll
        for (int e = 0; e < V; ++e) r[e] = __dadd_rn(__dmul_rn(a, widen_f(x[e])), b);
    }
};
struct FAffineI {   // wrap-around a*x + b (a = 1 / b = 0 when absent: exact)
    typedef int64_t Res;
    int64_t a, b;
    template <int V, class TX>
    __device__ __forceinline__ void operator()(const TX (&x)[V], int64_t, int64_t (&r)[V], int (&)[V]) const {
#pragma unroll
        for (int e = 0; e < V; ++e) r[e] = wadd(wmul(a, widen_i(x[e])), b);
    }
};

// ---------------------------------------------------- reduce operators
struct OAddF { typedef double A; __device__ static double id() { return 0.0; }
               __device__ static double f(double a, double b) { return __dadd_rn(a, b); } };
struct OMulF { typedef double A; __device__ static double id() { return 1.0; }
               __device__ static double f(double a, double b) { return __dmul_rn(a, b); } };
struct OMinF { typedef double A; __device__ static double id() { return __longlong_as_double(0x7ff0000000000000ll); }
               __device__ static double f(double a, double b) { return a < b ? a : b; } };
struct OMaxF { typedef double A; __device__ static double id() { return __longlong_as_double((long long)0xfff0000000000000ull); }
               __device__ static double f(double a, double b) { return a > b ? a : b; } };
struct OAddI { typedef int64_t A; __device__ static int64_t id() { return 0; }
               __device__ static int64_t f(int64_t a, int64_t b) { return wadd(a, b); } };
struct OMulI { typedef int64_t A; __device__ static int64_t id() { return 1; }
               __device__ static int64_t f(int64_t a, int64_t b) { return wmul(a, b); } };
struct OMinI { typedef int64_t A; __device__ static int64_t id() { return (int64_t)0x7fffffffffffffffll; }
               __device__ static int64_t f(int64_t a, int64_t b) { return a < b ? a : b; } };
struct OMaxI { typedef int64_t A; __device__ static int64_t id() { return (int64_t)(-0x7fffffffffffffffll - 1); }
               __device__ static int64_t f(int64_t a, int64_t b) { return a > b ? a : b; } };
// plain map: no reduction
struct NoReduce { typedef double A; __device__ static double id() { return 0.0; }
                  __device__ static double f(double a, double) { return a; } };

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
    return v;   // valid in every lane of warp 0
}

template <class Op>
struct OpFold {
    __device__ __forceinline__ typename Op::A operator()(typename Op::A a, typename Op::A b) const {
        return Op::f(a, b);
    }
};

// Last CTA to arrive folds the per-CTA partials in CTA order and applies init
// once. Resets the ticket so the workspace can be reused on the stream.
// With a peer group (pg.world > 0) the result is this rank's chunk partial;
// warp 0 then exchanges it with the other GPUs over peer memory and writes
// the rank-ordered fold of all chunk partials (peer.cuh).
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
    if (threadIdx.x < 32) {
        bool ok;
        int any;
        A tot = peer_exchange<A>(pg, Op::f(init, v), has, OpFold<Op>(), Op::id(), err, &ok, &any);
        if (threadIdx.x == 0) {
            *out = any ? tot : init;
            *ticket = 0u;
        }
    }
}

// Per packet: apply f, report errors, store y, accumulate.
template <class TX, class TY, class F, class Op, bool WRITE_Y, bool DO_REDUCE>
__device__ __forceinline__ void mr_packet(const Pack4<TX>& v, TY* y, int64_t j0, const F& f,
                                          typename Op::A& acc0, typename Op::A& acc1, uint64_t* err) {
    typedef typename F::Res R;
    R r[4];
    int code[4] = {0, 0, 0, 0};
    f(v.e, j0, r, code);
    if (WRITE_Y) {
        Pack4<TY> w;
#pragma unroll
        for (int e = 0; e < 4; ++e) cvt_store(r[e], w.e[e], code[e]);
        store_pack(y + j0, w);
    }
#pragma unroll
    for (int e = 0; e < 4; ++e)
        if (code[e]) raise_err(err, j0 + e, code[e]);
    if (DO_REDUCE) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            if (e & 1) acc1 = Op::f(acc1, (typename Op::A)r[e]);
            else acc0 = Op::f(acc0, (typename Op::A)r[e]);
        }
    }
}

// ---- vectorised fused map -> reduce (plain map: Op = NoReduce) -----------
// Grid = one resident wave (4 CTAs/SM, <= 64 registers: room for the element
// functor's fp64 registers without spills), grid-stride over 4-element
// packets. Read-only streams keep 128 B per thread in flight (measured 102% of
// the copy peak); read+write streams 64 B (the stores add their own
// parallelism).
template <class TX, class TY, class F, class Op, bool WRITE_Y, bool DO_REDUCE>
__global__ void __launch_bounds__(256, 4)
k_map_reduce_vec(const TX* __restrict__ x, TY* __restrict__ y, int64_t n, const F f,
                 typename Op::A* partials, unsigned* ticket, typename Op::A init,
                 typename Op::A* out, const __grid_constant__ pmx_peer_group pg, uint64_t* err) {
    typedef typename Op::A A;
    constexpr int U = WRITE_Y ? (sizeof(TX) >= 8 ? 2 : 4) : (sizeof(TX) >= 8 ? 4 : 8);
    const int64_t npk = n / 4;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    A acc0 = Op::id(), acc1 = Op::id();   // two chains: halves the dependent-op depth
    for (; p + (U - 1) * stride < npk; p += U * stride) {
        Pack4<TX> v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) load_pack(v[u], x + (p + u * stride) * 4);
        // Join point on every loaded packet: a (never taken) branch on a value
        // that depends on all U loads forces ptxas to issue all of them before
        // any consumer, so U packets per thread are in flight at once.
        if (!WRITE_Y) {
            unsigned j = 0;
#pragma unroll
            for (int u = 0; u < U; ++u) j += v[u].w[0];
            if (j == 0x7fc00001u && n == -1) __trap();
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
            mr_packet<TX, TY, F, Op, WRITE_Y, DO_REDUCE>(v[u], y, (p + u * stride) * 4, f, acc0, acc1, err);
    }
    for (; p < npk; p += stride) {
        Pack4<TX> v;
        load_pack(v, x + p * 4);
        mr_packet<TX, TY, F, Op, WRITE_Y, DO_REDUCE>(v, y, p * 4, f, acc0, acc1, err);
    }
    // scalar tail (< 4 elements)
    for (int64_t j = npk * 4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride) {
        typename F::Res r[1];
        int code[1] = {0};
        const TX xe[1] = {x[j]};
        f(xe, j, r, code);
        if (WRITE_Y) cvt_store(r[0], y[j], code[0]);
        if (code[0]) raise_err(err, j, code[0]);
        if (DO_REDUCE) acc0 = Op::f(acc0, (A)r[0]);
    }
    if (DO_REDUCE) {
        A bt = block_reduce<Op>(Op::f(acc0, acc1));
        grid_combine<Op>(bt, partials, ticket, init, out, pg, n > 0 || pg.rank == 0, err);
    }
}

// Scalar variant for misaligned views.
template <class TX, class TY, class F, class Op, bool WRITE_Y, bool DO_REDUCE>
__global__ void __launch_bounds__(256)
k_map_reduce_scalar(const TX* __restrict__ x, TY* __restrict__ y, int64_t n, const F f,
                    typename Op::A* partials, unsigned* ticket, typename Op::A init,
                    typename Op::A* out, const __grid_constant__ pmx_peer_group pg, uint64_t* err) {
    typedef typename Op::A A;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    A acc = Op::id();
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride) {
        typename F::Res r[1];
        int code[1] = {0};
        const TX xe[1] = {x[j]};
        f(xe, j, r, code);
        if (WRITE_Y) cvt_store(r[0], y[j], code[0]);
        if (code[0]) raise_err(err, j, code[0]);
        if (DO_REDUCE) acc = Op::f(acc, (A)r[0]);
    }
    if (DO_REDUCE) {
        A bt = block_reduce<Op>(acc);
        grid_combine<Op>(bt, partials, ticket, init, out, pg, n > 0 || pg.rank == 0, err);
    }
}

// ---- map2: z[j] = f(a[j], b[j]) -------------------------------------------
template <class TA, class TB, class TZ, class F, bool VEC>
__global__ void __launch_bounds__(256, 4)
k_map2_vec(const TA* __restrict__ a, const TB* __restrict__ b, TZ* __restrict__ z, int64_t n,
           const F f, uint64_t* err) {
    typedef typename F::Res R;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (VEC) {
        constexpr int U = 2;
        const int64_t npk = n / 4;
        for (; p + (U - 1) * stride < npk; p += U * stride) {
            Pack4<TA> va[U];
            Pack4<TB> vb[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                load_pack(va[u], a + (p + u * stride) * 4);
                load_pack(vb[u], b + (p + u * stride) * 4);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int64_t j0 = (p + u * stride) * 4;
                R r[4];
                int code[4] = {0, 0, 0, 0};
                f(va[u].e, vb[u].e, j0, r, code);
                Pack4<TZ> w;
#pragma unroll
                for (int e = 0; e < 4; ++e) cvt_store(r[e], w.e[e], code[e]);
                store_pack(z + j0, w);
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    if (code[e]) raise_err(err, j0 + e, code[e]);
            }
        }
        for (; p < npk; p += stride) {
            Pack4<TA> va;
            Pack4<TB> vb;
            load_pack(va, a + p * 4);
            load_pack(vb, b + p * 4);
            R r[4];
            int code[4] = {0, 0, 0, 0};
            f(va.e, vb.e, p * 4, r, code);
            Pack4<TZ> w;
#pragma unroll
            for (int e = 0; e < 4; ++e) cvt_store(r[e], w.e[e], code[e]);
            store_pack(z + p * 4, w);
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if (code[e]) raise_err(err, p * 4 + e, code[e]);
        }
        p = npk * 4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    }
    for (; p < n; p += stride) {
        R r[1];
        int code[1] = {0};
        const TA ae[1] = {a[p]};
        const TB be[1] = {b[p]};
        f(ae, be, p, r, code);
        cvt_store(r[0], z[p], code[0]);
        if (code[0]) raise_err(err, p, code[0]);
    }
}

// ---- parallel loop: body(i) for i in [0, n) --------------------------------
// Each thread runs B::U iterations at once, interleaved statement by
// statement (the body is straight-line; iterations are independent by the
// skeleton's contract, interp.py:346-358), so U tensor loads per thread are in
// flight. Lane u handles i = base + u * stride: coalesced across the warp.
template <class B>
__global__ void __launch_bounds__(256, 4)
k_loop_lanes(int64_t n, const B body, uint64_t* err) {
    constexpr int U = B::U;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; base < n; base += U * stride) {
        int64_t i[U];
        int code[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            i[u] = base + u * stride;
            code[u] = i[u] < n ? 0 : -1;    // -1: no iteration in this lane
        }
        body(i, code);
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (code[u] > 0) raise_err(err, i[u], code[u]);
    }
}

// ---- reduce with an arbitrary associative operator ---------------------------
// fold op init (map f x) for an operator the library does not recognise: the
// result must equal the sequential left fold for any associative op, so every
// combine keeps the left operand earlier in the sequence.  A CTA owns a
// contiguous range, split into one contiguous sub-range per warp; warps run
// independently (no CTA barrier per block): per 1024-element block each lane
// folds its 32 contiguous elements (16-byte loads, the next block's already in
// flight) as two 16-element chains joined left-to-right, an ordered shuffle
// tree (lower lane on the left) folds the lanes, and lane 0 folds the block
// into the warp's running value.  The warp values fold in warp order, the CTA
// values in CTA order after `init` (last CTA).  The ragged tail block keeps
// has-value bookkeeping; full blocks do not.
struct OPart { int64_t v; int has; };

template <class G>
__device__ __forceinline__ OPart op_combine(const G& g, OPart a, OPart b, uint64_t* err, int64_t idx) {
    if (!a.has) return b;
    if (!b.has) return a;
    const int64_t i0[1] = {a.v}, i1[1] = {b.v};
    int64_t o[1];
    int code[1] = {0};
    g.template run<1>(i0, i1, o, code);
    if (code[0]) raise_err(err, idx, code[0]);
    OPart r;
    r.v = o[0];
    r.has = 1;
    return r;
}

template <class G>
__device__ __forceinline__ int64_t op_apply(const G& g, int64_t a, int64_t b, uint64_t* err, int64_t idx) {
    const int64_t i0[1] = {a}, i1[1] = {b};
    int64_t o[1];
    int code[1] = {0};
    g.template run<1>(i0, i1, o, code);
    if (code[0]) raise_err(err, idx, code[0]);
    return o[0];
}

// Block loads.  COAL: packet u of lane l holds elements 128u + 4l .. +3 (every
// load instruction reads 32 contiguous packets — coalesced); otherwise packet
// u holds the lane's own elements 32l + 4u .. +3 (lane-contiguous: each
// instruction touches 32 cache lines, served through L1).
template <bool COAL, class TX>
__device__ __forceinline__ void ord_load_full(const TX* __restrict__ x, int64_t r0, int l, TX (&xe)[8][4]) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        const int64_t e0 = COAL ? r0 + 128 * u + 4 * l : r0 + 32 * l + 4 * u;
        Pack4<TX> v;
#pragma unroll
        for (int k = 0; k < (int)(sizeof(TX) >= 4 ? sizeof(TX) / 4 : 1); ++k)
            v.q[k] = __ldg(reinterpret_cast<const uint4*>(x + e0) + k);
#pragma unroll
        for (int e = 0; e < 4; ++e) xe[u][e] = v.e[e];
    }
}

template <class TX, class F, class G>
__global__ void __launch_bounds__(256, 2)
k_reduce_ordered(const TX* __restrict__ x, int64_t n, const F f, const G g, int64_t init, int64_t* out,
                 OPart* partials, unsigned* ticket, uint64_t* err) {
    constexpr int UP = 8;                         // 16-byte packets per lane per block
    constexpr int RW = 32 * 4 * UP;               // elements per warp block
    const int nw = blockDim.x >> 5;
    const int64_t RB = (int64_t)nw * RW;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    const int64_t per = ((n + gridDim.x - 1) / gridDim.x + RB - 1) / RB * RB;
    const int64_t lo = min(n, (int64_t)blockIdx.x * per), hi = min(n, lo + per);
    const int64_t wper = per / nw;
    const int64_t wlo = min(hi, lo + (int64_t)w * wper), whi = min(hi, wlo + wper);
    const bool aligned = ((uintptr_t)(x + wlo) % (4 * sizeof(TX))) == 0;
    __shared__ OPart s_w[32];
    OPart acc;                                    // the warp's running value (lane 0)
    acc.v = 0;
    acc.has = 0;
    // full blocks [wlo, wfull): software-pipelined (the next block's loads are in
    // flight while this one folds); the ragged tail block takes the general path
    const int64_t wfull = aligned ? wlo + (whi - wlo) / RW * RW : wlo;
    // 4-byte elements: coalesced loads, transposed to lane-contiguous runs
    // through a per-warp shared buffer (row pitch 33: conflict-free); 33 KiB
    // per CTA (8-byte elements would need 66 KiB of static shared memory)
    constexpr bool COAL = sizeof(TX) == 4;
    __shared__ TX s_tr[COAL ? 8 * (RW + RW / 32) : 1];
    TX* tr = s_tr + (COAL ? w * (RW + RW / 32) : 0);
    TX nx[UP][4];
    if (wlo < wfull) ord_load_full<COAL>(x, wlo, l, nx);
    for (int64_t r0 = wlo; r0 < wfull; r0 += RW) {
        const int64_t p0 = r0 + (int64_t)l * (4 * UP);
        TX xe[UP][4];
        if (COAL) {
            __syncwarp();                         // previous block's reads done
#pragma unroll
            for (int u = 0; u < UP; ++u)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int q = 128 * u + 4 * l + e;
                    tr[q + (q >> 5)] = nx[u][e];
                }
            __syncwarp();
#pragma unroll
            for (int u = 0; u < UP; ++u)
#pragma unroll
                for (int e = 0; e < 4; ++e) xe[u][e] = tr[33 * l + 4 * u + e];
        } else {
#pragma unroll
            for (int u = 0; u < UP; ++u)
#pragma unroll
                for (int e = 0; e < 4; ++e) xe[u][e] = nx[u][e];
        }
        if (r0 + RW < wfull) ord_load_full<COAL>(x, r0 + RW, l, nx);
        // two 16-element chains (elements 0..15 and 16..31 of the lane), joined left-to-right
        int64_t a = 0, b = 0;
#pragma unroll
        for (int u = 0; u < UP / 2; ++u) {
            typename F::Res ra[4], rb[4];
            int ca[4] = {0, 0, 0, 0}, cb[4] = {0, 0, 0, 0};
            f(xe[u], p0 + 4 * u, ra, ca);
            f(xe[u + UP / 2], p0 + 4 * (u + UP / 2), rb, cb);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int64_t qa = p0 + 4 * u + e, qb = qa + 2 * UP;
                if (ca[e]) raise_err(err, qa, ca[e]);
                if (cb[e]) raise_err(err, qb, cb[e]);
                if (u == 0 && e == 0) {
                    a = to_reg(ra[0]);
                    b = to_reg(rb[0]);
                } else {
                    a = op_apply(g, a, to_reg(ra[e]), err, qa);
                    b = op_apply(g, b, to_reg(rb[e]), err, qb);
                }
            }
        }
        int64_t lv = op_apply(g, a, b, err, p0 + UP * 4 - 1);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t rr = __shfl_down_sync(0xffffffffu, lv, o);
            if ((l & (2 * o - 1)) == 0) lv = op_apply(g, lv, rr, err, p0);
        }
        if (l == 0) {
            OPart bp;
            bp.v = lv;
            bp.has = 1;
            acc = op_combine(g, acc, bp, err, r0);
        }
    }
    if (wfull < whi) {                            // ragged / unaligned rest, element by element
        for (int64_t r0 = wfull; r0 < whi; r0 += RW) {
            const int64_t p0 = r0 + (int64_t)l * (4 * UP);
            OPart lp;
            lp.v = 0;
            lp.has = 0;
#pragma unroll
            for (int u = 0; u < UP; ++u) {
                TX xe4[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int64_t q = p0 + 4 * u + e;
                    xe4[e] = q < whi ? x[q] : x[wlo];
                }
                typename F::Res r[4];
                int code[4] = {0, 0, 0, 0};
                f(xe4, p0 + 4 * u, r, code);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int64_t q = p0 + 4 * u + e;
                    if (q >= whi) break;
                    if (code[e]) { raise_err(err, q, code[e]); continue; }
                    OPart v;
                    v.v = to_reg(r[e]);
                    v.has = 1;
                    lp = op_combine(g, lp, v, err, q);
                }
            }
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                OPart rr;
                rr.v = __shfl_down_sync(0xffffffffu, lp.v, o);
                rr.has = __shfl_down_sync(0xffffffffu, lp.has, o);
                if ((l & (2 * o - 1)) == 0 && l + o < 32) lp = op_combine(g, lp, rr, err, p0);
            }
            if (l == 0) acc = op_combine(g, acc, lp, err, r0);
        }
    }
    if (l == 0) s_w[w] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        OPart c = s_w[0];
        for (int q = 1; q < nw; ++q) c = op_combine(g, c, s_w[q], err, lo);
        acc = c;
    }
    __shared__ bool s_last;
    if (threadIdx.x == 0) {
        partials[blockIdx.x] = acc;
        __threadfence();
        s_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (s_last && threadIdx.x == 0) {
        __threadfence();
        OPart a;
        a.v = init;
        a.has = 1;                                   // init applied once, on the left
        for (int b = 0; b < (int)gridDim.x; ++b) {
            OPart q;
            q.v = __ldcg(&partials[b].v);
            q.has = __ldcg(&partials[b].has);
            a = op_combine(g, a, q, err, n > 0 ? n - 1 : 0);
        }
        *out = a.v;
        *ticket = 0u;
    }
}

// ---- seqLoop: persistent on-device iteration --------------------------------
// state'[j] = f(state[j], j, t) for t in [0, steps), f reading the previous
// state through arrays[0]; one resident wave of CTAs, a software grid barrier
// (monotonic arrival counter, zeroed by the host) between steps.
__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(bar, 1u);
        // spin with relaxed loads (an acquire load per iteration would invalidate
        // this SM's L1 each time, under the CTAs still working on it), then one
        // acquire fence
        unsigned v;
        do {
            asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
        } while (v < target);
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
    }
    __syncthreads();
}

template <class F>
__global__ void __launch_bounds__(256)
k_seq_loop_jit(const F f, const double* src, double* a, double* b, int64_t m, int64_t steps, unsigned* bar,
               uint64_t* err) {
    F fl = f;
    fl.T[0].offset = 0;
    fl.T[0].shape[0] = m;
    fl.T[0].rank = 1;
    fl.T[0].dtype = PMX_F64;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    // straight-line bodies: SQU = 8 elements per thread per pass (grid-strided, so
    // each of the SQU loads is coalesced across the warp), all loads and the
    // body's reads of the previous state issued before the stores
    constexpr int SQU = F::kStraight ? 8 : 1;
    for (int64_t t = 0; t < steps; ++t) {
        const double* cur = t == 0 ? src : ((t & 1) ? b : a);   // step 0 reads the caller's state
        double* nxt = (t & 1) ? a : b;
        fl.T[0].data = const_cast<double*>(cur);
        int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
        if (SQU > 1) {
            for (; j + (SQU - 1) * stride < m; j += SQU * stride) {
                int64_t x[SQU], jj[SQU], tt[SQU], o[SQU];
                int code[SQU];
#pragma unroll
                for (int u = 0; u < SQU; ++u) {
                    jj[u] = j + u * stride;
                    x[u] = __double_as_longlong(__ldcg(cur + jj[u]));
                    tt[u] = t;
                    code[u] = 0;
                }
                fl.template run<SQU>(x, jj, tt, o, code);
#pragma unroll
                for (int u = 0; u < SQU; ++u) {
                    if (code[u]) raise_err(err, jj[u], code[u]);
                    nxt[jj[u]] = F::kOutFloat ? __longlong_as_double(o[u]) : (double)o[u];
                }
            }
        }
        for (; j < m; j += stride) {
            const int64_t x[1] = {__double_as_longlong(__ldcg(cur + j))}, jj[1] = {j}, tt[1] = {t};
            int64_t o[1];
            int code[1] = {0};
            fl.template run<1>(x, jj, tt, o, code);
            if (code[0]) raise_err(err, j, code[0]);
            nxt[j] = F::kOutFloat ? __longlong_as_double(o[0]) : (double)o[0];
        }
        grid_barrier(bar, (unsigned)(gridDim.x * (t + 1)));
    }
}

// ---- elementwise parallel loop (tensor accesses at [i] only) ----------------
// Packets of 4 consecutive iterations with vector loads/stores (B::vec), VP
// packets per thread interleaved statement by statement; the < 4 tail
// iterations run through the bounds-checked lane path.
template <class B, int VP>
__global__ void __launch_bounds__(256, 4)
k_loop_vec(int64_t n, const B body, uint64_t* err) {
    const int64_t npk = n / 4;
    const int64_t gs = (int64_t)gridDim.x * blockDim.x;
    int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; p + (VP - 1) * gs < npk; p += VP * gs) {
        int64_t pk[VP];
        int code[4 * VP];
#pragma unroll
        for (int q = 0; q < VP; ++q) pk[q] = p + q * gs;
#pragma unroll
        for (int u = 0; u < 4 * VP; ++u) code[u] = 0;
        body.template vec<VP>(pk, code);
#pragma unroll
        for (int u = 0; u < 4 * VP; ++u)
            if (code[u]) raise_err(err, 4 * pk[u >> 2] + (u & 3), code[u]);
    }
    for (; p < npk; p += gs) {
        int64_t pk[1] = {p};
        int code[4] = {0, 0, 0, 0};
        body.template vec<1>(pk, code);
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (code[u]) raise_err(err, 4 * p + u, code[u]);
    }
    if (blockIdx.x == 0 && threadIdx.x < 4) {
        const int64_t i0 = 4 * npk + threadIdx.x;
        int64_t i[B::U];
        int code[B::U];
#pragma unroll
        for (int u = 0; u < B::U; ++u) {
            i[u] = i0;
            code[u] = (u == 0 && i0 < n) ? 0 : -1;
        }
        body(i, code);
        if (code[0] > 0) raise_err(err, i0, code[0]);
    }
}

}  // namespace pmx
