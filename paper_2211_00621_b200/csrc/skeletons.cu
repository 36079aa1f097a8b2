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
#include "skel_kernels.cuh"
#include "jit.h"

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
// Fast-path kinds: enum FastKind in jit.h.

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
        // Float forms must be exactly OMinF/OMaxF(acc, x) = acc CMP x ? acc : x
        // (lo = acc): the mirrored form returns the other operand on ties, which
        // differs for signed zeros and NaN. Int forms are equal either way.
        switch (C.op) {   // (lo < hi ? lo : hi) = min ; (lo > hi ? lo : hi) = max
            case PMX_OP_LTF: return lo == 0 ? K_MIN_F : K_VM;
            case PMX_OP_GTF: return lo == 0 ? K_MAX_F : K_VM;
            case PMX_OP_LTI: return K_MIN_I;
            case PMX_OP_GTI: return K_MAX_I;
        }
    }
    return K_VM;
}

// ==================================================================== device
// Streaming kernels (map / map2 / map->reduce / loop) live in skel_kernels.cuh,
// shared with the run-time compiled instantiations (jit.cu).

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

// map (lam row. reduce op acc (map g row)) rows — and foldl op acc row, reduce
// op acc row: one thread per row, the inner fold sequential in element order
// (inside a map body the reference's skeletons run sequentially,
// interp.py:82-84, so the fold is a left fold from acc).  g sees (x, index in
// the row), op sees (acc, x).  Errors report the row (the map's element).
__global__ void k_rows_fold_vm(const __grid_constant__ pmx_program G, int has_g,
                               const __grid_constant__ pmx_program OP, const void* x, int xt,
                               const int64_t* __restrict__ offs, int64_t nrows, int64_t init,
                               void* out, int ot, uint64_t* err) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nrows; r += stride) {
        int64_t acc = init;
        int code = 0;
        const int64_t lo = offs[r], hi = offs[r + 1];
        for (int64_t e = lo; e < hi && !code; ++e) {
            int64_t R[PMX_MAX_REGS];
            int64_t v = load_elem(x, xt, e);
            if (has_g) {
                R[0] = v;
                R[1] = e - lo;
                code = vm_run(G, R);
                if (code) break;
                v = vm_opnd(G, R, G.out);
            }
            R[0] = acc;
            R[1] = v;
            code = vm_run(OP, R);
            if (!code) acc = vm_opnd(OP, R, OP.out);
        }
        if (!code && !store_elem(out, ot, r, acc)) code = PMX_E_F32_RANGE;
        if (code) raise_err(err, r, code);
    }
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
__global__ void k_seq_loop(pmx_program P, const double* src, double* a, double* b, int64_t m, int64_t steps,
                           uint64_t* err) {
    cg::grid_group grid = cg::this_grid();
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t t = 0; t < steps; ++t) {
        const double* cur = t == 0 ? src : ((t & 1) ? b : a);   // step 0 reads the caller's state
        double* nxt = (t & 1) ? a : b;
        P.arrays[0].data = const_cast<double*>(cur);   // previous state visible to GET through arrays[0]
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

// offsets of a regular nested sequence: off[i] = i * row_len, i in [0, nrows]
__global__ void k_row_offsets(int64_t* off, int64_t nrows, int64_t row_len) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= nrows; i += (int64_t)gridDim.x * blockDim.x)
        off[i] = i * row_len;
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

// Grid of a streaming kernel over n elements: at least 8 four-element packets
// per thread, at most one resident wave (`cap` CTAs).
int stream_grid(int64_t n, int cap) {
    int64_t want = (n / 4 + kStreamThreads * 8 - 1) / (kStreamThreads * 8);
    if (want > cap) want = cap;
    return (int)(want < 1 ? 1 : want);
}

// Workspace layout: [ticket u32 | pad to 256][partials: grid * 16 bytes]
static const int kReduceThreads = kStreamThreads;


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

template <class TX, class TY, class F, class Op, bool WY, bool RED>
static int launch_mr(const TX* x, TY* y, int64_t n, F f, void* ws, typename Op::A init,
                     typename Op::A* out, cudaStream_t st, const pmx_peer_group* pgp = nullptr,
                     uint64_t* err = nullptr) {
    pmx_peer_group pg;
    if (pgp) pg = *pgp; else memset(&pg, 0, sizeof(pg));
    static int grid_cache[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!grid_cache[dev & 63])
        grid_cache[dev & 63] = occupancy_grid(k_map_reduce_vec<TX, TY, F, Op, WY, RED>, (int64_t)1 << 40, kReduceThreads);
    int grid = stream_grid(n, grid_cache[dev & 63]);
    unsigned* ticket = (unsigned*)ws;
    typename Op::A* partials = (typename Op::A*)((char*)ws + 256);
    bool aligned = ((uintptr_t)x % (4 * sizeof(TX)) == 0) && (!WY || (uintptr_t)y % (4 * sizeof(TY)) == 0);
    if (aligned)
        k_map_reduce_vec<TX, TY, F, Op, WY, RED><<<grid, kReduceThreads, 0, st>>>(x, y, n, f, partials, ticket, init, out, pg, err);
    else
        k_map_reduce_scalar<TX, TY, F, Op, WY, RED><<<grid, kReduceThreads, 0, st>>>(x, y, n, f, partials, ticket, init, out, pg, err);
    PMX_CHECK_LAUNCH("map_reduce");
    return 0;
}

// Dispatch on reduce operator for storage type T and functor F.
template <class T, class F>
static int dispatch_op(int okind, const T* x, T* y, int64_t n, F f, void* ws,
                       const void* init_host, void* out, cudaStream_t st,
                       const pmx_peer_group* pg = nullptr, uint64_t* err = nullptr) {
    const bool wy = y != nullptr;
#define PMX_MR(OP, ACC)                                                                              \
    {                                                                                                \
        ACC init; memcpy(&init, init_host, 8);                                                       \
        return wy ? launch_mr<T, T, F, OP, true, true>(x, y, n, f, ws, init, (ACC*)out, st, pg, err)  \
                  : launch_mr<T, T, F, OP, false, true>(x, y, n, f, ws, init, (ACC*)out, st, pg, err); \
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
static int dispatch_map_only(const T* x, T* y, int64_t n, F f, cudaStream_t st, uint64_t* err) {
    return launch_mr<T, T, F, NoReduce, true, false>(x, y, n, f, nullptr, 0.0, nullptr, st, nullptr, err);
}


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
            return dispatch_op<float>(ok, (const float*)x, (float*)y, n, FIdentity<double>{}, ws, init_host, out, st, pg, err);
        if (fk == K_AFFINE_F)
            return dispatch_op<float>(ok, (const float*)x, (float*)y, n, FAffineF{A.af, A.bf},
                                      ws, init_host, out, st, pg, err);
    } else if (xt == PMX_F64 && float_op) {
        if (fk == K_IDENTITY)
            return dispatch_op<double>(ok, (const double*)x, (double*)y, n, FIdentity<double>{}, ws, init_host, out, st, pg, err);
        if (fk == K_AFFINE_F)
            return dispatch_op<double>(ok, (const double*)x, (double*)y, n, FAffineF{A.af, A.bf},
                                       ws, init_host, out, st, pg, err);
    } else if (xt == PMX_I64 && int_op) {
        if (fk == K_IDENTITY)
            return dispatch_op<int64_t>(ok, (const int64_t*)x, (int64_t*)y, n, FIdentity<int64_t>{}, ws, init_host, out, st, pg, err);
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
        if (kind == K_AFFINE_F && xt == PMX_F32)
            return dispatch_map_only<float>((const float*)x, (float*)y, n,
                                            FAffineF{A.af, A.bf}, st, err);
        if (kind == K_AFFINE_F && xt == PMX_F64)
            return dispatch_map_only<double>((const double*)x, (double*)y, n,
                                             FAffineF{A.af, A.bf}, st, err);
        if (kind == K_AFFINE_I && xt == PMX_I64)
            return dispatch_map_only<int64_t>((const int64_t*)x, (int64_t*)y, n,
                                              FAffineI{A.ai, A.bi}, st, err);
    }
    PMX_REQUIRE(f, "pmx_map: null program with differing dtypes");
    int jr = jit_map(f, x, xt, y, yt, n, err, st);
    if (jr <= 0) return jr;
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
    int jr = jit_map2(f, x, xt, y, yt, z, zt, n, err, (cudaStream_t)stream);
    if (jr <= 0) return jr;
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
    const int okind = recognise_reduce(op);
    if (okind != K_VM && ((okind < K_ADD_I) == (acc_dtype == PMX_F64))) {
        r = jit_map_reduce(f, okind, x, xt, n, init_host, out, y, yt, ws, st, nullptr, err);
        if (r <= 0) return r;
    }
    if (okind == K_VM && y == nullptr) {     // unrecognised operator: ordered specialised kernel
        r = jit_reduce_generic(f, op, x, xt, n, init_host, acc_dtype, out, ws, st, err);
        if (r <= 0) return r;
    }
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
    const int okind = recognise_reduce(op);
    if (r == 1 && okind != K_VM && ((okind < K_ADD_I) == (acc_dtype == PMX_F64)))
        r = jit_map_reduce(f, okind, x, xt, n, init_host, out, nullptr, xt, ws, (cudaStream_t)stream, g, err);
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

int pmx_map_rows_fold(const pmx_program* g, const pmx_program* op, const void* x, int32_t xt,
                      const int64_t* offsets, int64_t nrows, const void* init_host, void* out, int32_t out_dtype,
                      uint64_t* err, void* stream) {
    PMX_REQUIRE(op && init_host && offsets && out, "pmx_map_rows_fold: null argument");
    PMX_REQUIRE(nrows >= 0, "pmx_map_rows_fold: negative row count");
    if (nrows == 0) return 0;
    int64_t init;
    memcpy(&init, init_host, 8);
    pmx_program none;
    memset(&none, 0, sizeof(none));
    k_rows_fold_vm<<<grid_for(nrows, 128, 8), 128, 0, (cudaStream_t)stream>>>(
        g ? *g : none, g ? 1 : 0, *op, x, xt, offsets, nrows, init, out, out_dtype, err);
    PMX_CHECK_LAUNCH("rows_fold");
    return 0;
}

int pmx_loop(const pmx_program* body, int64_t n, uint64_t* err, void* stream) {
    PMX_REQUIRE(body, "pmx_loop: null body");
    if (n <= 0) return 0;    // interp.py:347-348
    int jr = jit_loop(body, n, err, (cudaStream_t)stream);
    if (jr <= 0) return jr;
    int grid = grid_for(n, 256, 8);
    k_loop_vm<<<grid, 256, 0, (cudaStream_t)stream>>>(*body, n, err);
    PMX_CHECK_LAUNCH("loop_vm");
    return 0;
}

int pmx_seq_loop_from(const pmx_program* f, const double* init, double* state, double* scratch, int64_t m,
                      int64_t steps, uint64_t* err, void* stream) {
    PMX_REQUIRE(f && init && state && scratch, "pmx_seq_loop: null argument");
    PMX_REQUIRE(f->n_arrays >= 1, "pmx_seq_loop: program must reserve arrays[0] for the state");
    if (m <= 0) return 0;
    cudaStream_t st = (cudaStream_t)stream;
    if (steps <= 0) {
        if (init != state) {
            cudaError_t e = cudaMemcpyAsync(state, init, (size_t)m * sizeof(double), cudaMemcpyDeviceToDevice, st);
            if (e != cudaSuccess) { set_last_error("seq_loop: %s", cudaGetErrorString(e)); return -2; }
        }
        return 0;
    }
    // run-time specialised persistent kernel (jit.cu); its grid-barrier word is
    // the 8-byte slot after the m scratch values (scratch holds m + 8 doubles)
    {
        unsigned* bar = reinterpret_cast<unsigned*>(scratch + m);
        int jr = jit_seq_loop(f, init, state, scratch, m, steps, bar, err, st);
        if (jr < 0) return jr;
        if (jr == 0) {
            if (steps & 1) {
                k_copy_f64<<<grid_for(m, 256, 4), 256, 0, st>>>(scratch, state, m);
                PMX_CHECK_LAUNCH("seq_loop copy");
            }
            return 0;
        }
    }
    int dev = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_seq_loop, 256, 0);
    if (per_sm < 1) per_sm = 1;
    int grid = grid_for(m, 256, per_sm);
    pmx_program P = *f;
    void* args[] = {&P, &init, &state, &scratch, &m, &steps, &err};
    cudaError_t e = cudaLaunchCooperativeKernel((void*)k_seq_loop, grid, 256, args, 0, st);
    if (e != cudaSuccess) { set_last_error("seq_loop: %s", cudaGetErrorString(e)); return -2; }
    if (steps & 1) {   // result landed in scratch: copy back so `state` holds it
        k_copy_f64<<<grid_for(m, 256, 4), 256, 0, st>>>(scratch, state, m);
        PMX_CHECK_LAUNCH("seq_loop copy");
    }
    return 0;
}

int pmx_seq_loop(const pmx_program* f, double* state, double* scratch, int64_t m, int64_t steps,
                 uint64_t* err, void* stream) {
    return pmx_seq_loop_from(f, state, state, scratch, m, steps, err, stream);
}

int pmx_row_offsets(int64_t* offsets, int64_t nrows, int64_t row_len, void* stream) {
    PMX_REQUIRE(offsets, "pmx_row_offsets: null offsets");
    PMX_REQUIRE(nrows >= 0 && row_len >= 0, "pmx_row_offsets: negative size");
    k_row_offsets<<<grid_for(nrows + 1, 256, 4), 256, 0, (cudaStream_t)stream>>>(offsets, nrows, row_len);
    PMX_CHECK_LAUNCH("row_offsets");
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
