// Viterbi decoding at scale: the reference's HMM program (programs/viterbi.pmx
// :23-59; oracle tests/test_acceptance.py:307-354) batched over signals, for
// state counts where the one-CTA-per-signal kernel (hmm.cu k_viterbi) leaves
// the FP64 pipe idle.
//
// Semantics kept bit for bit (fp64, like the reference's Float):
//   chi0[i]   = log(init i) + logEmit[i][obs 0]                 (:31-33)
//   scores_i  = chi[i] + logTrans[i][j]                          (:38-39)
//   best      = argmax scores, first index on ties (strict >)   (:26-29)
//   chi'[j]   = scores_best + logEmit[j][obs t]                  (:42)
//   path      = backtrack from argmax chiFinal                   (:53-57)
// Every score is one rounded fp64 add and the max is order-independent
// except for ties, which the increasing-i strict comparison resolves to the
// smallest index exactly as the reference's foldl does.
//
// B200 design: a CTA owns MS = 8192/S signals for all T steps (persistent in
// time, no grid sync); chi lives in shared memory (transposed, MS signals
// contiguous per state); log A streams from L2 through a cp.async double
// buffer of KT rows (A is step-invariant, so the buffer prefetches across
// steps); each thread keeps a 4-signal x 8-state tile of (best score, argmax)
// in registers, so one A row chunk and one chi chunk feed 32 max-plus cells.
// Per cell: one DADD + one DSETP (FP64 pipe) + two selects: the kernel is
// FP64-pipe bound (64 lanes/clk/SM => 32 cells/clk/SM).
// Back pointers go to the caller's workspace [nsig][T-1][S] int32; a second
// kernel (one warp per signal) takes the final argmax and walks them back.
#include "common.cuh"

namespace pmx {

constexpr int VT_NT = 256;     // threads per CTA
constexpr int VT_KT = 8;       // log A rows per pipeline stage

__device__ __forceinline__ void vt_cp_async16(void* smem, const void* gmem) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void vt_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void vt_wait() { asm volatile("cp.async.wait_group %0;" :: "n"(N) : "memory"); }

template <int S>
__device__ __forceinline__ void vt_load_stage(double* dst, const double* __restrict__ lA, int kt) {
    constexpr int VEC = VT_KT * S / 2;     // 16-byte chunks per stage
    const double* src = lA + (int64_t)kt * VT_KT * S;
#pragma unroll 4
    for (int v = threadIdx.x; v < VEC; v += VT_NT) vt_cp_async16(dst + v * 2, src + v * 2);
}

template <int S>
__global__ void __launch_bounds__(VT_NT, 1)
k_viterbi_tiled(const double* __restrict__ log_pi, const double* __restrict__ log_A,
                const double* __restrict__ log_E, int K, const int* __restrict__ obs, int64_t nsig, int T,
                int* __restrict__ back, double* __restrict__ chi_out) {
    constexpr int GT = S / 8;              // threads per signal group (8 states each)
    constexpr int NG = VT_NT / GT;         // signal groups
    constexpr int MS = NG * 4;             // signals per CTA
    constexpr int NKT = S / VT_KT;
    extern __shared__ __align__(16) double vsm[];
    double* chiT = vsm;                    // [S][MS]
    double* As = vsm + S * MS;             // [2][KT][S]
    __shared__ int s_sym[MS];

    const int tid = threadIdx.x;
    const int sg = tid / GT, jg = tid % GT;
    const int j0 = jg * 4, j1 = S / 2 + jg * 4;
    const int64_t s0 = (int64_t)blockIdx.x * MS;
    const int64_t steps = T > 1 ? T - 1 : 0;

    // chi0 (viterbi.pmx:31-33)
    for (int v = tid; v < S * MS; v += VT_NT) {
        const int i = v / MS, m = v % MS;
        const int64_t sig = s0 + m;
        const int o = sig < nsig ? obs[sig * T] : 0;
        chiT[v] = __dadd_rn(log_pi[i], log_E[(int64_t)i * K + o]);
    }
    if (T > 1) { vt_load_stage<S>(As, log_A, 0); vt_commit(); }
    __syncthreads();

    for (int t = 1; t < T; ++t) {
        if (tid < MS) {
            const int64_t sig = s0 + tid;
            s_sym[tid] = sig < nsig ? obs[sig * T + t] : 0;
        }
        double best[4][8];
        int arg[4][8];
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
            for (int y = 0; y < 8; ++y) { best[x][y] = __longlong_as_double(0xfff0000000000000ll); arg[x][y] = 0; }
        for (int kt = 0; kt < NKT; ++kt) {
            const int stage = kt & 1;
            const bool more = (kt + 1 < NKT) || (t + 1 < T);
            if (more) {
                vt_load_stage<S>(As + (stage ^ 1) * VT_KT * S, log_A, (kt + 1) % NKT);
                vt_commit();
                vt_wait<1>();
            } else {
                vt_wait<0>();
            }
            __syncthreads();
            const double* At = As + stage * VT_KT * S;
#pragma unroll
            for (int kk = 0; kk < VT_KT; ++kk) {
                const int k = kt * VT_KT + kk;
                const double2 a01 = *reinterpret_cast<const double2*>(chiT + k * MS + sg * 4);
                const double2 a23 = *reinterpret_cast<const double2*>(chiT + k * MS + sg * 4 + 2);
                const double2 b01 = *reinterpret_cast<const double2*>(At + kk * S + j0);
                const double2 b23 = *reinterpret_cast<const double2*>(At + kk * S + j0 + 2);
                const double2 b45 = *reinterpret_cast<const double2*>(At + kk * S + j1);
                const double2 b67 = *reinterpret_cast<const double2*>(At + kk * S + j1 + 2);
                const double av[4] = {a01.x, a01.y, a23.x, a23.y};
                const double bv[8] = {b01.x, b01.y, b23.x, b23.y, b45.x, b45.y, b67.x, b67.y};
#pragma unroll
                for (int x = 0; x < 4; ++x)
#pragma unroll
                    for (int y = 0; y < 8; ++y) {
                        const double sc = __dadd_rn(av[x], bv[y]);
                        if (sc > best[x][y]) { best[x][y] = sc; arg[x][y] = k; }   // first max wins
                    }
            }
            __syncthreads();   // stage buffer (and, at the last kt, chiT) reads complete
        }
        // chi'[j] = best + logEmit[j][obs t]; back pointers (viterbi.pmx:40-47)
#pragma unroll
        for (int x = 0; x < 4; ++x) {
            const int m = sg * 4 + x;
            const int64_t sig = s0 + m;
            const int o = s_sym[m];
            int* bk = back + (sig * steps + (t - 1)) * (int64_t)S;
#pragma unroll
            for (int y = 0; y < 8; ++y) {
                const int j = y < 4 ? j0 + y : j1 + y - 4;
                best[x][y] = __dadd_rn(best[x][y], __ldg(log_E + (int64_t)j * K + o));
            }
            if (sig < nsig) {
                *reinterpret_cast<int4*>(bk + j0) = make_int4(arg[x][0], arg[x][1], arg[x][2], arg[x][3]);
                *reinterpret_cast<int4*>(bk + j1) = make_int4(arg[x][4], arg[x][5], arg[x][6], arg[x][7]);
            }
        }
#pragma unroll
        for (int y = 0; y < 8; ++y) {
            const int j = y < 4 ? j0 + y : j1 + y - 4;
            *reinterpret_cast<double2*>(chiT + j * MS + sg * 4) = make_double2(best[0][y], best[1][y]);
            *reinterpret_cast<double2*>(chiT + j * MS + sg * 4 + 2) = make_double2(best[2][y], best[3][y]);
        }
        __syncthreads();
    }
    for (int v = tid; v < S * MS; v += VT_NT) {
        const int i = v / MS, m = v % MS;
        const int64_t sig = s0 + m;
        if (sig < nsig) chi_out[sig * S + i] = chiT[v];
    }
}

// One warp per signal: bestLast = argmax chiFinal (first max), logp, and the
// walk back through the pointers (viterbi.pmx:50-57).
__global__ void k_viterbi_backtrack(const double* __restrict__ chi, const int* __restrict__ back, int S,
                                    int64_t nsig, int T, int* __restrict__ path, double* __restrict__ logp) {
    const int64_t sig = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (sig >= nsig) return;
    const double* c = chi + sig * S;
    double bv = __longlong_as_double(0xfff0000000000000ll);
    int bi = 0x7fffffff;
    for (int i = lane; i < S; i += 32) {
        const double v = c[i];
        if (v > bv || (v == bv && i < bi)) { bv = v; bi = i; }
    }
    for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    if (bi == 0x7fffffff) bi = 0;             // all -inf / NaN: the reference keeps index 0
    if (lane != 0) return;
    const int64_t steps = T > 1 ? T - 1 : 0;
    int* p = path + sig * T;
    p[T - 1] = bi;
    int s = bi;
    const int* bk = back + sig * steps * (int64_t)S;
    for (int t = T - 2; t >= 0; --t) {
        s = bk[(int64_t)t * S + s];
        p[t] = s;
    }
    logp[sig] = c[bi];
}

bool viterbi_tiled_eligible(int S) { return S == 256 || S == 512 || S == 1024; }

int viterbi_tiled_launch(const double* log_pi, const double* log_A, const double* log_E, int S, int K,
                         const int* obs, int64_t nsig, int T, int* path, double* logp, int* back,
                         double* chi_final, cudaStream_t st) {
#define PMX_VT(SS)                                                                                 \
    if (S == SS) {                                                                                 \
        constexpr int MS = 4 * (VT_NT / (SS / 8));                                                 \
        const size_t smem = ((size_t)SS * MS + 2 * (size_t)VT_KT * SS) * sizeof(double);           \
        cudaFuncSetAttribute(k_viterbi_tiled<SS>, cudaFuncAttributeMaxDynamicSharedMemorySize,     \
                             (int)smem);                                                           \
        k_viterbi_tiled<SS><<<(unsigned)((nsig + MS - 1) / MS), VT_NT, smem, st>>>(                \
            log_pi, log_A, log_E, K, obs, nsig, T, back, chi_final);                               \
        PMX_CHECK_LAUNCH("viterbi_tiled");                                                         \
    }
    PMX_VT(1024)
    PMX_VT(512)
    PMX_VT(256)
#undef PMX_VT
    k_viterbi_backtrack<<<(unsigned)((nsig + 7) / 8), 256, 0, st>>>(chi_final, back, S, nsig, T, path, logp);
    PMX_CHECK_LAUNCH("viterbi_backtrack");
    return 0;
}

}  // namespace pmx
