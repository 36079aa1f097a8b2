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
// Per cell: one DADD + one DSETP (FP64 pipe) + three selects (SASS: DADD,
// DSETP.GT, 2x FSEL, SEL) — five issue slots per cell, so the kernel is
// issue-bound at <= 25.6 cells/clk/SM (4 schedulers x 32 lanes / 5) before
// the FP64 pipe's 32 cells/clk/SM (64 lanes, 2 FP64 ops per cell).
// Back pointers go to the caller's workspace [nsig][T-1][S] int32; a second
// kernel (one warp per signal) takes the final argmax and walks them back.
#include <stdlib.h>
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

// ARGMAX = true: (score, argmax) per cell in registers, back pointers stored
// [nsig][T-1][S] int32 (DADD + DSETP + 3 selects per cell: issue-bound).
// ARGMAX = false: scores only (DADD + DMNMX per cell) and the chi vectors of
// every step stored [nsig][T-1][S] fp64; the backtrack recomputes the one
// argmax per step it needs (viterbi.pmx's back pointer for the state on the
// path) from chi_{t-1} and a column of log A — bit-identical scores, 1/S of
// the forward work.
template <int S, bool ARGMAX>
__global__ void __launch_bounds__(VT_NT, 1)
k_viterbi_tiled(const double* __restrict__ log_pi, const double* __restrict__ log_A,
                const double* __restrict__ log_E, int K, const int* __restrict__ obs, int64_t nsig, int T,
                int* __restrict__ back, double* __restrict__ hist, double* __restrict__ chi_out) {
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
        if (!ARGMAX && T > 1 && sig < nsig) hist[sig * steps * S + i] = chiT[v];
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
                        if (ARGMAX) {
                            if (sc > best[x][y]) { best[x][y] = sc; arg[x][y] = k; }   // first max wins
                        } else {
                            best[x][y] = fmax(best[x][y], sc);
                        }
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
            if (ARGMAX && sig < nsig) {
                *reinterpret_cast<int4*>(bk + j0) = make_int4(arg[x][0], arg[x][1], arg[x][2], arg[x][3]);
                *reinterpret_cast<int4*>(bk + j1) = make_int4(arg[x][4], arg[x][5], arg[x][6], arg[x][7]);
            }
            if (!ARGMAX && sig < nsig && t + 1 < T) {      // chi_t, read back by the backtrack
                double* h = hist + (sig * steps + t) * (int64_t)S;
                *reinterpret_cast<double2*>(h + j0) = make_double2(best[x][0], best[x][1]);
                *reinterpret_cast<double2*>(h + j0 + 2) = make_double2(best[x][2], best[x][3]);
                *reinterpret_cast<double2*>(h + j1) = make_double2(best[x][4], best[x][5]);
                *reinterpret_cast<double2*>(h + j1 + 2) = make_double2(best[x][6], best[x][7]);
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

// Recomputing backtrack: s_{t-1} = first argmax_i (chi_{t-1}[i] + logA[i][s_t])
// with logA^T rows contiguous (lAT[j][i]); one warp per signal.
__global__ void k_viterbi_backtrack_recompute(const double* __restrict__ chi, const double* __restrict__ hist,
                                              const double* __restrict__ lAT, int S, int64_t nsig, int T,
                                              int* __restrict__ path, double* __restrict__ logp) {
    const int64_t sig = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (sig >= nsig) return;
    auto warp_argmax = [&](double bv, int bi) {
        for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
        }
        return bi == 0x7fffffff ? 0 : bi;
    };
    const double* c = chi + sig * S;
    double bv = __longlong_as_double(0xfff0000000000000ll);
    int bi = 0x7fffffff;
    for (int i = lane; i < S; i += 32) {
        const double v = c[i];
        if (v > bv) { bv = v; bi = i; }        // lanes scan increasing i: strict > keeps the first
    }
    int s = warp_argmax(bv, bi);
    const int64_t steps = T > 1 ? T - 1 : 0;
    int* p = path + sig * T;
    if (lane == 0) { p[T - 1] = s; logp[sig] = c[s]; }
    for (int t = T - 1; t >= 1; --t) {
        const double* h = hist + (sig * steps + (t - 1)) * (int64_t)S;
        const double* col = lAT + (int64_t)s * S;
        bv = __longlong_as_double(0xfff0000000000000ll);
        bi = 0x7fffffff;
#pragma unroll 4
        for (int i = lane; i < S; i += 32) {
            const double v = __dadd_rn(h[i], col[i]);
            if (v > bv) { bv = v; bi = i; }
        }
        s = warp_argmax(bv, bi);
        if (lane == 0) p[t - 1] = s;
    }
}

// ---- pruned max-plus (branch and bound over each column's sorted entries) ----
// chi'[j] = max_i (chi[i] + logA[i][j]).  With the entries of column j visited in
// decreasing logA order (ties: increasing i) and M = max_i chi[i], every
// candidate from rank r on scores at most M (+) logA_r (rounded addition is
// monotonic), so the scan of (signal, j) stops at the first r with
// M (+) logA_r < best: nothing later can beat or tie the best found.  The
// best keeps the reference's first-index tie rule explicitly (score >, or ==
// with a smaller i), so paths and scores are the dense kernel's bit for bit.
// On the bench model ~7% of the candidates are visited (measured on the
// Dirichlet(1) model in numpy: 4-14% per step).
template <int S>
__global__ void __launch_bounds__(S / 2) k_viterbi_sort_cols(const double* __restrict__ lA, double* __restrict__ lAs,
                                                             uint16_t* __restrict__ perm) {
    __shared__ double v[S];
    __shared__ int ix[S];
    const int j = blockIdx.x;
    for (int i = threadIdx.x; i < S; i += blockDim.x) { v[i] = lA[(int64_t)i * S + j]; ix[i] = i; }
    __syncthreads();
    for (int k = 2; k <= S; k <<= 1)                    // bitonic: "before" = larger, then smaller i
        for (int jj = k >> 1; jj > 0; jj >>= 1) {
            for (int t = threadIdx.x; t < S / 2; t += blockDim.x) {
                const int i = (t / jj) * 2 * jj + (t % jj), q = i + jj;
                const double a = v[i], b = v[q];
                const int ia = ix[i], ib = ix[q];
                // NaN entries (a NaN log A) sort after every number: they never win
                // (score > best is false) and never end a scan early (the bound
                // test is false), as in the dense kernel
                const bool na = a != a, nb = b != b;
                const bool a_first = (na != nb) ? nb : (na ? ia < ib : (a > b || (a == b && ia < ib)));
                if (((i & k) == 0) ? !a_first : a_first) { v[i] = b; v[q] = a; ix[i] = ib; ix[q] = ia; }
            }
            __syncthreads();
        }
    for (int r = threadIdx.x; r < S; r += blockDim.x) {
        lAs[(int64_t)j * S + r] = v[r];
        perm[(int64_t)j * S + r] = (uint16_t)ix[r];
    }
}

// A CTA owns VP_MS = 8 signals (chi double-buffered in shared memory,
// [state][signal]); warp w scans columns jb + 4w + g for its four lane groups
// g (8 lanes = the 8 signals), the warp stepping on until every lane's bound
// is met.
constexpr int VP_MS = 8, VP_NT = 512;
template <int S>
__global__ void __launch_bounds__(VP_NT, 1)
k_viterbi_pruned(const double* __restrict__ log_pi, const double* __restrict__ lAs,
                 const uint16_t* __restrict__ perm, const double* __restrict__ log_E, int K,
                 const int* __restrict__ obs, int64_t nsig, int T, int* __restrict__ back,
                 double* __restrict__ chi_out, unsigned long long* __restrict__ visited) {
    extern __shared__ __align__(16) double vsm[];
    uint32_t rounds = 0;                   // candidate rounds this lane's scans ran (roofline counter)
    double* cur = vsm;                     // [S][VP_MS]
    double* nxt = vsm + S * VP_MS;
    __shared__ int s_sym[VP_MS];
    __shared__ double s_red[VP_NT / 32][VP_MS];
    __shared__ double s_M[VP_MS];
    __shared__ int s_next;                 // next group of 4 target states (dynamic, per step)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int m = lane & 7, g = lane >> 3;
    const int64_t s0 = (int64_t)blockIdx.x * VP_MS;
    const int64_t steps = T > 1 ? T - 1 : 0;
    const int64_t sig = s0 + m;
    const double NEG_INF = __longlong_as_double(0xfff0000000000000ll);
    for (int v = tid; v < S * VP_MS; v += VP_NT) {          // chi0 (viterbi.pmx:31-33)
        const int i = v / VP_MS, mm = v % VP_MS;
        const int64_t sg = s0 + mm;
        const int o = sg < nsig ? obs[sg * T] : 0;
        cur[v] = __dadd_rn(log_pi[i], log_E[(int64_t)i * K + o]);
    }
    __syncthreads();
    for (int t = 1; t < T; ++t) {
        if (tid < VP_MS) s_sym[tid] = s0 + tid < nsig ? obs[(s0 + tid) * T + t] : 0;
        if (tid == 0) s_next = 0;
        // M = max_i chi[i] per signal
        double mx = NEG_INF;
        for (int i = tid >> 3; i < S; i += VP_NT / 8) mx = fmax(mx, cur[i * VP_MS + (tid & 7)]);
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 8));
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
        if (lane < 8) s_red[warp][lane] = mx;
        __syncthreads();
        if (tid < VP_MS) {
            double r = s_red[0][tid];
            for (int w = 1; w < VP_NT / 32; ++w) r = fmax(r, s_red[w][tid]);
            s_M[tid] = r;
        }
        __syncthreads();
        const double M = s_M[m];
        const int o = s_sym[m];
        // groups of 4 target states handed out dynamically: scans stop at different
        // ranks, so a static split leaves warps idle at the step's barrier
        for (;;) {
            int jg = 0;
            if (lane == 0) jg = atomicAdd(&s_next, 1);
            jg = __shfl_sync(0xffffffffu, jg, 0);
            if (jg >= S / 4) break;
            const int j = jg * 4 + g;
            const double* col = lAs + (int64_t)j * S;
            const uint16_t* pc = perm + (int64_t)j * S;
            double best = NEG_INF;
            int arg = 0;
            bool act = true;
            // VP_R candidates per round: sorted values and indices by vector loads, the
            // scores independent; one warp vote per round
            constexpr int VP_R = 16;
            for (int r0 = 0; r0 < S; r0 += VP_R) {
                double lv[VP_R];
                uint32_t pw[VP_R / 2];
#pragma unroll
                for (int u = 0; u < VP_R; u += 2) {
                    const double2 l2 = __ldg(reinterpret_cast<const double2*>(col + r0 + u));
                    lv[u] = l2.x;
                    lv[u + 1] = l2.y;
                }
#pragma unroll
                for (int u = 0; u < VP_R / 8; ++u) {
                    const uint4 pk = __ldg(reinterpret_cast<const uint4*>(pc + r0) + u);
                    pw[4 * u] = pk.x; pw[4 * u + 1] = pk.y; pw[4 * u + 2] = pk.z; pw[4 * u + 3] = pk.w;
                }
                double sc[VP_R];
#pragma unroll
                for (int u = 0; u < VP_R; ++u) {
                    const int i = (int)((pw[u >> 1] >> (16 * (u & 1))) & 0xffffu);
                    sc[u] = __dadd_rn(cur[i * VP_MS + m], lv[u]);
                }
#pragma unroll
                for (int u = 0; u < VP_R; ++u) {
                    if (act && __dadd_rn(M, lv[u]) < best) act = false;   // nothing later can tie
                    const int i = (int)((pw[u >> 1] >> (16 * (u & 1))) & 0xffffu);
                    if (act && (sc[u] > best || (sc[u] == best && i < arg))) { best = sc[u]; arg = i; }
                }
                ++rounds;
                if (!__any_sync(0xffffffffu, act)) break;
            }
            nxt[j * VP_MS + m] = __dadd_rn(best, __ldg(log_E + (int64_t)j * K + o));   // (:42)
            if (sig < nsig) back[(sig * steps + (t - 1)) * (int64_t)S + j] = arg;
        }
        __syncthreads();
        double* tmp = cur; cur = nxt; nxt = tmp;
    }
    for (int v = tid; v < S * VP_MS; v += VP_NT) {
        const int i = v / VP_MS, mm = v % VP_MS;
        if (s0 + mm < nsig) chi_out[(s0 + mm) * S + i] = cur[v];
    }
    unsigned long long cells = (unsigned long long)rounds * 16ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cells += __shfl_xor_sync(0xffffffffu, cells, o);
    if (lane == 0) atomicAdd(visited, cells);
}

__global__ void k_transpose_f64(const double* __restrict__ a, double* __restrict__ at, int S) {
    __shared__ double tile[32][33];
    const int bi = blockIdx.y * 32, bj = blockIdx.x * 32;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) tile[r][threadIdx.x] = a[(int64_t)(bi + r) * S + bj + threadIdx.x];
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) at[(int64_t)(bj + r) * S + bi + threadIdx.x] = tile[threadIdx.x][r];
}

bool viterbi_tiled_eligible(int S) { return S == 256 || S == 512 || S == 1024; }

// workspace of the tiled path: max(back pointers int32, chi history fp64) | final chi | log A^T
// | sorted-column permutation | visited-cell counter (pruned kernel)
static size_t viterbi_counter_offset(int S, int64_t nsig, int T) {
    const size_t steps = (size_t)(T > 1 ? T - 1 : 0);
    const size_t h = ((size_t)nsig * steps * (size_t)S * sizeof(double) + 255) & ~(size_t)255;
    const size_t c = ((size_t)nsig * (size_t)S * sizeof(double) + 255) & ~(size_t)255;
    return (h + c + (size_t)S * S * sizeof(double) + (size_t)S * S * sizeof(uint16_t) + 7) & ~(size_t)7;
}

unsigned long long* viterbi_visited_counter(void* ws, int S, int64_t nsig, int T) {
    return (unsigned long long*)((char*)ws + viterbi_counter_offset(S, nsig, T));
}

size_t viterbi_tiled_workspace(int S, int64_t nsig, int T) {
    const size_t steps = (size_t)(T > 1 ? T - 1 : 0);
    const size_t h = ((size_t)nsig * steps * (size_t)S * sizeof(double) + 255) & ~(size_t)255;
    const size_t c = ((size_t)nsig * (size_t)S * sizeof(double) + 255) & ~(size_t)255;
    return h + c + (size_t)S * S * sizeof(double) + (size_t)S * S * sizeof(uint16_t) + 512;
}

int viterbi_tiled_launch(const double* log_pi, const double* log_A, const double* log_E, int S, int K,
                         const int* obs, int64_t nsig, int T, int* path, double* logp, void* ws,
                         cudaStream_t st) {
    // Default: argmax kept in the forward (back pointers). PMX_VITERBI_RECOMPUTE=1:
    // scores only + recomputing backtrack — measured slower (476 vs 353 ms at
    // the bench config): sm_100 has no fp64 max instruction, fmax lowers to
    // DSETP + selects, so a cell costs the same issue slots either way.
    static const bool argmax = !(getenv("PMX_VITERBI_RECOMPUTE") && getenv("PMX_VITERBI_RECOMPUTE")[0] == '1');
    const size_t steps = (size_t)(T > 1 ? T - 1 : 0);
    const size_t h = ((size_t)nsig * steps * (size_t)S * sizeof(double) + 255) & ~(size_t)255;
    const size_t c = ((size_t)nsig * (size_t)S * sizeof(double) + 255) & ~(size_t)255;
    int* back = (int*)ws;
    double* hist = (double*)ws;
    double* chi_final = (double*)((char*)ws + h);
    double* lAT = (double*)((char*)ws + h + c);
#define PMX_VT(SS, AM)                                                                             \
    if (S == SS) {                                                                                 \
        constexpr int MS = 4 * (VT_NT / (SS / 8));                                                 \
        const size_t smem = ((size_t)SS * MS + 2 * (size_t)VT_KT * SS) * sizeof(double);           \
        cudaFuncSetAttribute(k_viterbi_tiled<SS, AM>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                             (int)smem);                                                           \
        k_viterbi_tiled<SS, AM><<<(unsigned)((nsig + MS - 1) / MS), VT_NT, smem, st>>>(            \
            log_pi, log_A, log_E, K, obs, nsig, T, back, hist, chi_final);                         \
        PMX_CHECK_LAUNCH("viterbi_tiled");                                                         \
    }
    // default: the pruned scan over sorted columns; PMX_VITERBI_DENSE=1: every cell
    static const bool dense = getenv("PMX_VITERBI_DENSE") && getenv("PMX_VITERBI_DENSE")[0] == '1';
    unsigned long long* visited = viterbi_visited_counter(ws, S, nsig, T);
    cudaMemsetAsync(visited, 0, sizeof(unsigned long long), st);
    if (argmax && !dense) {
        uint16_t* perm = (uint16_t*)((char*)lAT + (size_t)S * S * sizeof(double));
#define PMX_VP(SS)                                                                                 \
        if (S == SS) {                                                                             \
            k_viterbi_sort_cols<SS><<<SS, SS / 2, 0, st>>>(log_A, lAT, perm);                       \
            PMX_CHECK_LAUNCH("viterbi_sort");                                                      \
            const size_t smem = 2 * (size_t)SS * VP_MS * sizeof(double);                           \
            cudaFuncSetAttribute(k_viterbi_pruned<SS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
            k_viterbi_pruned<SS><<<(unsigned)((nsig + VP_MS - 1) / VP_MS), VP_NT, smem, st>>>(     \
                log_pi, lAT, perm, log_E, K, obs, nsig, T, back, chi_final, visited);             \
            PMX_CHECK_LAUNCH("viterbi_pruned");                                                    \
        }
        PMX_VP(1024) PMX_VP(512) PMX_VP(256)
#undef PMX_VP
        k_viterbi_backtrack<<<(unsigned)((nsig + 7) / 8), 256, 0, st>>>(chi_final, back, S, nsig, T, path, logp);
        PMX_CHECK_LAUNCH("viterbi_backtrack");
        return 0;
    }
    if (argmax) {
        PMX_VT(1024, true)
        PMX_VT(512, true)
        PMX_VT(256, true)
        k_viterbi_backtrack<<<(unsigned)((nsig + 7) / 8), 256, 0, st>>>(chi_final, back, S, nsig, T, path, logp);
        PMX_CHECK_LAUNCH("viterbi_backtrack");
        return 0;
    }
    PMX_VT(1024, false)
    PMX_VT(512, false)
    PMX_VT(256, false)
#undef PMX_VT
    k_transpose_f64<<<dim3(S / 32, S / 32), dim3(32, 8), 0, st>>>(log_A, lAT, S);
    PMX_CHECK_LAUNCH("viterbi_transpose");
    k_viterbi_backtrack_recompute<<<(unsigned)((nsig + 7) / 8), 256, 0, st>>>(chi_final, hist, lAT, S, nsig, T,
                                                                             path, logp);
    PMX_CHECK_LAUNCH("viterbi_backtrack");
    return 0;
}

}  // namespace pmx
