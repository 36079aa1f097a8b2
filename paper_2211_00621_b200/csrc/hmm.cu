// HMM case studies: forward algorithm (BASELINE config) and Viterbi.
//
// Reference anchors
//   Viterbi: programs/viterbi.pmx:23-59 (the reference's HMM program; oracle
//            tests/test_acceptance.py:307-354).  Per step, `create numStates`
//            of per-state max/argmax over predecessors (viterbi.pmx:37-44),
//            then the `forward` recursion (35-48) and the backtrack (53-57).
//   Forward: SURVEY Appendix A.1 `hmm_forward.pmx` — the same trellis with
//            log-sum-exp in place of max (lse with max shift, A.1 lines 15-17),
//            batched over signals by `map`, ll = lse(alpha_{T-1}).
//
// B200 design (forward)
//   The log-space recursion alpha_t[j] = LSE_i(alpha_{t-1}[i] + log A_ij) +
//   log E_j,o_t is evaluated as the equivalent scaled linear recursion
//       a_t[j] = (sum_i ahat_{t-1}[i] * A_ij) * E_j,o_t ,  c_t = sum_j a_t[j],
//       ahat_t = a_t / c_t ,  ll = sum_t log c_t           (fp64 running sum)
//   so the S^2 work per step is a multiply-add contraction instead of S^2
//   exp/log.  Signals are independent, so a CTA owns a
//   tile of 32 signals for all T steps (persistent over time, no grid sync):
//   ahat lives in shared memory, A streams from L2 in k-tiles through a
//   cp.async double buffer, each thread accumulates an 8-signal x 8-state
//   register tile.  A general small-S kernel (one CTA per signal) covers
//   other state counts.
#include <stdlib.h>
#include <string.h>
#include "common.cuh"

namespace pmx {

// ------------------------------------------------------------------ prep
// E_lin[k*S + j] = exp(log_E[j*K + k]); pi_lin[j] = exp(log_pi[j])
__global__ void k_hmm_prep(const float* __restrict__ log_pi, const float* __restrict__ log_E,
                           int S, int K, float* __restrict__ E_lin, float* __restrict__ pi_lin) {
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < S * K; idx += gridDim.x * blockDim.x) {
        const int j = idx % S, k = idx / S;
        E_lin[idx] = expf(log_E[j * K + k]);
        if (k == 0) pi_lin[j] = expf(log_pi[j]);
    }
}

// ------------------------------------------------------- small-S forward
// One CTA per signal; thread-strided states; A read through L1/L2.
__global__ void k_hmm_fwd_small(const float* __restrict__ pi_lin, const float* __restrict__ A,
                                const float* __restrict__ E_lin, int S, const int* __restrict__ obs,
                                int64_t nsig, int T, double* __restrict__ out_ll) {
    extern __shared__ float sm[];
    float* ah = sm;          // [S] normalised alpha
    float* nw = sm + S;      // [S] next alpha
    __shared__ float s_red[32];
    __shared__ float s_c;
    const int64_t sig = blockIdx.x;
    if (sig >= nsig) return;
    const int* o = obs + sig * (int64_t)T;
    double ll = 0.0;
    for (int t = 0; t < T; ++t) {
        const int sym = o[t];
        const float* e = E_lin + (int64_t)sym * S;
        float part = 0.f;
        for (int j = threadIdx.x; j < S; j += blockDim.x) {
            float v;
            if (t == 0) {
                v = pi_lin[j] * e[j];
            } else {
                float acc = 0.f;
                for (int i = 0; i < S; ++i) acc = fmaf(ah[i], A[(int64_t)i * S + j], acc);
                v = acc * e[j];
            }
            nw[j] = v;
            part += v;
        }
        // block sum
        for (int off = 16; off > 0; off >>= 1) part += __shfl_xor_sync(0xffffffffu, part, off);
        if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = part;
        __syncthreads();
        if (threadIdx.x == 0) {
            float c = 0.f;
            for (int w = 0; w < (int)((blockDim.x + 31) >> 5); ++w) c += s_red[w];
            s_c = c;
            ll += log_scale((double)c);
        }
        __syncthreads();
        const float inv = 1.0f / s_c;
        for (int j = threadIdx.x; j < S; j += blockDim.x) ah[j] = nw[j] * inv;
        __syncthreads();
    }
    if (threadIdx.x == 0) out_ll[sig] = ll;
}

// ------------------------------------------------------- tiled forward
// S in {256, 512, 1024}; 32 signals per CTA; S/2 threads.
// Thread (sg, jg): signals sg*8 .. sg*8+7, states jg*4 + {0..3} and
// S/2 + jg*4 + {0..3}.  A warp shares sg, so ahat loads are broadcasts and
// A-tile loads are contiguous 16-byte lanes (conflict-free).
constexpr int HMM_MS = 32;   // signals per CTA
constexpr int HMM_KT = 8;    // A rows per pipeline stage

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" :: "n"(N) : "memory"); }

template <int S>
__device__ __forceinline__ void hmm_load_stage(float* dst, const float* __restrict__ A, int kt) {
    constexpr int NT = S / 2;
    constexpr int VEC = HMM_KT * S / 4;   // 16-byte chunks per stage
    const float* src = A + (int64_t)kt * HMM_KT * S;
#pragma unroll
    for (int v = threadIdx.x; v < VEC; v += NT) cp_async16(dst + v * 4, src + v * 4);
}

template <int S>
__global__ void __launch_bounds__(S / 2, 1)
k_hmm_fwd_tiled(const float* __restrict__ pi_lin, const float* __restrict__ A,
                const float* __restrict__ E_lin, const int* __restrict__ obs,
                int64_t nsig, int T, double* __restrict__ out_ll,
                const int* __restrict__ list = nullptr, const int* __restrict__ count = nullptr) {
    // list != nullptr: the fp16 tensor-core path's guard re-run — this CTA takes
    // entries [32 b, 32 b + 32) of the list of flagged signals (*count of them)
    constexpr int NT = S / 2;
    constexpr int GT = S / 8;              // threads per signal group
    constexpr int NW = NT / 32;
    constexpr int NKT = S / HMM_KT;
    extern __shared__ __align__(16) float smem[];
    float* aT = smem;                          // [S][32] ahat transposed
    float* As = smem + S * HMM_MS;             // [2][KT][S]
    __shared__ float s_red[NW][8];
    __shared__ float s_inv[HMM_MS];
    __shared__ int s_sym[HMM_MS];

    const int tid = threadIdx.x;
    const int sg = tid / GT, jg = tid % GT;
    const int warp = tid >> 5, lane = tid & 31;
    const int64_t s0 = (int64_t)blockIdx.x * HMM_MS;
    if (list) {
        nsig = *count;
        if (s0 >= nsig) return;
    }
    auto sig = [&](int64_t i) -> int64_t { return list ? (int64_t)list[i] : i; };
    const int j0 = jg * 4, j1 = S / 2 + jg * 4;
    double ll = 0.0;                           // thread tid < 32 owns signal s0 + tid

    // prefetch stage 0 of step 1
    if (T > 1) { hmm_load_stage<S>(As, A, 0); cp_async_commit(); }

    for (int t = 0; t < T; ++t) {
        if (tid < HMM_MS) {
            const int64_t s = s0 + tid;
            s_sym[tid] = (s < nsig) ? obs[sig(s) * T + t] : 0;
        }
        float acc[8][8];
#pragma unroll
        for (int a = 0; a < 8; ++a)
#pragma unroll
            for (int b = 0; b < 8; ++b) acc[a][b] = 0.f;

        if (t == 0) {
            float p[8];
#pragma unroll
            for (int q = 0; q < 4; ++q) { p[q] = pi_lin[j0 + q]; p[4 + q] = pi_lin[j1 + q]; }
#pragma unroll
            for (int a = 0; a < 8; ++a)
#pragma unroll
                for (int b = 0; b < 8; ++b) acc[a][b] = p[b];
        } else {
            for (int kt = 0; kt < NKT; ++kt) {
                const int stage = kt & 1;
                // issue the next stage (wrapping to stage 0 of the next step: A is step-invariant)
                const bool more = (kt + 1 < NKT) || (t + 1 < T);
                if (more) {
                    hmm_load_stage<S>(As + (stage ^ 1) * HMM_KT * S, A, (kt + 1) % NKT);
                    cp_async_commit();
                    cp_async_wait<1>();
                } else {
                    cp_async_wait<0>();
                }
                __syncthreads();
                const float* At = As + stage * HMM_KT * S;
#pragma unroll
                for (int kk = 0; kk < HMM_KT; ++kk) {
                    const int k = kt * HMM_KT + kk;
                    const float4 a0 = *reinterpret_cast<const float4*>(aT + k * HMM_MS + sg * 8);
                    const float4 a1 = *reinterpret_cast<const float4*>(aT + k * HMM_MS + sg * 8 + 4);
                    const float4 b0 = *reinterpret_cast<const float4*>(At + kk * S + j0);
                    const float4 b1 = *reinterpret_cast<const float4*>(At + kk * S + j1);
                    const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
                    const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
                    for (int a = 0; a < 8; ++a)
#pragma unroll
                        for (int b = 0; b < 8; ++b) acc[a][b] = fmaf(av[a], bv[b], acc[a][b]);
                }
                __syncthreads();   // stage buffer and aT reads complete
            }
        }
        __syncthreads();   // s_sym visible; all aT reads of this step done
        // emission, per-signal row sums
        float rs[8];
#pragma unroll
        for (int a = 0; a < 8; ++a) {
            const float* e = E_lin + (int64_t)s_sym[sg * 8 + a] * S;
            const float4 e0 = __ldg(reinterpret_cast<const float4*>(e + j0));
            const float4 e1 = __ldg(reinterpret_cast<const float4*>(e + j1));
            const float ev[8] = {e0.x, e0.y, e0.z, e0.w, e1.x, e1.y, e1.z, e1.w};
            float r = 0.f;
#pragma unroll
            for (int b = 0; b < 8; ++b) { acc[a][b] *= ev[b]; r += acc[a][b]; }
            rs[a] = r;
        }
#pragma unroll
        for (int a = 0; a < 8; ++a)
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) rs[a] += __shfl_xor_sync(0xffffffffu, rs[a], off);
        if (lane == 0)
#pragma unroll
            for (int a = 0; a < 8; ++a) s_red[warp][a] = rs[a];
        __syncthreads();
        if (tid < HMM_MS) {
            const int g = tid / 8, a = tid % 8;
            float c = 0.f;
            for (int w = g * (GT / 32); w < (g + 1) * (GT / 32); ++w) c += s_red[w][a];
            s_inv[tid] = 1.0f / c;
            ll += log_scale((double)c);
        }
        __syncthreads();
        // ahat_t -> aT (transposed: 8 signals contiguous per state)
#pragma unroll
        for (int b = 0; b < 8; ++b) {
            const int j = (b < 4) ? (j0 + b) : (j1 + b - 4);
            float4 lo, hi;
            lo.x = acc[0][b] * s_inv[sg * 8 + 0]; lo.y = acc[1][b] * s_inv[sg * 8 + 1];
            lo.z = acc[2][b] * s_inv[sg * 8 + 2]; lo.w = acc[3][b] * s_inv[sg * 8 + 3];
            hi.x = acc[4][b] * s_inv[sg * 8 + 4]; hi.y = acc[5][b] * s_inv[sg * 8 + 5];
            hi.z = acc[6][b] * s_inv[sg * 8 + 6]; hi.w = acc[7][b] * s_inv[sg * 8 + 7];
            *reinterpret_cast<float4*>(aT + j * HMM_MS + sg * 8) = lo;
            *reinterpret_cast<float4*>(aT + j * HMM_MS + sg * 8 + 4) = hi;
        }
        __syncthreads();
    }
    if (tid < HMM_MS && s0 + tid < nsig) out_ll[sig(s0 + tid)] = ll;
}

// ------------------------------------------- tensor-core guard re-run
// The fp16 tensor-core kernel (hmm_quad.cu) leaves, per signal, a range flag
// (some step's predicted emission mass fell below 2^-8) and a count of
// concentration events (an entry of u' holding >= 1/64 of the mass: its 2^-11
// rounding error recurs instead of averaging out).  A signal is re-run in fp32
// when it hit the range flag, its result is not finite, or the events' worst-case
// error (2^-11 each) exceeds a quarter of the 1e-5 budget on |ll|.
__global__ void k_hmm_guard_select(const int* __restrict__ rflag, const int* __restrict__ events,
                                   const double* __restrict__ ll, int64_t nsig, int* __restrict__ list,
                                   int* __restrict__ count) {
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nsig; s += (int64_t)gridDim.x * blockDim.x) {
        const double v = ll[s];
        const bool bad = rflag[s] != 0 || !isfinite(v) || (double)events[s] * 0x1p-11 > 2.5e-6 * fabs(v);
        if (bad) list[atomicAdd(count, 1)] = (int)s;
    }
}

int* hmm_guard_words(void* ws, int S);

int hmm_guard_rerun(const float* A, const float* E_lin, const float* pi_lin, int S, const int* obs, int64_t nsig,
                    int T, double* out_ll, int* guard, cudaStream_t st) {
    int* count = guard;
    const int* rflag = guard + 4;
    const int* events = rflag + nsig;
    int* list = const_cast<int*>(events) + nsig;
    const unsigned gsel = (unsigned)((nsig + 255) / 256 < 148 ? (nsig + 255) / 256 : 148);
    k_hmm_guard_select<<<gsel, 256, 0, st>>>(rflag, events, out_ll, nsig, list, count);
    PMX_CHECK_LAUNCH("hmm_guard_select");
    if (S != 1024) { set_last_error("hmm guard re-run: S != 1024"); return -2; }
    const size_t smem = (size_t)(1024 * HMM_MS + 2 * HMM_KT * 1024) * sizeof(float);
    cudaFuncSetAttribute(k_hmm_fwd_tiled<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const unsigned grid = (unsigned)((nsig + HMM_MS - 1) / HMM_MS);
    k_hmm_fwd_tiled<1024><<<grid, 512, smem, st>>>(pi_lin, A, E_lin, obs, nsig, T, out_ll, list, count);
    PMX_CHECK_LAUNCH("hmm_guard_rerun");
    return 0;
}

// ------------------------------------------------------------ Viterbi
// One CTA per signal, fp64 like the reference; thread-strided states.
// back pointers in workspace [nsig][T-1][S] int32; thread 0 backtracks.
__global__ void k_viterbi(const double* __restrict__ log_pi, const double* __restrict__ log_A,
                          const double* __restrict__ log_E, int S, int K,
                          const int* __restrict__ obs, int64_t nsig, int T,
                          int* __restrict__ path, double* __restrict__ logp,
                          int* __restrict__ back) {
    extern __shared__ double dsm[];
    double* chi = dsm;        // [S]
    double* nxt = dsm + S;    // [S]
    const int64_t sig = blockIdx.x;
    if (sig >= nsig) return;
    const int* o = obs + sig * (int64_t)T;
    int* bk = back + sig * (int64_t)(T > 1 ? T - 1 : 0) * S;
    // chi0[i] = log(init i) + logEmit[i][obs 0]            (viterbi.pmx:147-149)
    for (int i = threadIdx.x; i < S; i += blockDim.x) chi[i] = __dadd_rn(log_pi[i], log_E[i * K + o[0]]);
    __syncthreads();
    for (int t = 1; t < T; ++t) {
        const int sym = o[t];
        for (int j = threadIdx.x; j < S; j += blockDim.x) {
            // scores i = chi i + logTrans i j ; argmax = first index of the max
            int best = 0;
            double bs = __dadd_rn(chi[0], log_A[j]);
            for (int i = 1; i < S; ++i) {
                const double sc = __dadd_rn(chi[i], log_A[(int64_t)i * S + j]);
                if (sc > bs) { bs = sc; best = i; }
            }
            nxt[j] = __dadd_rn(bs, log_E[j * K + sym]);
            bk[(int64_t)(t - 1) * S + j] = best;
        }
        __syncthreads();
        for (int j = threadIdx.x; j < S; j += blockDim.x) chi[j] = nxt[j];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        int best = 0;
        for (int i = 1; i < S; ++i) if (chi[i] > chi[best]) best = i;   // argmax chiFinal
        int* pth = path + sig * (int64_t)T;
        pth[T - 1] = best;
        int s = best;
        for (int t = T - 2; t >= 0; --t) { s = bk[(int64_t)t * S + s]; pth[t] = s; }   // walkBack
        logp[sig] = chi[best];
    }
}

bool viterbi_tiled_eligible(int S);
size_t viterbi_tiled_workspace(int S, int64_t nsig, int T);
int viterbi_tiled_launch(const double* log_pi, const double* log_A, const double* log_E, int S, int K,
                         const int* obs, int64_t nsig, int T, int* path, double* logp, void* ws,
                         cudaStream_t st);
unsigned long long* viterbi_visited_counter(void* ws, int S, int64_t nsig, int T);
size_t hmm_tc_workspace(int S, int K);
bool hmm_tc_eligible(int S, int K);
int* hmm_guard_words(void* ws, int S);
int hmm_tc_launch(const float* log_pi, const float* A, const float* log_E, int S, int K, const int* obs,
                  int64_t nsig, int T, double* out_ll, void* ws, cudaStream_t st);

}  // namespace pmx

using namespace pmx;

extern "C" {

size_t pmx_hmm_forward_workspace_bytes(int32_t S, int64_t nsig) {
    // E_lin [K<=64][S] + pi_lin [S], generous K bound; + the tensor-core path's A^T
    size_t simt = (size_t)S * 65 * sizeof(float) + 256;
    // + the guard's words (hmm_guard_words): a count and three ints per signal
    size_t tc = hmm_tc_workspace(S, 8) + 16 + 12 * (size_t)nsig;
    return simt > tc ? simt : tc;
}

int pmx_hmm_forward_f32(const float* log_pi, const float* A, const float* log_E, int32_t S, int32_t K,
                        const int32_t* obs, int64_t nsig, int32_t T, double* out_ll, void* ws,
                        size_t ws_bytes, void* stream) {
    PMX_REQUIRE(S > 0 && K > 0 && K <= 64 && T > 0 && nsig >= 0, "pmx_hmm_forward_f32: bad sizes");
    PMX_REQUIRE(ws && ws_bytes >= pmx_hmm_forward_workspace_bytes(S, nsig), "pmx_hmm_forward_f32: workspace too small");
    if (nsig == 0) return 0;
    cudaStream_t st = (cudaStream_t)stream;
    // tensor-core path (hmm_tc.cu) for the BASELINE state count; PMX_HMM_SIMT=1
    // forces the SIMT kernel (A/B comparisons)
    static const bool force_simt = getenv("PMX_HMM_SIMT") && getenv("PMX_HMM_SIMT")[0] == '1';
    if (!force_simt && hmm_tc_eligible(S, K))
        return hmm_tc_launch(log_pi, A, log_E, S, K, obs, nsig, T, out_ll, ws, st);
    float* E_lin = (float*)ws;
    float* pi_lin = E_lin + (size_t)S * 64;
    k_hmm_prep<<<(S * K + 255) / 256, 256, 0, st>>>(log_pi, log_E, S, K, E_lin, pi_lin);
    PMX_CHECK_LAUNCH("hmm_prep");
    const unsigned grid = (unsigned)((nsig + HMM_MS - 1) / HMM_MS);
#define PMX_HMM_TILED(SS)                                                                          \
    if (S == SS) {                                                                                 \
        const size_t smem = (size_t)(SS * HMM_MS + 2 * HMM_KT * SS) * sizeof(float);               \
        cudaFuncSetAttribute(k_hmm_fwd_tiled<SS>, cudaFuncAttributeMaxDynamicSharedMemorySize,     \
                             (int)smem);                                                           \
        k_hmm_fwd_tiled<SS><<<grid, SS / 2, smem, st>>>(pi_lin, A, E_lin, obs, nsig, T, out_ll);   \
        PMX_CHECK_LAUNCH("hmm_fwd_tiled");                                                         \
        return 0;                                                                                  \
    }
    PMX_HMM_TILED(1024)
    PMX_HMM_TILED(512)
    PMX_HMM_TILED(256)
#undef PMX_HMM_TILED
    PMX_REQUIRE(S <= 12288, "pmx_hmm_forward_f32: S too large for the one-CTA-per-signal kernel");
    int threads = S >= 1024 ? 1024 : ((S + 31) / 32) * 32;
    const size_t smem = 2 * (size_t)S * sizeof(float);
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(k_hmm_fwd_small, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_hmm_fwd_small<<<(unsigned)nsig, threads, smem, st>>>(pi_lin, A, E_lin, S, obs, nsig, T, out_ll);
    PMX_CHECK_LAUNCH("hmm_fwd_small");
    return 0;
}

int64_t pmx_hmm_forward_rerun_count(const void* ws, int32_t S, int64_t nsig, void* stream) {
    // signals of the last pmx_hmm_forward_f32 call on `ws` that the fp16 path's
    // guard re-ran in fp32 (0 when another path ran)
    PMX_REQUIRE(ws && nsig >= 0, "pmx_hmm_forward_rerun_count: bad arguments");
    if (!hmm_tc_eligible(S, 8) || nsig == 0) return 0;
    static const char* mode = getenv("PMX_HMM_TC");
    if (mode && strcmp(mode, "quad")) return 0;
    int n = 0;
    if (cudaMemcpyAsync(&n, hmm_guard_words(const_cast<void*>(ws), S), sizeof(int), cudaMemcpyDeviceToHost,
                        (cudaStream_t)stream) != cudaSuccess ||
        cudaStreamSynchronize((cudaStream_t)stream) != cudaSuccess)
        return -1;
    return n;
}

int64_t pmx_viterbi_visited_cells(const void* ws, int32_t S, int64_t nsig, int32_t T, void* stream) {
    // max-plus cells the last pmx_viterbi_f64 call on `ws` evaluated in the
    // pruned kernel (0 when another kernel ran); synchronises `stream`
    PMX_REQUIRE(ws && nsig >= 0, "pmx_viterbi_visited_cells: bad arguments");
    if (!viterbi_tiled_eligible(S) || nsig == 0) return 0;
    unsigned long long n = 0;
    if (cudaMemcpyAsync(&n, viterbi_visited_counter(const_cast<void*>(ws), S, nsig, T), sizeof(n),
                        cudaMemcpyDeviceToHost, (cudaStream_t)stream) != cudaSuccess ||
        cudaStreamSynchronize((cudaStream_t)stream) != cudaSuccess)
        return -1;
    return (int64_t)n;
}

size_t pmx_viterbi_workspace_bytes(int32_t S, int64_t nsig, int32_t T) {
    // simple kernel: back pointers [nsig][T-1][S] int32; tiled kernels (S in
    // {256, 512, 1024}): chi history / back pointers + final chi + log A^T
    const size_t simple = (size_t)nsig * (size_t)(T > 1 ? T - 1 : 0) * (size_t)S * sizeof(int32_t) + 256;
    const size_t tiled = viterbi_tiled_eligible(S) ? viterbi_tiled_workspace(S, nsig, T) : 0;
    return simple > tiled ? simple : tiled;
}

int pmx_viterbi_f64(const double* log_pi, const double* log_A, const double* log_E, int32_t S, int32_t K,
                    const int32_t* obs, int64_t nsig, int32_t T, int32_t* path, double* logp,
                    void* ws, size_t ws_bytes, void* stream) {
    PMX_REQUIRE(S > 0 && K > 0 && T > 0 && nsig >= 0, "pmx_viterbi_f64: bad sizes");
    PMX_REQUIRE(ws && ws_bytes >= pmx_viterbi_workspace_bytes(S, nsig, T), "pmx_viterbi_f64: workspace too small");
    if (nsig == 0) return 0;
    // S in {256, 512, 1024}: batched register-tiled kernel (viterbi.cu);
    // PMX_VITERBI_SIMPLE=1 forces the one-CTA-per-signal kernel (A/B checks)
    static const bool simple = getenv("PMX_VITERBI_SIMPLE") && getenv("PMX_VITERBI_SIMPLE")[0] == '1';
    if (!simple && viterbi_tiled_eligible(S))
        return viterbi_tiled_launch(log_pi, log_A, log_E, S, K, obs, nsig, T, path, logp, ws,
                                    (cudaStream_t)stream);
    const size_t smem = 2 * (size_t)S * sizeof(double);
    PMX_REQUIRE(smem <= 200 * 1024, "pmx_viterbi_f64: S too large");
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(k_viterbi, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int threads = S >= 256 ? 256 : ((S + 31) / 32) * 32;
    k_viterbi<<<(unsigned)nsig, threads, smem, (cudaStream_t)stream>>>(log_pi, log_A, log_E, S, K, obs, nsig,
                                                                       T, path, logp, (int*)ws);
    PMX_CHECK_LAUNCH("viterbi");
    return 0;
}

}  // extern "C"
