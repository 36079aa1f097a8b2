// HMM forward on the tensor cores (tcgen05 kind::f16 or kind::tf32, TMEM, TMA).
//
// Reference anchor: SURVEY Appendix A.1 hmm_forward.pmx — the log-space
// forward recursion batched over signals by `map` (see hmm.cu for the SIMT
// kernel and the linear-space reformulation).  Here the per-step contraction
//     a_t[j, s] = sum_i A[i, j] * u_{t-1}[i, s]          (all signals s of a CTA)
// runs as UMMA with the transposed transition matrix as the A operand
// (M = 128 states per block, K = states i) and the CTA's state vectors as the
// B operand (N = 32 signals), accumulating in TMEM.
//
// Scaling (no normalisation barrier inside a step): with c_t = sum_j u_t[j],
//     u_0 = pi * E(o_0),   u_t = (u_{t-1} A) * E(o_t) / c_{t-1},
//     ll = sum_{t=0}^{T-1} log c_t        (fp64)
// which equals log sum_j alpha_{T-1}[j] exactly in real arithmetic.
//
// Operand precision (ET): fp16 (default) or TF32 — both carry a 10-bit
// mantissa; fp16 halves the shared-memory bytes per multiply-add, which bounds
// this kernel, and doubles the tensor-core rate.  fp16's exponent range is
// handled by exact power-of-two scaling: the operands are A' = 2^10 A and
// u' = 2^10 u (row sums of A are 1, entries of u sum to c_t ~ 1, so both sit
// in fp16's normal range; entries below 2^-14 lose relative precision but not
// absolute, ~1e-8 against a row sum of 2^10), and the epilogue removes 2^20.
// Operands are rounded to nearest (RNE for fp16, RNA for TF32) — truncation
// would bias every row sum of A low and the bias compounds over T steps.
// Accumulation is fp32 in TMEM.  The error is checked against the fp64
// log-space oracle in tests (rel 1e-5 budget).
//
// CTA layout (384 threads): warp 0 TMA producer (A^T tiles of 128 states x
// 128 bytes of K, SW128, 4-stage ring multicast across a 4-CTA cluster,
// streamed from L2 every step — A is step-invariant, so the ring keeps
// prefetching into the next step), warp 1 MMA issuer, warp 2 TMEM allocator,
// warps 4-11 epilogue (TMEM lane = state within a 128-state block, two warps
// per lane quadrant, 16 signals each): scale by E(o_t)/c_{t-1}, round, write
// u_t back into the B-operand buffer in shared memory (in place: the step's
// MMAs are complete), per-signal row sums -> c_t, log c_t.
//
// Measured per step at the BASELINE config (tools/hmm_time.py, PMX_HMM_DBG):
// TMA stream alone 13.6 us, + UMMA 20.4 us, + epilogue 25.0 us (fp16); the
// UMMA phase is bound by shared-memory bandwidth — per step every SM writes
// (TMA) and reads (UMMA) the 2 MiB A^T and re-reads 512 KiB of B: 4.5 MiB at
// 128 B/clk = 18.8 us.
#include <cuda_fp16.h>
#include <stdlib.h>
#include "common.cuh"
#include "tc.cuh"

namespace pmx {

constexpr int HT_N = 32;            // signals per CTA (UMMA N)
constexpr int HT_M = 128;           // states per UMMA M block
constexpr int HT_THREADS = 384;    // 4 control warps + 8 epilogue warps
constexpr int HT_KMAX = 8;          // symbols staged in shared memory

__device__ __forceinline__ float tf32_rna(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

// Operand element: storage type, K elements per 128-byte swizzle row, UMMA
// format, and the power-of-two scalings (A' = A * kScaleA; the epilogue writes
// u' = D * e / c * kOut; c = sum(u') * kSum; t = 0 feeds pi * kInit as D).
template <class ET> struct HmmElem;
template <> struct HmmElem<float> {
    static constexpr int KB = 32, FMT = 2, KSTEP = 8;       // kind::tf32, K = 8 per UMMA
    static constexpr float kScaleA = 1.f, kOut = 1.f, kSum = 1.f, kInit = 1.f;
    __device__ static float round(float x) { return tf32_rna(x); }
    __device__ static float widen(float x) { return x; }
};
template <> struct HmmElem<__half> {
    static constexpr int KB = 64, FMT = 0, KSTEP = 16;      // kind::f16 (fp16 in), K = 16 per UMMA
    static constexpr float kScaleA = 1024.f, kOut = 1.f / 1024.f, kSum = 1.f / 1024.f, kInit = 1048576.f;
    __device__ static __half round(float x) { return __float2half_rn(x); }
    __device__ static float widen(__half x) { return __half2float(x); }
};

// Configuration: CL = CTAs of a cluster sharing each A^T tile by TMA
// multicast (each loads HT_M / CL rows), ST = pipeline stages, ESM = emissions
// staged in shared memory (else read through L1).
template <class ET, int S, int CL, int ST, bool ESM>
struct __align__(1024) HmmSmem {
    static constexpr int KB = HmmElem<ET>::KB;
    ET U[S / KB][HT_N * KB];                      // B operand: K-major SW128, [kblock][signal][KB]
    ET At[ST][HT_M * KB];                         // A operand tiles: [state j][KB i], SW128
    float E[ESM ? HT_KMAX : 1][ESM ? S : 1];      // linear emissions E[k][j]
    float wsum[4][HT_N];                          // per-warp row-sum partials
    float inv_c[HT_N];
    int sym[HT_N];
    uint64_t full[ST], empty[ST];
    uint64_t dfull, bready;
    uint32_t tmem_base;
};

// At[j][i] = round(A[i][j] * kScaleA); E_lin[k][j] = exp(log_E[j][k]); pi = exp(log_pi)
template <class ET>
__global__ void k_hmm_tc_prep(const float* __restrict__ A, const float* __restrict__ log_E,
                              const float* __restrict__ log_pi, int S, int K, ET* __restrict__ At,
                              float* __restrict__ E_lin, float* __restrict__ pi_lin) {
    __shared__ float tile[32][33];
    const int bi = blockIdx.y * 32, bj = blockIdx.x * 32;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) tile[r][threadIdx.x] = A[(int64_t)(bi + r) * S + bj + threadIdx.x];
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y)
        At[(int64_t)(bj + r) * S + bi + threadIdx.x] = HmmElem<ET>::round(tile[threadIdx.x][r] * HmmElem<ET>::kScaleA);
    if (blockIdx.y == 0) {
        for (int r = threadIdx.y; r < 32; r += blockDim.y) {
            const int j = bj + threadIdx.x;
            if (r < K) E_lin[(int64_t)r * S + j] = expf(log_E[(int64_t)j * K + r]);
            if (r == 0) pi_lin[j] = expf(log_pi[j]);
        }
    }
}

// byte offset of element (signal s, state i) in the SW128 K-major B buffer
template <class ET>
__device__ __forceinline__ uint32_t u_offset(int s, int i) {
    constexpr int KB = HmmElem<ET>::KB;
    const int kb = i / KB;
    const uint32_t byte = (uint32_t)(i % KB) * (uint32_t)sizeof(ET);
    const uint32_t chunk = (byte >> 4) ^ (uint32_t)(s & 7);
    return (uint32_t)kb * (HT_N * 128) + (uint32_t)s * 128 + (chunk << 4) + (byte & 15);
}

template <class ET, int S, int HT_CLUSTER, int HT_STAGES, bool ESM>
__global__ void __cluster_dims__(HT_CLUSTER, 1, 1) __launch_bounds__(HT_THREADS, 1)
k_hmm_fwd_tc(const __grid_constant__ CUtensorMap tmA, const float* __restrict__ E_lin,
             const float* __restrict__ pi_lin, int K, const int* __restrict__ obs, int64_t nsig, int T,
             double* __restrict__ out_ll, int dbg) {
    typedef HmmElem<ET> EL;
    constexpr int HT_KB = EL::KB;          // K elements per 128-byte row
    constexpr int NJB = S / HT_M;          // 128-state blocks (M)
    constexpr int NKB = S / HT_KB;         // K blocks
    constexpr uint32_t TILE_BYTES = HT_M * 128;
    constexpr int HT_ROWS = HT_M / HT_CLUSTER;   // tile rows loaded (and multicast) per CTA
    extern __shared__ uint8_t smem_raw[];
    typedef HmmSmem<ET, S, HT_CLUSTER, HT_STAGES, ESM> Smem;
    // 1 KiB-aligned by pointer arithmetic on the __shared__ array itself, so every
    // access through it stays in the shared space (STS/LDS, not generic ST/LD)
    Smem& Sm = *reinterpret_cast<Smem*>(
        smem_raw + ((1024u - ((uint32_t)__cvta_generic_to_shared(smem_raw) & 1023u)) & 1023u));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t s0 = (int64_t)blockIdx.x * HT_N;

    // ---- setup
    if (ESM)
        for (int v = threadIdx.x; v < K * S; v += blockDim.x) (&Sm.E[0][0])[v] = E_lin[v];
    if (threadIdx.x < HT_N) Sm.inv_c[threadIdx.x] = 1.f;
    if (threadIdx.x == 0) {
        // empty[s] completes when the MMAs of EVERY CTA of the cluster consumed
        // stage s (each CTA's multicast writes into all of them)
        for (int s = 0; s < HT_STAGES; ++s) { tc::mbar_init(&Sm.full[s], 1); tc::mbar_init(&Sm.empty[s], HT_CLUSTER); }
        tc::mbar_init(&Sm.dfull, 1);
        tc::mbar_init(&Sm.bready, 1);
        tc::fence_mbar_init();
        tc::tma_prefetch(&tmA);
    }
    if (warp == 2) tc::tmem_alloc(&Sm.tmem_base, 512);
    tc::tc_fence_before();
    tc::cluster_sync();                      // all barriers of the cluster initialised
    tc::tc_fence_after();
    const uint32_t rank = tc::cluster_ctarank();
    const uint32_t tmem = Sm.tmem_base;

    if (warp == 0) {
        if (lane == 0) {                                     // ---- TMA producer
            int stage = 0; uint32_t phase = 0;
            for (int t = 1; t < T; ++t)
                for (int kb = 0; kb < NKB; ++kb)
                    for (int jb = 0; jb < NJB; ++jb) {
                        tc::mbar_wait(&Sm.empty[stage], phase ^ 1);
                        tc::mbar_arrive_expect_tx(&Sm.full[stage], TILE_BYTES);
                        // this CTA's quarter of the tile, multicast to the whole cluster
                        tc::tma_load_2d_mc(Sm.At[stage] + rank * HT_ROWS * HT_KB, &tmA, &Sm.full[stage],
                                           kb * HT_KB, jb * HT_M + (int)rank * HT_ROWS,
                                           (uint16_t)((1u << HT_CLUSTER) - 1));
                        if (++stage == HT_STAGES) { stage = 0; phase ^= 1; }
                    }
        }
    } else if (warp == 1) {
        // ---- MMA issuer: the whole warp walks the pipeline (warp-uniform state
        // stays in uniform registers); one elected lane issues the UMMAs.
        constexpr uint32_t idesc = tc::instr_desc(HT_M, HT_N, EL::FMT);
        int stage = 0; uint32_t phase = 0, bpar = 0;
        const uint64_t u_desc = tc::sw128_kmajor_desc(tc::smem_u32(&Sm.U[0][0]));
        const uint64_t at_desc = tc::sw128_kmajor_desc(tc::smem_u32(Sm.At[0]));
        for (int t = 1; t < T; ++t) {
            tc::mbar_wait(&Sm.bready, bpar); bpar ^= 1;   // u_{t-1} written (and D drained)
            tc::tc_fence_after();
            for (int kb = 0; kb < NKB; ++kb)
                for (int jb = 0; jb < NJB; ++jb) {
                    tc::mbar_wait(&Sm.full[stage], phase);
                    tc::tc_fence_after();
                    if (tc::elect_one()) {
                        if (!(dbg & 2)) {
                        // descriptor start addresses are in 16-byte units
                        const uint64_t ad = at_desc + (uint64_t)(stage * (TILE_BYTES >> 4));
                        const uint64_t bd = u_desc + (uint64_t)(kb * ((HT_N * 128) >> 4));
                        // two accumulator sets (even / odd K blocks), summed in the
                        // epilogue: halves the chain of truncating tensor-core
                        // accumulations per output (a low bias that compounds over T)
                        const uint32_t d = tmem + (uint32_t)((kb & 1) * (NJB * HT_N) + jb * HT_N);
#pragma unroll
                        for (int kk = 0; kk < HT_KB / EL::KSTEP; ++kk) {   // 32 B of K per UMMA
                            if (EL::FMT == 2) tc::umma_tf32(d, ad + 2 * kk, bd + 2 * kk, idesc, (kb >= 2) || (kk != 0));
                            else tc::umma_f16(d, ad + 2 * kk, bd + 2 * kk, idesc, (kb >= 2) || (kk != 0));
                        }
                        }
                        tc::umma_commit_mc(&Sm.empty[stage], (uint16_t)((1u << HT_CLUSTER) - 1));
                    }
                    __syncwarp();
                    if (++stage == HT_STAGES) { stage = 0; phase ^= 1; }
                }
            if (tc::elect_one()) tc::umma_commit(&Sm.dfull);
            __syncwarp();
        }
    } else if (warp >= 4) {
        // ---- epilogue: 8 warps; warp w reads TMEM lane quadrant w % 4 (state
        // j = jb*128 + 32*(w%4) + lane) for signal half h = (w-4)/4 (16 signals)
        const int q = warp & 3;
        const int ew = warp - 4;
        const int h = ew >> 2;
        double ll = 0.0;                                       // lane s of warp 4 owns signal s
        uint32_t dpar = 0;
        const float* Ef = &Sm.E[0][0];
        for (int t = 0; t < T; ++t) {
            // stage this step's symbols
            if (ew == 0) {
                const int64_t sg = s0 + lane;
                Sm.sym[lane] = (sg < nsig) ? obs[sg * T + t] : 0;
            }
            asm volatile("bar.sync 1, 256;" ::: "memory");
            if (t > 0) {
                tc::mbar_wait(&Sm.dfull, dpar); dpar ^= 1;
                tc::tc_fence_after();
            }
            // per-signal constants of this step, in registers
            int eoff[16];
            float ic[16], csum[16];
#pragma unroll
            for (int s = 0; s < 16; ++s) {
                eoff[s] = Sm.sym[h * 16 + s] * S;
                ic[s] = Sm.inv_c[h * 16 + s] * EL::kOut;
                csum[s] = 0.f;
            }
#pragma unroll 1
            for (int jb = 0; jb < ((dbg & 1) ? 0 : NJB); ++jb) {
                const int j = jb * HT_M + q * 32 + lane;
                float d[16];
                if (t > 0) {
                    uint32_t r[16], r2[16];
                    const uint32_t col = (uint32_t)(jb * HT_N + h * 16);
                    tc::tmem_ld_32x32b_x16(tmem + ((uint32_t)(q * 32) << 16) + col, r);
                    tc::tmem_ld_32x32b_x16(tmem + ((uint32_t)(q * 32) << 16) + NJB * HT_N + col, r2);
                    tc::tmem_ld_wait();
#pragma unroll
                    for (int s = 0; s < 16; ++s) d[s] = __uint_as_float(r[s]) + __uint_as_float(r2[s]);
                } else {
                    const float p = pi_lin[j] * EL::kInit;
#pragma unroll
                    for (int s = 0; s < 16; ++s) d[s] = p;
                }
                // row address of state j in the SW128 K-major B buffer: fixed
                // part + per-signal (s * 128, chunk ^ (s & 7)) with s unrolled
                const uint32_t byte = (uint32_t)(j % HT_KB) * (uint32_t)sizeof(ET);
                const uint32_t chunkj = byte >> 4;
                uint8_t* rowp = reinterpret_cast<uint8_t*>(&Sm.U[0][0]) + (j / HT_KB) * (HT_N * 128) + (byte & 15);
#pragma unroll
                for (int s = 0; s < 16; ++s) {
                    const int sg = h * 16 + s;
                    const float u = d[s] * Ef[eoff[s] + j] * ic[s];
                    const ET ur = EL::round(u);
                    csum[s] += EL::widen(ur);
                    *reinterpret_cast<ET*>(rowp + sg * 128 + ((chunkj ^ (uint32_t)(sg & 7)) << 4)) = ur;
                }
            }
            // per-signal sums over the warp's 32 states: fold lane halves, then
            // transpose-reduce 16 values over 16 lanes (lane l < 16 ends with
            // signal h*16 + l in csum[0]; 16 + 15 shuffles)
#pragma unroll
            for (int s = 0; s < 16; ++s) csum[s] += __shfl_xor_sync(0xffffffffu, csum[s], 16);
#pragma unroll
            for (int w = 8; w > 0; w >>= 1) {
                const bool upper = (lane & w) != 0;
#pragma unroll
                for (int s = 0; s < w; ++s) {
                    const float send = upper ? csum[s] : csum[s + w];
                    const float keep = upper ? csum[s + w] : csum[s];
                    csum[s] = keep + __shfl_xor_sync(0xffffffffu, send, w);
                }
            }
            if (lane < 16) Sm.wsum[q][h * 16 + lane] = csum[0];
            tc::fence_proxy_async();                 // u_t visible to the UMMA async proxy
            tc::tc_fence_before();                   // TMEM reads ordered before the hand-off
            asm volatile("bar.sync 1, 256;" ::: "memory");
            if (ew == 0) {
                const float c = (Sm.wsum[0][lane] + Sm.wsum[1][lane] + Sm.wsum[2][lane] + Sm.wsum[3][lane]) * EL::kSum;
                Sm.inv_c[lane] = 1.f / c;
                ll += log_scale((double)c);
            }
            asm volatile("bar.sync 1, 256;" ::: "memory");
            if (threadIdx.x == 128 && t + 1 < T) {
                tc::tc_fence_before();
                tc::mbar_arrive(&Sm.bready);
            }
        }
        if (ew == 0 && s0 + lane < nsig) out_ll[s0 + lane] = ll;
    }
    tc::tc_fence_before();
    tc::cluster_sync();                      // no CTA leaves while peers may still multicast into it
    if (warp == 2) tc::tmem_dealloc(tmem, 512);
}

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
bool make_tmap_2d(CUtensorMap* m, const void* base, CUtensorMapDataType dt, int elem_bytes, uint64_t rows,
                  uint64_t cols, uint32_t box_rows, uint32_t box_cols, CUtensorMapSwizzle swz);

size_t hmm_tc_workspace(int S, int K) { return (size_t)S * S * 4 + (size_t)HT_KMAX * S * 4 + (size_t)S * 4 + 1024; }

// precision / range guard words after the tensor-core workspace (hmm_quad.cu):
// [0] number of flagged signals, [4 ...] range flags, event counts and the list
// of flagged signals (nsig each)
int* hmm_guard_words(void* ws, int S) { return (int*)((char*)ws + hmm_tc_workspace(S, HT_KMAX)); }

bool hmm_tc_eligible(int S, int K) { return S == 1024 && K <= HT_KMAX; }

// PMX_HMM_DBG (timing experiments only, results invalid): bit 0 skips the
// epilogue's per-state work, bit 1 skips the UMMA issue.
static int dbg_flags() {
    static const int v = getenv("PMX_HMM_DBG") ? atoi(getenv("PMX_HMM_DBG")) : 0;
    return v;
}

int hmm_quad_launch(const float* log_pi, const float* A, const float* log_E, int S, int K, const int* obs,
                    int64_t nsig, int T, double* out_ll, void* ws, cudaStream_t st);
int hmm_pair_launch(const float* log_pi, const float* A, const float* log_E, int S, int K, const int* obs,
                    int64_t nsig, int T, double* out_ll, void* ws, cudaStream_t st);

template <class ET, int CL, int ST>
static int hmm_tc_run(const float* log_pi, const float* A, const float* log_E, int S, int K, const int* obs,
                      int64_t nsig, int T, double* out_ll, void* ws, cudaStream_t st) {
    ET* At = (ET*)ws;
    float* E_lin = (float*)((char*)ws + (size_t)S * S * 4);
    float* pi_lin = E_lin + (size_t)HT_KMAX * S;
    k_hmm_tc_prep<ET><<<dim3(S / 32, S / 32), dim3(32, 8), 0, st>>>(A, log_E, log_pi, S, K, At, E_lin, pi_lin);
    PMX_CHECK_LAUNCH("hmm_tc_prep");
    CUtensorMap tmA;
    const bool half = sizeof(ET) == 2;
    if (!make_tmap_2d(&tmA, At, half ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                      (int)sizeof(ET), (uint64_t)S, (uint64_t)S, HT_M / CL, HmmElem<ET>::KB,
                      CU_TENSOR_MAP_SWIZZLE_128B)) {
        set_last_error("hmm: cuTensorMapEncodeTiled failed");
        return -2;
    }
    unsigned grid = (unsigned)((nsig + HT_N - 1) / HT_N);
    grid = (grid + CL - 1) / CL * CL;        // whole clusters (padding CTAs run on masked signals)
    const size_t smem = sizeof(HmmSmem<ET, 1024, CL, ST, true>) + 1024;
    cudaFuncSetAttribute(k_hmm_fwd_tc<ET, 1024, CL, ST, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_hmm_fwd_tc<ET, 1024, CL, ST, true><<<grid, HT_THREADS, smem, st>>>(tmA, E_lin, pi_lin, K, obs, nsig, T, out_ll,
                                                                        dbg_flags());
    PMX_CHECK_LAUNCH("hmm_fwd_tc");
    return 0;
}


int hmm_tc_launch(const float* log_pi, const float* A, const float* log_E, int S, int K, const int* obs,
                  int64_t nsig, int T, double* out_ll, void* ws, cudaStream_t st) {
    // Operands: fp16 (default) or TF32 (PMX_HMM_TC=tf32, for comparison).
    // TF32 configuration measured at the BASELINE config (4096 x 10^4 x 1024):
    //   cluster 4 / 4 stages / E in smem  487 ms   (chosen: also cuts L2 reads 4x)
    //   cluster 1 / 4 stages / E in smem  487 ms
    //   cluster 1 or 4 / 6 stages / E via L1  653 ms
    // The step is bound by shared-memory traffic: every SM streams the whole
    // A^T through smem once per step (TMA write + UMMA read) for only 32
    // signals — fp16 operands halve those bytes.
    // Default: the 4-CTA pair-UMMA kernel (hmm_quad.cu, 10.4 us/step at the BASELINE
    // config); PMX_HMM_TC=pair: CTA pairs with single-SM UMMAs (hmm_pair.cu, 13.2).
    static const char* mode = getenv("PMX_HMM_TC");
    if (!mode || !strcmp(mode, "quad"))
        return hmm_quad_launch(log_pi, A, log_E, S, K, obs, nsig, T, out_ll, ws, st);
    if (!strcmp(mode, "pair"))
        return hmm_pair_launch(log_pi, A, log_E, S, K, obs, nsig, T, out_ll, ws, st);
    if (mode && !strcmp(mode, "tf32"))
        return hmm_tc_run<float, 4, 4>(log_pi, A, log_E, S, K, obs, nsig, T, out_ll, ws, st);
    if (mode && !strcmp(mode, "f16s6"))
        return hmm_tc_run<__half, 4, 6>(log_pi, A, log_E, S, K, obs, nsig, T, out_ll, ws, st);
    if (mode && !strcmp(mode, "f16s8"))
        return hmm_tc_run<__half, 4, 8>(log_pi, A, log_E, S, K, obs, nsig, T, out_ll, ws, st);
    if (mode && !strcmp(mode, "f16c1"))
        return hmm_tc_run<__half, 1, 4>(log_pi, A, log_E, S, K, obs, nsig, T, out_ll, ws, st);
    return hmm_tc_run<__half, 4, 4>(log_pi, A, log_E, S, K, obs, nsig, T, out_ll, ws, st);
}

}  // namespace pmx
