// HMM forward on the tensor cores, 4-CTA variant with CTA-pair UMMA
// (tcgen05 cta_group::2).  Same recursion, scaling and fp16 operands as
// hmm_tc.cu / hmm_pair.cu (see hmm_tc.cu for the reference anchor and the
// precision argument).
//
// Why: at M = 128, N = 64 (hmm_pair.cu) a UMMA needs 6 KiB of shared-memory
// operands per 32 clocks — more than the 128 B/clk an SM's shared memory
// delivers (tools/umma_rate.cu: N = 64 issues at 1.46 PFLOP/s, N = 128 at
// 2.2) — and every SM also streams 1 MiB of A^T per step.  A pair UMMA
// (M = 256, N = 128) takes its A rows from both SMs of a pair and splits the
// N = 128 signal columns of u between them (64 each: the 128 KiB B buffer of
// hmm_pair.cu), so each SM reads 6 KiB per 64 clocks; two pairs in a cluster
// split the states, so each SM streams 256 rows (512 KiB) of A^T per step.
//
// Layout (cluster of 4, 128 signals): CTA c = 2p + h.  Pair p owns output
// states [512p, 512p + 512) as two M blocks of 256 rows; in M block mb, CTA h
// holds rows 512p + 256mb + 128h + [0, 128) of A^T (its TMEM lanes) and B
// columns (signals) 64h + [0, 64) for all 1024 states (K).  D (fp32, TMEM):
// lanes = this CTA's 128 states of the M block, columns = the 128 signals.
//
// Per step t (u_{t-1} complete in all four B buffers):
//   producers (both CTAs of a pair): A^T tiles by TMA (cta_group::2: the
//                bytes complete on the pair leader's `full`)
//   MMA (leader): 2 M blocks x 16 K blocks x 4 UMMA (K = 16), commit to both
//                CTAs' `empty`, finally to both CTAs' `dfull`
//   epilogue (16 warps per CTA: TMEM lane quadrant x signal quarter):
//     a. wait dfull(t) (D of step t complete)
//     b. per M block: u_t = D * E(o_t) * 1/c_{t-1} -> fp16, once both pairs'
//        MMAs consumed my rows of u_{t-1} (`gdone[mb]`, multicast commits of the
//        two leaders): my signal half into my own B (then one bulk copy to the
//        other pair's CTA of my half), the other half straight to the two CTAs
//        holding it by 4-byte st.async; all complete on their `ur[me][mb]`
//     c. per-signal partial sums -> all four CTAs (st.async, `psum`); c_{t} =
//        the four partials added in CTA order (identical everywhere), folded at
//        the next step (nobody waits for the slowest CTA)
//   the leader's MMAs of t+1 consume u_t group by group as `ur` / `pr` (the
//   partner's arrivals, forwarded) complete; D is double-buffered in TMEM.
#include <cuda_fp16.h>
#include <stdio.h>
#include <stdlib.h>
#include "common.cuh"
#include "tc.cuh"

namespace pmx {

constexpr int HQ_N = 128;            // signals per cluster (UMMA N)
constexpr int HQ_NH = 64;            // signals in one CTA's B buffer
constexpr int HQ_M = 128;            // A^T rows per CTA per UMMA (M = 256 per pair)
constexpr int HQ_KB = 64;            // fp16 per 128-byte swizzle row
constexpr int HQ_S = 1024;
constexpr int HQ_NKB = HQ_S / HQ_KB;   // 16 K blocks
constexpr int HQ_MB = 2;             // M blocks (256 states) per pair
constexpr int HQ_ST = 5;             // TMA ring stages (the MMAs are latency-bound on A^T tiles)
constexpr int HQ_KMAX = 8;
constexpr int HQ_EW = 16;            // epilogue warps (4 TMEM lane quadrants x 4 signal quarters)
constexpr int HQ_THREADS = 128 + 32 * HQ_EW;
constexpr uint32_t HQ_TILE = HQ_M * 128;                 // 16 KiB of A^T per CTA per stage
constexpr uint32_t HQ_ROWS = 2 * HQ_NH * 128;            // 16 KiB: 2 K blocks x 64 signals (128 states)

struct __align__(1024) HqSmem {
    __half U[HQ_NKB][HQ_NH * HQ_KB];     // B operand: K-major SW128 [kblock][signal][64]
    __half At[HQ_ST][HQ_M * HQ_KB];      // A operand tiles
    float Es[HQ_KMAX][HQ_MB * HQ_M];     // emission probabilities of my 256 states
    float wsum[4][HQ_N];                 // per TMEM lane quadrant partial sums
    float psum_in[2][4][HQ_N];           // [step parity][source CTA][signal]
    float inv_c[HQ_N];
    int sym[HQ_N];
    float escl[HQ_KMAX];                 // exact power-of-two emission scale per symbol
    int eex[HQ_KMAX];                    // its exponent (escl = 2^eex)
    uint64_t full[HQ_ST], empty[HQ_ST];
    uint64_t ur[4][2];                   // rows of u_t from CTA c's M block mb in my B (local or copied)
    uint64_t pr[4][2];                   // (pair leader) the same group landed in the partner's B
    uint64_t gdone[HQ_MB];               // both pairs' MMAs consumed my rows of M block mb (u_{t-1})
    uint64_t dfull, psum[2];
    uint32_t tmem_base;
};

__device__ __forceinline__ void hq_bulk_to(uint32_t remote_dst, const void* src, uint32_t bytes, uint32_t remote_bar) {
    asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(remote_dst), "r"(tc::smem_u32(src)), "r"(bytes), "r"(remote_bar) : "memory");
}
__device__ __forceinline__ void hq_bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void hq_bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }

__global__ void __cluster_dims__(4, 1, 1) __launch_bounds__(HQ_THREADS, 1)
k_hmm_fwd_quad(const __grid_constant__ CUtensorMap tmA, const float* __restrict__ E_lin,
               const float* __restrict__ pi_lin, int K, const int* __restrict__ obs, int64_t nsig, int T,
               double* __restrict__ out_ll, int* __restrict__ rflag, int* __restrict__ events,
               unsigned long long* __restrict__ trace) {
    constexpr float kOut = 1.f / 1024.f, kSum = 1.f / 1024.f, kInit = 1048576.f;
    extern __shared__ uint8_t smem_raw[];
    // 1 KiB-aligned by pointer arithmetic on the __shared__ array itself, so every
    // access through it stays in the shared space (STS/LDS, not generic ST/LD)
    HqSmem& Sm = *reinterpret_cast<HqSmem*>(
        smem_raw + ((1024u - ((uint32_t)__cvta_generic_to_shared(smem_raw) & 1023u)) & 1023u));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t crank = tc::cluster_ctarank();
    const uint32_t p = crank >> 1, h = crank & 1u;
    const uint32_t leader = crank & ~1u;                       // this pair's MMA issuer
    const uint16_t pair_mask = (uint16_t)(3u << (2 * p));
    const int64_t s0 = (int64_t)(blockIdx.x >> 2) * HQ_N;
    // PMX_HMM_QUAD_TRACE: %globaltimer stamps of cluster 0, CTA 0, steps < 64 (timeline debugging)
    auto stamp = [&](int t, int k) {
        if (trace && blockIdx.x < 4 && t < 64) {
            unsigned long long g;
            asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g));
            trace[blockIdx.x * 1024 + t * 16 + k] = g;
        }
    };
    auto jbase = [&](int mb) { return (int)(512 * p + 256 * mb + 128 * h); };   // my first state of M block mb
    // K blocks of u_t produced by CTA c's M block mb (its 128 states)
    auto kbgrp = [](uint32_t c, int mb) { return (int)(8 * (c >> 1) + 4 * mb + 2 * (c & 1)); };
    // The MMAs of a step consume K in the order the rows of u_{t-1} become ready:
    // source M block 0 of the four CTAs (own pair first), then M block 1.

    if (threadIdx.x < HQ_N) Sm.inv_c[threadIdx.x] = 1.f;
    // Range guard, part 1: every symbol's emission column is scaled by an exact
    // power of two so that its largest entry lies in [1, 2) (log-likelihoods get
    // the exponent back).  A symbol that is rare in every state then no longer
    // drives u_t into fp16's subnormal range.
    if (warp < HQ_KMAX) {
        float m = 0.f;
        if (warp < K)
            for (int j = lane; j < HQ_S; j += 32) m = fmaxf(m, E_lin[warp * HQ_S + j]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (lane == 0) {
            // m = 1.f x 2^(E - 127): x = 127 - E puts m * 2^x in [1, 2)
            const int E = (int)((__float_as_uint(m) >> 23) & 0xffu);
            const int x = (m > 0.f && E < 255) ? min(max(127 - E, -126), 126) : 0;
            Sm.eex[warp] = x;
            Sm.escl[warp] = __uint_as_float((uint32_t)(x + 127) << 23);
        }
    }
    __syncthreads();
    for (int v = threadIdx.x; v < HQ_KMAX * HQ_MB * HQ_M; v += blockDim.x) {
        const int k = v / (HQ_MB * HQ_M), jl = v % (HQ_MB * HQ_M);
        Sm.Es[k][jl] = k < K ? E_lin[k * HQ_S + jbase(jl / HQ_M) + jl % HQ_M] * Sm.escl[k] : 0.f;
    }
    if (threadIdx.x == 0) {
        for (int s = 0; s < HQ_ST; ++s) { tc::mbar_init(&Sm.full[s], 1); tc::mbar_init(&Sm.empty[s], 1); }
        tc::mbar_init(&Sm.dfull, 1);
        for (int c = 0; c < 4; ++c)
            for (int b = 0; b < HQ_MB; ++b) { tc::mbar_init(&Sm.ur[c][b], 1); tc::mbar_init(&Sm.pr[c][b], 1); }
        for (int b = 0; b < HQ_MB; ++b) tc::mbar_init(&Sm.gdone[b], 2);
        tc::mbar_init(&Sm.psum[0], 1);
        tc::mbar_init(&Sm.psum[1], 1);
        // Arm the first phases of the barriers that receive remote bytes: every later
        // phase is armed by the thread that consumed the previous one, which happens
        // before any CTA can send the next phase's bytes (a transaction never lands
        // on an unarmed phase)
        if (T > 1)
            for (int c = 0; c < 4; ++c)
                if (c != (int)crank)
                    for (int b = 0; b < HQ_MB; ++b) tc::mbar_arrive_expect_tx(&Sm.ur[c][b], HQ_ROWS);
        tc::mbar_arrive_expect_tx(&Sm.psum[0], 3 * HQ_N * 4);
        if (T > 1) tc::mbar_arrive_expect_tx(&Sm.psum[1], 3 * HQ_N * 4);
        tc::fence_mbar_init();
        tc::tma_prefetch(&tmA);
    }
    if (warp == 2) tc::tmem_alloc2(&Sm.tmem_base, 512);   // D double-buffered by step parity
    tc::tc_fence_before();
    tc::cluster_sync();
    tc::tc_fence_after();
    const uint32_t tmem = Sm.tmem_base;

    if (warp == 0) {
        if (lane == 0) {                                     // ---- TMA producer (both CTAs of a pair)
            const uint32_t lead_full0 = tc::mapa(tc::smem_u32(&Sm.full[0]), leader);
            int stage = 0; uint32_t phase = 0;
            for (int t = 1; t < T; ++t)
                for (int mbs = 0; mbs < HQ_MB; ++mbs)
                    for (int i = 0; i < 4; ++i)
                        for (int k2 = 0; k2 < 2; ++k2)
                            for (int mbo = 0; mbo < HQ_MB; ++mbo) {
                                const int kb = kbgrp(leader ^ (uint32_t)i, mbs) + k2;
                                tc::mbar_wait(&Sm.empty[stage], phase ^ 1);
                                if (h == 0) tc::mbar_arrive_expect_tx(&Sm.full[stage], 2 * HQ_TILE);
                                tc::tma_load_2d_pair(Sm.At[stage], &tmA, lead_full0 + (uint32_t)(stage * sizeof(uint64_t)),
                                             kb * HQ_KB, jbase(mbo));
                                if (++stage == HQ_ST) { stage = 0; phase ^= 1; }
                            }
        }
    } else if (warp == 1) {
        if (h == 0) {                                        // ---- MMA issuer (pair leader)
            constexpr uint32_t idesc = tc::instr_desc(2 * HQ_M, HQ_N, 0);
            int stage = 0; uint32_t phase = 0;
            const uint64_t u_desc = tc::sw128_kmajor_desc(tc::smem_u32(&Sm.U[0][0]));
            const uint64_t at_desc = tc::sw128_kmajor_desc(tc::smem_u32(Sm.At[0]));
            for (int t = 1; t < T; ++t) {
                const uint32_t dstep = tmem + (uint32_t)((t & 1) * (HQ_MB * HQ_N));
                bool first[HQ_MB] = {true, true};
                for (int mbs = 0; mbs < HQ_MB; ++mbs)
                    for (int i = 0; i < 4; ++i) {
                        const uint32_t c = leader ^ (uint32_t)i;
                        tc::mbar_wait(&Sm.ur[c][mbs], (uint32_t)((t - 1) & 1));      // in my B
                        if (c != crank && t + 1 < T && lane == 0)                      // arm u_t's phase
                            tc::mbar_arrive_expect_tx(&Sm.ur[c][mbs], HQ_ROWS);
                        __syncwarp();
                        tc::mbar_wait_cluster(&Sm.pr[c][mbs], (uint32_t)((t - 1) & 1));    // and the partner's
                        tc::tc_fence_after();
                        if (t < 64 && mbs == 0 && i == 0 && lane == 0) stamp(t, 8);
                        for (int k2 = 0; k2 < 2; ++k2)
                            for (int mbo = 0; mbo < HQ_MB; ++mbo) {
                                const int kb = kbgrp(c, mbs) + k2;
                                tc::mbar_wait(&Sm.full[stage], phase);
                                tc::tc_fence_after();
                                if (tc::elect_one()) {
                                    const uint64_t ad = at_desc + (uint64_t)(stage * (HQ_TILE >> 4));
                                    const uint64_t bd = u_desc + (uint64_t)(kb * ((HQ_NH * 128) >> 4));
                                    const uint32_t d = dstep + (uint32_t)(mbo * HQ_N);
#pragma unroll
                                    for (int kk = 0; kk < HQ_KB / 16; ++kk)
                                        tc::umma2_f16(d, ad + 2 * kk, bd + 2 * kk, idesc, (!first[mbo]) || (kk != 0));
                                    tc::umma2_commit_mc(&Sm.empty[stage], pair_mask);
                                }
                                __syncwarp();
                                first[mbo] = false;
                                if (++stage == HQ_ST) { stage = 0; phase ^= 1; }
                            }
                        // CTA c may overwrite these rows (in every B) once both pairs consumed them
                        if (tc::elect_one()) tc::umma2_commit_mc(&Sm.gdone[mbs], (uint16_t)(1u << c));
                        __syncwarp();
                    }
                if (lane == 0) stamp(t, 10);
                if (tc::elect_one()) tc::umma2_commit_mc(&Sm.dfull, pair_mask);
                __syncwarp();
            }
        } else if (lane == 0) {                              // partner: forward "my B is ready"
            for (int t = 1; t < T; ++t)
                for (int mbs = 0; mbs < HQ_MB; ++mbs)
                    for (int i = 0; i < 4; ++i) {
                        const uint32_t c = leader ^ (uint32_t)i;
                        tc::mbar_wait(&Sm.ur[c][mbs], (uint32_t)((t - 1) & 1));
                        if (c != crank && t + 1 < T) tc::mbar_arrive_expect_tx(&Sm.ur[c][mbs], HQ_ROWS);
                        tc::arrive_remote(tc::mapa(tc::smem_u32(&Sm.pr[c][mbs]), leader));
                    }
        }
    } else if (warp >= 4) {
        // ---- epilogue: warp w reads TMEM lane quadrant q (states jbase(mb) + 32q + lane)
        // and the signal half hh (signals 64 hh .. 64 hh + 63, in two chunks of 32)
        const int q = warp & 3;
        const int ew = warp - 4;
        const int hq = ew >> 2;                          // signal quarter: signals 32 hq .. 32 hq + 31
        const int hh = hq >> 1;                          // ... in signal half hh
        const bool lead = threadIdx.x == 128;
        double ll = 0.0, cprod = 1.0;
        int esum = 0;                                    // sum of the emission-scale exponents
        bool out_of_range = false;
        uint32_t dpar = 0;
        // c_t of step tt (partials of all four CTAs, added in CTA order): 1/c_t for the
        // next epilogue, log c_t into ll.  Done one step late, after the next dfull, so
        // no CTA waits for the slowest one's partials.
        auto finish_c = [&](int tt) {
            if (ew < 4) {
                tc::mbar_wait_cluster(&Sm.psum[tt & 1], (uint32_t)((tt >> 1) & 1));
                if (lead && tt + 2 < T) tc::mbar_arrive_expect_tx(&Sm.psum[tt & 1], 3 * HQ_N * 4);
                const int m = ew * 32 + lane;
                const float c = ((Sm.psum_in[tt & 1][0][m] + Sm.psum_in[tt & 1][1][m]) +
                                 (Sm.psum_in[tt & 1][2][m] + Sm.psum_in[tt & 1][3][m])) * kSum;
                Sm.inv_c[m] = 1.f / c;
                // Range guard, part 2: c_t is the predicted emission mass (scaled as
                // above).  Below 2^-8 the fp16 rounding of u_t (subnormal entries, and
                // the subnormal entries of 2^10 A) could cost more than the 1e-5
                // budget; such a signal is re-run by the fp32 kernel.
                if (!(c >= 0.00390625f)) out_of_range = true;
                cprod *= (double)c;                          // one fp64 log per 16 steps
                if ((tt & 15) == 15 || tt == T - 1) { ll += log_scale(cprod); cprod = 1.0; }
            }
            asm volatile("bar.sync 1, %0;" :: "n"(32 * HQ_EW) : "memory");
        };
        const uint32_t same_half_other_pair = crank ^ 2u, other_half_same_pair = crank ^ 1u,
                       other_half_other_pair = crank ^ 3u;
        const uint32_t rU_osp = tc::mapa(tc::smem_u32(&Sm.U[0][0]), other_half_same_pair);
        const uint32_t rU_oop = tc::mapa(tc::smem_u32(&Sm.U[0][0]), other_half_other_pair);
        uint32_t rB_osp[HQ_MB], rB_oop[HQ_MB];
#pragma unroll
        for (int b = 0; b < HQ_MB; ++b) {
            rB_osp[b] = tc::mapa(tc::smem_u32(&Sm.ur[crank][b]), other_half_same_pair);
            rB_oop[b] = tc::mapa(tc::smem_u32(&Sm.ur[crank][b]), other_half_other_pair);
        }
        for (int t = 0; t < T; ++t) {
            if (ew < 4) {
                const int m = ew * 32 + lane;
                const int64_t sg = s0 + m;
                const int o = (sg < nsig) ? obs[sg * T + t] : 0;
                Sm.sym[m] = o;
                esum += Sm.eex[(unsigned)o < (unsigned)HQ_KMAX ? o : 0];
            }
            for (int v = ew * 32 + lane; v < 4 * HQ_N; v += 32 * HQ_EW) (&Sm.wsum[0][0])[v] = 0.f;
            if (lead) stamp(t, 0);
            if (t > 0) {
                tc::mbar_wait(&Sm.dfull, dpar); dpar ^= 1;
                tc::tc_fence_after();
                if (lead) stamp(t, 1);
                finish_c(t - 1);
            } else {
                asm volatile("bar.sync 1, %0;" :: "n"(32 * HQ_EW) : "memory");
            }
#pragma unroll 1
            for (int mb = 0; mb < HQ_MB; ++mb) {
                const int j = jbase(mb) + q * 32 + lane;
                const int kb0 = jbase(mb) / HQ_KB;           // first of my two K blocks
                const uint32_t byte = (uint32_t)(j % HQ_KB) * 2u;
                const uint32_t chunkj = byte >> 4;
                uint8_t* dst = reinterpret_cast<uint8_t*>(&Sm.U[0][0]) + (j / HQ_KB) * (HQ_NH * 128) + (byte & 15);
                // the other signal half goes straight to the two CTAs holding it: 4-byte
                // st.async of a state pair (j & ~1, j | 1), complete_tx on their ur[me][mb]
                const uint32_t pair_off = (uint32_t)(j / HQ_KB) * (HQ_NH * 128) + ((byte & ~3u) & 15u);
                // (1) u_t of this M block into registers (32 signals, packed fp16)
                __half2 uh[16];
#pragma unroll
                for (int ch = 0; ch < 2; ++ch) {             // 16 signals at a time
                    const int sb = hq * 32 + ch * 16;        // first signal (of the cluster's 128)
                    float ev[16], ic[16];
#pragma unroll
                    for (int s = 0; s < 16; ++s) {
                        ev[s] = Sm.Es[Sm.sym[sb + s]][mb * HQ_M + q * 32 + lane];
                        ic[s] = Sm.inv_c[sb + s] * kOut;
                    }
                    float d[16];
                    if (t > 0) {
                        uint32_t r[16];
                        tc::tmem_ld_32x32b_x16(tmem + ((uint32_t)(q * 32) << 16) +
                                               (uint32_t)((t & 1) * (HQ_MB * HQ_N) + mb * HQ_N + sb), r);
                        tc::tmem_ld_wait();
#pragma unroll
                        for (int s = 0; s < 16; ++s) d[s] = __uint_as_float(r[s]);
                    } else {
                        const float pv = pi_lin[j] * kInit;
#pragma unroll
                        for (int s = 0; s < 16; ++s) d[s] = pv;
                    }
                    float v[16];
#pragma unroll
                    for (int s = 0; s < 16; ++s) v[s] = d[s] * ev[s] * ic[s];
                    // Precision guard: an entry >= 32 of u' (which sums to 2^10 c_t <= 2^11)
                    // means >= 1/64 of the predicted mass sits in one state.  Rounding
                    // errors of such entries (2^-11 relative) do not average out over the
                    // states and recur step after step; these events are counted per
                    // signal and weighed against the log-likelihood after the kernel.
                    float vmax = v[0];
#pragma unroll
                    for (int s = 1; s < 16; ++s) vmax = fmaxf(vmax, v[s]);
                    if (__any_sync(0xffffffffu, vmax >= 32.f)) {
#pragma unroll
                        for (int s = 0; s < 16; ++s)
                            if (v[s] >= 32.f && s0 + sb + s < nsig) atomicAdd(&events[s0 + sb + s], 1);
                    }
#pragma unroll
                    for (int s = 0; s < 16; s += 2) uh[ch * 8 + s / 2] = __floats2half2_rn(v[s], v[s + 1]);
                }
                if (lead) stamp(t, 4 * mb);
                // (2) store, once both pairs' MMAs of t consumed my rows of u_{t-1} (gdone):
                // my signal half into my B, the other half into the other-half CTAs' B
                if (t > 0) tc::mbar_wait_cluster(&Sm.gdone[mb], (uint32_t)((t - 1) & 1));
                if (hh == (int)h) {
#pragma unroll
                    for (int s = 0; s < 32; ++s) {
                        const int sl = (hq & 1) * 32 + s;    // B column (signal within the half)
                        const __half v = (s & 1) ? __high2half(uh[s / 2]) : __low2half(uh[s / 2]);
                        *reinterpret_cast<__half*>(dst + sl * 128 + ((chunkj ^ (uint32_t)(sl & 7)) << 4)) = v;
                    }
                } else if (t + 1 < T) {
                    const bool odd = (lane & 1) != 0;
#pragma unroll
                    for (int k = 0; k < 16; ++k) {
                        const __half2 mine = uh[k];              // signals 2k, 2k+1 at state j
                        const __half2 other = __shfl_xor_sync(0xffffffffu, mine, 1);   // at state j ^ 1
                        // even lane: signal 2k (states j, j+1); odd lane: signal 2k+1 (j-1, j)
                        const __half2 pr = odd ? __halves2half2(__high2half(other), __high2half(mine))
                                               : __halves2half2(__low2half(mine), __low2half(other));
                        const int sl = (hq & 1) * 32 + 2 * k + (odd ? 1 : 0);
                        const uint32_t off = pair_off + (uint32_t)sl * 128 + ((chunkj ^ (uint32_t)(sl & 7)) << 4);
                        const float bits = __uint_as_float(*reinterpret_cast<const uint32_t*>(&pr));
                        tc::st_async_b32(rU_osp + off, __float_as_uint(bits), rB_osp[mb]);
                        tc::st_async_b32(rU_oop + off, __float_as_uint(bits), rB_oop[mb]);
                    }
                }
                tc::tc_fence_before();
                tc::fence_proxy_async();                     // u_t rows visible to the async proxy
                asm volatile("bar.sync 1, %0;" :: "n"(32 * HQ_EW) : "memory");
                if (lead && t + 1 < T) {
                    tc::mbar_arrive(&Sm.ur[crank][mb]);      // my own rows are in my B
                    const uint32_t off = (uint32_t)kb0 * (HQ_NH * 128);
                    const uint8_t* mine = reinterpret_cast<const uint8_t*>(&Sm.U[0][0]) + off;
                    const uint32_t u0 = tc::smem_u32(&Sm.U[0][0]) + off;
                    const uint32_t urb = tc::smem_u32(&Sm.ur[crank][mb]);
                    hq_bulk_to(tc::mapa(u0, same_half_other_pair), mine, HQ_ROWS, tc::mapa(urb, same_half_other_pair));
                    hq_bulk_commit();
                }
                if (lead) stamp(t, 3 + 2 * mb);
                // (3) per-signal sums of the stored (fp16-rounded) values over the warp's 32
                // states — after the stores, off the path to the next step's first UMMAs
                // (the sums are folded one step late): fold the lane halves, then
                // transpose-reduce 16 values over 16 lanes (lane l < 16 ends with signal
                // sb + l)
#pragma unroll
                for (int ch = 0; ch < 2; ++ch) {
                    const int sb = hq * 32 + ch * 16;
                    float csum[16];
#pragma unroll
                    for (int s = 0; s < 16; s += 2) {
                        const float2 f2 = __half22float2(uh[ch * 8 + s / 2]);
                        csum[s] = f2.x;
                        csum[s + 1] = f2.y;
                    }
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
                    if (lane < 16) Sm.wsum[q][sb + lane] += csum[0];   // M block 0, then 1 (same warp)
                }
            }
            if (lead && t + 1 < T) hq_bulk_wait_read();      // my rows free for the next step
            asm volatile("bar.sync 1, %0;" :: "n"(32 * HQ_EW) : "memory");   // every warp's sums in wsum
            // my partial of every signal -> all four CTAs (own slot written locally)
            float part = 0.f;
            if (ew < 4) {
                const int m = ew * 32 + lane;
                part = (Sm.wsum[0][m] + Sm.wsum[1][m]) + (Sm.wsum[2][m] + Sm.wsum[3][m]);
                Sm.psum_in[t & 1][crank][m] = part;
#pragma unroll
                for (int c = 0; c < 4; ++c)
                    if (c != (int)crank)
                        tc::st_async_b32(tc::mapa(tc::smem_u32(&Sm.psum_in[t & 1][crank][m]), (uint32_t)c), __float_as_uint(part),
                                    tc::mapa(tc::smem_u32(&Sm.psum[t & 1]), (uint32_t)c));
            }
            asm volatile("bar.sync 1, %0;" :: "n"(32 * HQ_EW) : "memory");
            if (lead) stamp(t, 11);
        }
        finish_c(T - 1);
        if (crank == 0 && ew < 4 && s0 + ew * 32 + lane < nsig) {
            const int64_t sg = s0 + ew * 32 + lane;
            out_ll[sg] = ll - (double)esum * 0.69314718055994530942;
            rflag[sg] = out_of_range ? 1 : 0;
        }
    }
    tc::tc_fence_before();
    tc::cluster_sync();                      // no CTA leaves while a peer may still write into it
    if (warp == 2) tc::tmem_dealloc2(tmem, 512);
}

bool make_tmap_2d(CUtensorMap* m, const void* base, CUtensorMapDataType dt, int elem_bytes, uint64_t rows,
                  uint64_t cols, uint32_t box_rows, uint32_t box_cols, CUtensorMapSwizzle swz);
template <class ET>
__global__ void k_hmm_tc_prep(const float* __restrict__ A, const float* __restrict__ log_E,
                              const float* __restrict__ log_pi, int S, int K, ET* __restrict__ At,
                              float* __restrict__ E_lin, float* __restrict__ pi_lin);
int* hmm_guard_words(void* ws, int S);
int hmm_guard_rerun(const float* A, const float* E_lin, const float* pi_lin, int S, const int* obs, int64_t nsig,
                    int T, double* out_ll, int* guard, cudaStream_t st);

int hmm_quad_launch(const float* log_pi, const float* A, const float* log_E, int S, int K, const int* obs,
                    int64_t nsig, int T, double* out_ll, void* ws, cudaStream_t st) {
    __half* At = (__half*)ws;
    float* E_lin = (float*)((char*)ws + (size_t)S * S * 4);
    float* pi_lin = E_lin + (size_t)HQ_KMAX * S;
    int* guard = hmm_guard_words(ws, S);       // [count, pad] [range flag x nsig] [events x nsig] [list x nsig]
    int* rflag = guard + 4;
    int* events = rflag + nsig;
    cudaMemsetAsync(guard, 0, sizeof(int) * (4 + 2 * (size_t)nsig), st);
    k_hmm_tc_prep<__half><<<dim3(S / 32, S / 32), dim3(32, 8), 0, st>>>(A, log_E, log_pi, S, K, At, E_lin, pi_lin);
    PMX_CHECK_LAUNCH("hmm_quad_prep");
    CUtensorMap tmA;
    if (!make_tmap_2d(&tmA, At, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, (uint64_t)S, (uint64_t)S, HQ_M, HQ_KB,
                      CU_TENSOR_MAP_SWIZZLE_128B)) {
        set_last_error("hmm_quad: cuTensorMapEncodeTiled failed");
        return -2;
    }
    const unsigned grid = (unsigned)(4 * ((nsig + HQ_N - 1) / HQ_N));
    const size_t smem = sizeof(HqSmem) + 1024;
    cudaFuncSetAttribute(k_hmm_fwd_quad, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    static unsigned long long* trace = nullptr;
    static const bool want_trace = getenv("PMX_HMM_QUAD_TRACE") != nullptr;
    if (want_trace && !trace) cudaMalloc(&trace, 4 * 64 * 16 * sizeof(unsigned long long));
    k_hmm_fwd_quad<<<grid, HQ_THREADS, smem, st>>>(tmA, E_lin, pi_lin, K, obs, nsig, T, out_ll, rflag, events,
                                                   trace);
    if (want_trace) {
        static unsigned long long h[4 * 64 * 16];
        cudaStreamSynchronize(st);
        cudaMemcpy(h, trace, sizeof(h), cudaMemcpyDeviceToHost);
        for (int c = 0; c < 4; ++c)
            for (int t = 8; t < 11; ++t) {
                fprintf(stderr, "cta%d t=%2d", c, t);
                for (int k = 0; k < 12; ++k) fprintf(stderr, " %6lld", (long long)(h[c * 1024 + t * 16 + k] - h[t * 16]));
                fprintf(stderr, "\n");
            }
    }
    PMX_CHECK_LAUNCH("hmm_fwd_quad");
    // signals the guard flags are recomputed by the fp32 SIMT kernel, selected on
    // the device (the re-run's CTAs return at once when no signal was flagged)
    return hmm_guard_rerun(A, E_lin, pi_lin, S, obs, nsig, T, out_ll, guard, st);
}

}  // namespace pmx
