// HMM forward on the tensor cores, CTA-pair variant: the two CTAs of a
// cluster share 64 signals and split the OUTPUT STATES (CTA r owns states
// [512 r, 512 r + 512)).  Same recursion, scaling and fp16 operands as
// hmm_tc.cu (see there for the reference anchor and the precision argument).
//
// Why: the single-CTA kernel is bound by shared-memory bytes — every SM
// streams the whole 2 MiB A^T through smem each step (TMA write + UMMA read)
// for its 32 signals.  Here each SM streams only the A^T rows of its own 512
// output states (1 MiB) for 64 signals, so A bytes per signal-step halve; the
// u operand (64 signals x 1024 states, 128 KiB fp16) is held by both CTAs.
//
// Per step t (u_{t-1} complete in both CTAs' B buffers):
//   MMA warp   : 4 M-blocks x 16 K-blocks of UMMA M=128 (states) N=64
//                (signals) K=64, A^T tiles through a 3-stage TMA ring, two
//                accumulator sets (even/odd K blocks), commit -> dfull.
//   epilogue   : (8 warps: TMEM lane quadrant x signal half)
//     a. wait dfull(t); arrive on the PEER's peer_done (my MMAs of t are done);
//        wait my peer_done (the peer's MMAs of t are done: it no longer reads
//        u_{t-1} in my region of its buffer, and my copy of u_{t-1} landed)
//     b. u_t for my 512 states -> my region of my own B buffer (in place),
//        per-signal partial sums of u_t
//     c. partial sums -> the peer (st.async, completes tx on its psum barrier)
//     d. bulk copy of my region (64 KiB) into the peer's B buffer (completes
//        tx on the peer's uready); arrive.expect_tx on my uready for the
//        peer's copy into mine
//     e. wait psum: c_t = own + peer partials, 1/c_t, ll += log c_t
//   MMA(t+1) waits my uready (my epilogue's arrival + the peer's copy).
#include <cuda_fp16.h>
#include <stdlib.h>
#include "common.cuh"
#include "tc.cuh"

namespace pmx {

constexpr int HP_N = 64;             // signals per pair (UMMA N)
constexpr int HP_M = 128;            // states per UMMA M block
constexpr int HP_KB = 64;            // fp16 per 128-byte swizzle row
constexpr int HP_S = 1024;
constexpr int HP_HALF = HP_S / 2;    // output states per CTA
constexpr int HP_MB = HP_HALF / HP_M;   // 4 M blocks per CTA
constexpr int HP_NKB = HP_S / HP_KB;    // 16 K blocks
constexpr int HP_ST = 5;             // TMA ring stages (the emission table is read through L1,
                                     // leaving shared memory to the ring: 80 KiB of A^T in flight)
constexpr int HP_KMAX = 8;
constexpr int HP_EW = 8;             // epilogue warps (16 measured: 13.8 vs 13.4 us/step) (4 TMEM lane quadrants x HP_EW/4 signal groups)
constexpr int HP_SPW = HP_N / (HP_EW / 4);   // signals per epilogue warp
constexpr int HP_THREADS = 128 + 32 * HP_EW; // 4 control warps + the epilogue warps
constexpr uint32_t HP_TILE = HP_M * 128;                 // 16 KiB A^T tile
constexpr uint32_t HP_REGION = (HP_NKB / 2) * HP_N * 128;  // 64 KiB: one CTA's K blocks of u
constexpr uint32_t HP_CHUNK = 2 * HP_N * 128;              // 16 KiB: the two K blocks of one M block

struct __align__(1024) HpSmem {
    __half U[HP_NKB][HP_N * HP_KB];      // B operand: K-major SW128 [kblock][signal][64]
    __half At[HP_ST][HP_M * HP_KB];      // A operand tiles
    float wsum[4][HP_N];
    float psum_in[2][HP_N];              // the peer's partial sums (by step parity)
    float inv_c[HP_N];
    int sym[HP_N];
    uint64_t full[HP_ST], empty[HP_ST];
    uint64_t dfull, uready, peer_done, psum;
    uint64_t ublk[HP_MB];                // OVL: my u_t rows of M block mb written
    uint64_t upeer[HP_MB];               // OVL: the peer's M block mb of u_t landed (bulk copy tx)
    uint32_t tmem_base;
};

__device__ __forceinline__ uint32_t mapa_peer(uint32_t smem_addr, uint32_t peer) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_addr), "r"(peer));
    return r;
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t remote_bar) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" :: "r"(remote_bar) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}"
        :: "r"(tc::smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void st_async_f32(uint32_t remote_addr, float v, uint32_t remote_bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];"
                 :: "r"(remote_addr), "r"(__float_as_uint(v)), "r"(remote_bar) : "memory");
}
__device__ __forceinline__ void bulk_copy_to_peer(uint32_t remote_dst, const void* src, uint32_t bytes,
                                                  uint32_t remote_bar) {
    asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(remote_dst), "r"(tc::smem_u32(src)), "r"(bytes), "r"(remote_bar) : "memory");
}

__device__ __forceinline__ void tmem_ld_spw(uint32_t taddr, uint32_t (&r)[32]) { tc::tmem_ld_32x32b_x32(taddr, r); }
__device__ __forceinline__ void tmem_ld_spw(uint32_t taddr, uint32_t (&r)[16]) { tc::tmem_ld_32x32b_x16(taddr, r); }

__device__ __forceinline__ uint32_t hp_u_offset(int s, int i) {
    const int kb = i / HP_KB;
    const uint32_t byte = (uint32_t)(i % HP_KB) * 2u;
    const uint32_t chunk = (byte >> 4) ^ (uint32_t)(s & 7);
    return (uint32_t)kb * (HP_N * 128) + (uint32_t)s * 128 + (chunk << 4) + (byte & 15);
}

// OVL: the UMMAs of step t+1 overlap the epilogue of step t.  D is double
// buffered in TMEM by step parity (one accumulator set each).  As the
// epilogue finishes M block mb it releases those rows of u_t to its own UMMAs
// (ublk[mb]) and bulk-copies them (16 KiB) to the peer (upeer[mb] there); the
// K blocks of a step run per M block: mine, then the peer's.
// CL = 4: two pairs per cluster (different signals); the CTAs holding the same
// half of the states in both pairs need the same A^T tiles, so each loads half
// of every tile (64 rows) and multicasts it to both: A^T is read from L2 once
// per two pairs (the pair kernel is L2 -> SM bound: ncu xbar2l1 ~10.5 TB/s).
template <bool OVL, int CL>
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(HP_THREADS, 1)
k_hmm_fwd_pair(const __grid_constant__ CUtensorMap tmA, const float* __restrict__ E_lin,
               const float* __restrict__ pi_lin, int K, const int* __restrict__ obs, int64_t nsig, int T,
               double* __restrict__ out_ll) {
    constexpr float kOut = 1.f / 1024.f, kSum = 1.f / 1024.f, kInit = 1048576.f;
    extern __shared__ uint8_t smem_raw[];
    // 1 KiB-aligned by pointer arithmetic on the __shared__ array itself, so every
    // access through it stays in the shared space (STS/LDS, not generic ST/LD)
    HpSmem& Sm = *reinterpret_cast<HpSmem*>(
        smem_raw + ((1024u - ((uint32_t)__cvta_generic_to_shared(smem_raw) & 1023u)) & 1023u));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t crank = tc::cluster_ctarank();
    const uint32_t peer = crank ^ 1u;                // the other half of my pair
    const uint32_t rank = crank & 1u;                // my half of the states
    const uint32_t pidx = crank >> 1;                // my pair within the cluster (CL = 4)
    const uint16_t mc_mask = (uint16_t)((1u << rank) | (1u << (rank + 2)));   // same half, both pairs
    const int64_t s0 = (int64_t)(blockIdx.x >> 1) * HP_N;
    const int j0 = (int)rank * HP_HALF;              // first output state of this CTA

    if (threadIdx.x < HP_N) Sm.inv_c[threadIdx.x] = 1.f;
    if (threadIdx.x == 0) {
        // CL = 4: a stage is free when the MMAs of both CTAs sharing its tiles consumed it
        for (int s = 0; s < HP_ST; ++s) { tc::mbar_init(&Sm.full[s], 1); tc::mbar_init(&Sm.empty[s], CL == 4 ? 2 : 1); }
        tc::mbar_init(&Sm.dfull, 1);
        // uready: two arrivals (armed with the peer copy's bytes; own u written) + the copy's tx
        tc::mbar_init(&Sm.uready, OVL ? 1 : 2);
        for (int b = 0; b < HP_MB; ++b) { tc::mbar_init(&Sm.ublk[b], 1); tc::mbar_init(&Sm.upeer[b], 1); }
        tc::mbar_init(&Sm.peer_done, 1);
        tc::mbar_init(&Sm.psum, 1);
        tc::fence_mbar_init();
        tc::tma_prefetch(&tmA);
        // arm step 0 before any peer can deliver (the cluster barrier below orders it)
        tc::mbar_arrive_expect_tx(&Sm.psum, HP_N * 4);
        if (T > 1 && !OVL) tc::mbar_arrive_expect_tx(&Sm.uready, HP_REGION);
        if (T > 1 && OVL)
            for (int b = 0; b < HP_MB; ++b) tc::mbar_arrive_expect_tx(&Sm.upeer[b], HP_CHUNK);
    }
    if (warp == 2) tc::tmem_alloc(&Sm.tmem_base, 512);
    tc::tc_fence_before();
    tc::cluster_sync();
    tc::tc_fence_after();
    const uint32_t tmem = Sm.tmem_base;

    if (warp == 0) {
        if (lane == 0) {                                     // ---- TMA producer
            int stage = 0; uint32_t phase = 0;
            for (int t = 1; t < T; ++t)
                for (int ki = 0; ki < HP_NKB; ++ki)
                    for (int mb = 0; mb < HP_MB; ++mb) {
                        // K block order: mine first (OVL), then the peer's
                        // OVL K block order: per M block g of the producing epilogue, my
                        // two K blocks then the peer's two
                        const int kb = OVL ? (int)((ki & 3) < 2 ? rank : (rank ^ 1u)) * 8 + 2 * (ki >> 2) + (ki & 1) : ki;
                        tc::mbar_wait(&Sm.empty[stage], phase ^ 1);
                        tc::mbar_arrive_expect_tx(&Sm.full[stage], HP_TILE);
                        if (CL == 4)                 // my 64 rows of the tile, to both CTAs of my half
                            tc::tma_load_2d_mc(Sm.At[stage] + pidx * (HP_M / 2) * HP_KB, &tmA, &Sm.full[stage],
                                               kb * HP_KB, j0 + mb * HP_M + (int)pidx * (HP_M / 2), mc_mask);
                        else
                            tc::tma_load_2d(Sm.At[stage], &tmA, &Sm.full[stage], kb * HP_KB, j0 + mb * HP_M);
                        if (++stage == HP_ST) { stage = 0; phase ^= 1; }
                    }
        }
    } else if (warp == 1) {                                  // ---- MMA issuer
        constexpr uint32_t idesc = tc::instr_desc(HP_M, HP_N, 0);
        int stage = 0; uint32_t phase = 0, upar = 0;
        const uint64_t u_desc = tc::sw128_kmajor_desc(tc::smem_u32(&Sm.U[0][0]));
        const uint64_t at_desc = tc::sw128_kmajor_desc(tc::smem_u32(Sm.At[0]));
        for (int t = 1; t < T; ++t) {
            if (!OVL) {
                tc::mbar_wait(&Sm.uready, upar); upar ^= 1;  // u_{t-1} complete (own half + peer's copy)
                tc::tc_fence_after();
            }
            const uint32_t dbase = OVL ? tmem + (uint32_t)((t & 1) * (HP_MB * HP_N)) : tmem;
            for (int ki = 0; ki < HP_NKB; ++ki) {
                int kb = ki;
                if (OVL) {
                    const int g = ki >> 2, w = ki & 3;
                    kb = (int)(w < 2 ? rank : (rank ^ 1u)) * 8 + 2 * g + (w & 1);
                    if (w == 0) {                                 // my M block g of u_{t-1} written
                        tc::mbar_wait(&Sm.ublk[g], (uint32_t)((t - 1) & 1));
                        tc::tc_fence_after();
                    } else if (w == 2) {                          // the peer's M block g landed
                        tc::mbar_wait(&Sm.upeer[g], (uint32_t)((t - 1) & 1));
                        tc::tc_fence_after();
                    }
                }
                for (int mb = 0; mb < HP_MB; ++mb) {
                    tc::mbar_wait(&Sm.full[stage], phase);
                    tc::tc_fence_after();
                    if (tc::elect_one()) {
                        const uint64_t ad = at_desc + (uint64_t)(stage * (HP_TILE >> 4));
                        const uint64_t bd = u_desc + (uint64_t)(kb * ((HP_N * 128) >> 4));
                        if (OVL) {
                            const uint32_t d = dbase + (uint32_t)(mb * HP_N);
#pragma unroll
                            for (int kk = 0; kk < HP_KB / 16; ++kk)
                                tc::umma_f16(d, ad + 2 * kk, bd + 2 * kk, idesc, (ki > 0) || (kk != 0));
                        } else {
                            const uint32_t d = tmem + (uint32_t)((kb & 1) * (HP_MB * HP_N) + mb * HP_N);
#pragma unroll
                            for (int kk = 0; kk < HP_KB / 16; ++kk)
                                tc::umma_f16(d, ad + 2 * kk, bd + 2 * kk, idesc, (kb >= 2) || (kk != 0));
                        }
                        if (CL == 4) tc::umma_commit_mc(&Sm.empty[stage], mc_mask);
                        else tc::umma_commit(&Sm.empty[stage]);
                    }
                    __syncwarp();
                    if (++stage == HP_ST) { stage = 0; phase ^= 1; }
                }
            }
            if (tc::elect_one()) tc::umma_commit(&Sm.dfull);
            __syncwarp();
        }
    } else if (warp >= 4) {
        // ---- epilogue: warp w reads TMEM lane quadrant q = w % 4 (state
        // j0 + mb*128 + 32q + lane), signals h*32 .. h*32+31 (h = (w-4)/4)
        const int q = warp & 3;
        const int ew = warp - 4;
        const int h = ew >> 2;
        const bool lead = threadIdx.x == 128;
        double ll = 0.0;                                     // thread ew*32+lane < 64 owns signal
        uint32_t dpar = 0, ppar = 0, spar = 0;
        const float* __restrict__ Ef = E_lin;
        const uint32_t peer_uready = mapa_peer(tc::smem_u32(&Sm.uready), peer);
        const uint32_t peer_done_bar = mapa_peer(tc::smem_u32(&Sm.peer_done), peer);
        const uint32_t peer_psum_bar = mapa_peer(tc::smem_u32(&Sm.psum), peer);
        const uint32_t region_off = rank * HP_REGION;       // my K blocks of u
        const uint32_t peer_region = mapa_peer(tc::smem_u32(&Sm.U[0][0]) + region_off, peer);
        for (int t = 0; t < T; ++t) {
            if (ew < 2) {
                const int m = ew * 32 + lane;
                const int64_t sg = s0 + m;
                Sm.sym[m] = (sg < nsig) ? obs[sg * T + t] : 0;
            }
            asm volatile("bar.sync 1, %0;" :: "n"(32 * HP_EW) : "memory");
            if (t > 0) {
                tc::mbar_wait(&Sm.dfull, dpar); dpar ^= 1;
                tc::tc_fence_after();
                if (lead) {
                    // uready / upeer of step t-1 completed before my MMAs of t ran: arm
                    // step t for the peer's copies, then let the peer overwrite my
                    // region of its buffer
                    if (t + 1 < T) {
                        if (OVL)
                            for (int b = 0; b < HP_MB; ++b) tc::mbar_arrive_expect_tx(&Sm.upeer[b], HP_CHUNK);
                        else
                            tc::mbar_arrive_expect_tx(&Sm.uready, HP_REGION);
                    }
                    mbar_arrive_remote(peer_done_bar);
                }
                mbar_wait_cluster(&Sm.peer_done, ppar); ppar ^= 1;
            }
            float ic[HP_SPW], csum[HP_SPW];
            int eoff[HP_SPW];
#pragma unroll
            for (int s = 0; s < HP_SPW; ++s) {
                eoff[s] = Sm.sym[h * HP_SPW + s] * HP_S;
                ic[s] = Sm.inv_c[h * HP_SPW + s] * kOut;
                csum[s] = 0.f;
            }
#pragma unroll 1
            for (int mb = 0; mb < HP_MB; ++mb) {
                const int j = j0 + mb * HP_M + q * 32 + lane;
                float d[HP_SPW];
                if (t > 0 && OVL) {
                    uint32_t r[HP_SPW];
                    const uint32_t col = (uint32_t)((t & 1) * (HP_MB * HP_N) + mb * HP_N + h * HP_SPW);
                    tmem_ld_spw(tmem + ((uint32_t)(q * 32) << 16) + col, r);
                    tc::tmem_ld_wait();
#pragma unroll
                    for (int s = 0; s < HP_SPW; ++s) d[s] = __uint_as_float(r[s]);
                } else if (t > 0) {
                    uint32_t r[HP_SPW], r2[HP_SPW];
                    const uint32_t col = (uint32_t)(mb * HP_N + h * HP_SPW);
                    tmem_ld_spw(tmem + ((uint32_t)(q * 32) << 16) + col, r);
                    tmem_ld_spw(tmem + ((uint32_t)(q * 32) << 16) + HP_MB * HP_N + col, r2);
                    tc::tmem_ld_wait();
#pragma unroll
                    for (int s = 0; s < HP_SPW; ++s) d[s] = __uint_as_float(r[s]) + __uint_as_float(r2[s]);
                } else {
                    const float p = pi_lin[j] * kInit;
#pragma unroll
                    for (int s = 0; s < HP_SPW; ++s) d[s] = p;
                }
                const uint32_t byte = (uint32_t)(j % HP_KB) * 2u;
                const uint32_t chunkj = byte >> 4;
                uint8_t* rowp = reinterpret_cast<uint8_t*>(&Sm.U[0][0]) + (j / HP_KB) * (HP_N * 128) + (byte & 15);
#pragma unroll
                for (int s = 0; s < HP_SPW; ++s) {
                    const int sg = h * HP_SPW + s;
                    const __half ur = __float2half_rn(d[s] * __ldg(Ef + eoff[s] + j) * ic[s]);
                    csum[s] += __half2float(ur);
                    *reinterpret_cast<__half*>(rowp + sg * 128 + ((chunkj ^ (uint32_t)(sg & 7)) << 4)) = ur;
                }
                if (OVL && t + 1 < T) {                      // release M block mb of u_t to my MMA
                    tc::fence_proxy_async();
                    tc::tc_fence_before();
                    asm volatile("bar.sync 1, %0;" :: "n"(32 * HP_EW) : "memory");
                    if (lead) {
                        tc::mbar_arrive(&Sm.ublk[mb]);
                        // this M block's two K blocks of u_t -> the peer (16 KiB)
                        const uint32_t off = (uint32_t)(rank * 8 + 2 * mb) * (HP_N * 128);
                        bulk_copy_to_peer(mapa_peer(tc::smem_u32(&Sm.U[0][0]) + off, peer),
                                          reinterpret_cast<const uint8_t*>(&Sm.U[0][0]) + off, HP_CHUNK,
                                          mapa_peer(tc::smem_u32(&Sm.upeer[mb]), peer));
                    }
                }
            }
            // per-signal sums over the warp's 32 states: fold the lane halves while
            // there are fewer signals than lanes, then transpose-reduce HP_SPW
            // values over HP_SPW lanes (lane l < HP_SPW ends with signal h*HP_SPW + l)
#pragma unroll
            for (int w = 16; w >= HP_SPW; w >>= 1)
#pragma unroll
                for (int s = 0; s < HP_SPW; ++s) csum[s] += __shfl_xor_sync(0xffffffffu, csum[s], w);
#pragma unroll
            for (int w = HP_SPW / 2; w > 0; w >>= 1) {
                const bool upper = (lane & w) != 0;
#pragma unroll
                for (int s = 0; s < w; ++s) {
                    const float send = upper ? csum[s] : csum[s + w];
                    const float keep = upper ? csum[s + w] : csum[s];
                    csum[s] = keep + __shfl_xor_sync(0xffffffffu, send, w);
                }
            }
            if (lane < HP_SPW) Sm.wsum[q][h * HP_SPW + lane] = csum[0];
            tc::fence_proxy_async();                 // u_t visible to the async proxy (UMMA, bulk copy)
            tc::tc_fence_before();
            asm volatile("bar.sync 1, %0;" :: "n"(32 * HP_EW) : "memory");
            float part = 0.f;
            if (ew < 2) {                            // this CTA's partial of signal m
                const int m = ew * 32 + lane;
                part = (Sm.wsum[0][m] + Sm.wsum[1][m]) + (Sm.wsum[2][m] + Sm.wsum[3][m]);
                st_async_f32(mapa_peer(tc::smem_u32(&Sm.psum_in[t & 1][m]), peer), part, peer_psum_bar);
            }
            if (!OVL && lead && t + 1 < T) {
                tc::mbar_arrive(&Sm.uready);                                // my own u_t is written
                bulk_copy_to_peer(peer_region, reinterpret_cast<const uint8_t*>(&Sm.U[0][0]) + region_off,
                                  HP_REGION, peer_uready);
            }
            if (ew < 2) {
                mbar_wait_cluster(&Sm.psum, spar);
                const int m = ew * 32 + lane;
                // own + peer, added in rank order so both CTAs get the same c_t
                const float c = (rank == 0 ? part + Sm.psum_in[t & 1][m] : Sm.psum_in[t & 1][m] + part) * kSum;
                Sm.inv_c[m] = 1.f / c;
                ll += log_scale((double)c);
            }
            spar ^= 1;
            asm volatile("bar.sync 1, %0;" :: "n"(32 * HP_EW) : "memory");
            // arm the next step's partial-sum exchange (the peer can only send it
            // after my next peer_done arrival)
            if (lead && t + 1 < T) tc::mbar_arrive_expect_tx(&Sm.psum, HP_N * 4);
        }
        if (rank == 0 && ew < 2 && s0 + ew * 32 + lane < nsig) out_ll[s0 + ew * 32 + lane] = ll;
    }
    tc::tc_fence_before();
    tc::cluster_sync();                      // no CTA leaves while a peer may still write into it
    if (warp == 2) tc::tmem_dealloc(tmem, 512);
}

bool make_tmap_2d(CUtensorMap* m, const void* base, CUtensorMapDataType dt, int elem_bytes, uint64_t rows,
                  uint64_t cols, uint32_t box_rows, uint32_t box_cols, CUtensorMapSwizzle swz);
template <class ET>
__global__ void k_hmm_tc_prep(const float* __restrict__ A, const float* __restrict__ log_E,
                              const float* __restrict__ log_pi, int S, int K, ET* __restrict__ At,
                              float* __restrict__ E_lin, float* __restrict__ pi_lin);

int hmm_pair_launch(const float* log_pi, const float* A, const float* log_E, int S, int K, const int* obs,
                    int64_t nsig, int T, double* out_ll, void* ws, cudaStream_t st) {
    __half* At = (__half*)ws;
    float* E_lin = (float*)((char*)ws + (size_t)S * S * 4);
    float* pi_lin = E_lin + (size_t)HP_KMAX * S;
    k_hmm_tc_prep<__half><<<dim3(S / 32, S / 32), dim3(32, 8), 0, st>>>(A, log_E, log_pi, S, K, At, E_lin, pi_lin);
    PMX_CHECK_LAUNCH("hmm_pair_prep");
    CUtensorMap tmA;
    static const bool mc_map = !(getenv("PMX_HMM_PAIR_MC") && getenv("PMX_HMM_PAIR_MC")[0] == '0') &&
                               !(getenv("PMX_HMM_PAIR_SERIAL") && getenv("PMX_HMM_PAIR_SERIAL")[0] == '1');
    if (!make_tmap_2d(&tmA, At, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, (uint64_t)S, (uint64_t)S,
                      mc_map ? HP_M / 2 : HP_M, HP_KB, CU_TENSOR_MAP_SWIZZLE_128B)) {
        set_last_error("hmm_pair: cuTensorMapEncodeTiled failed");
        return -2;
    }
    const size_t smem = sizeof(HpSmem) + 1024;
    static const bool serial = getenv("PMX_HMM_PAIR_SERIAL") && getenv("PMX_HMM_PAIR_SERIAL")[0] == '1';
    static const bool mc = !(getenv("PMX_HMM_PAIR_MC") && getenv("PMX_HMM_PAIR_MC")[0] == '0');
    const int64_t pairs = (nsig + HP_N - 1) / HP_N;
    if (serial) {
        const unsigned grid = (unsigned)(2 * pairs);
        cudaFuncSetAttribute(k_hmm_fwd_pair<false, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_hmm_fwd_pair<false, 2><<<grid, HP_THREADS, smem, st>>>(tmA, E_lin, pi_lin, K, obs, nsig, T, out_ll);
    } else if (!mc) {
        const unsigned grid = (unsigned)(2 * pairs);
        cudaFuncSetAttribute(k_hmm_fwd_pair<true, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_hmm_fwd_pair<true, 2><<<grid, HP_THREADS, smem, st>>>(tmA, E_lin, pi_lin, K, obs, nsig, T, out_ll);
    } else {
        // whole clusters of two pairs (a padding pair runs on masked signals)
        const unsigned grid = (unsigned)(4 * ((pairs + 1) / 2));
        cudaFuncSetAttribute(k_hmm_fwd_pair<true, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_hmm_fwd_pair<true, 4><<<grid, HP_THREADS, smem, st>>>(tmA, E_lin, pi_lin, K, obs, nsig, T, out_ll);
    }
    PMX_CHECK_LAUNCH("hmm_fwd_pair");
    return 0;
}

}  // namespace pmx
