// k-mer (de Bruijn) HMM forward — the "nanopore scale" BASELINE config.
//
// Reference anchor: the trellis is the forward recursion of SURVEY Appendix
// A.1 (log-sum-exp over predecessors, `map one sigs` over signals) with the
// sparse transition structure pinned in SURVEY §8(d): S = 4^kmer states; the
// predecessors of j are j itself (stay, p_stay) and (j >> 2) | (b << (2k-2)),
// b = 0..3 (step, p_step each).  The paper's Viterbi case study uses this
// k-mer model.
//
// Design: the 5-point stencil per state is memory-bound on the alpha vector
// (256 KiB per signal at S = 65536 — larger than one SM's shared memory), so
// each CTA keeps its signal's alpha double-buffered in a private global
// workspace slice that stays L2-resident (148 CTAs x 512 KiB = 76 MiB < L2),
// reads it with L2-only loads (ld.global.cg), and normalises lazily: step t
// multiplies by 1/c_{t-1} while computing a_t, and accumulates log c_t in
// fp64.  Small S (alpha fits in shared memory) uses a shared-memory variant.
#include <stdlib.h>
#include "common.cuh"
#include "tc.cuh"

namespace pmx {

__global__ void k_kmer_prep(const float* __restrict__ log_E, int S, int K, float* __restrict__ E_lin) {
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < (int64_t)S * K;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = idx % S, k = idx / S;
        E_lin[idx] = expf(log_E[j * K + k]);
    }
}

template <bool SMEM>
__global__ void __launch_bounds__(1024)
k_kmer_fwd(int kmer, float p_stay, float p_step, const float* __restrict__ E_lin,
           const int* __restrict__ obs, int64_t nsig, int T, double* __restrict__ out_ll,
           float* __restrict__ ws) {
    extern __shared__ float sm[];
    __shared__ float s_red[32];
    __shared__ float s_c;
    const int S = 1 << (2 * kmer);
    const int hi_shift = 2 * kmer - 2;
    float* bufA = SMEM ? sm : ws + (int64_t)blockIdx.x * 2 * S;
    float* bufB = bufA + S;
    for (int64_t sig = blockIdx.x; sig < nsig; sig += gridDim.x) {
        const int* o = obs + sig * (int64_t)T;
        double ll = 0.0;
        float inv = 1.0f / (float)S;    // uniform initial distribution
        float* cur = bufA;
        float* nxt = bufB;
        for (int t = 0; t < T; ++t) {
            const float* e = E_lin + (int64_t)o[t] * S;
            float part = 0.f;
            for (int j = threadIdx.x; j < S; j += blockDim.x) {
                float v;
                if (t == 0) {
                    v = inv * e[j];
                } else {
                    const int base = j >> 2;
                    float a0, a1, a2, a3, a4;
                    if (SMEM) {
                        a0 = cur[j];
                        a1 = cur[base]; a2 = cur[base | (1 << hi_shift)];
                        a3 = cur[base | (2 << hi_shift)]; a4 = cur[base | (3 << hi_shift)];
                    } else {
                        a0 = __ldcg(cur + j);
                        a1 = __ldcg(cur + base); a2 = __ldcg(cur + (base | (1 << hi_shift)));
                        a3 = __ldcg(cur + (base | (2 << hi_shift))); a4 = __ldcg(cur + (base | (3 << hi_shift)));
                    }
                    const float stepsum = (a1 + a2) + (a3 + a4);
                    v = inv * e[j] * fmaf(p_stay, a0, p_step * stepsum);
                }
                if (SMEM) nxt[j] = v; else __stcg(nxt + j, v);
                part += v;
            }
            for (int off = 16; off > 0; off >>= 1) part += __shfl_xor_sync(0xffffffffu, part, off);
            if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = part;
            __syncthreads();
            if (threadIdx.x == 0) {
                float c = 0.f;
                for (int w = 0; w < (int)(blockDim.x >> 5); ++w) c += s_red[w];
                s_c = c;
                ll += log_scale((double)c);
            }
            __syncthreads();
            inv = 1.0f / s_c;
            float* tmp = cur; cur = nxt; nxt = tmp;
        }
        if (threadIdx.x == 0) out_ll[sig] = ll;
        __syncthreads();
    }
}

// L2 policy: keep the alpha slices resident (evict_last); the emission table
// is read once per step and may go first.
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ float4 ld_keep4(const float* a, uint64_t pol) {
    float4 v;
    asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(a), "l"(pol));
    return v;
}
__device__ __forceinline__ float ld_keep(const float* a, uint64_t pol) {
    float v;
    asm volatile("ld.global.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(a), "l"(pol));
    return v;
}
__device__ __forceinline__ void st_keep4(float* a, float4 v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;"
                 :: "l"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol) : "memory");
}

// Global-alpha path, 4 states per thread: j = 4q .. 4q+3 share the step
// predecessors (j >> 2 = q): alpha[q | b << (2k-2)], b = 0..3 — four scalar
// loads, coalesced across the warp (consecutive q) and reused by the four
// states; the stay terms, emissions and the new alpha are 16-byte vectors.
// Same arithmetic per state as k_kmer_fwd (fmaf(p_stay, a_j, p_step *
// ((a1 + a2) + (a3 + a4)))).
__global__ void __launch_bounds__(1024)
k_kmer_fwd_vec(int kmer, float p_stay, float p_step, const float* __restrict__ E_lin,
               const int* __restrict__ obs, int64_t nsig, int T, double* __restrict__ out_ll,
               float* __restrict__ ws) {
    __shared__ float s_red[32];
    __shared__ float s_c;
    const int S = 1 << (2 * kmer);
    const int Q = S >> 2;
    const int hi = 2 * kmer - 2;
    const uint64_t pol = l2_policy_evict_last();
    float* bufA = ws + (int64_t)blockIdx.x * 2 * S;
    float* bufB = bufA + S;
    for (int64_t sig = blockIdx.x; sig < nsig; sig += gridDim.x) {
        const int* o = obs + sig * (int64_t)T;
        double ll = 0.0;
        float inv = 1.0f / (float)S;
        float* cur = bufA;
        float* nxt = bufB;
        for (int t = 0; t < T; ++t) {
            const float* e = E_lin + (int64_t)o[t] * S;
            float part = 0.f;
            // KU state quads per thread per iteration, all loads issued before any
            // store (the cache-hinted accesses are ordered asm statements: without the
            // batching each quad's loads would wait behind the previous quad's store)
            constexpr int KU = 2;
            for (int q0 = threadIdx.x; q0 < Q; q0 += KU * blockDim.x) {
                float4 ev[KU], a0[KU];
                float a1[KU], a2[KU], a3[KU], a4[KU];
#pragma unroll
                for (int u = 0; u < KU; ++u) {
                    const int q = q0 + u * blockDim.x;
                    if (q < Q) {
                        ev[u] = __ldg(reinterpret_cast<const float4*>(e) + q);
                        if (t > 0) {
                            a0[u] = ld_keep4(cur + 4 * q, pol);
                            a1[u] = ld_keep(cur + q, pol);
                            a2[u] = ld_keep(cur + (q | (1 << hi)), pol);
                            a3[u] = ld_keep(cur + (q | (2 << hi)), pol);
                            a4[u] = ld_keep(cur + (q | (3 << hi)), pol);
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < KU; ++u) {
                    const int q = q0 + u * blockDim.x;
                    if (q >= Q) break;
                    float4 v;
                    if (t == 0) {
                        v = make_float4(inv * ev[u].x, inv * ev[u].y, inv * ev[u].z, inv * ev[u].w);
                    } else {
                        const float st = p_step * ((a1[u] + a2[u]) + (a3[u] + a4[u]));
                        v.x = inv * ev[u].x * fmaf(p_stay, a0[u].x, st);
                        v.y = inv * ev[u].y * fmaf(p_stay, a0[u].y, st);
                        v.z = inv * ev[u].z * fmaf(p_stay, a0[u].z, st);
                        v.w = inv * ev[u].w * fmaf(p_stay, a0[u].w, st);
                    }
                    st_keep4(nxt + 4 * q, v, pol);
                    part += (v.x + v.y) + (v.z + v.w);
                }
            }
            for (int off = 16; off > 0; off >>= 1) part += __shfl_xor_sync(0xffffffffu, part, off);
            if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = part;
            __syncthreads();
            if (threadIdx.x == 0) {
                float c = 0.f;
                for (int w = 0; w < (int)(blockDim.x >> 5); ++w) c += s_red[w];
                s_c = c;
                ll += log_scale((double)c);
            }
            __syncthreads();
            inv = 1.0f / s_c;
            float* tmp = cur; cur = nxt; nxt = tmp;
        }
        if (threadIdx.x == 0) out_ll[sig] = ll;
        __syncthreads();
    }
}

// ------------------------------------------------------------------------
// k = 8 (S = 65,536): CTA pairs with alpha in registers.
//
// The two CTAs of a cluster hold one signal's alpha: CTA r the states
// [r * 2^15, (r + 1) * 2^15) as 8192 local quads (4 states sharing their step
// predecessors), thread t the quads 512 u + t (u = 4 v + k: chunk v = 0..3,
// k = 0..3; a warp's emission loads are 512 contiguous bytes): 64 floats in
// registers.  State j's step predecessors q | b << 14
// (q = j >> 2, b = 0..3) live in CTA b >> 1 at local index q + (b & 1) * 2^14,
// so each step CTA c ships to CTA R the pair sums alpha_c[q] + alpha_c[q + 2^14]
// for R's 8192 q values — chunk R plus chunk R + 2 of every thread, element by
// element (the (a1 + a2) and (a3 + a4) of the global kernel; their sum is the
// same rounded stepsum).  The peer's chunks are computed first and
// sent by 16-byte st.async while the own chunks are computed.  The per-step
// sum c_t travels as 16 per-warp partials per CTA (sums of the pair sums);
// both CTAs fold the 32 partials in the same order, so both divide by the same
// c_t.  Outside the SM per step: the emission row (128 KiB per CTA, an
// L2-resident table; the peer-bound chunks of the next step are loaded into
// registers, the own chunks staged by cp.async) and the 32 KiB exchange.  No
// __syncthreads: one mbarrier per receive slot (two slots by step parity)
// counts the 512 threads' arrivals plus the peer's bytes.
namespace kp {
#ifndef KP_THREADS
#define KP_THREADS 512
#endif
constexpr int THREADS = KP_THREADS, WARPS = THREADS / 32;
constexpr int S = 1 << 16, HALF = 1 << 15, QL = HALF / 4;   // states, per CTA, quads per CTA
constexpr int QPT = QL / THREADS;                            // quads per thread (16 at 512 threads)
constexpr int SPC = QPT / 4;                                 // slots (quads) per chunk: 4 chunks per thread
constexpr uint32_t REMOTE_BYTES = SPC * THREADS * 16 + WARPS * 4;   // pair sums (32 KiB) + partials
struct Smem {
    float recv[2][2][QL];           // [slot][source CTA][local q]: pair sums
    float4 estage[2][SPC][THREADS];   // the own chunks' emissions of the next step (cp.async)
    float part[2][2][WARPS];        // [slot][source CTA][warp]: partial sums of alpha
    uint64_t bar[2];
};
__device__ __forceinline__ float4 ld_e4(const float4* p) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
    return v;
}
__device__ __forceinline__ void st_async_v4(uint32_t remote_addr, float4 v, uint32_t remote_bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1,%2,%3,%4}, [%5];"
                 :: "r"(remote_addr), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "r"(remote_bar) : "memory");
}
__device__ __forceinline__ void expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" :: "r"(tc::smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ float4 add4(float4 a, float4 b) {
    return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}
// chunk V: alpha_t from alpha_{t-1}, the received pair sums and the emissions
template <int V>
__device__ __forceinline__ void step_chunk(float4 (&a)[QPT], const float4 (&e)[SPC], const float* r0, const float* r1,
                                           int tid, float inv, float p_stay, float p_step) {
    float x[SPC], y[SPC];
#pragma unroll
    for (int k = 0; k < SPC; ++k) {
        x[k] = r0[(SPC * V + k) * THREADS + tid];
        y[k] = r1[(SPC * V + k) * THREADS + tid];
    }
#pragma unroll
    for (int k = 0; k < SPC; ++k) {
        const float st = p_step * (x[k] + y[k]);
        float4& v = a[SPC * V + k];
        v.x = inv * e[k].x * fmaf(p_stay, v.x, st);
        v.y = inv * e[k].y * fmaf(p_stay, v.y, st);
        v.z = inv * e[k].z * fmaf(p_stay, v.z, st);
        v.w = inv * e[k].w * fmaf(p_stay, v.w, st);
    }
}
template <int V>
__device__ __forceinline__ void first_chunk(float4 (&a)[QPT], const float4 (&e)[SPC], float inv) {
#pragma unroll
    for (int k = 0; k < SPC; ++k)
        a[SPC * V + k] = make_float4(inv * e[k].x, inv * e[k].y, inv * e[k].z, inv * e[k].w);
}
template <int V>
__device__ __forceinline__ void load_chunk(float4 (&e)[SPC], const float4* row, int tid) {
#pragma unroll
    for (int k = 0; k < SPC; ++k) e[k] = ld_e4(row + (SPC * V + k) * THREADS + tid);
}
template <int V>
__device__ __forceinline__ void stage_chunk(float4 (*stage)[THREADS], const float4* row, int tid) {
#pragma unroll
    for (int k = 0; k < SPC; ++k) {
        const uint32_t d = tc::smem_u32(&stage[k][tid]);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(d), "l"(row + (SPC * V + k) * THREADS + tid)
                     : "memory");
    }
}
__device__ __forceinline__ void unstage(float4 (&e)[SPC], float4 (*stage)[THREADS], int tid) {
#pragma unroll
    for (int k = 0; k < SPC; ++k) e[k] = stage[k][tid];
}
// pair sums for target CTA R (chunks R and R + 2): float4s 512 k + t of R's buffer; returns their sum
template <int R, bool REMOTE>
__device__ __forceinline__ float send_pairs(const float4 (&a)[QPT], float* own_slot, uint32_t remote_slot,
                                            uint32_t remote_bar, int tid) {
    float part = 0.f;
#pragma unroll
    for (int k = 0; k < SPC; ++k) {
        const float4 v = add4(a[SPC * R + k], a[SPC * (R + 2) + k]);
        const int idx = 4 * (k * THREADS + tid);
        if (REMOTE) st_async_v4(remote_slot + 4u * idx, v, remote_bar);
        else *reinterpret_cast<float4*>(own_slot + idx) = v;
        part += (v.x + v.y) + (v.z + v.w);
    }
    return part;
}

// the whole signal loop of CTA rank R
template <int R>
__device__ __forceinline__ void pair_run(Smem& sm, float p_stay, float p_step, const float* __restrict__ E_lin,
                                         const int* __restrict__ obs, int64_t nsig, int T,
                                         double* __restrict__ out_ll) {
    constexpr int P = 1 - R;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t recv_peer = tc::mapa(tc::smem_u32(&sm.recv[0][R][0]), P);   // my rows in the peer
    const uint32_t part_peer = tc::mapa(tc::smem_u32(&sm.part[0][R][warp]), P);
    const uint32_t bar_peer = tc::mapa(tc::smem_u32(&sm.bar[0]), P);
    constexpr uint32_t SLOT_RECV = 2 * QL * 4, SLOT_PART = 2 * WARPS * 4;
    const int64_t ncl = gridDim.x >> 1;
    const float4* Erank = reinterpret_cast<const float4*>(E_lin + (size_t)R * HALF);
    float4 a[QPT];
    float4 eP0[SPC], eP1[SPC];   // emissions of the peer-bound chunks P, P + 2 (registers)
    uint32_t g = 0;            // step counter across signals (slot and barrier phase)
    double ll = 0.0;
    int64_t prev = -1;
    int64_t sig = blockIdx.x >> 1;
    if (sig < nsig) {
        const float4* row0 = Erank + (size_t)__ldg(obs + sig * (int64_t)T) * (S / 4);
        load_chunk<P>(eP0, row0, tid);
        load_chunk<P + 2>(eP1, row0, tid);
        stage_chunk<R>(sm.estage[0], row0, tid);
        stage_chunk<R + 2>(sm.estage[1], row0, tid);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    for (; sig < nsig; sig += ncl) {
        const int* o = obs + sig * (int64_t)T;
        for (int t = 0; t < T; ++t, ++g) {
            int onext = -1;
            if (t + 1 < T) onext = __ldg(o + t + 1);
            else if (sig + ncl < nsig) onext = __ldg(obs + (sig + ncl) * (int64_t)T);
            float inv = 1.0f / (float)S;
            const uint32_t ps = (g - 1) & 1u;
            if (g > 0) {
                tc::mbar_wait(&sm.bar[ps], ((g - 1) >> 1) & 1u);
                if (tid == 0) expect_tx(&sm.bar[ps], REMOTE_BYTES);   // re-arm for step g + 1's bytes
                float c = 0.f;
#pragma unroll
                for (int w = lane; w < 2 * WARPS; w += 32) c += sm.part[ps][w / WARPS][w % WARPS];
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) c += __shfl_xor_sync(0xffffffffu, c, off);
                if (R == 0 && tid == 0) {
                    ll += log_scale((double)c);
                    if (t == 0) { out_ll[prev] = ll; ll = 0.0; }
                }
                if (t > 0) inv = 1.0f / c;
            }
            const uint32_t s = g & 1u;
            const uint32_t rslot = recv_peer + s * SLOT_RECV, rbar = bar_peer + s * 8u;
            float* own = &sm.recv[s][R][0];
            const float* r0 = &sm.recv[ps][0][0];
            const float* r1 = &sm.recv[ps][1][0];
            // peer-bound chunks first, then send
            if (t == 0) {
                first_chunk<P>(a, eP0, inv);
                first_chunk<P + 2>(a, eP1, inv);
            } else {
                step_chunk<P>(a, eP0, r0, r1, tid, inv, p_stay, p_step);
                step_chunk<P + 2>(a, eP1, r0, r1, tid, inv, p_stay, p_step);
            }
            float part = send_pairs<P, true>(a, own, rslot, rbar, tid);
            // own chunks (emissions staged in shared memory by the previous step)
            asm volatile("cp.async.wait_group 0;" ::: "memory");
            float4 e0[SPC];
            unstage(e0, sm.estage[0], tid);
            if (t == 0) first_chunk<R>(a, e0, inv);
            else step_chunk<R>(a, e0, r0, r1, tid, inv, p_stay, p_step);
            unstage(e0, sm.estage[1], tid);
            if (t == 0) first_chunk<R + 2>(a, e0, inv);
            else step_chunk<R + 2>(a, e0, r0, r1, tid, inv, p_stay, p_step);
            // the next step's emissions
            const float4* nrow = Erank + (size_t)(onext < 0 ? 0 : onext) * (S / 4);
            if (onext >= 0) {
                stage_chunk<R>(sm.estage[0], nrow, tid);
                stage_chunk<R + 2>(sm.estage[1], nrow, tid);
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
            part += send_pairs<R, false>(a, own, rslot, rbar, tid);
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) part += __shfl_xor_sync(0xffffffffu, part, off);
            if (lane == 0) {
                sm.part[s][R][warp] = part;
                tc::st_async_b32(part_peer + s * SLOT_PART, __float_as_uint(part), rbar);
            }
            tc::mbar_arrive(&sm.bar[s]);
            if (onext >= 0) {   // in flight during the exchange wait
                load_chunk<P>(eP0, nrow, tid);
                load_chunk<P + 2>(eP1, nrow, tid);
            }
        }
        prev = sig;
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    if (g > 0) {   // the last step's c
        const uint32_t ps = (g - 1) & 1u;
        tc::mbar_wait(&sm.bar[ps], ((g - 1) >> 1) & 1u);
        float c = 0.f;
#pragma unroll
        for (int w = lane; w < 2 * WARPS; w += 32) c += sm.part[ps][w / WARPS][w % WARPS];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) c += __shfl_xor_sync(0xffffffffu, c, off);
        if (R == 0 && tid == 0) out_ll[prev] = ll + log_scale((double)c);
    }
}
}  // namespace kp

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kp::THREADS, 1)
k_kmer_fwd_pair(float p_stay, float p_step, const float* __restrict__ E_lin, const int* __restrict__ obs,
                int64_t nsig, int T, double* __restrict__ out_ll) {
    using namespace kp;
    extern __shared__ __align__(16) uint8_t kp_smem[];
    Smem& sm = *reinterpret_cast<Smem*>(kp_smem);
    if (threadIdx.x == 0) {
        tc::mbar_init(&sm.bar[0], THREADS);
        tc::mbar_init(&sm.bar[1], THREADS);
        expect_tx(&sm.bar[0], REMOTE_BYTES);
        expect_tx(&sm.bar[1], REMOTE_BYTES);
        tc::fence_mbar_init();
    }
    tc::cluster_sync();
    if (tc::cluster_ctarank() == 0) pair_run<0>(sm, p_stay, p_step, E_lin, obs, nsig, T, out_ll);
    else pair_run<1>(sm, p_stay, p_step, E_lin, obs, nsig, T, out_ll);
    tc::cluster_sync();   // neither CTA leaves while the other may still write into it
}

}  // namespace pmx

using namespace pmx;

extern "C" {

size_t pmx_hmm_kmer_workspace_bytes(int32_t kmer, int64_t nsig) {
    const int64_t S = 1ll << (2 * kmer);
    int64_t ctas = nsig < 148 * 2 ? nsig : 148 * 2;
    return (size_t)(S * 64 + ctas * 2 * S) * sizeof(float) + 256;
}

int pmx_hmm_kmer_forward_f32(int32_t kmer, float p_stay, float p_step, const float* log_E, int32_t K,
                             const int32_t* obs, int64_t nsig, int32_t T, double* out_ll, void* ws,
                             size_t ws_bytes, void* stream) {
    PMX_REQUIRE(kmer >= 1 && kmer <= 10 && K >= 1 && K <= 64 && T > 0 && nsig >= 0,
                "pmx_hmm_kmer_forward_f32: bad sizes");
    PMX_REQUIRE(ws && ws_bytes >= pmx_hmm_kmer_workspace_bytes(kmer, nsig),
                "pmx_hmm_kmer_forward_f32: workspace too small");
    if (nsig == 0) return 0;
    cudaStream_t st = (cudaStream_t)stream;
    const int S = 1 << (2 * kmer);
    float* E_lin = (float*)ws;
    float* alpha = E_lin + (size_t)S * 64;
    k_kmer_prep<<<(unsigned)imin64(4096, ((int64_t)S * K + 255) / 256), 256, 0, st>>>(log_E, S, K, E_lin);
    PMX_CHECK_LAUNCH("kmer_prep");
    const int threads = S >= 1024 ? 1024 : ((S + 31) / 32) * 32;
    const size_t smem = 2 * (size_t)S * sizeof(float);
    if (smem <= 200 * 1024) {
        if (smem > 48 * 1024)
            cudaFuncSetAttribute(k_kmer_fwd<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        const unsigned grid = (unsigned)nsig;
        k_kmer_fwd<true><<<grid, threads, smem, st>>>(kmer, p_stay, p_step, E_lin, obs, nsig, T, out_ll, alpha);
    } else {
        // one CTA per SM keeps all alpha slices L2-resident (148 x 512 KiB)
        const unsigned grid = (unsigned)(nsig < sm_count() ? nsig : sm_count());
        static const bool old = getenv("PMX_KMER_SCALAR") && getenv("PMX_KMER_SCALAR")[0] == '1';
        static const bool vec = getenv("PMX_KMER_VEC") && getenv("PMX_KMER_VEC")[0] == '1';
        if (kmer == 8 && !old && !vec) {
            // CTA pairs, alpha in registers: one signal per cluster at a time
            const size_t psm = sizeof(kp::Smem);
            // per call: the attribute is per device (one process may drive several)
            cudaFuncSetAttribute(k_kmer_fwd_pair, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psm);
            const int64_t clusters = nsig < sm_count() / 2 ? nsig : sm_count() / 2;
            k_kmer_fwd_pair<<<(unsigned)(2 * clusters), kp::THREADS, psm, st>>>(p_stay, p_step, E_lin, obs, nsig, T,
                                                                                 out_ll);
        } else if (old || S < 4096)
            k_kmer_fwd<false><<<grid, threads, 0, st>>>(kmer, p_stay, p_step, E_lin, obs, nsig, T, out_ll, alpha);
        else
            k_kmer_fwd_vec<<<grid, 1024, 0, st>>>(kmer, p_stay, p_step, E_lin, obs, nsig, T, out_ll, alpha);
    }
    PMX_CHECK_LAUNCH("kmer_fwd");
    return 0;
}

}  // extern "C"
