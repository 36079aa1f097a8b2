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
                ll += log((double)c);
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
                ll += log((double)c);
            }
            __syncthreads();
            inv = 1.0f / s_c;
            float* tmp = cur; cur = nxt; nxt = tmp;
        }
        if (threadIdx.x == 0) out_ll[sig] = ll;
        __syncthreads();
    }
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
        if (old || S < 4096)
            k_kmer_fwd<false><<<grid, threads, 0, st>>>(kmer, p_stay, p_step, E_lin, obs, nsig, T, out_ll, alpha);
        else
            k_kmer_fwd_vec<<<grid, 1024, 0, st>>>(kmer, p_stay, p_step, E_lin, obs, nsig, T, out_ll, alpha);
    }
    PMX_CHECK_LAUNCH("kmer_fwd");
    return 0;
}

}  // extern "C"
