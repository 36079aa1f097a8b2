// k-NN on the 5th-generation tensor cores (tcgen05 + TMEM + TMA).
//
// Same contract as the SIMT kernel in knn.cu (reference anchor: SURVEY
// Appendix A.2 knn.pmx — top-k by (distance, train index), vote ties to the
// smaller label).  Used when d == 64, k <= 8 and the data are exact in the
// tensor-core formulation below (the BASELINE config: integer coordinates in
// [-8, 8]); then every distance is computed exactly and the answer is
// bit-identical to the fp64 reference.  Otherwise a device flag set by the
// prep kernel turns these kernels into no-ops and the SIMT kernel runs (no
// host synchronisation).
//
// Formulation: the accumulator holds the exact squared distance plus 2^23,
//     D[q, p] = sum_k q_k * (-2 x_pk) + (||x_p||^2 + ||q||^2 + 2^23)
// four UMMA k-steps over the 64 coordinates (SWIZZLE_128B operands) plus one
// over a 16-wide augmentation (SWIZZLE_32B): query rows [256, 1, hi_q, lo_q,
// 2^23, 0...], train rows [hi_x, lo_x, 256, 1, 1, 0...] with the norms split
// into bf16-exact integers (||v||^2 = 256 hi + lo).  Every partial sum is an
// integer below 2^24, so fp32 accumulation is exact, and the low 16 bits of D
// are the distance: tcgen05.ld .pack::16b hands the epilogue two candidates
// per register and the scan is packed 16-bit integer work.
//
// Structure (persistent, one CTA per SM, 18 warps):
//   warp 0   TMA producer: the 256-query block A (2 x 128 rows) and its
//            augmentation rows once per work item; train tiles B (128 x 64
//            bf16 of -2x) + B_aug (128 x 16) through a 4-stage ring
//   warp 1   TMEM allocator and MMA issuer (one thread): per train tile, two
//            128 x 128 accumulators (one per 128-query half) into one of two
//            TMEM buffers (2 buffers x 2 halves x 128 columns = all 512 columns);
//            each half has its own full / empty barriers, so the two groups of
//            8 epilogue warps never wait for each other
//   warps 2-17 epilogue: warp w owns TMEM lane quadrant w%4 (one query per
//            thread), query half ((w-2)>>2)&1 and column half (w-2)>>3; it
//            loads its 64 candidates of the tile (one packed tcgen05.ld),
//            releases the accumulator, and scans them: a min tree and a warp
//            vote per 64, and the rare insertion into a register-resident
//            sorted top-8 of packed (distance, index) keys
// Work item = (256-query block, contiguous range of train tiles).  Reusing
// each B tile for 256 queries halves L2 traffic versus 128; the split count
// is chosen so the items fill whole rounds of the SMs (all SMs with the same
// split stream the same train tiles in lockstep, so B tiles hit in L2).  Each
// CTA takes a contiguous run of items, so the splits of one query block meet
// in one CTA and carry their thresholds.  Per-item partial top-8 lists (two
// per query: one per column half) go to global memory; k_knn_merge merges
// them and votes.
//
// Bounds (measured): TMEM reads are not the limit (tools/
// tmem_probe.cu: 450 B/clk/SM with 16 warps reading, 128 KiB per tile ->
// ~290 clk); the UMMAs read 80 KiB of shared-memory operands per tile and TMA
// writes 20 KiB, ~780 clk at 128 B/clk against 640 clk of tensor work.  A
// CTA-pair variant (cta_group::2, M = N = 256: 60 KiB of shared-memory traffic
// per tile) measured no faster (9.8 ms): with two accumulator buffers, a
// warp in the rare insertion path delays the release of the next tile for
// everyone; that coupling, not a pipe, sets the remaining gap.
#include <cuda_bf16.h>
#include "common.cuh"
#include "tc.cuh"

namespace pmx {

constexpr int KT_M = 128;                 // UMMA M (queries per half)
constexpr int KT_Q = 256;                 // queries per work item
constexpr int KT_N = 128;                 // train points per tile (UMMA N)
constexpr int KT_D = 64;
constexpr int KT_AUG = 16;
constexpr int KT_STAGES = 4;
constexpr int KT_KMAX = 8;
constexpr int KT_EW = 16;                 // epilogue warps
constexpr int KT_THREADS = 64 + 32 * KT_EW;
constexpr int KT_LPQ = 2;                 // partial lists per query per item (column halves)
// Operand formats of the tensor-core kernel.  Rows are K-major byte strings:
// 64 coordinates (bf16: 128 B, SWIZZLE_128B; int8: 64 B, SWIZZLE_64B) and a
// 32-byte augmentation row (SWIZZLE_32B).  Every UMMA consumes 32 bytes of K.
//   BF16: kind::f16, fp32 accumulation, D = dist + 2^23 (low 16 bits = dist)
//   I8:   kind::i8, int32 accumulation, D = dist (exact by construction)
#ifndef KT_SPLIT
#define KT_SPLIT 1                        // accumulator regions per query half (N = 128 / KT_SPLIT per UMMA; 2: 10.0 ms)
#endif
constexpr int KT_NU = KT_N / KT_SPLIT;    // UMMA N
struct OpsBF16 {
    static constexpr int ROWB = 128, KSTEPS = 4;
    static constexpr uint32_t IDESC = tc::instr_desc(128, KT_NU, 1);
    static constexpr unsigned FLAG_RUN = 8;       // runs when only the int8 form is inexact
};
struct OpsI8 {
    static constexpr int ROWB = 64, KSTEPS = 2;
    // c_format S32 (2), a/b signed int8 (1), K-major, N >> 3, M >> 4
    static constexpr uint32_t IDESC = (2u << 4) | (1u << 7) | (1u << 10) | (((uint32_t)KT_NU >> 3) << 17) |
                                      ((128u >> 4) << 24);
    static constexpr unsigned FLAG_RUN = 0;
};
constexpr int KT_AUGB = 32;                       // augmentation row bytes (16 bf16 / 32 int8)

template <class Ops>
struct __align__(1024) KnnSmem {
    uint8_t A[KT_Q * Ops::ROWB];                        // 2 halves of 128 query rows
    uint8_t B[KT_STAGES][KT_N * Ops::ROWB];             // train rows per tile
    uint8_t Aaug[KT_Q * KT_AUGB];                       // query augmentation rows (2 halves)
    uint8_t Baug[KT_STAGES][KT_N * KT_AUGB];
    uint64_t full[KT_STAGES], empty[KT_STAGES];
    uint64_t a_full, a_empty;
    uint64_t tfull[2][2][KT_SPLIT], tempty[2][2][KT_SPLIT];   // [buffer][query half][column region]
    uint32_t tmem_base;
};

__device__ __forceinline__ uint32_t ord_f32(float f) {
    uint32_t b = __float_as_uint(f);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float unord_f32(uint32_t u) {
    return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}

// Sorted top-8 of one thread, in registers, as packed 32-bit keys
//     key = dist << 17 | local
// dist = the exact squared distance (an integer <= 32766, checked per launch
// by k_knn_bound) and local = the candidate's position in this thread's part of
// the work item (< 2^17: at most 2048 tiles x 64 columns, see knn_tc_nsplit).
// Keys order exactly like (distance, train index), so an insertion is a
// min/max network (16 IMNMX, no selects or branches) and ties keep the
// smaller index.
//
// The accumulator holds dist + 2^23 (the augmentation adds ||x||^2, ||q||^2
// and 2^23), an fp32 whose low 16 bits are dist; tcgen05.ld .pack::16b
// delivers two candidates' distances per register (column 2j in bits 0-15,
// column 2j+1 in bits 16-31; tools/tmem_probe.cu layout check), so the scan
// is packed 16-bit integer work (VIMNMX3.U16x2: four candidates per op).
constexpr uint32_t KT_LOCAL_BITS = 17;
constexpr uint32_t KT_EMPTY = 0xffffffffu;
constexpr int KT_MAX_ITEM_TILES = (1 << KT_LOCAL_BITS) / 64;             // 2048 tiles of 64 per thread
constexpr float KT_DIST_MAX = 32766.f;                                    // dist 32767 = empty / padding

struct Top8 {
    uint32_t d[KT_KMAX];
    __device__ __forceinline__ void reset() {
#pragma unroll
        for (int i = 0; i < KT_KMAX; ++i) d[i] = KT_EMPTY;
    }
    // distances below this may enter (candidates arrive in increasing index,
    // so one equal to the 8th's distance never does)
    __device__ __forceinline__ uint32_t thr() const { return d[KT_KMAX - 1] >> KT_LOCAL_BITS; }
    // Next split of the same query block (later train indices): the 8 best so
    // far were written with the previous split, so only distances below the
    // current 8th can still matter.  The list restarts as 8 copies of the key
    // (that distance, local 2^17 - 1); entries still equal to it at the end are
    // empty (a real candidate with that key ties an earlier one at a larger
    // index, so it is never needed).
    __device__ __forceinline__ uint32_t carry() {
        const uint32_t pk = (d[KT_KMAX - 1] | ((1u << KT_LOCAL_BITS) - 1));
#pragma unroll
        for (int i = 0; i < KT_KMAX; ++i) d[i] = pk;
        return pk;
    }
    __device__ __forceinline__ void insert(uint32_t key) {   // no-op when key > d[7]
#pragma unroll
        for (int i = 0; i < KT_KMAX; ++i) {
            const uint32_t lo = min(d[i], key);
            key = max(d[i], key);
            d[i] = lo;
        }
    }
};

__device__ __forceinline__ uint32_t vmin2(uint32_t a, uint32_t b) {
    uint32_t r;
    asm("min.u16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
    return r;
}
// min of N packed u16x2 words as a tree of 3-input mins (VIMNMX3.U16x2)
template <int N>
__device__ __forceinline__ uint32_t min_tree16(const uint32_t* v) {
    if constexpr (N == 1) {
        return v[0];
    } else if constexpr (N == 2) {
        return vmin2(v[0], v[1]);
    } else {
        constexpr int M = (N + 2) / 3;
        uint32_t m[M];
#pragma unroll
        for (int i = 0; i < N / 3; ++i) m[i] = vmin2(vmin2(v[3 * i], v[3 * i + 1]), v[3 * i + 2]);
        if constexpr (N % 3 == 1) m[M - 1] = v[N - 1];
        if constexpr (N % 3 == 2) m[M - 1] = vmin2(v[N - 2], v[N - 1]);
        return min_tree16<M>(m);
    }
}
__device__ __forceinline__ uint32_t min_halves(uint32_t m) { return min(m & 0xffffu, m >> 16); }

// Scan 64 candidates (32 packed words; local positions lbase + j) into the
// list: one min tree and one vote per 64 against the threshold; in a group
// some lane needs, a vote per 16 and then per candidate gates the (warp-wide)
// insert.
__device__ __forceinline__ void knn_scan64p(const uint32_t (&r)[32], uint32_t lbase, Top8& L) {
    if (!__any_sync(0xffffffffu, min_halves(min_tree16<32>(r)) < L.thr())) return;
#pragma unroll
    for (int g = 0; g < 4; ++g) {
        if (!__any_sync(0xffffffffu, min_halves(min_tree16<8>(r + g * 8)) < L.thr())) continue;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const uint32_t w = r[g * 8 + (j >> 1)];
            const uint32_t dist = (j & 1) ? (w >> 16) : (w & 0xffffu);
            const uint32_t key = (dist << KT_LOCAL_BITS) | (lbase + (uint32_t)(g * 16 + j));
            if (__any_sync(0xffffffffu, key < L.d[KT_KMAX - 1])) L.insert(key);
        }
    }
}

// prep (d == 64), 16 lanes per row, one float4 per lane (coalesced):
//   train:  xb = bf16(-2 x), xaug = [hi, lo, 256, 1, 1, 0 x 11] with ||x||^2 = 256 hi + lo
//   query:  xb = bf16(q),    xaug = [256, 1, hi, lo, 2^23, 0 x 11] with ||q||^2 = 256 hi + lo
// so that the augmentation k-step adds ||x||^2 + ||q||^2 + 2^23.
// norms (fp32) feed the SIMT fallback; flag |= 1 when the exact formulation
// does not hold (a coordinate not exact in bf16, or ||x||^2 not an integer
// below 2^16).
__global__ void k_knn_prep(const float* __restrict__ x, int64_t rows, float scale, bool is_query,
                           __nv_bfloat16* __restrict__ xb, __nv_bfloat16* __restrict__ xaug,
                           float* __restrict__ norms, unsigned* __restrict__ flag, unsigned* __restrict__ maxn) {
    const int sub = threadIdx.x & 15;
    const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    bool inexact = false;
    float nmax = 0.f;
    const bool write_ops = (*flag & 8u) != 0;   // bf16 operands only when the int8 form is inexact
    for (int64_t w = wid; w * 2 < rows; w += nw) {          // warp-uniform trip count
        const int64_t r = w * 2 + ((threadIdx.x >> 4) & 1);
        const bool valid = r < rows;
        const float4 v = valid ? __ldg(reinterpret_cast<const float4*>(x + r * 64) + sub)
                               : make_float4(0.f, 0.f, 0.f, 0.f);
        const float f[4] = {v.x, v.y, v.z, v.w};
        __nv_bfloat16 h[4];
        float s = 0.f;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const float sv = scale * f[e];
            h[e] = __float2bfloat16_rn(sv);
            inexact |= (__bfloat162float(h[e]) != sv) || (sv / scale != f[e]);
            s = fmaf(f[e], f[e], s);
        }
        uint2 packed;
        packed.x = (uint32_t)__bfloat16_as_ushort(h[0]) | ((uint32_t)__bfloat16_as_ushort(h[1]) << 16);
        packed.y = (uint32_t)__bfloat16_as_ushort(h[2]) | ((uint32_t)__bfloat16_as_ushort(h[3]) << 16);
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o, 16);
        if (valid) {
            if (sub == 0) inexact |= !(s >= 0.f && s < 65536.f && s == floorf(s));
            if (write_ops) reinterpret_cast<uint2*>(xb + r * 64)[sub] = packed;
            nmax = fmaxf(nmax, s);
            if (sub == 0) norms[r] = s;
            if (sub < 4 && write_ops) {
                // hi, lo are exact in bf16 when s is an integer in [0, 2^16)
                const float hi = floorf(s / 256.f), lo = s - 256.f * hi;
                auto bf = [](float v) { return (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(v)); };
                uint2 a = make_uint2(0u, 0u);
                if (sub == 0) {
                    a = is_query ? make_uint2(bf(256.f) | (bf(1.f) << 16), bf(hi) | (bf(lo) << 16))
                                 : make_uint2(bf(hi) | (bf(lo) << 16), bf(256.f) | (bf(1.f) << 16));
                } else if (sub == 1) {
                    a.x = bf(is_query ? 8388608.f : 1.f);
                }
                reinterpret_cast<uint2*>(xaug + r * KT_AUG)[sub] = a;
            }
        }
    }
    if (__any_sync(0xffffffffu, inexact) && (threadIdx.x & 31) == 0) atomicOr(flag, 1u);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nmax = fmaxf(nmax, __shfl_xor_sync(0xffffffffu, nmax, o));
    if ((threadIdx.x & 31) == 0) atomicMax(maxn, __float_as_uint(nmax));    // norms >= 0: bits order as values
}

// int8 operands (the default tensor-core form): train -2x, query q as signed
// 8-bit integers, augmentation rows (32 bytes) train [a, b, 64, 1, 0...] and
// query [64, 1, a, b, 0...] with ||v||^2 = 64 a + b, so the int32 accumulator
// is exactly ||x||^2 - 2 q.x + ||q||^2.  flag |= 8 when a scaled coordinate is
// not an integer in [-128, 127] or a norm not an integer below 8192 (the bf16
// form then runs).
__global__ void k_knn_prep8(const float* __restrict__ x, int64_t rows, float scale, bool is_query,
                            int8_t* __restrict__ xb, int8_t* __restrict__ xaug, unsigned* __restrict__ flag) {
    const int sub = threadIdx.x & 15;
    const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    bool inexact = false;
    for (int64_t w = wid; w * 2 < rows; w += nw) {
        const int64_t r = w * 2 + ((threadIdx.x >> 4) & 1);
        const bool valid = r < rows;
        const float4 v = valid ? __ldg(reinterpret_cast<const float4*>(x + r * 64) + sub)
                               : make_float4(0.f, 0.f, 0.f, 0.f);
        const float f[4] = {v.x, v.y, v.z, v.w};
        uint32_t packed = 0;
        float s = 0.f;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const float sv = scale * f[e];
            inexact |= !(sv == rintf(sv) && sv >= -128.f && sv <= 127.f);
            packed |= (uint32_t)(uint8_t)(int8_t)(int)fminf(fmaxf(sv, -128.f), 127.f) << (8 * e);
            s = fmaf(f[e], f[e], s);
        }
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o, 16);
        if (valid) {
            reinterpret_cast<uint32_t*>(xb + r * 64)[sub] = packed;
            if (sub < 2) {
                const bool ok = s >= 0.f && s < 8192.f && s == floorf(s);
                if (sub == 0) inexact |= !ok;
                const uint32_t a = ok ? (uint32_t)(s / 64.f) : 0u, b = ok ? (uint32_t)s - 64u * a : 0u;
                uint4 row = make_uint4(0u, 0u, 0u, 0u);
                if (sub == 0) row.x = is_query ? (64u | (1u << 8) | (a << 16) | (b << 24)) : (a | (b << 8) | (64u << 16) | (1u << 24));
                reinterpret_cast<uint4*>(xaug + r * KT_AUGB)[sub] = row;
            }
        }
    }
    if (__any_sync(0xffffffffu, inexact) && (threadIdx.x & 31) == 0) atomicOr(flag, 8u);
}

// The packed keys hold squared distances up to KT_DIST_MAX: with the largest
// norms (sqrt(max ||x||^2) + sqrt(max ||q||^2))^2 bounds every distance; above
// it the SIMT kernel answers (flag bit 2).
__global__ void k_knn_bound(const unsigned* __restrict__ maxn, unsigned* __restrict__ flag) {
    if (threadIdx.x == 0) {
        const double b = sqrt((double)__uint_as_float(maxn[0])) + sqrt((double)__uint_as_float(maxn[1]));
        if (!(b * b <= (double)KT_DIST_MAX)) atomicOr(flag, 2u);
    }
}

template <class Ops>
__global__ void __maxnreg__(96)
k_knn_tc(const __grid_constant__ CUtensorMap tmq, const __grid_constant__ CUtensorMap tmqa,
         const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmxa, int64_t ntr, int64_t nq,
         int k, int nsplit, uint64_t* __restrict__ lists, const unsigned* __restrict__ flag) {
    if (*flag != Ops::FLAG_RUN) return;      // the other format (or the SIMT kernel) answers
    constexpr uint32_t A_BYTES = KT_Q * Ops::ROWB, AAUG_BYTES = KT_Q * KT_AUGB;
    constexpr uint32_t B_BYTES = KT_N * Ops::ROWB, BAUG_BYTES = KT_N * KT_AUGB;
    extern __shared__ uint8_t smem_raw[];
    // 1 KiB-aligned by pointer arithmetic on the __shared__ array itself, so every
    // access through it stays in the shared space (STS/LDS, not generic ST/LD)
    KnnSmem<Ops>& S = *reinterpret_cast<KnnSmem<Ops>*>(
        smem_raw + ((1024u - ((uint32_t)__cvta_generic_to_shared(smem_raw) & 1023u)) & 1023u));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nblk = (int)((nq + KT_Q - 1) / KT_Q);
    const int ntiles = (int)((ntr + KT_N - 1) / KT_N);
    const int nitems = nblk * nsplit;
    // each CTA takes a contiguous run of items, so consecutive splits of one
    // query block meet in one CTA and the epilogue carries its thresholds
    // across them (all runs advance through equal-length items in step, so at
    // any time the SMs stream nsplit train regions, as B tiles hit in L2)
    const int it_begin = (int)((int64_t)blockIdx.x * nitems / gridDim.x);
    const int it_end = (int)((int64_t)(blockIdx.x + 1) * nitems / gridDim.x);

    if (threadIdx.x == 0) {
        for (int s = 0; s < KT_STAGES; ++s) { tc::mbar_init(&S.full[s], 1); tc::mbar_init(&S.empty[s], 1); }
        tc::mbar_init(&S.a_full, 1);
        tc::mbar_init(&S.a_empty, 1);
        for (int b = 0; b < 2; ++b)
            for (int h = 0; h < 2; ++h)
                for (int c = 0; c < KT_SPLIT; ++c) {
                    tc::mbar_init(&S.tfull[b][h][c], 1);
                    tc::mbar_init(&S.tempty[b][h][c], KT_EW / (2 * KT_SPLIT));
                }
        tc::fence_mbar_init();
        tc::tma_prefetch(&tmq);
        tc::tma_prefetch(&tmqa);
        tc::tma_prefetch(&tmx);
        tc::tma_prefetch(&tmxa);
    }
    tc::fence_proxy_async();                 // generic-proxy smem writes -> UMMA (async proxy)
    if (warp == 1) tc::tmem_alloc(&S.tmem_base, 512);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = S.tmem_base;

    if (warp == 0) {
        if (lane == 0) {                                    // ---- TMA producer
            int stage = 0; uint32_t phase = 0, a_par = 0;
            bool first = true;
            for (int it = it_begin; it < it_end; ++it) {
                const int qb = it / nsplit, sp = it % nsplit;
                const int t0 = (int)((int64_t)sp * ntiles / nsplit), t1 = (int)((int64_t)(sp + 1) * ntiles / nsplit);
                if (!first) { tc::mbar_wait(&S.a_empty, a_par); a_par ^= 1; }
                first = false;
                tc::mbar_arrive_expect_tx(&S.a_full, A_BYTES + AAUG_BYTES);
                tc::tma_load_2d(S.A, &tmq, &S.a_full, 0, qb * KT_Q);
                tc::tma_load_2d(S.Aaug, &tmqa, &S.a_full, 0, qb * KT_Q);
                for (int t = t0; t < t1; ++t) {
                    tc::mbar_wait(&S.empty[stage], phase ^ 1);
                    tc::mbar_arrive_expect_tx(&S.full[stage], B_BYTES + BAUG_BYTES);
                    tc::tma_load_2d(S.B[stage], &tmx, &S.full[stage], 0, t * KT_N);
                    tc::tma_load_2d(S.Baug[stage], &tmxa, &S.full[stage], 0, t * KT_N);
                    if (++stage == KT_STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ---- MMA issuer: the whole warp walks the pipeline (uniform registers),
        // one elected lane issues; descriptors advance in 16-byte units
        constexpr uint32_t idesc = Ops::IDESC;
        int stage = 0; uint32_t phase = 0, a_par = 0;
        int b = 0; uint32_t acc_phase = 0;
        auto main_desc = [](const void* p) {
            return Ops::ROWB == 128 ? tc::sw128_kmajor_desc(tc::smem_u32(p)) : tc::sw64_kmajor_desc(tc::smem_u32(p));
        };
        const uint64_t a_desc = main_desc(S.A);
        const uint64_t b_desc0 = main_desc(S.B[0]);
        const uint64_t aaug_desc = tc::sw32_kmajor_desc(tc::smem_u32(S.Aaug));
        const uint64_t baug_desc0 = tc::sw32_kmajor_desc(tc::smem_u32(S.Baug[0]));
        const uint32_t full_a = tc::smem_u32(&S.full[0]), empty_a = tc::smem_u32(&S.empty[0]);
        const uint32_t tfull_a = tc::smem_u32(&S.tfull[0][0][0]), tempty_a = tc::smem_u32(&S.tempty[0][0][0]);
        for (int it = it_begin; it < it_end; ++it) {
            const int sp = it % nsplit;
            const int t0 = (int)((int64_t)sp * ntiles / nsplit), t1 = (int)((int64_t)(sp + 1) * ntiles / nsplit);
            tc::mbar_wait(&S.a_full, a_par); a_par ^= 1;
            for (int t = t0; t < t1; ++t) {
                tc::mbar_wait_addr(full_a + 8u * stage, phase);
                const uint64_t bd = b_desc0 + (uint64_t)(stage * (B_BYTES >> 4));
                const uint64_t bad = baug_desc0 + (uint64_t)(stage * (BAUG_BYTES >> 4));
                // per query half: its accumulator free (its 8 epilogue warps), its
                // UMMAs, its own commit — the halves' epilogue groups do not wait
                // for each other
#pragma unroll
                for (int h = 0; h < 2; ++h)
#pragma unroll
                    for (int c = 0; c < KT_SPLIT; ++c) {
                        const uint32_t bo = 8u * ((b * 2 + h) * KT_SPLIT + c);
                        tc::mbar_wait_addr(tempty_a + bo, acc_phase ^ 1);
                        tc::tc_fence_after();
                        if (tc::elect_one()) {
                            const uint32_t d = tmem + (uint32_t)((b * 2 + h) * KT_N + c * KT_NU);
                            const uint64_t ad = a_desc + (uint64_t)(h * ((KT_M * Ops::ROWB) >> 4));
                            const uint64_t bdc = bd + (uint64_t)(c * ((KT_NU * Ops::ROWB) >> 4));
                            const uint64_t badc = bad + (uint64_t)(c * ((KT_NU * KT_AUGB) >> 4));
                            // K advances 32 bytes (2 descriptor units) per UMMA
#pragma unroll
                            for (int kk = 0; kk < Ops::KSTEPS; ++kk) {
                                if (Ops::ROWB == 128) tc::umma_f16(d, ad + 2 * kk, bdc + 2 * kk, idesc, kk > 0);
                                else tc::umma_i8(d, ad + 2 * kk, bdc + 2 * kk, idesc, kk > 0);
                            }
                            // + ||x||^2 + ||q||^2 (+ 2^23 for the bf16 form)
                            const uint64_t aad = aaug_desc + (uint64_t)(h * ((KT_M * KT_AUGB) >> 4));
                            if (Ops::ROWB == 128) tc::umma_f16(d, aad, badc, idesc, 1);
                            else tc::umma_i8(d, aad, badc, idesc, 1);
                            tc::umma_commit_addr(tfull_a + bo);
                            if (h == 1 && c == KT_SPLIT - 1) tc::umma_commit_addr(empty_a + 8u * stage);
                        }
                        __syncwarp();
                    }
                if (++stage == KT_STAGES) { stage = 0; phase ^= 1; }
                b ^= 1;
                if (b == 0) acc_phase ^= 1;
            }
            if (tc::elect_one()) tc::umma_commit(&S.a_empty);
            __syncwarp();
        }
    } else {                                                 // ---- epilogue (warps 2..17)
        const int ew = warp - 2;
        const int quad = warp & 3, h = (ew >> 2) & 1, ch = ew >> 3;
        const int row = h * KT_M + quad * 32 + lane;           // query within the block
        int b = 0; uint32_t acc_phase = 0;
        // shared addresses of the accumulator barriers, once (the smem struct is
        // reached through a generic pointer: converting it per tile costs an
        // S2UR of the CTA id and address arithmetic on every wait / arrive)
        // my 64 columns lie in column region ch * 64 / KT_NU of my half
        const uint32_t tfull_a = tc::smem_u32(&S.tfull[0][h][ch * 64 / KT_NU]),
                       tempty_a = tc::smem_u32(&S.tempty[0][h][ch * 64 / KT_NU]);
        Top8 L;
        int prev_qb = -1;
        uint32_t pseudo = KT_EMPTY;
        for (int it = it_begin; it < it_end; ++it) {
            const int qb = it / nsplit, sp = it % nsplit;
            const int t0 = (int)((int64_t)sp * ntiles / nsplit), t1 = (int)((int64_t)(sp + 1) * ntiles / nsplit);
            const int64_t q = (int64_t)qb * KT_Q + row;
            if (qb != prev_qb) { L.reset(); pseudo = KT_EMPTY; }
            else pseudo = L.carry();
            prev_qb = qb;
            for (int t = t0; t < t1; ++t) {
                tc::mbar_wait_addr(tfull_a + 8u * (2 * KT_SPLIT) * b, acc_phase);
                tc::tc_fence_after();
                const uint32_t taddr = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)((b * 2 + h) * KT_N + ch * 64);
                uint32_t r[32];
                tc::tmem_ld_32x32b_x32_pack16(taddr, r);          // 64 columns, two per register
                tc::tmem_ld_wait();
                // my 64 columns are in registers: release the accumulator at once, so
                // the MMAs of tile t + 2 overlap this scan (a slow warp delays nobody
                // until it falls a whole tile behind)
                tc::tc_fence_before();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive_addr(tempty_a + 8u * (2 * KT_SPLIT) * b);
                if (t == ntiles - 1) {                       // last tile: padded rows never enter
                    const int64_t colbase = (int64_t)t * KT_N + ch * 64;
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        if (colbase + 2 * j >= ntr) r[j] = (r[j] & 0xffff0000u) | 0x7fffu;
                        if (colbase + 2 * j + 1 >= ntr) r[j] = (r[j] & 0xffffu) | 0x7fff0000u;
                    }
                }
                knn_scan64p(r, (uint32_t)((t - t0) * 64), L);
                b ^= 1;
                if (b == 0) acc_phase ^= 1;
            }
            if (q < nq) {
                uint64_t* dst = lists + ((q * nsplit + sp) * KT_LPQ + ch) * KT_KMAX;
#pragma unroll
                for (int i = 0; i < KT_KMAX; ++i) {
                    const uint32_t dist = L.d[i] >> KT_LOCAL_BITS, loc = L.d[i] & ((1u << KT_LOCAL_BITS) - 1);
                    const uint64_t gidx = (uint64_t)(t0 + (int)(loc >> 6)) * KT_N + (uint64_t)(ch * 64) + (loc & 63u);
                    dst[i] = (dist >= 32767u || L.d[i] == pseudo) ? ~0ull : (((uint64_t)dist << 32) | gidx);
                }
            }
        }
    }
    tc::tc_fence_before();
    __syncthreads();
    if (warp == 1) tc::tmem_dealloc(tmem, 512);
}

// Merge the nsplit sorted partial lists of each query and vote (ties -> the
// smaller label, `foldl (... gti ...) 0 classIdx`).
__global__ void k_knn_merge(const uint64_t* __restrict__ lists, int nlists, const int* __restrict__ labels,
                            int64_t nq, int k, int ncls, int* __restrict__ out_label, int* __restrict__ out_idx,
                            const unsigned* __restrict__ flag) {
    if (*flag & 7u) return;                  // the SIMT kernel answers
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nq) return;
    const uint64_t* P = lists + q * nlists * KT_KMAX;
    int head[64];
    for (int l = 0; l < nlists; ++l) head[l] = 0;
    int votes[64];
    for (int c = 0; c < ncls; ++c) votes[c] = 0;
    for (int r = 0; r < k; ++r) {
        uint64_t best = ~0ull;
        int bl = 0;
        for (int l = 0; l < nlists; ++l) {
            const uint64_t v = head[l] < k ? P[l * KT_KMAX + head[l]] : ~0ull;
            if (v < best) { best = v; bl = l; }
        }
        head[bl]++;
        const int idx = best == ~0ull ? -1 : (int)(uint32_t)(best & 0xffffffffu);
        if (out_idx) out_idx[q * k + r] = idx;
        if (idx >= 0) {
            const int lab = labels[idx];
            if (lab >= 0 && lab < ncls) votes[lab]++;
        }
    }
    int best = 0;
    for (int c = 1; c < ncls; ++c) if (votes[c] > votes[best]) best = c;
    out_label[q] = best;
}

// ---------------------------------------------------------------- host side
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

PFN_encodeTiled get_encode_tiled() {
    static PFN_encodeTiled fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PFN_encodeTiled)p;
    }
    return fn;
}

// 2-D row-major [rows][cols] tensor, box [box_rows][box_cols], given swizzle.
bool make_tmap_2d(CUtensorMap* m, const void* base, CUtensorMapDataType dt, int elem_bytes, uint64_t rows,
                  uint64_t cols, uint32_t box_rows, uint32_t box_cols, CUtensorMapSwizzle swz) {
    PFN_encodeTiled enc = get_encode_tiled();
    if (!enc) return false;
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {cols * (uint64_t)elem_bytes};
    cuuint32_t box[2] = {box_cols, box_rows};
    cuuint32_t estr[2] = {1, 1};
    return enc(m, dt, 2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Split count: items fill whole rounds of the SMs (rounds x tiles per item is
// the kernel's length in tile times), with a 1% charge per split for the
// per-item restart of the top-8 lists (early tiles insert often).
int knn_tc_nsplit(int64_t ntr, int64_t nq) {
    const int64_t nblk = (nq + KT_Q - 1) / KT_Q;
    const int64_t ntiles = (ntr + KT_N - 1) / KT_N;
    const int64_t sms = sm_count();
    int best = -1;                                      // none: more than 32 x 2048 tiles
    double best_cost = 1e300;
    for (int ns = 1; ns <= 32 && ns <= ntiles; ++ns) {
        const int64_t rounds = (nblk * ns + sms - 1) / sms;
        const int64_t per = (ntiles + ns - 1) / ns;
        if (per > KT_MAX_ITEM_TILES) continue;          // local positions must fit the key
        const double cost = (double)(rounds * per) * (1.0 + 0.01 * ns);
        if (cost < best_cost) { best_cost = cost; best = ns; }
    }
    return best;
}

// workspace: xb (ntr x 64 bf16) | xaug (ntr x 16 bf16) | qb (nq x 64 bf16) | qaug (nq x 16 bf16) | lists
// Operand buffers are padded to whole TMA boxes (a box may not exceed the
// tensor): rows beyond nq / ntr hold garbage that is never reported (queries)
// or masked to +inf (train columns) in the epilogue.
static inline int64_t pad_to(int64_t n, int64_t m) { return (n + m - 1) / m * m; }

// workspace: bf16 operands (train 64 + 16 aug, query 64 + 16 aug per row) |
// int8 operands (64 + 32 bytes per row each) | lists | maxn
size_t knn_tc_workspace(int64_t ntr, int64_t nq) {
    const int ns = knn_tc_nsplit(ntr, nq) > 0 ? knn_tc_nsplit(ntr, nq) : 0;
    const int64_t ntr_p = pad_to(ntr, KT_N), nq_p = pad_to(nq, KT_Q);
    return (size_t)(ntr_p + nq_p) * (KT_D + KT_AUG) * 2 + (size_t)(ntr_p + nq_p) * (64 + KT_AUGB) + 2048 +
           (size_t)nq * ns * KT_LPQ * KT_KMAX * 8 + 256 + 256;
}

template <class Ops>
static int knn_tc_launch(const CUtensorMap& tmq, const CUtensorMap& tmqa, const CUtensorMap& tmx,
                         const CUtensorMap& tmxa, int64_t ntr, int64_t nq, int k, int nsplit, uint64_t* lists,
                         const unsigned* flag, cudaStream_t st) {
    const int nitems = (int)((nq + KT_Q - 1) / KT_Q) * nsplit;
    const size_t smem = sizeof(KnnSmem<Ops>) + 1024;
    cudaFuncSetAttribute(k_knn_tc<Ops>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int grid = nitems < sm_count() ? nitems : sm_count();
    k_knn_tc<Ops><<<grid, KT_THREADS, smem, st>>>(tmq, tmqa, tmx, tmxa, ntr, nq, k, nsplit, lists, flag);
    PMX_CHECK_LAUNCH("knn_tc");
    return 0;
}

int knn_tc_run(const float* train, const float* query, const int* labels, int64_t ntr, int64_t nq, int k, int ncls,
               int* out_label, int* out_idx, float* tnorm, float* qnorm, unsigned* flag, void* ws, cudaStream_t st) {
    const int64_t ntr_p = pad_to(ntr, KT_N), nq_p = pad_to(nq, KT_Q);
    char* w = (char*)ws;
    __nv_bfloat16* xb = (__nv_bfloat16*)w;
    __nv_bfloat16* xaug = xb + (size_t)ntr_p * KT_D;
    __nv_bfloat16* qb = xaug + (size_t)ntr_p * KT_AUG;
    __nv_bfloat16* qaug = qb + (size_t)nq_p * KT_D;
    int8_t* xb8 = (int8_t*)(((uintptr_t)(qaug + (size_t)nq_p * KT_AUG) + 1023) & ~(uintptr_t)1023);
    int8_t* xaug8 = xb8 + (size_t)ntr_p * 64;
    int8_t* qb8 = xaug8 + (size_t)ntr_p * KT_AUGB;
    int8_t* qaug8 = qb8 + (size_t)nq_p * 64;
    uint64_t* lists = (uint64_t*)(((uintptr_t)(qaug8 + (size_t)nq_p * KT_AUGB) + 1023) & ~(uintptr_t)1023);
    const int nsplit = knn_tc_nsplit(ntr, nq);
    if (nsplit < 0) {                                   // train set too long for the packed keys: SIMT
        cudaError_t e = cudaMemsetAsync(flag, 0x04, 1, st);
        if (e != cudaSuccess) { set_last_error("knn flag: %s", cudaGetErrorString(e)); return -2; }
        return 0;
    }
    unsigned* maxn = (unsigned*)(lists + (size_t)nq * nsplit * KT_LPQ * KT_KMAX);
    cudaMemsetAsync(maxn, 0, 2 * sizeof(unsigned), st);
    const int pgrid = 4 * sm_count();
    const unsigned gtr = (unsigned)imin64(pgrid, (ntr + 15) / 16), gq = (unsigned)imin64(pgrid, (nq + 15) / 16);
    // int8 operands first (flag bit 8 when inexact); then norms, the bf16
    // exactness bit and — only if the int8 form is inexact — the bf16 operands
    k_knn_prep8<<<gtr, 256, 0, st>>>(train, ntr, -2.f, false, xb8, xaug8, flag);
    k_knn_prep8<<<gq, 256, 0, st>>>(query, nq, 1.f, true, qb8, qaug8, flag);
    k_knn_prep<<<gtr, 256, 0, st>>>(train, ntr, -2.f, false, xb, xaug, tnorm, flag, maxn);
    k_knn_prep<<<gq, 256, 0, st>>>(query, nq, 1.f, true, qb, qaug, qnorm, flag, maxn + 1);
    PMX_CHECK_LAUNCH("knn_prep");
    CUtensorMap tmq, tmqa, tmx, tmxa, tmq8, tmqa8, tmx8, tmxa8;
    const CUtensorMapDataType BF = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, U8 = CU_TENSOR_MAP_DATA_TYPE_UINT8;
    if (!make_tmap_2d(&tmq, qb, BF, 2, (uint64_t)nq_p, KT_D, KT_Q, KT_D, CU_TENSOR_MAP_SWIZZLE_128B) ||
        !make_tmap_2d(&tmqa, qaug, BF, 2, (uint64_t)nq_p, KT_AUG, KT_Q, KT_AUG, CU_TENSOR_MAP_SWIZZLE_32B) ||
        !make_tmap_2d(&tmx, xb, BF, 2, (uint64_t)ntr_p, KT_D, KT_N, KT_D, CU_TENSOR_MAP_SWIZZLE_128B) ||
        !make_tmap_2d(&tmxa, xaug, BF, 2, (uint64_t)ntr_p, KT_AUG, KT_N, KT_AUG, CU_TENSOR_MAP_SWIZZLE_32B) ||
        !make_tmap_2d(&tmq8, qb8, U8, 1, (uint64_t)nq_p, 64, KT_Q, 64, CU_TENSOR_MAP_SWIZZLE_64B) ||
        !make_tmap_2d(&tmqa8, qaug8, U8, 1, (uint64_t)nq_p, KT_AUGB, KT_Q, KT_AUGB, CU_TENSOR_MAP_SWIZZLE_32B) ||
        !make_tmap_2d(&tmx8, xb8, U8, 1, (uint64_t)ntr_p, 64, KT_N, 64, CU_TENSOR_MAP_SWIZZLE_64B) ||
        !make_tmap_2d(&tmxa8, xaug8, U8, 1, (uint64_t)ntr_p, KT_AUGB, KT_N, KT_AUGB, CU_TENSOR_MAP_SWIZZLE_32B)) {
        set_last_error("knn: cuTensorMapEncodeTiled unavailable or failed");
        return -2;
    }
    k_knn_bound<<<1, 32, 0, st>>>(maxn, flag);
    // exactly one of these does the work (flag == 0: int8, flag == 8: bf16); the
    // other returns at once, as both do when the SIMT kernel answers
    int rc = knn_tc_launch<OpsI8>(tmq8, tmqa8, tmx8, tmxa8, ntr, nq, k, nsplit, lists, flag, st);
    if (rc) return rc;
    rc = knn_tc_launch<OpsBF16>(tmq, tmqa, tmx, tmxa, ntr, nq, k, nsplit, lists, flag, st);
    if (rc) return rc;
    k_knn_merge<<<(unsigned)((nq + 127) / 128), 128, 0, st>>>(lists, nsplit * KT_LPQ, labels, nq, k, ncls, out_label,
                                                              out_idx, flag);
    PMX_CHECK_LAUNCH("knn_merge");
    return 0;
}

}  // namespace pmx
