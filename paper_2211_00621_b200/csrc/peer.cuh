// Cross-GPU combine of reduce partials over NVLink peer memory, fused into
// the reduce kernel's last CTA (no NCCL call on the data path).
//
// The reference folds its per-chunk partials left to right in chunk order
// (pmx/interp.py:334-336) after dropping empty chunks (:276). Across GPUs the
// chunks are the ranks' shards (`_chunks(n, world)`), so after a rank's last
// CTA has its shard's partial it:
//   1. stores (value, flag) into slot [parity][rank] of EVERY rank's mailbox
//      (peer mailboxes are cudaIpc-mapped; one lane per destination), the flag
//      with st.release.sys after the value;
//   2. polls its own mailbox slots [parity][0..world) with ld.acquire.sys until
//      every flag carries this launch's epoch;
//   3. folds the non-empty partials in rank order.
// Every rank ends with the same total, in one kernel. The parity of the epoch
// double-buffers the slots: a rank can run at most one launch ahead of a peer
// (it needs that peer's partial of the current epoch to finish), so the slot
// it writes for epoch e+1 is never the one the peer is still reading for e.
#pragma once
#include "device_common.cuh"

namespace pmx {

// flag word = epoch << 1 | has (has = 0: this rank's shard was empty)
__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_sys(uint64_t* p, uint64_t v) {
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_relaxed_sys(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint64_t globaltimer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ uint64_t bits_of(double v) { return (uint64_t)__double_as_longlong(v); }
__device__ __forceinline__ uint64_t bits_of(int64_t v) { return (uint64_t)v; }
template <class A> __device__ __forceinline__ A from_bits(uint64_t b);
template <> __device__ __forceinline__ double from_bits<double>(uint64_t b) { return __longlong_as_double((long long)b); }
template <> __device__ __forceinline__ int64_t from_bits<int64_t>(uint64_t b) { return (int64_t)b; }

__device__ __forceinline__ uint64_t* mbox_slot(uint64_t* mbox, uint64_t epoch, int src) {
    return mbox + ((int)(epoch & 1) * PMX_MAX_PEERS + src) * 2;
}

// Executed by one full warp. `local` is this rank's partial (bits of a 64-bit
// value), `has` whether its shard was non-empty. Returns the rank-ordered fold
// of the non-empty partials (valid in every lane) and sets *ok = false on a
// peer timeout (error word PMX_E_PEER_TIMEOUT).
template <class A, class Fold>
__device__ A peer_exchange(const pmx_peer_group& g, A local, int has, Fold fold, A empty, uint64_t* err,
                           bool* ok, int* any_out) {
    const int lane = threadIdx.x & 31;
    const uint64_t bits = bits_of(local);
    const uint64_t flag = (g.epoch << 1) | (uint64_t)(has != 0);
    if (lane < g.world) {
        uint64_t* s = mbox_slot(g.mbox[lane], g.epoch, g.rank);
        st_relaxed_sys(s, bits);
        st_release_sys(s + 1, flag);
    }
    uint64_t got = 0, f = 0;
    int timed_out = 0;
    if (lane < g.world) {
        const uint64_t* s = mbox_slot(g.mbox[g.rank], g.epoch, lane);
        const uint64_t t0 = globaltimer_ns();
        while (((f = ld_acquire_sys(s + 1)) >> 1) != g.epoch) {
            if (globaltimer_ns() - t0 > 20ull * 1000 * 1000 * 1000) { timed_out = 1; break; }
            __nanosleep(64);
        }
        got = ld_relaxed_sys(s);
    }
    timed_out = __any_sync(0xffffffffu, timed_out);
    *ok = !timed_out;
    *any_out = 0;
    if (timed_out) {
        if (lane == 0) raise_err(err, 0, PMX_E_PEER_TIMEOUT);
        return empty;
    }
    A total = empty;
    int any = 0;
    for (int r = 0; r < g.world; ++r) {
        uint64_t vb = __shfl_sync(0xffffffffu, got, r);
        uint64_t fb = __shfl_sync(0xffffffffu, f, r);
        if (!(fb & 1)) continue;               // empty chunk: dropped (interp.py:276)
        const A v = from_bits<A>(vb);
        total = any ? fold(total, v) : v;
        any = 1;
    }
    *any_out = any;
    return total;
}

}  // namespace pmx
