// DSMEM exchange probe for the k-mer pair kernel: two CTAs of a cluster swap
// 32 KiB per round (double-buffered slots, one mbarrier per slot), 512 threads,
// all 74 clusters at once.  Modes:
//   0  st.async 16 B per thread-store, complete_tx on the peer's barrier
//   1  threads store their 64 B locally, __syncthreads, one thread issues a
//      bulk copy shared::cta -> shared::cluster (2 x 16 KiB) completing on the peer
//   2  plain remote stores (st.shared::cluster.v4) + per-thread remote arrive (release.cluster)
//   3  st.async, as 0, but 8 B per store (v2)
// Reports SM clocks per round (round trip of a full exchange, no compute).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2211_00621_b200/csrc \
//        -o /tmp/dsmem_probe tools/dsmem_probe.cu && /tmp/dsmem_probe
#include <cstdio>
#include <cuda_runtime.h>
#include "tc.cuh"

using namespace pmx;

constexpr int THREADS = 512, BYTES = 32768, ROUNDS = 2000;

struct Smem {
    float4 slot[2][BYTES / 16];
    float4 stage[BYTES / 16];
    uint64_t bar[2];
};

__device__ __forceinline__ void st_async_v4(uint32_t a, float4 v, uint32_t bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1,%2,%3,%4}, [%5];"
                 :: "r"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "r"(bar) : "memory");
}
__device__ __forceinline__ void st_async_v2(uint32_t a, float x, float y, uint32_t bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f32 [%0], {%1,%2}, [%3];"
                 :: "r"(a), "f"(x), "f"(y), "r"(bar) : "memory");
}
__device__ __forceinline__ void expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" :: "r"(tc::smem_u32(bar)), "r"(bytes)
                 : "memory");
}

template <int MODE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1) k_probe(long long* out, float* sink) {
    extern __shared__ __align__(16) uint8_t raw[];
    Smem& sm = *reinterpret_cast<Smem*>(raw);
    const uint32_t rank = tc::cluster_ctarank(), peer = rank ^ 1u;
    const int tid = threadIdx.x;
    if (tid == 0) {
        tc::mbar_init(&sm.bar[0], MODE == 2 ? THREADS : 1);
        tc::mbar_init(&sm.bar[1], MODE == 2 ? THREADS : 1);
        if (MODE != 2) {
            expect_tx(&sm.bar[0], BYTES);
            expect_tx(&sm.bar[1], BYTES);
        }
        tc::fence_mbar_init();
    }
    tc::cluster_sync();
    const uint32_t slot_peer = tc::mapa(tc::smem_u32(&sm.slot[0][0]), peer);
    const uint32_t bar_peer = tc::mapa(tc::smem_u32(&sm.bar[0]), peer);
    float4 v = make_float4(tid, rank, 1.f, 2.f);
    float acc = 0.f;
    long long t0 = 0;
    for (int r = 0; r < ROUNDS; ++r) {
        if (r == 16) t0 = clock64();
        const uint32_t s = r & 1;
        if (MODE == 0) {
#pragma unroll
            for (int k = 0; k < 4; ++k)
                st_async_v4(slot_peer + s * BYTES + 16u * (k * THREADS + tid), v, bar_peer + 8u * s);
        } else if (MODE == 3) {
#pragma unroll
            for (int k = 0; k < 8; ++k)
                st_async_v2(slot_peer + s * BYTES + 8u * (k * THREADS + tid), v.x, v.y, bar_peer + 8u * s);
        } else if (MODE == 1) {
#pragma unroll
            for (int k = 0; k < 4; ++k) sm.stage[k * THREADS + tid] = v;
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncthreads();
            if (tid == 0) {
                for (int h = 0; h < 2; ++h)
                    asm volatile(
                        "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                        :: "r"(slot_peer + s * BYTES + h * (BYTES / 2)),
                           "r"(tc::smem_u32(&sm.stage[0]) + h * (BYTES / 2)), "n"(BYTES / 2),
                           "r"(bar_peer + 8u * s) : "memory");
                asm volatile("cp.async.bulk.commit_group;\n\tcp.async.bulk.wait_group.read 0;" ::: "memory");
            }
            __syncthreads();
        } else {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint32_t a = slot_peer + s * BYTES + 16u * (k * THREADS + tid);
                asm volatile("st.shared::cluster.v4.f32 [%0], {%1,%2,%3,%4};" :: "r"(a), "f"(v.x), "f"(v.y),
                             "f"(v.z), "f"(v.w) : "memory");
            }
            tc::arrive_remote(bar_peer + 8u * s);
        }
        if (MODE != 2 && tid == 0) tc::mbar_arrive(&sm.bar[s]);   // the one local arrival
        tc::mbar_wait(&sm.bar[s], (r >> 1) & 1);
        if (MODE != 2 && tid == 0) expect_tx(&sm.bar[s], BYTES);  // re-arm for round r + 2
        const float4 w = sm.slot[s][tid];
        acc += w.x;
        v.x += 1.f;
    }
    const long long t1 = clock64();
    if (tid == 0) out[blockIdx.x] = (t1 - t0) / (ROUNDS - 16);
    if (acc == -1.f) *sink = acc;
    tc::cluster_sync();
}

template <int MODE>
void run(const char* name) {
    const int grid = 148;
    long long* d;
    float* sink;
    cudaMalloc(&d, grid * sizeof(long long));
    cudaMalloc(&sink, 4);
    cudaFuncSetAttribute(k_probe<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Smem));
    for (int g : {2, grid}) {
        k_probe<MODE><<<g, THREADS, sizeof(Smem)>>>(d, sink);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); return; }
        long long h[148];
        cudaMemcpy(h, d, g * sizeof(long long), cudaMemcpyDeviceToHost);
        double m = 0;
        for (int i = 0; i < g; ++i) m += h[i];
        m /= g;
        printf("%-44s clusters %3d: %7.0f clk per 32 KiB round (%5.1f B/clk/SM each way)\n", name, g / 2, m,
               BYTES / m);
    }
    cudaFree(d);
}

int main() {
    run<0>("st.async v4 (complete_tx)");
    run<3>("st.async v2 (complete_tx)");
    run<1>("local STS + bulk copy 2 x 16 KiB");
    run<2>("st.shared::cluster v4 + remote arrive");
    return 0;
}
