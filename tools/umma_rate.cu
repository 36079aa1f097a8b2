// UMMA issue-rate probe: one CTA per SM issues back-to-back tcgen05.mma
// kind::f16 (M = 128, N in {32, 64, 128, 256}, K = 16, A and B from shared
// memory, fp32 accumulation in TMEM) and reports TFLOP/s — the ceiling the HMM
// pair kernel's UMMA shape (M = 128, N = 64) can reach.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2211_00621_b200/csrc -lcuda \
//        -o gpurun_out/umma_rate tools/umma_rate.cu && gpurun_out/umma_rate
#include <cstdio>
#include <cuda_runtime.h>
#include "tc.cuh"

using namespace pmx;

constexpr int ITER = 4096;

template <int N, bool I8>
__global__ void __launch_bounds__(128, 1) k_umma(int* sink) {
    extern __shared__ uint8_t raw[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    uint8_t* A = base;                         // 4 stages x 128 x 64 fp16 (16 KiB each)
    uint8_t* B = base + 4 * 16384;             // N x 64 fp16
    __shared__ uint64_t done;
    __shared__ uint32_t tbase;
    for (int i = threadIdx.x; i < (4 * 16384 + N * 128) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(base)[i] = 0;
    if (threadIdx.x == 0) { tc::mbar_init(&done, 1); tc::fence_mbar_init(); }
    if ((threadIdx.x >> 5) == 0) tc::tmem_alloc(&tbase, 512);
    tc::fence_proxy_async();
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = tbase;
    if (threadIdx.x == 0) {
        // kind::f16 (fp16, K = 16 per UMMA) or kind::i8 (signed int8, int32 accumulate, K = 32)
        constexpr uint32_t idesc = I8 ? ((2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24))
                                      : tc::instr_desc(128, N, 0);
        const uint64_t bd = tc::sw128_kmajor_desc(tc::smem_u32(B));
        for (int it = 0; it < ITER; ++it) {
            const uint64_t ad = tc::sw128_kmajor_desc(tc::smem_u32(A + (it & 3) * 16384));
            const uint32_t d = tmem + (uint32_t)((it & 1) * 256);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                if (I8) tc::umma_i8(d, ad + 2 * kk, bd + 2 * kk, idesc, kk != 0);
                else tc::umma_f16(d, ad + 2 * kk, bd + 2 * kk, idesc, kk != 0);
            }
        }
        tc::umma_commit(&done);
    }
    __syncwarp();
    tc::mbar_wait(&done, 0);
    tc::tc_fence_after();
    __syncthreads();
    if ((threadIdx.x >> 5) == 0) tc::tmem_dealloc(tmem, 512);
    if (threadIdx.x == 0 && tmem == 12345u) *sink = 1;
}

template <int N, bool I8 = false>
static void run(int sms) {
    const size_t smem = 4 * 16384 + N * 128 + 2048;
    cudaFuncSetAttribute(k_umma<N, I8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int* sink;
    cudaMalloc(&sink, 4);
    k_umma<N, I8><<<sms, 128, smem>>>(sink);
    cudaDeviceSynchronize();
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(a);
        k_umma<N, I8><<<sms, 128, smem>>>(sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    const int K = I8 ? 32 : 16;
    const double flop = (double)sms * ITER * 4 * 2.0 * 128 * N * K;
    printf("{\"kind\": \"%s\", \"M\": 128, \"N\": %d, \"K\": %d, \"tflops\": %.1f, \"ms\": %.4f, \"err\": \"%s\"}\n",
           I8 ? "i8" : "f16", N, K, flop / (best * 1e-3) / 1e12, best, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<32>(sms);
    run<64>(sms);
    run<128>(sms);
    run<256>(sms);
    run<64, true>(sms);
    run<80, true>(sms);
    run<96, true>(sms);
    run<112, true>(sms);
    run<128, true>(sms);
    run<256, true>(sms);
    return 0;
}
