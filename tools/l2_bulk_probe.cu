// L2 -> SM ingress probe with TMA bulk copies (cp.async.bulk global -> shared):
// one CTA per SM, one thread keeps a ring of 32 KiB copies in flight (no
// register or LSU limits), the data is never read.  Two sources:
//   table : every CTA streams the same 2 MiB table (the k-mer emission rows /
//           the HMM's A^T: L2-resident, shared by all SMs)
//   slice : every CTA streams its own 512 KiB slice of a 74 MiB buffer
// Reports bytes per second over all SMs and bytes per clock per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2211_00621_b200/csrc \
//        -o /tmp/l2_bulk_probe tools/l2_bulk_probe.cu && /tmp/l2_bulk_probe
#include <cstdio>
#include <cuda_runtime.h>
#include "tc.cuh"

using namespace pmx;

constexpr int CHUNK = 32768;

template <int STAGES>
__global__ void __launch_bounds__(32, 1) k_bulk(const uint8_t* __restrict__ src, size_t span, size_t cta_stride,
                                                int iters, long long* clk) {
    extern __shared__ __align__(128) uint8_t sm[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + STAGES * CHUNK);
    if (threadIdx.x != 0) return;
    for (int s = 0; s < STAGES; ++s) tc::mbar_init(&bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const uint8_t* base = src + (size_t)blockIdx.x * cta_stride;
    const size_t nchunks = span / CHUNK;
    const long long t0 = clock64();
    size_t c = blockIdx.x % nchunks;
    for (int s = 0; s < STAGES; ++s) {
        tc::mbar_arrive_expect_tx(&bar[s], CHUNK);
        tc::bulk_load_1d(sm + s * CHUNK, base + c * CHUNK, CHUNK, &bar[s]);
        c = c + 1 == nchunks ? 0 : c + 1;
    }
    for (int i = STAGES; i < iters; ++i) {
        const int s = i % STAGES;
        tc::mbar_wait(&bar[s], (uint32_t)((i / STAGES - 1) & 1));
        tc::mbar_arrive_expect_tx(&bar[s], CHUNK);
        tc::bulk_load_1d(sm + s * CHUNK, base + c * CHUNK, CHUNK, &bar[s]);
        c = c + 1 == nchunks ? 0 : c + 1;
    }
    for (int i = iters; i < iters + STAGES; ++i) tc::mbar_wait(&bar[i % STAGES], (uint32_t)((i / STAGES - 1) & 1));
    clk[blockIdx.x] = clock64() - t0;
}

template <int STAGES>
void run(const char* name, const uint8_t* src, size_t span, size_t cta_stride, int sms) {
    const int iters = 4096;
    const size_t smem = STAGES * CHUNK + STAGES * 8;
    cudaFuncSetAttribute(k_bulk<STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    long long* dclk;
    cudaMalloc(&dclk, sms * sizeof(long long));
    k_bulk<STAGES><<<sms, 32, smem>>>(src, span, cta_stride, 64, dclk);   // warm the L2
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k_bulk<STAGES><<<sms, 32, smem>>>(src, span, cta_stride, iters, dclk);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    long long h[148];
    cudaMemcpy(h, dclk, sms * sizeof(long long), cudaMemcpyDeviceToHost);
    double mclk = 0;
    for (int i = 0; i < sms; ++i) mclk += h[i];
    mclk /= sms;
    const double bytes = (double)iters * CHUNK * sms;
    printf("%-6s %d stages x 32 KiB: %7.2f TB/s over %d SMs, %6.1f B/clk/SM\n", name, STAGES,
           bytes / (ms * 1e-3) / 1e12, sms, (double)iters * CHUNK / mclk);
    cudaFree(dclk);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint8_t* buf;
    const size_t big = (size_t)148 * 512 * 1024;
    cudaMalloc(&buf, big);
    cudaMemset(buf, 1, big);
    run<4>("table", buf, 2u << 20, 0, sms);
    run<6>("table", buf, 2u << 20, 0, sms);
    run<4>("slice", buf, 512u << 10, 512u << 10, sms);
    run<6>("slice", buf, 512u << 10, 512u << 10, sms);
    return 0;
}
