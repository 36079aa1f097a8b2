// Pipe-throughput probes for the rooflines bench.py quotes beside the
// driver-measured HBM / bf16 peaks (MEASURED_PEAKS.json): FP64 add and FMA,
// FP32 FMA, MUFU ex2, shared-memory load bandwidth.  Each kernel runs 8
// independent chains per thread on 8 x 148 CTAs of 256 threads; the rate is
// best-of-5 with CUDA events.  Build + run on the box:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gpurun_out/peaks tools/peaks.cu && gpurun_out/peaks
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096, CH = 8;

__global__ void k_dadd(double* out, double s) {
    double a[CH];
    for (int c = 0; c < CH; ++c) a[c] = threadIdx.x + c;
    for (int i = 0; i < ITERS; ++i)
#pragma unroll
        for (int c = 0; c < CH; ++c) a[c] = __dadd_rn(a[c], s);
    double r = 0;
    for (int c = 0; c < CH; ++c) r += a[c];
    if (r == 1.2345) out[0] = r;
}
__global__ void k_dfma(double* out, double s) {
    double a[CH];
    for (int c = 0; c < CH; ++c) a[c] = threadIdx.x + c;
    for (int i = 0; i < ITERS; ++i)
#pragma unroll
        for (int c = 0; c < CH; ++c) a[c] = __fma_rn(a[c], s, 0.5);
    double r = 0;
    for (int c = 0; c < CH; ++c) r += a[c];
    if (r == 1.2345) out[0] = r;
}
__global__ void k_ffma(double* out, float s) {
    float a[CH];
    for (int c = 0; c < CH; ++c) a[c] = threadIdx.x + c;
    for (int i = 0; i < ITERS; ++i)
#pragma unroll
        for (int c = 0; c < CH; ++c) a[c] = __fmaf_rn(a[c], s, 0.5f);
    float r = 0;
    for (int c = 0; c < CH; ++c) r += a[c];
    if (r == 1.2345f) out[0] = r;
}
__global__ void k_ex2(double* out, float s) {
    float a[CH];
    for (int c = 0; c < CH; ++c) a[c] = (threadIdx.x + c) * 1e-3f;
    for (int i = 0; i < ITERS; ++i)
#pragma unroll
        for (int c = 0; c < CH; ++c) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[c]));
    float r = 0;
    for (int c = 0; c < CH; ++c) r += a[c];
    if (r == 1.2345f) out[0] = r;
}
__global__ void k_lds(double* out, int s) {
    __shared__ float4 buf[2048];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) buf[i] = make_float4(i, i, i, i);
    __syncthreads();
    float4 acc = make_float4(0, 0, 0, 0);
    int idx = threadIdx.x;
    for (int i = 0; i < ITERS / 4; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            const float4 v = buf[(idx + c * 256) & 2047];
            acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
        idx += s;
    }
    if (acc.x + acc.y + acc.z + acc.w == 1.2345f) out[0] = acc.x;
}

// L2 read bandwidth: the grid streams an L2-resident buffer (ld.global.cg,
// 16-B vectors, 4 independent loads per thread per iteration), `passes` times.
__global__ void k_l2(const float4* __restrict__ buf, size_t n4, int passes, double* out) {
    float4 acc = make_float4(0, 0, 0, 0);
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (int p = 0; p < passes; ++p)
        for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i + 3 * stride < n4; i += 4 * stride) {
            const float4 v0 = __ldcg(buf + i), v1 = __ldcg(buf + i + stride);
            const float4 v2 = __ldcg(buf + i + 2 * stride), v3 = __ldcg(buf + i + 3 * stride);
            acc.x += v0.x + v1.x; acc.y += v0.y + v2.y; acc.z += v1.z + v3.z; acc.w += v2.w + v3.w;
        }
    if (acc.x + acc.y + acc.z + acc.w == 1.2345f) out[0] = acc.x;
}

template <class F>
static double best_ms(F launch) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    launch();
    cudaDeviceSynchronize();
    double best = 1e30;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(a);
        launch();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    return best;
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double* out;
    cudaMalloc(&out, 8);
    const int grid = 8 * sms, thr = 256;
    const double lanes_ops = (double)grid * thr * ITERS * CH;
    const double dadd = lanes_ops / (best_ms([&] { k_dadd<<<grid, thr>>>(out, 1e-9); }) * 1e-3);
    const double dfma = lanes_ops / (best_ms([&] { k_dfma<<<grid, thr>>>(out, 0.999); }) * 1e-3);
    const double ffma = lanes_ops / (best_ms([&] { k_ffma<<<grid, thr>>>(out, 0.999f); }) * 1e-3);
    const double ex2 = lanes_ops / (best_ms([&] { k_ex2<<<grid, thr>>>(out, 0.f); }) * 1e-3);
    const double lds = (double)grid * thr * (ITERS / 4) * CH * 16 /
                       (best_ms([&] { k_lds<<<grid, thr>>>(out, 1); }) * 1e-3);
    const size_t l2n4 = (size_t)4 * sms * 512 * 4 * 24;   // 24 iterations per thread: ~58 MiB
    float4* l2buf;
    cudaMalloc(&l2buf, l2n4 * 16);
    cudaMemset(l2buf, 0, l2n4 * 16);
    const double l2 = 8.0 * l2n4 * 16 / (best_ms([&] { k_l2<<<4 * sms, 512>>>(l2buf, l2n4, 8, out); }) * 1e-3);
    const size_t l2s = l2n4 / 4;                           // ~14.5 MiB: inside one die's L2 half
    const double l2small = 32.0 * l2s * 16 / (best_ms([&] { k_l2<<<4 * sms, 512>>>(l2buf, l2s, 32, out); }) * 1e-3);
    const double hz = clk * 1e3;
    printf("{\"sms\": %d, \"clock_mhz_attr\": %.0f, "
           "\"fp64_add_ops_per_s\": %.4e, \"fp64_fma_flops_per_s\": %.4e, \"fp32_fma_flops_per_s\": %.4e, "
           "\"mufu_ex2_per_s\": %.4e, \"smem_load_bytes_per_s\": %.4e, \"l2_read_bytes_per_s\": %.4e, \"l2_read_bytes_per_s_14MiB\": %.4e, "
           "\"per_sm_per_clk_at_attr_clock\": {\"fp64_add\": %.1f, \"fp64_fma\": %.1f, \"fp32_fma\": %.1f, "
           "\"mufu_ex2\": %.1f, \"smem_load_B\": %.1f}}\n",
           sms, hz / 1e6, dadd, 2 * dfma, 2 * ffma, ex2, lds, l2, l2small, dadd / sms / hz, dfma / sms / hz, ffma / sms / hz,
           ex2 / sms / hz, lds / sms / hz);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { fprintf(stderr, "%s\n", cudaGetErrorString(e)); return 1; }
    return 0;
}
