// TMEM -> register read-bandwidth probe (the k-NN epilogue's candidate bound).
// One CTA per SM allocates all 512 TMEM columns; W warps each read their lane
// quadrant (warp % 4) with tcgen05.ld in a loop and fold the words into a sink
// so nothing is dead.  Reports bytes per SM clock for each shape / warp count /
// loads-in-flight, with and without a per-word min (the k-NN scan's ALU work).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2211_00621_b200/csrc -lcuda \
//        -o /tmp/tmem_probe tools/tmem_probe.cu && /tmp/tmem_probe
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <cstring>
#include "tc.cuh"

using namespace pmx;

constexpr int ITER = 8192;

__device__ __forceinline__ void ld_16x256b_x16(uint32_t taddr, uint32_t (&r)[64]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.16x256b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,"
        "%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,"
        "%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]),
          "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]),
          "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]),
          "=r"(r[48]), "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]),
          "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
        : "r"(taddr));
}

#define PMX_LD64(SHAPE_STR)                                                                          \
    asm volatile(                                                                                    \
        "tcgen05.ld.sync.aligned." SHAPE_STR ".b32 "                                                 \
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"                                    \
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,"                           \
        "%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,"                           \
        "%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"                   \
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), \
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),     \
          "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),   \
          "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),   \
          "=r"(r[29]), "=r"(r[30]), "=r"(r[31]), "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]),   \
          "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]), "=r"(r[40]), "=r"(r[41]), "=r"(r[42]),   \
          "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]), "=r"(r[48]), "=r"(r[49]),   \
          "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]), "=r"(r[56]),   \
          "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])    \
        : "r"(taddr))
__device__ __forceinline__ void ld_16x64b_x64(uint32_t taddr, uint32_t (&r)[64]) { PMX_LD64("16x64b.x64"); }
__device__ __forceinline__ void ld_16x128b_x32(uint32_t taddr, uint32_t (&r)[64]) { PMX_LD64("16x128b.x32"); }

// SHAPE 0: 32x32b.x64 (8 KiB per warp-load, 64 columns), 1: 32x32b.x32 (4 KiB),
// 2: 16x256b.x16, 3: 16x128b.x32, 4: 16x64b.x64 (8 KiB each over 16 lanes x 128 columns)
// INFL: loads issued before one wait (1 or 2; 2 needs 128 registers)
// WORK: 0 = xor fold, 1 = float min over each word (the k-NN scan)
template <int SHAPE, int INFL, int WORK>
__global__ void k_tmem(uint32_t* sink, long long* clk) {
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) tc::tmem_alloc(&tbase, 512);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = tbase;
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    const int nw4 = (blockDim.x >> 5) >> 2;
    constexpr uint32_t span = SHAPE >= 2 ? 128u : 64u;           // columns one load covers
    const uint32_t col0 = (uint32_t)(((warp >> 2) * span) & 511);
    uint32_t acc = 0;
    float m = 3.0e38f;
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < ITER; ++it) {
        const uint32_t col = (col0 + (uint32_t)(it * nw4) * span) & 511u;
        if (SHAPE == 1) {
            uint32_t r[32];
            tc::tmem_ld_32x32b_x32(tmem + lane_base + col, r);
            tc::tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                if (WORK) m = fminf(m, __uint_as_float(r[j])); else acc ^= r[j];
            }
        } else {
            uint32_t r[INFL][64];
#pragma unroll
            for (int f = 0; f < INFL; ++f) {
                const uint32_t c = (col + (uint32_t)f * span) & 511u;
                if (SHAPE == 0) tc::tmem_ld_32x32b_x64(tmem + lane_base + c, r[f]);
                else if (SHAPE == 2) ld_16x256b_x16(tmem + lane_base + c, r[f]);
                else if (SHAPE == 3) ld_16x128b_x32(tmem + lane_base + c, r[f]);
                else ld_16x64b_x64(tmem + lane_base + c, r[f]);
            }
            tc::tmem_ld_wait();
#pragma unroll
            for (int f = 0; f < INFL; ++f)
#pragma unroll
                for (int j = 0; j < 64; ++j) {
                    if (WORK) m = fminf(m, __uint_as_float(r[f][j])); else acc ^= r[f][j];
                }
        }
    }
    const long long t1 = clock64();
    if (acc == 0x12345678u || m == 1.2345f) sink[blockIdx.x] = acc;
    if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
    tc::tc_fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tmem, 512);
}

// Layout check for a 16-bit (F16) accumulator: one M=128 N=128 K=16 UMMA with
// fp16 A = 1 and B row p = p, so D[q][p] = 16 p (an F16 accumulator needs fp16
// operands; bf16 ones require F32).  Lane 0's 128 TMEM words tell
// whether two 16-bit results share a 32-bit column (packed) or not.
__global__ void k_f16acc_layout(uint32_t* out) {
    __shared__ __align__(1024) __half A[128 * 64];
    __shared__ __align__(1024) __half B[128 * 64];
    __shared__ uint64_t done;
    __shared__ uint32_t tbase;
    for (int i = threadIdx.x; i < 128 * 64; i += blockDim.x) {
        A[i] = __float2half_rn(1.f);
        B[i] = __float2half_rn((float)(i / 64));
    }
    if (threadIdx.x == 0) { tc::mbar_init(&done, 1); tc::fence_mbar_init(); }
    if ((threadIdx.x >> 5) == 0) tc::tmem_alloc(&tbase, 512);
    tc::fence_proxy_async();
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = tbase;
    if (threadIdx.x == 0) {
        constexpr uint32_t idesc = ((128u >> 3) << 17) | ((128u >> 4) << 24);  // c = F16, a = b = F16
        tc::umma_f16(tmem, tc::sw128_kmajor_desc(tc::smem_u32(A)), tc::sw128_kmajor_desc(tc::smem_u32(B)), idesc, 0);
        tc::umma_commit(&done);
    }
    __syncwarp();
    tc::mbar_wait(&done, 0);
    tc::tc_fence_after();
    if ((threadIdx.x >> 5) == 0) {
        uint32_t r[64];
        tc::tmem_ld_32x32b_x64(tmem, r);
        tc::tmem_ld_wait();
        uint32_t r2[64];
        tc::tmem_ld_32x32b_x64(tmem + 64, r2);
        tc::tmem_ld_wait();
        if (threadIdx.x == 0)
            for (int j = 0; j < 64; ++j) { out[j] = r[j]; out[64 + j] = r2[j]; }
    }
    tc::tc_fence_before();
    __syncthreads();
    if ((threadIdx.x >> 5) == 0) tc::tmem_dealloc(tmem, 512);
}

static void f16acc_layout() {
    uint32_t* d;
    cudaMalloc(&d, 128 * 4);
    cudaMemset(d, 0, 128 * 4);
    k_f16acc_layout<<<1, 128>>>(d);
    uint32_t h[128];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("{\"f16_accumulator_lane0_words\": [");
    for (int j = 0; j < 128; ++j) printf("%s\"%08x\"", j ? ", " : "", h[j]);
    printf("], \"err\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
}

// .pack::16b check: store 32-bit words (column c of lane l = 0x4b000000 | (l << 8 | c))
// with tcgen05.st, read back with 32x32b.x32.pack::16b (64 columns into 32
// registers) and print lane 0's registers: expected pairs of low halves.
__global__ void k_pack16_layout(uint32_t* out) {
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) tc::tmem_alloc(&tbase, 512);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = tbase;
    if (warp == 0) {
        for (int c = 0; c < 64; ++c) {
            const uint32_t v = 0x4b000000u | ((uint32_t)lane << 8) | (uint32_t)c;
            asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" :: "r"(tmem + (uint32_t)c), "r"(v) : "memory");
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        uint32_t r[32];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.pack::16b.b32 "
            "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
              "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
              "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
            : "r"(tmem));
        tc::tmem_ld_wait();
        if (lane == 0 || lane == 5)
            for (int j = 0; j < 32; ++j) out[(lane ? 32 : 0) + j] = r[j];
    }
    tc::tc_fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tmem, 512);
}

static void pack16_layout() {
    uint32_t* d;
    cudaMalloc(&d, 64 * 4);
    cudaMemset(d, 0, 64 * 4);
    k_pack16_layout<<<1, 128>>>(d);
    uint32_t h[64];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("{\"pack16b_lane0\": [");
    for (int j = 0; j < 32; ++j) printf("%s\"%08x\"", j ? ", " : "", h[j]);
    printf("], \"pack16b_lane5\": [");
    for (int j = 0; j < 32; ++j) printf("%s\"%08x\"", j ? ", " : "", h[32 + j]);
    printf("], \"err\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
}

// 3-input packed 16-bit min, if the toolchain has it
__global__ void k_min3_u16x2(const uint32_t* a, uint32_t* o) {
    uint32_t r;
    asm("min.u16x2 %0, %1, %2;" : "=r"(r) : "r"(a[0]), "r"(a[1]));
    o[0] = r;
}

template <int SHAPE, int INFL, int WORK>
static void run(int sms, int warps, const char* name) {
    uint32_t* sink;
    long long* clk;
    cudaMalloc(&sink, sms * 4);
    cudaMalloc(&clk, sms * 8);
    k_tmem<SHAPE, INFL, WORK><<<sms, warps * 32>>>(sink, clk);
    cudaDeviceSynchronize();
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k_tmem<SHAPE, INFL, WORK><<<sms, warps * 32>>>(sink, clk);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    long long h[1024];
    cudaMemcpy(h, clk, sms * 8, cudaMemcpyDeviceToHost);
    double cmax = 0;
    for (int i = 0; i < sms; ++i) cmax = h[i] > cmax ? (double)h[i] : cmax;
    const int words = SHAPE == 1 ? 32 : 64 * INFL;
    const double bytes_sm = (double)warps * ITER * 32.0 * words * 4.0;
    const cudaError_t e = cudaGetLastError();
    printf("{\"shape\": \"%s\", \"warps\": %d, \"loads_in_flight\": %d, \"work\": \"%s\", \"B_per_clk_per_SM\": %.1f, "
           "\"TB_per_s_chip\": %.2f, \"err\": \"%s\"}\n",
           name, warps, INFL, WORK ? "fmin" : "xor", bytes_sm / cmax, bytes_sm * sms / (ms * 1e-3) / 1e12,
           cudaGetErrorString(e));
    cudaFree(sink);
    cudaFree(clk);
}

int main(int argc, char** argv) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    if (argc > 1 && !strcmp(argv[1], "layout")) { f16acc_layout(); pack16_layout(); return 0; }
    for (int w : {4, 8, 16}) {
        run<0, 1, 0>(sms, w, "32x32b.x64");
        run<0, 2, 0>(sms, w, "32x32b.x64");
        run<1, 1, 0>(sms, w, "32x32b.x32");
        run<2, 1, 0>(sms, w, "16x256b.x16");
        run<3, 1, 0>(sms, w, "16x128b.x32");
        run<4, 1, 0>(sms, w, "16x64b.x64");
        run<2, 2, 0>(sms, w, "16x256b.x16");
        run<0, 1, 1>(sms, w, "32x32b.x64");
    }
    return 0;
}
