// Softmax-regression loss and analytic gradients: the reference's NN case
// study (programs/nn.pmx:22-49; oracle tests/test_acceptance.py:399-441),
// fused into one kernel over the points.
//
// Reference, per point p (all fp64, CPython rounding of each op):
//   z_j   = foldl (acc + x_i * w_ij) b_j over i = 0..nin-1        (:24-27)
//   total = reduce addf 0.0 (map exp z)   -- sequential inside a map (:30)
//   loss_p = log total - z_y                                       (:31)
//   dz_j  = exp z_j / total - [j == y]                            (:34-38)
// and over points: loss = (sum_p loss_p) / n, dw_ij = (sum_p x_pi dz_pj) / n,
// db_j = (sum_p dz_pj) / n (:40-48).  z, total, loss_p and dz are evaluated in
// the reference's order (bit-identical up to CUDA vs glibc exp/log, <= 2 ulp);
// the three sums over points are the reference's top-level reduces, whose
// order depends on its worker count — here a fixed tree (per-warp sequential,
// warps and CTAs folded in index order), deterministic run to run.
//
// B200 design: points in tiles of 64 staged in shared memory (x is the only
// HBM stream, 8 * nin bytes per point, read once); phase 1 runs the z chains
// with lane j = class j and PT points per thread (independent sequential
// chains hide the fp64 latency), softmax through lane-group shuffles, dz to
// shared memory; phase 2 accumulates x^T dz into per-thread (i, j) registers.
// Per-CTA partials go to the workspace and the last CTA folds them in CTA
// order (one launch).
#include "common.cuh"

namespace pmx {

constexpr int NN_THREADS = 256;
constexpr int NN_MAXIN = 64;
constexpr int NN_MAXOUT = 32;
constexpr int NN_TILE = 64;          // points per tile (x tile 64 x 64 fp64 = 32 KiB)
constexpr int NN_PAIRS = 8;          // (i, j) dw accumulators per thread (nin*nout <= 2048)

// Thread layout for the per-point phase: lane group of CW = next pow2 >= nout
// (>= 4) lanes per point (lane j = class j), NP = 256 / CW point rows, each thread
// runs PT = NN_TILE / NP points (independent fp64 chains: ILP for the
// sequential foldl of z).  Per-(i,j) dw accumulators live in registers of the
// gradient phase (thread t owns pairs t, t + 256, ...).
template <int CW>
__global__ void __launch_bounds__(NN_THREADS)
k_nn_grad(const double* __restrict__ x, const int* __restrict__ y, const double* __restrict__ w,
          const double* __restrict__ b, int64_t npts, int nin, int nout, double* __restrict__ partials,
          unsigned* ticket, double* __restrict__ loss_out, double* __restrict__ dw_out,
          double* __restrict__ db_out, uint64_t* err) {
    constexpr int NP = NN_THREADS / CW;
    constexpr int PT = NN_TILE / NP > 0 ? NN_TILE / NP : 1;
    constexpr int TILE = NP * PT;
    static_assert(TILE == NN_TILE, "tile");
    extern __shared__ double nsm[];
    double* ws = nsm;                                  // [NN_MAXIN * NN_MAXOUT]
    double* xs = ws + NN_MAXIN * NN_MAXOUT;            // [TILE * nin]
    double* dzs = xs + TILE * NN_MAXIN;                // [TILE * NN_MAXOUT]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int j = tid % CW, row = tid / CW;
    const bool act = j < nout;
    const int npairs = nin * nout;
    for (int v = tid; v < npairs; v += NN_THREADS) ws[v] = w[v];
    const double bj = act ? b[j] : 0.0;
    double dwacc[NN_PAIRS];
#pragma unroll
    for (int k = 0; k < NN_PAIRS; ++k) dwacc[k] = 0.0;
    double dbacc = 0.0, lossacc = 0.0;
    const int64_t ntiles = (npts + TILE - 1) / TILE;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t p0 = tile * TILE;
        const int npt = (int)(npts - p0 < TILE ? npts - p0 : TILE);
        __syncthreads();                                   // previous tile's xs / dzs reads done
        const double* xt = x + p0 * nin;
        for (int v = tid; v < npt * nin; v += NN_THREADS) xs[v] = __ldcs(xt + v);   // coalesced stream
        if (npt < TILE)                                    // tail tile: zero the unused rows
            for (int v = npt * nin + tid; v < TILE * nin; v += NN_THREADS) xs[v] = 0.0;
        __syncthreads();
        // ---- per point: z (reference foldl order), softmax, loss, dz
        double z[PT];
#pragma unroll
        for (int k = 0; k < PT; ++k) z[k] = bj;
        // rows past the tile end hold zeros and are never used
        const double* xr = xs + row * nin;
        const double* wc = ws + (act ? j : 0);             // w[i][j]: lanes j contiguous
        int i = 0;
        if ((nin & 1) == 0) {                               // x as 16-byte pairs over i
#pragma unroll 4
            for (; i < nin; i += 2) {
                const double w0 = wc[i * nout], w1 = wc[(i + 1) * nout];
#pragma unroll
                for (int k = 0; k < PT; ++k) {
                    const double2 x2 = *reinterpret_cast<const double2*>(xr + k * NP * nin + i);
                    z[k] = __dadd_rn(z[k], __dmul_rn(x2.x, w0));
                    z[k] = __dadd_rn(z[k], __dmul_rn(x2.y, w1));
                }
            }
        }
        for (; i < nin; ++i) {
            const double wij = wc[i * nout];
#pragma unroll
            for (int k = 0; k < PT; ++k) z[k] = __dadd_rn(z[k], __dmul_rn(xr[k * NP * nin + i], wij));
        }
#pragma unroll
        for (int k = 0; k < PT; ++k) {
            const int pl = row + k * NP;
            const bool live = pl < npt;
            const double e = act ? exp(z[k]) : 0.0;
            int code = (live && act && is_inf(e) && !is_inf(z[k])) ? PMX_E_EXP_RANGE : 0;
            double total = 0.0;                            // left fold over classes
            const int base = lane & ~(CW - 1);
            for (int c = 0; c < nout; ++c) total = __dadd_rn(total, __shfl_sync(0xffffffffu, e, base + c));
            const int yp = live ? __ldg(y + p0 + pl) : 0;
            if (live && (yp < 0 || yp >= nout) && !code) code = PMX_E_OOB;
            const int ys_ = (yp >= 0 && yp < nout) ? yp : 0;
            const double zy = __shfl_sync(0xffffffffu, z[k], base + ys_);
            if (code && j == 0) raise_err(err, p0 + pl, code);
            double dz = __ddiv_rn(e, total);
            if (j == yp) dz = __dsub_rn(dz, 1.0);
            if (live && act) {
                dzs[pl * NN_MAXOUT + j] = dz;
                dbacc = __dadd_rn(dbacc, dz);
            }
            if (live && j == 0) lossacc = __dadd_rn(lossacc, __dsub_rn(log(total), zy));
        }
        __syncthreads();
        // ---- dw partials: pair (i, jj) = t + 256 q, sequential over the tile's points
#pragma unroll
        for (int q = 0; q < NN_PAIRS; ++q) {
            const int pr = tid + q * NN_THREADS;
            if (pr < npairs) {
                const int ii = pr / nout, jj = pr % nout;
                // two partial chains (even / odd points) halve the dependent-add
                // depth; folded in order at the end of the tile
                double a0 = 0.0, a1 = 0.0;
                const double* xc = xs + ii;
                const double* dc = dzs + jj;
                int pl = 0;
#pragma unroll 4
                for (; pl + 1 < npt; pl += 2) {
                    a0 = __dadd_rn(a0, __dmul_rn(xc[pl * nin], dc[pl * NN_MAXOUT]));
                    a1 = __dadd_rn(a1, __dmul_rn(xc[(pl + 1) * nin], dc[(pl + 1) * NN_MAXOUT]));
                }
                if (pl < npt) a0 = __dadd_rn(a0, __dmul_rn(xc[pl * nin], dc[pl * NN_MAXOUT]));
                dwacc[q] = __dadd_rn(dwacc[q], __dadd_rn(a0, a1));
            }
        }
    }
    // ---- CTA partial: dw (per thread), db and loss (fold the point rows in order)
    double* part = partials + (int64_t)blockIdx.x * (npairs + nout + 1);
#pragma unroll
    for (int q = 0; q < NN_PAIRS; ++q) {
        const int pr = tid + q * NN_THREADS;
        if (pr < npairs) part[pr] = dwacc[q];
    }
    __shared__ double rowsum[NP][NN_MAXOUT + 1];
    if (act) rowsum[row][j] = dbacc;
    if (j == 0) rowsum[row][NN_MAXOUT] = lossacc;
    __syncthreads();
    if (tid < nout || tid == NN_MAXOUT) {
        const int c = tid;
        double s = rowsum[0][c];
        for (int r = 1; r < NP; ++r) s = __dadd_rn(s, rowsum[r][c]);
        part[c < nout ? npairs + c : npairs + nout] = s;
    }
    (void)warp;
    __threadfence();
    __syncthreads();
    __shared__ bool s_last;
    if (tid == 0) s_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    const double n = (double)npts;
    const int stride = npairs + nout + 1;
    for (int v = tid; v < stride; v += NN_THREADS) {
        double s = __ldcg(partials + v);
        for (int c = 1; c < (int)gridDim.x; ++c) s = __dadd_rn(s, __ldcg(partials + (int64_t)c * stride + v));
        const double r = __ddiv_rn(s, n);               // divf (...) n  (:40, 45, 48)
        if (v < npairs) dw_out[v] = r;
        else if (v < npairs + nout) db_out[v - npairs] = r;
        else *loss_out = r;
    }
    if (tid == 0) *ticket = 0u;
}

}  // namespace pmx

using namespace pmx;

extern "C" {

size_t pmx_nn_workspace_bytes(int64_t npts, int32_t nin, int32_t nout) {
    (void)npts;
    return 256 + (size_t)2 * sm_count() * ((size_t)nin * nout + nout + 1) * sizeof(double);
}

int pmx_nn_softmax_grad_f64(const double* x, const int32_t* y, const double* w, const double* b, int64_t npts,
                            int32_t nin, int32_t nout, double* loss, double* dw, double* db, void* ws,
                            size_t ws_bytes, uint64_t* err, void* stream) {
    PMX_REQUIRE(npts >= 0 && nin > 0 && nout > 0, "pmx_nn_softmax_grad_f64: bad sizes");
    PMX_REQUIRE(nin <= NN_MAXIN && nout <= NN_MAXOUT, "pmx_nn_softmax_grad_f64: nin <= 64 and nout <= 32");
    PMX_REQUIRE(ws && ws_bytes >= pmx_nn_workspace_bytes(npts, nin, nout), "pmx_nn_softmax_grad_f64: workspace");
    cudaStream_t st = (cudaStream_t)stream;
    if (npts == 0) {   // n = 0.0: divf _ n is the reference's "float division by zero"
        if (err) {
            const uint64_t w0 = ((uint64_t)0 << 8) | PMX_E_DIVF0;
            cudaError_t e = cudaMemcpyAsync(err, &w0, 8, cudaMemcpyHostToDevice, st);
            if (e != cudaSuccess) { set_last_error("nn: %s", cudaGetErrorString(e)); return -2; }
            cudaStreamSynchronize(st);
        }
        return 0;
    }
    int64_t want = (npts + NN_TILE - 1) / NN_TILE;
    int grid = (int)(want < 2 * sm_count() ? (want < 1 ? 1 : want) : 2 * sm_count());
    unsigned* ticket = (unsigned*)ws;
    double* partials = (double*)((char*)ws + 256);
    cudaError_t me = cudaMemsetAsync(ticket, 0, sizeof(unsigned), st);
    if (me != cudaSuccess) { set_last_error("nn: %s", cudaGetErrorString(me)); return -2; }
    const int cw = nout <= 4 ? 4 : nout <= 8 ? 8 : nout <= 16 ? 16 : 32;
    const size_t smem = (size_t)(NN_MAXIN * NN_MAXOUT + NN_TILE * NN_MAXIN + NN_TILE * NN_MAXOUT) * sizeof(double);
#define PMX_NN(CW)                                                                                         \
    if (cw == CW) {                                                                                        \
        cudaFuncSetAttribute(k_nn_grad<CW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);        \
        k_nn_grad<CW><<<grid, NN_THREADS, smem, st>>>(x, y, w, b, npts, nin, nout, partials, ticket, loss,  \
                                                      dw, db, err);                                        \
    }
    PMX_NN(4) PMX_NN(8) PMX_NN(16) PMX_NN(32)
#undef PMX_NN
    PMX_CHECK_LAUNCH("nn_grad");
    return 0;
}

}  // extern "C"
