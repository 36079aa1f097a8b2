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
// warps and CTAs folded in index order), deterministic run to run.  The dw
// terms x_pi * dz_pj enter their sums through fused multiply-add (one rounding
// per term instead of two, half the FP64 issue slots): those sums have no
// single reference value to be bit-identical to, and the parity bar for them is
// the north star's 1e-9 relative.  z, the softmax and dz keep the reference's
// separately rounded operations.
//
// B200 design: points in tiles of 64 (x is the only HBM stream, 8 * nin bytes
// per point, read once).  A tile is brought into shared memory by one 1-D bulk
// copy (TMA engine, mbarrier completion) into a double buffer, so the next
// tile streams in while this one is computed.  Phase 1 runs the z chains with
// lane j = class j and PT points per thread (independent sequential chains
// hide the fp64 latency), softmax through lane-group shuffles, dz to shared
// memory.  Phase 2 accumulates x^T dz in 4 x 4 register tiles per thread
// (four x and four dz values feed 16 MACs) over G interleaved point groups;
// the one-pair-per-thread form was shared-memory bound (2 wavefronts per MAC).
// Per-CTA partials go to the workspace and the last CTA folds them in CTA
// order (one launch).
#include "common.cuh"
#include "tc.cuh"

namespace pmx {

constexpr int NN_THREADS = 256;
constexpr int NN_MAXIN = 64;
constexpr int NN_MAXOUT = 32;
constexpr int NN_TILE = 64;          // points per tile (x tile 64 x 64 fp64 = 32 KiB)
constexpr size_t NN_SMEM = (size_t)(NN_MAXIN * NN_MAXOUT + 2 * NN_TILE * NN_MAXIN + NN_TILE * NN_MAXOUT +
                                   2 * NN_TILE) * sizeof(double) + 64;

// Thread layout for the per-point phase: lane group of CW = next pow2 >= nout
// (>= 4) lanes per point (lane j = class j), NP = 256 / CW point rows, each thread
// runs PT = NN_TILE / NP points (independent fp64 chains: ILP for the
// sequential foldl of z).  BULK: x is 16-B aligned (tiles by bulk copy; the
// tail tile and unaligned x are loaded by the threads).
template <int CW, bool BULK>
__global__ void __launch_bounds__(NN_THREADS, 2)
k_nn_grad(const double* __restrict__ x, const int* __restrict__ y, const double* __restrict__ w,
          const double* __restrict__ b, int64_t npts, int nin, int nout, double* __restrict__ partials,
          unsigned* ticket, double* __restrict__ loss_out, double* __restrict__ dw_out,
          double* __restrict__ db_out, uint64_t* err) {
    constexpr int NP = NN_THREADS / CW;
    constexpr int PT = NN_TILE / NP > 0 ? NN_TILE / NP : 1;
    constexpr int TILE = NP * PT;
    static_assert(TILE == NN_TILE, "tile");
    extern __shared__ __align__(16) double nsm[];
    double* ws = nsm;                                  // [NN_MAXIN * NN_MAXOUT]
    double* xbuf = ws + NN_MAXIN * NN_MAXOUT;          // [2][TILE * NN_MAXIN]
    double* dzs = xbuf + 2 * TILE * NN_MAXIN;          // [TILE * NN_MAXOUT]
    double* tot = dzs + TILE * NN_MAXOUT;              // [TILE] softmax totals
    double* zys = tot + TILE;                          // [TILE] z_y
    uint64_t* bar = reinterpret_cast<uint64_t*>(zys + TILE);   // [2]
    constexpr int RW = 32 / CW;                        // point rows per warp
    const int tid = threadIdx.x, lane = tid & 31;
    const int j = tid % CW, row = tid / CW;
    const bool act = j < nout;
    const int npairs = nin * nout;
    // phase-2 thread tiles: 4 x 4 (i, j) pairs, G point groups
    const int nbj = (nout + 3) >> 2, ntl = ((nin + 3) >> 2) * nbj;
    const int G = NN_THREADS / ntl, tl = tid % ntl, g = tid / ntl;
    const int tbi = tl / nbj, tbj = tl % nbj;
    for (int v = tid; v < npairs; v += NN_THREADS) ws[v] = w[v];
    const double bj = act ? b[j] : 0.0;
    const int64_t ntiles = (npts + TILE - 1) / TILE;
    auto full = [&](int64_t t) { return (t + 1) * TILE <= npts; };
    auto issue = [&](int it) {                          // thread 0: tile of local iteration `it`
        const int64_t t = blockIdx.x + (int64_t)it * gridDim.x;
        if (BULK && t < ntiles && full(t)) {
            const uint32_t bytes = (uint32_t)(TILE * nin * sizeof(double));
            tc::mbar_arrive_expect_tx(&bar[it & 1], bytes);
            tc::bulk_load_1d(xbuf + (it & 1) * TILE * NN_MAXIN, x + t * TILE * nin, bytes, &bar[it & 1]);
        }
    };
    if (BULK && tid == 0) {
        tc::mbar_init(&bar[0], 1);
        tc::mbar_init(&bar[1], 1);
        tc::fence_mbar_init();
    }
    __syncthreads();
    if (BULK && tid == 0) { issue(0); issue(1); }
    double dwacc[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) dwacc[c] = 0.0;
    double dbacc = 0.0, lossacc = 0.0;
    int it = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const int64_t p0 = tile * TILE;
        const int npt = (int)(npts - p0 < TILE ? npts - p0 : TILE);
        double* xs = xbuf + (it & 1) * TILE * NN_MAXIN;
        if (BULK && full(tile)) {
            tc::mbar_wait(&bar[it & 1], (uint32_t)(it >> 1) & 1u);
        } else {
            const double* xt = x + p0 * nin;
            for (int v = tid; v < npt * nin; v += NN_THREADS) xs[v] = __ldcs(xt + v);   // coalesced stream
            for (int v = npt * nin + tid; v < TILE * nin; v += NN_THREADS) xs[v] = 0.0;  // tail rows
            __syncthreads();
        }
        // ---- per point: z (reference foldl order), softmax, loss, dz
        int yk[PT];                                        // labels, loaded ahead of the z chains
#pragma unroll
        for (int k = 0; k < PT; ++k) yk[k] = row + k * NP < npt ? __ldg(y + p0 + row + k * NP) : 0;
        double z[PT];
#pragma unroll
        for (int k = 0; k < PT; ++k) z[k] = bj;
        // rows past the tile end are never used
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
        // softmax in three warp-local steps (a point's CW class lanes are in one
        // warp): (1) e = exp z to shared memory, z_y noted by the lane j == y;
        // (2) one lane per point folds the totals left to right over the
        // classes (the reference's sequential reduce) and adds the point's loss;
        // (3) dz = e / total - [j == y].  Runtime errors: exp overflow, log of a
        // zero total, y out of bounds — codes ordered as the reference meets
        // them within a point (raise_err keeps the smallest (point, code)).
        double ek[PT];
#pragma unroll
        for (int k = 0; k < PT; ++k) {
            const int pl = row + k * NP;
            const bool live = pl < npt;
            ek[k] = act ? exp(z[k]) : 0.0;
            if (live && act) {
                if (is_inf(ek[k]) && !is_inf(z[k])) raise_err(err, p0 + pl, PMX_E_EXP_RANGE);
                dzs[pl * NN_MAXOUT + j] = ek[k];
                if (j == yk[k]) zys[pl] = z[k];
            }
            if (live && j == 0 && (yk[k] < 0 || yk[k] >= nout)) raise_err(err, p0 + pl, PMX_E_OOB);
        }
        __syncwarp();
        if (lane < RW * PT) {
            const int pl = (tid >> 5) * RW + lane / PT + (lane % PT) * NP;
            if (pl < npt) {
                const double* er = dzs + pl * NN_MAXOUT;
                double total = 0.0;                        // left fold over classes
                for (int c = 0; c < nout; ++c) total = __dadd_rn(total, er[c]);
                tot[pl] = total;
                if (total == 0.0) raise_err(err, p0 + pl, PMX_E_LOG_DOMAIN);
                lossacc = __dadd_rn(lossacc, __dsub_rn(log(total), zys[pl]));
            }
        }
        __syncwarp();
#pragma unroll
        for (int k = 0; k < PT; ++k) {
            const int pl = row + k * NP;
            if (pl < npt && act) {
                double dz = __ddiv_rn(ek[k], tot[pl]);
                if (j == yk[k]) dz = __dsub_rn(dz, 1.0);
                dzs[pl * NN_MAXOUT + j] = dz;
                dbacc = __dadd_rn(dbacc, dz);
            }
        }
        __syncthreads();
        // ---- dw: thread tile (bi, bj) = pairs (4bi + 0..3, 4bj + 0..3), point
        // group g = points g, g + G, ... of every tile: one sequential chain per
        // (pair, group); out-of-range members of an edge tile read padding and
        // are never stored
        if (g < G) {
            const double* xc = xs + 4 * tbi + g * nin;
            const double* dc = dzs + 4 * tbj + g * NN_MAXOUT;
            const int xstep = G * nin, dstep = G * NN_MAXOUT;
            auto mac = [&](const double (&xv)[4], const double* d) {
                const double2 d01 = *reinterpret_cast<const double2*>(d);
                const double2 d23 = *reinterpret_cast<const double2*>(d + 2);
                const double dv[4] = {d01.x, d01.y, d23.x, d23.y};
#pragma unroll
                for (int u = 0; u < 4; ++u)
#pragma unroll
                    for (int v = 0; v < 4; ++v) dwacc[u * 4 + v] = __fma_rn(xv[u], dv[v], dwacc[u * 4 + v]);
            };
            if ((nin & 1) == 0) {                          // x rows 16-byte aligned
#pragma unroll 4
                for (int pl = g; pl < npt; pl += G, xc += xstep, dc += dstep) {
                    const double2 a = *reinterpret_cast<const double2*>(xc);
                    const double2 c = *reinterpret_cast<const double2*>(xc + 2);
                    const double xv[4] = {a.x, a.y, c.x, c.y};
                    mac(xv, dc);
                }
            } else {
#pragma unroll 4
                for (int pl = g; pl < npt; pl += G, xc += xstep, dc += dstep) {
                    const double xv[4] = {xc[0], xc[1], xc[2], xc[3]};
                    mac(xv, dc);
                }
            }
        }
        __syncthreads();                                   // xs[it & 1] and dzs free
        if (BULK && tid == 0) issue(it + 2);
    }
    // ---- CTA partial: dw (the G group chains of a pair folded in group order),
    // db and loss (fold the point rows in order)
    double* part = partials + (int64_t)blockIdx.x * (npairs + nout + 1);
    double* red = xbuf;                                    // all copies consumed: reuse the x buffers
    if (g < G)
#pragma unroll
        for (int c = 0; c < 16; ++c) red[(g * ntl + tl) * 16 + c] = dwacc[c];
    __syncthreads();
    for (int pr = tid; pr < npairs; pr += NN_THREADS) {
        const int ii = pr / nout, jj = pr % nout;
        const int t = (ii >> 2) * nbj + (jj >> 2), c = (ii & 3) * 4 + (jj & 3);
        double sum = red[t * 16 + c];
        for (int q = 1; q < G; ++q) sum = __dadd_rn(sum, red[(q * ntl + t) * 16 + c]);
        part[pr] = sum;
    }
    __shared__ double rowsum[NP][NN_MAXOUT];
    __shared__ double lsum[NN_THREADS];
    if (act) rowsum[row][j] = dbacc;
    lsum[tid] = lossacc;
    __syncthreads();
    if (tid < nout) {
        double s = rowsum[0][tid];
        for (int r = 1; r < NP; ++r) s = __dadd_rn(s, rowsum[r][tid]);
        part[npairs + tid] = s;
    } else if (tid == NN_MAXOUT) {
        double s = lsum[0];
        for (int r = 1; r < NN_THREADS; ++r) s = __dadd_rn(s, lsum[r]);
        part[npairs + nout] = s;
    }
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
    const bool bulk = ((uintptr_t)x & 15) == 0;
#define PMX_NN(CW, B)                                                                                      \
    if (cw == CW && bulk == B) {                                                                           \
        cudaFuncSetAttribute(k_nn_grad<CW, B>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)NN_SMEM);  \
        k_nn_grad<CW, B><<<grid, NN_THREADS, NN_SMEM, st>>>(x, y, w, b, npts, nin, nout, partials, ticket,  \
                                                            loss, dw, db, err);                            \
    }
    PMX_NN(4, true) PMX_NN(8, true) PMX_NN(16, true) PMX_NN(32, true)
    PMX_NN(4, false) PMX_NN(8, false) PMX_NN(16, false) PMX_NN(32, false)
#undef PMX_NN
    PMX_CHECK_LAUNCH("nn_grad");
    return 0;
}

}  // extern "C"
