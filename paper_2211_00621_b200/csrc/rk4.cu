// Batched RK4 parameter sweep — the case study of programs/rk4.pmx.
//
// Reference: programs/rk4.pmx:11-45 runs `map (lam p. integrate p init M) ps`
// (one eval_map fan-out, pmx/interp.py:294-304); each worker then performs the
// `integrate` recursion (rk4.pmx:38-40) — M dependent RK4 steps of the 4-state
// system `deriv` (rk4.pmx:11-22) with `axpy` = map2 (rk4.pmx:23-25, sequential
// under flattening) — on a thread.  Oracle: tests/test_acceptance.py:359-394.
//
// B200 design: one thread per parameter set, state in registers, the step
// loop on the device (the "seqLoop" of the north star).  Every fp64 operation
// is issued with an explicit round-to-nearest intrinsic so nvcc cannot fuse
// a*b+c into an FMA: the arithmetic is the program's, in the program's order.
// sin/cos of the same angle are computed once per `deriv` (pure functions, so
// common-subexpression elimination does not change any value).
// The kernel is latency-bound at N = 10^4 (68 threads/SM); see DESIGN.md.
#include "common.cuh"

namespace pmx {

#define M_(a, b) __dmul_rn((a), (b))
#define A_(a, b) __dadd_rn((a), (b))
#define S_(a, b) __dsub_rn((a), (b))

struct St { double x0, x1, x2, x3; };

// deriv p s (rk4.pmx:11-22)
__device__ __forceinline__ St deriv(double p, const St& s) {
    double sp, cp;
    sincos(s.x2, &sp, &cp);
    const double sa = sin(s.x0);
    St d;
    d.x0 = s.x1;
    // subf (mulf p (mulf (sin pend) (cos pend))) (addf (mulf 0.2 armVel) (mulf 0.3 (sin arm)))
    d.x1 = S_(M_(p, M_(sp, cp)), A_(M_(0.2, s.x1), M_(0.3, sa)));
    d.x2 = s.x3;
    // subf (negf (mulf 9.81 (sin pend))) (addf (mulf 0.1 pendVel) (mulf p (mulf armVel (cos pend))))
    d.x3 = S_(-M_(9.81, sp), A_(M_(0.1, s.x3), M_(p, M_(s.x1, cp))));
    return d;
}

// axpy s c d = map2 (lam x. lam dx. addf x (mulf c dx)) s d   (rk4.pmx:23-25)
__device__ __forceinline__ St axpy(const St& s, double c, const St& d) {
    return St{A_(s.x0, M_(c, d.x0)), A_(s.x1, M_(c, d.x1)), A_(s.x2, M_(c, d.x2)), A_(s.x3, M_(c, d.x3))};
}

// s_i + (h/6) * (k1_i + (2*k2_i + (2*k3_i + k4_i)))   (rk4.pmx:31-36)
__device__ __forceinline__ double comb(double s, double h6, double k1, double k2, double k3, double k4) {
    return A_(s, M_(h6, A_(k1, A_(M_(2.0, k2), A_(M_(2.0, k3), k4)))));
}

// TRACE: also record state component `comp` after every step into
// trace[k * steps + m] (the paper's N x M tensor of one measured state,
// PAPER.md:1435-1440, written by its accelerated `loop` through tensorSet).
template <bool TRACE>
__global__ void __launch_bounds__(64)
k_rk4(const double* __restrict__ ps, int64_t n, const double* __restrict__ init4,
      int steps, double h, double* __restrict__ out, int comp, double* __restrict__ trace) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const double p = ps[k];
    const double h2 = __ddiv_rn(h, 2.0);   // divf h 2.0
    const double h6 = __ddiv_rn(h, 6.0);   // divf h 6.0
    St s{init4[0], init4[1], init4[2], init4[3]};
    for (int m = 0; m < steps; ++m) {   // integrate p s m  (rk4.pmx:38-40)
        const St k1 = deriv(p, s);
        const St k2 = deriv(p, axpy(s, h2, k1));
        const St k3 = deriv(p, axpy(s, h2, k2));
        const St k4 = deriv(p, axpy(s, h, k3));
        s = St{comb(s.x0, h6, k1.x0, k2.x0, k3.x0, k4.x0), comb(s.x1, h6, k1.x1, k2.x1, k3.x1, k4.x1),
               comb(s.x2, h6, k1.x2, k2.x2, k3.x2, k4.x2), comb(s.x3, h6, k1.x3, k2.x3, k3.x3, k4.x3)};
        if (TRACE) {
            const double v = comp == 0 ? s.x0 : comp == 1 ? s.x1 : comp == 2 ? s.x2 : s.x3;
            __stcs(trace + k * (int64_t)steps + m, v);
        }
    }
    double* o = out + 4 * k;
    o[0] = s.x0; o[1] = s.x1; o[2] = s.x2; o[3] = s.x3;
}

}  // namespace pmx

using namespace pmx;

extern "C" int pmx_rk4_sweep_f64(const double* params, int64_t n, const double* init4,
                                 int32_t steps, double h, double* out, void* stream) {
    PMX_REQUIRE(n >= 0 && steps >= 0, "pmx_rk4_sweep_f64: negative size");
    if (n == 0) return 0;
    PMX_REQUIRE(params && init4 && out, "pmx_rk4_sweep_f64: null buffer");
    // 64 threads per CTA spreads the few warps of an N=10^4 sweep over all SMs.
    const int threads = 64;
    const int64_t grid = (n + threads - 1) / threads;
    k_rk4<false><<<(unsigned)grid, threads, 0, (cudaStream_t)stream>>>(params, n, init4, steps, h, out, 0, nullptr);
    PMX_CHECK_LAUNCH("rk4");
    return 0;
}

extern "C" int pmx_rk4_trace_f64(const double* params, int64_t n, const double* init4, int32_t steps, double h,
                                 int32_t comp, double* trace, double* out, void* stream) {
    PMX_REQUIRE(n >= 0 && steps >= 0, "pmx_rk4_trace_f64: negative size");
    PMX_REQUIRE(comp >= 0 && comp < 4, "pmx_rk4_trace_f64: state component must be 0..3");
    if (n == 0) return 0;
    PMX_REQUIRE(params && init4 && out && (trace || steps == 0), "pmx_rk4_trace_f64: null buffer");
    const int threads = 64;
    const int64_t grid = (n + threads - 1) / threads;
    k_rk4<true><<<(unsigned)grid, threads, 0, (cudaStream_t)stream>>>(params, n, init4, steps, h, out, comp, trace);
    PMX_CHECK_LAUNCH("rk4_trace");
    return 0;
}
