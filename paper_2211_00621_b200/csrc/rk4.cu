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

// Branch-free sin/cos for the two angles of `deriv`.  CUDA's sin/sincos carry
// a Payne-Hanek branch for huge arguments, which keeps the compiler from
// interleaving the independent transcendental chains of one RK4 step (sin of
// the arm angle, sin/cos of the pendulum angle, and the k2/k4 evaluations that
// are off the critical path) — at 68 threads/SM that ILP is the only
// parallelism the SM has.  Here: Cody-Waite reduction by pi/2 in three 33-bit
// pieces (each k*piece exact for |k| < 2^20) and the fdlibm minimax
// polynomials on [-pi/4, pi/4]; accuracy ~1 ulp, like glibc's and CUDA's (the
// oracle runs glibc; the parity bar is 1e-9 relative).  Arguments outside
// |x| <= 2^18 (and NaN/inf) take CUDA's sincos after the fast path.
struct SinCos { double s, c; };

__device__ __forceinline__ SinCos sincos_cw(double x) {
    const double k = rint(x * 6.36619772367581382433e-01);           // x * 2/pi
    double r = fma(-k, 1.57079632673412561417e+00, x);                // pio2_1 (33 bits)
    r = fma(-k, 6.07710050630396597660e-11, r);                       // pio2_2
    r = fma(-k, 2.02226624871116645580e-21, r);                       // pio2_3
    const double z = r * r;
    // Horner (Estrin's shallower tree measured no faster here)
    const double ps = fma(z, fma(z, fma(z, fma(z, fma(z, 1.58969099521155010221e-10, -2.50507602534068634195e-08),
                                               2.75573137070700676789e-06), -1.98412698298579493134e-04),
                                 8.33333333332248946124e-03), -1.66666666666666324348e-01);
    const double pc = fma(z, fma(z, fma(z, fma(z, fma(z, -1.13596475577881948265e-11, 2.08757232129817482790e-09),
                                               -2.75573143513906633035e-07), 2.48015872894767294178e-05),
                                 -1.38888888888741095749e-03), 4.16666666666666019037e-02);
    const double sr = fma(r * z, ps, r);
    const double cr = fma(z * z, pc, fma(-0.5, z, 1.0));
    const int q = (int)k & 3;
    double sv = (q & 1) ? cr : sr, cv = (q & 1) ? sr : cr;
    sv = (q & 2) ? -sv : sv;
    cv = ((q + 1) & 2) ? -cv : cv;
    sv = x == 0.0 ? x : sv;                                           // sin(-0) = -0
    return SinCos{sv, cv};
}

// Trig modes.  LIBM: CUDA's sin/sincos.  FAST: sincos_cw of both angles,
// recording in `bad` whether an angle left its range; the caller then redoes
// the whole step with LIBM, so the step itself is straight-line code.
// (Measured on B200, N = 10^4 x 10^3: LIBM 0.99 ms, FAST 0.62 ms; a lane pair
// per parameter set splitting the two reductions, with shuffles, 0.63 ms;
// Estrin instead of Horner 0.63 ms; 32/64/128-thread CTAs all equal — the
// time is one warp's dependent chain, ~1200 cycles per RK4 step.)
enum { RK4_LIBM = 0, RK4_FAST = 1, RK4_ADD = 2 };
#ifndef RK4_ADD_BLOCK
#define RK4_ADD_BLOCK 4      // steps per full sin/cos in RK4_ADD (one straight-line block)
#endif

// sin and cos of a small increment d (|d| <= 1/16, checked by the caller: the
// omitted terms are below 2^-64 relative), Taylor series to d^9 / d^8 in
// Estrin form on z = d^2 (dependent depth 4-5 instead of 7).
__device__ __forceinline__ SinCos sincos_small(double d) {
    const double z = d * d, z2 = z * z;
    const double ps = fma(z2, fma(z, -2.7557319223985890653e-06, 1.9841269841269841270e-04),
                          fma(z, -8.3333333333333333333e-03, 1.6666666666666666667e-01));
    const double pc = fma(z2 * z2, -2.7557319223985890653e-07,
                          fma(z2, fma(z, 2.4801587301587301587e-05, -1.3888888888888888889e-03),
                              fma(z, 4.1666666666666666667e-02, -0.5)));
    return SinCos{fma(-d * z, ps, d), fma(z, pc, 1.0)};
}

// sin/cos(x0 + d) from sin/cos(x0) and of the small increment d:
// angle addition, two fused products each (the result is within ~2 ulp, like
// a direct evaluation; parity is checked at 1e-9 relative)
__device__ __forceinline__ SinCos sincos_add(const SinCos& b, const SinCos& e) {
    return SinCos{fma(b.s, e.c, b.c * e.s), fma(b.c, e.c, -(b.s * e.s))};
}

template <int MODE>
__device__ __forceinline__ void trig(const St& s, double& sa, double& sp, double& cp, bool& bad) {
    if (MODE == RK4_FAST) {
        const SinCos a = sincos_cw(s.x0), b = sincos_cw(s.x2);
        sa = a.s; sp = b.s; cp = b.c;
        bad |= !(fabs(s.x0) <= 262144.0 && fabs(s.x2) <= 262144.0);
    } else {
        sincos(s.x2, &sp, &cp);
        sa = sin(s.x0);
    }
}

// deriv p s (rk4.pmx:11-22)
template <int MODE>
__device__ __forceinline__ St deriv(double p, const St& s, bool& bad) {
    double sa, sp, cp;
    trig<MODE>(s, sa, sp, cp, bad);
    St d;
    d.x0 = s.x1;
    // subf (mulf p (mulf (sin pend) (cos pend))) (addf (mulf 0.2 armVel) (mulf 0.3 (sin arm)))
    d.x1 = S_(M_(p, M_(sp, cp)), A_(M_(0.2, s.x1), M_(0.3, sa)));
    d.x2 = s.x3;
    // subf (negf (mulf 9.81 (sin pend))) (addf (mulf 0.1 pendVel) (mulf p (mulf armVel (cos pend))))
    d.x3 = S_(-M_(9.81, sp), A_(M_(0.1, s.x3), M_(p, M_(s.x1, cp))));
    return d;
}

// deriv with the trig values supplied (RK4_ADD computes them by angle addition)
__device__ __forceinline__ St deriv_t(double p, const St& s, double sa, double sp, double cp) {
    St d;
    d.x0 = s.x1;
    d.x1 = S_(M_(p, M_(sp, cp)), A_(M_(0.2, s.x1), M_(0.3, sa)));
    d.x2 = s.x3;
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

// step p s with RK4_ADD trig: one full sin/cos of the step's two angles; the
// stage arguments s_i = s + c k (rk4.pmx:27-29) are the base angles plus a
// small increment (h/2 or h times a velocity; at most 0.015 on the bench sweep), whose sin/cos is a short series
// available as soon as the increment is — so the three later stages no
// longer wait on a full argument reduction and polynomial.
// (A, B): sin/cos of the step's two angles s.x0 and s.x2
__device__ __forceinline__ St step_add_t(double p, const St& s, const SinCos& A, const SinCos& B, double h,
                                         double h2, double h6, bool& bad) {
    auto stage_trig = [&](const St& si, double& sa, double& sp, double& cp) {
        const double da = __dsub_rn(si.x0, s.x0), dp = __dsub_rn(si.x2, s.x2);
        bad |= !(fabs(da) <= 0.0625 && fabs(dp) <= 0.0625);
        const SinCos a = sincos_add(A, sincos_small(da)), b = sincos_add(B, sincos_small(dp));
        sa = a.s; sp = b.s; cp = b.c;
    };
    const St k1 = deriv_t(p, s, A.s, B.s, B.c);
    double sa, sp, cp;
    const St s2 = axpy(s, h2, k1);
    stage_trig(s2, sa, sp, cp);
    const St k2 = deriv_t(p, s2, sa, sp, cp);
    const St s3 = axpy(s, h2, k2);
    stage_trig(s3, sa, sp, cp);
    const St k3 = deriv_t(p, s3, sa, sp, cp);
    const St s4 = axpy(s, h, k3);
    stage_trig(s4, sa, sp, cp);
    const St k4 = deriv_t(p, s4, sa, sp, cp);
    return St{comb(s.x0, h6, k1.x0, k2.x0, k3.x0, k4.x0), comb(s.x1, h6, k1.x1, k2.x1, k3.x1, k4.x1),
              comb(s.x2, h6, k1.x2, k2.x2, k3.x2, k4.x2), comb(s.x3, h6, k1.x3, k2.x3, k3.x3, k4.x3)};
}

__device__ __forceinline__ St step_add(double p, const St& s, double h, double h2, double h6, bool& bad) {
    const SinCos A = sincos_cw(s.x0), B = sincos_cw(s.x2);
    bad |= !(fabs(s.x0) <= 262144.0 && fabs(s.x2) <= 262144.0);
    return step_add_t(p, s, A, B, h, h2, h6, bad);
}

// two steps with one full sin/cos: the second step's angles are the first
// step's plus a small increment, so its base sin/cos come by angle addition
// too (a full reduction every other step bounds the accumulated rounding)
template <int NS>
__device__ __forceinline__ St stepn_add(double p, St s, double h, double h2, double h6, bool& bad) {
    SinCos A = sincos_cw(s.x0), B = sincos_cw(s.x2);
    bad |= !(fabs(s.x0) <= 262144.0 && fabs(s.x2) <= 262144.0);
#pragma unroll
    for (int i = 0; i < NS; ++i) {
        const St s1 = step_add_t(p, s, A, B, h, h2, h6, bad);
        if (i + 1 < NS) {
            const double da = __dsub_rn(s1.x0, s.x0), dp = __dsub_rn(s1.x2, s.x2);
            bad |= !(fabs(da) <= 0.0625 && fabs(dp) <= 0.0625);
            A = sincos_add(A, sincos_small(da));
            B = sincos_add(B, sincos_small(dp));
        }
        s = s1;
    }
    return s;
}

// step p s (rk4.pmx:26-37)
template <int MODE>
__device__ __forceinline__ St step(double p, const St& s, double h, double h2, double h6, bool& bad) {
    if (MODE == RK4_ADD) return step_add(p, s, h, h2, h6, bad);
    const St k1 = deriv<MODE>(p, s, bad);
    const St k2 = deriv<MODE>(p, axpy(s, h2, k1), bad);
    const St k3 = deriv<MODE>(p, axpy(s, h2, k2), bad);
    const St k4 = deriv<MODE>(p, axpy(s, h, k3), bad);
    return St{comb(s.x0, h6, k1.x0, k2.x0, k3.x0, k4.x0), comb(s.x1, h6, k1.x1, k2.x1, k3.x1, k4.x1),
              comb(s.x2, h6, k1.x2, k2.x2, k3.x2, k4.x2), comb(s.x3, h6, k1.x3, k2.x3, k3.x3, k4.x3)};
}

// TRACE: also record state component `comp` after every step into
// trace[k * steps + m] (the paper's N x M tensor of one measured state,
// PAPER.md:1435-1440, written by its accelerated `loop` through tensorSet).
template <bool TRACE, int MODE>
__global__ void __launch_bounds__(64)
k_rk4(const double* __restrict__ ps, int64_t n, const double* __restrict__ init4,
      int steps, double h, double* __restrict__ out, int comp, double* __restrict__ trace) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const double p = ps[k];
    const double h2 = __ddiv_rn(h, 2.0);   // divf h 2.0
    const double h6 = __ddiv_rn(h, 6.0);   // divf h 6.0
    St s{init4[0], init4[1], init4[2], init4[3]};
    int m = 0;
    if (MODE != RK4_LIBM && !TRACE) {
        // two steps as one straight-line block (the next step's first derivative
        // overlaps this step's last one), both redone with libm if an angle left
        // the fast reduction's range in either.  Measured 0.615 -> 0.532 ms; three
        // steps per block 0.624, a rolled 2- or 4-step loop 0.58 / 0.64 (ptxas
        // schedules the explicit pair best).
        constexpr int NB = MODE == RK4_ADD ? RK4_ADD_BLOCK : 2;
        for (; m + NB - 1 < steps; m += NB) {
            bool bad = false;
            St sn;
            if (MODE == RK4_ADD) {
                sn = stepn_add<NB>(p, s, h, h2, h6, bad);
            } else {
                const St s1 = step<MODE>(p, s, h, h2, h6, bad);
                sn = step<MODE>(p, s1, h, h2, h6, bad);
            }
            if (bad) {
                bool unused = false;
#pragma unroll 1
                for (int i = 0; i < NB; ++i) s = step<RK4_LIBM>(p, s, h, h2, h6, unused);
            } else {
                s = sn;
            }
        }
    }
    for (; m < steps; ++m) {   // integrate p s m  (rk4.pmx:38-40)
        bool bad = false;
        const St next = step<MODE>(p, s, h, h2, h6, bad);
        if (MODE != RK4_LIBM && bad) {     // an angle left sincos_cw's range (or is NaN/inf)
            bool unused = false;
            s = step<RK4_LIBM>(p, s, h, h2, h6, unused);
        } else {
            s = next;
        }
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

// PMX_RK4_MODE=0 selects CUDA's libm sin/sincos, 1 the per-stage fast sin/cos
// (A/B and tests); default 2 (one fast sin/cos per step + angle addition).
static int rk4_mode() {
    static const int v = [] {
        const char* e = getenv("PMX_RK4_MODE");
        return e && (e[0] == '0' || e[0] == '1') ? e[0] - '0' : 2;
    }();
    return v;
}

template <bool TRACE>
static void rk4_launch(const double* params, int64_t n, const double* init4, int steps, double h, double* out,
                       int comp, double* trace, cudaStream_t st) {
    // 64 threads per CTA spreads the few warps of an N=10^4 sweep over all SMs.
    const int threads = 64;
    const int64_t grid = (n + threads - 1) / threads;
    if (rk4_mode() == RK4_LIBM)
        k_rk4<TRACE, RK4_LIBM><<<(unsigned)grid, threads, 0, st>>>(params, n, init4, steps, h, out, comp, trace);
    else if (rk4_mode() == RK4_FAST)
        k_rk4<TRACE, RK4_FAST><<<(unsigned)grid, threads, 0, st>>>(params, n, init4, steps, h, out, comp, trace);
    else
        k_rk4<TRACE, RK4_ADD><<<(unsigned)grid, threads, 0, st>>>(params, n, init4, steps, h, out, comp, trace);
}

extern "C" int pmx_rk4_sweep_f64(const double* params, int64_t n, const double* init4,
                                 int32_t steps, double h, double* out, void* stream) {
    PMX_REQUIRE(n >= 0 && steps >= 0, "pmx_rk4_sweep_f64: negative size");
    if (n == 0) return 0;
    PMX_REQUIRE(params && init4 && out, "pmx_rk4_sweep_f64: null buffer");
    rk4_launch<false>(params, n, init4, steps, h, out, 0, nullptr, (cudaStream_t)stream);
    PMX_CHECK_LAUNCH("rk4");
    return 0;
}

extern "C" int pmx_rk4_trace_f64(const double* params, int64_t n, const double* init4, int32_t steps, double h,
                                 int32_t comp, double* trace, double* out, void* stream) {
    PMX_REQUIRE(n >= 0 && steps >= 0, "pmx_rk4_trace_f64: negative size");
    PMX_REQUIRE(comp >= 0 && comp < 4, "pmx_rk4_trace_f64: state component must be 0..3");
    if (n == 0) return 0;
    PMX_REQUIRE(params && init4 && out && (trace || steps == 0), "pmx_rk4_trace_f64: null buffer");
    rk4_launch<true>(params, n, init4, steps, h, out, comp, trace, (cudaStream_t)stream);
    PMX_CHECK_LAUNCH("rk4_trace");
    return 0;
}
