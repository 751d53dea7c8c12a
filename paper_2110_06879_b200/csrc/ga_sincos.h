/* ga_sincos.h — the pinned sine/cosine shared by the host oracle shim and the
 * sm_100a kernels.
 *
 * Why this exists: the reference evaluates cos/sin of branch angle
 * differences inside every branch-NLP evaluation (reference
 * proj/src/kernels.cpp:30-31, proj/src/netdata.cpp:37-38) and at parse time
 * (std::polar in proj/src/netdata.cpp:20).  GCC fuses those calls into glibc
 * `sincos`, an IFUNC whose result bits depend on the host CPU, and the ADMM
 * trajectory is chaotic at the ULP level.  A GPU libm
 * cannot reproduce glibc's bits, so both sides call THIS routine instead:
 * the oracle links it in place of libm's sin/cos/sincos (oracle/sincos_shim.c)
 * and the device code inlines it.
 *
 * Determinism contract: only IEEE-754 double operations that are correctly
 * rounded on every target are used — add, multiply, and explicit fma() (DFMA
 * on sm_100a, glibc fma() on the host).  Host code must be compiled with
 * -ffp-contract=off and device code with -fmad=false so the compiler never
 * fuses a written a*b+c.  Accuracy: < 1 ulp for |x| <= 2^20 (Cody-Waite
 * reduction with a 3-part pi/2, fdlibm-style minimax kernels on
 * [-pi/4, pi/4]).  Arguments seen by the solver are bounded by 4*pi
 * (angle box +-2pi, reference proj/src/kernels.cpp:94-95).
 */
#ifndef GA_SINCOS_H
#define GA_SINCOS_H

#include <math.h>

#if defined(__CUDACC__)
#define GA_HD __host__ __device__ __forceinline__
#else
#define GA_HD static inline
#endif

/* 2/pi and pi/2 split into three parts (the first two have trailing zero
 * bits so k*P1 and k*P2 are exact for |k| < 2^20). */
#define GA_TWO_OVER_PI 6.36619772367581382433e-01
#define GA_PIO2_1 1.57079632673412561417e+00  /* first 33 bits of pi/2 */
#define GA_PIO2_2 6.07710050630396597660e-11  /* next 33 bits */
#define GA_PIO2_3 2.02226624879595063154e-21  /* pi/2 - (P1 + P2), rounded */
#define GA_ROUND_MAGIC 6.75539944105574400000e+15 /* 1.5 * 2^52 */

/* Polynomial coefficients of the classic fdlibm kernels (minimax on
 * [-pi/4, pi/4]); public mathematical constants. */
#define GA_S1 -1.66666666666666324348e-01
#define GA_S2 8.33333333332248946124e-03
#define GA_S3 -1.98412698298579493134e-04
#define GA_S4 2.75573137070700676789e-06
#define GA_S5 -2.50507602534068634195e-08
#define GA_S6 1.58969099521155010221e-10

#define GA_C1 4.16666666666666019037e-02
#define GA_C2 -1.38888888888741095749e-03
#define GA_C3 2.48015872894767294178e-05
#define GA_C4 -2.75573143513906633035e-07
#define GA_C5 2.08757232129817482790e-09
#define GA_C6 -1.13596475577881948265e-11

/* sin and cos of a reduced argument r = hi + lo, |r| <= ~pi/4. */
GA_HD void ga_kernel_sincos(double r, double lo, double* s, double* c) {
    const double z = r * r;
    /* sin: r + r^3 (S1 + z P(z)) + lo correction (fdlibm __kernel_sin). */
    double ps = fma(z, GA_S6, GA_S5);
    ps = fma(z, ps, GA_S4);
    ps = fma(z, ps, GA_S3);
    ps = fma(z, ps, GA_S2);
    const double v = z * r;
    /* r - ((z*(0.5*lo - v*ps) - lo) - v*S1) */
    const double t1 = 0.5 * lo - v * ps;
    const double t2 = z * t1 - lo;
    const double t3 = t2 - v * GA_S1;
    *s = r - t3;
    /* cos: fdlibm __kernel_cos, 1 - z/2 + z^2 C(z) - r*lo. */
    double pc = fma(z, GA_C6, GA_C5);
    pc = fma(z, pc, GA_C4);
    pc = fma(z, pc, GA_C3);
    pc = fma(z, pc, GA_C2);
    pc = fma(z, pc, GA_C1);
    const double rr = z * pc;
    const double hz = 0.5 * z;
    const double w = 1.0 - hz;
    const double corr = ((1.0 - w) - hz) + (z * rr - r * lo);
    *c = w + corr;
}

/* Pinned sincos.  Non-finite input gives NaN for both outputs. */
GA_HD void ga_sincos(double x, double* s, double* c) {
    if (!(x - x == 0.0)) { /* inf or nan */
        const double nan = x - x;
        *s = nan;
        *c = nan;
        return;
    }
    /* k = nearest integer to x*2/pi (round-half-even via the 1.5*2^52 trick;
     * both the multiply and the adds are correctly rounded everywhere). */
    const double kd = (x * GA_TWO_OVER_PI + GA_ROUND_MAGIC) - GA_ROUND_MAGIC;
    /* r = x - k*pi/2 in three exact-product steps; lo carries the rounding
     * error of the final subtraction so the kernel sees ~2 doubles. */
    const double r1 = x - kd * GA_PIO2_1;   /* exact: k*P1 exact, Sterbenz */
    const double w2 = kd * GA_PIO2_2;       /* exact */
    const double r2 = r1 - w2;
    const double e2 = (r1 - r2) - w2;       /* error of r1 - w2 */
    const double w3 = kd * GA_PIO2_3;
    const double r = r2 - (w3 - e2);
    const double lo = (r2 - r) - (w3 - e2);
    double sr, cr;
    ga_kernel_sincos(r, lo, &sr, &cr);
    const long long k = (long long)kd;
    switch ((int)(k & 3)) {
        case 0: *s = sr; *c = cr; break;
        case 1: *s = cr; *c = -sr; break;
        case 2: *s = -sr; *c = -cr; break;
        default: *s = -cr; *c = sr; break;
    }
}

GA_HD double ga_sin(double x) { double s, c; ga_sincos(x, &s, &c); return s; }
GA_HD double ga_cos(double x) { double s, c; ga_sincos(x, &s, &c); return c; }

#if defined(__CUDACC__)
/* Out-of-line device copy: the branch kernels call sincos from ~10 sites and
 * their hot loop must fit the instruction cache.  Same operations, same bits. */
static __device__ __noinline__ double2 ga_sincos_call(double x) {
    double s, c;
    ga_sincos(x, &s, &c);
    return make_double2(s, c);
}
/* sincos for code compiled for both sides: out-of-line on the device. */
__host__ __device__ __forceinline__ void ga_sincos_ool(double x, double* s, double* c) {
#if defined(__CUDA_ARCH__)
    const double2 r = ga_sincos_call(x);
    *s = r.x;
    *c = r.y;
#else
    ga_sincos(x, s, c);
#endif
}
#endif

#endif /* GA_SINCOS_H */
