// ga_math.h — scalar helpers with the exact semantics of the libstdc++
// algorithms the reference uses, so host and device give identical bits
// (including NaN propagation, which differs from fmin/fmax):
//   std::min(a, b)        = (b < a) ? b : a
//   std::max(a, b)        = (a < b) ? b : a
//   std::clamp(v, lo, hi) = (v < lo) ? lo : (hi < v) ? hi : v
// Reference call sites: proj/src/tron.cpp:25,233,250-252,280-281,293,304-307;
// proj/src/kernels.cpp:203,206,261-266,428-436; proj/src/decomp.cpp:67.
#ifndef GA_MATH_H
#define GA_MATH_H

#include <math.h>

#if defined(__CUDACC__)
#define GA_FN __host__ __device__ __forceinline__
#else
#define GA_FN inline
#endif

namespace ga {

GA_FN double smin(double a, double b) { return (b < a) ? b : a; }
GA_FN double smax(double a, double b) { return (a < b) ? b : a; }
GA_FN double sclamp(double v, double lo, double hi) {
    return (v < lo) ? lo : ((hi < v) ? hi : v);
}
GA_FN bool sfinite(double v) { return v - v == 0.0; }
// |v| that drops NaN to 0 — the effect of std::max(acc, std::abs(v)) on a
// running non-negative max (proj/src/decomp.cpp:67, driver.cpp:117-120,179-186).
GA_FN double abs_or_zero(double v) { return (v == v) ? fabs(v) : 0.0; }

// Largest double t with fl(sqrt(t)) <= d, so that for every double y
//   (sqrt(y) <= d)  ==  (y <= t)
// (sqrt is correctly rounded and monotone; NaN y fails both sides).  The
// trust-region test ||s|| <= delta of the Cauchy search (tron.cpp:111,130)
// then costs one compare per trial instead of a square root.  Valid for
// d in [2^-400, 2^400]: fl(d*d) is normal there and fl(sqrt(fl(d*d))) == d
// (round-to-nearest), and at most two successors of fl(d*d) still round to
// d; *ok is false outside that range (the caller keeps the square root).
// tests/c/sqrt_bound_check.cpp checks maximality and the equivalence.
GA_FN double sqrt_le_bound(double d, bool* ok) {
    *ok = d >= 0x1p-400 && d <= 0x1p400;
    if (!*ok) return 0.0;
    double t = d * d;
#if defined(__CUDACC__)
#pragma unroll 1
#endif
    for (int k = 0; k < 4; ++k) {  // one square-root site (code size)
        long long bits;
        __builtin_memcpy(&bits, &t, sizeof t);
        ++bits;
        double n;
        __builtin_memcpy(&n, &bits, sizeof n);
        if (!(sqrt(n) <= d)) break;
        t = n;
    }
    return t;
}

}  // namespace ga

#endif
