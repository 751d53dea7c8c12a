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

}  // namespace ga

#endif
