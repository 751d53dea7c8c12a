// Checks ga::sqrt_le_bound (csrc/ga_math.h): for every tested d, the bound t
// satisfies sqrt(t) <= d and sqrt(nextup(t)) > d (so it is the largest such
// double, by monotonicity of the correctly rounded sqrt), and for random y
// near d*d the two forms of the trust-region test agree.  Prints the number
// of failures (0 expected).  Built and run by tests/test_host.py.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <random>

#include "ga_math.h"

static double bump(double v, long long k) {
    long long b;
    std::memcpy(&b, &v, sizeof b);
    b += k;
    std::memcpy(&v, &b, sizeof v);
    return v;
}

int main(int argc, char** argv) {
    const long n = argc > 1 ? std::atol(argv[1]) : 2000000;
    std::mt19937_64 rng(2110);
    std::uniform_real_distribution<double> mant(1.0, 2.0);
    std::uniform_int_distribution<int> expo(-400, 399);
    long fails = 0, checked = 0;
    for (long i = 0; i < n; ++i) {
        double d;
        if (i % 4 == 0) d = std::ldexp(mant(rng), expo(rng));        // any binade
        else if (i % 4 == 1) d = std::ldexp(mant(rng), expo(rng) % 50);  // solver range
        else if (i % 4 == 2) d = bump(std::ldexp(1.0, expo(rng) % 60), (long long)(rng() % 7) - 3);
        else d = std::ldexp(mant(rng), -48 + (int)(rng() % 90));      // 2.5e-13 .. 1e10
        bool ok;
        const double t = ga::sqrt_le_bound(d, &ok);
        if (!ok) continue;
        ++checked;
        if (!(std::sqrt(t) <= d) || std::sqrt(bump(t, 1)) <= d) ++fails;
        for (int k = -6; k <= 6; ++k) {
            const double y = bump(d * d, k);
            if ((std::sqrt(y) <= d) != (y <= t)) ++fails;
        }
    }
    // out-of-range and special values fall back
    const double specials[] = {0.0, -1.0, std::ldexp(1.0, -401), std::ldexp(1.0, 401), INFINITY, NAN};
    for (double d : specials) {
        bool ok = true;
        ga::sqrt_le_bound(d, &ok);
        if (ok) ++fails;
    }
    std::printf("%ld %ld\n", fails, checked);
    return 0;
}
