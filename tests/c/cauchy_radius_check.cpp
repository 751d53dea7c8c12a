// Checks the radius-test skip of the Cauchy search (csrc/tron.cuh
// cauchy_point / TileSearch::cauchy): for x inside its box, every trial at
// alpha0 * 2^-k with k >= 2 has fl(sqrt(t.t)) <= delta, the reference's test
// (tron.cpp:111,130) — so skipping it cannot change a result.  Random and
// adversarial instances: x on or next to the bounds, gradients spanning many
// binades, steps far below ulp(x), clipped components, tiny / huge radii.
// Also counts failures at k = 0 (alpha0 itself): the test is live there.
// Prints "<violations> <k0_failures> <instances>".  Run by tests/test_host.py.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>

#include "ga_math.h"

int main(int argc, char** argv) {
    constexpr int N = 6;
    const long n = argc > 1 ? std::atol(argv[1]) : 1000000;
    std::mt19937_64 rng(2110);
    std::uniform_real_distribution<double> U(0.0, 1.0);
    long viol = 0, k1_fail = 0;  // k1_fail: failures at k = 0
    for (long it = 0; it < n; ++it) {
        double x[N], g[N], l[N], u[N];
        for (int i = 0; i < N; ++i) {
            const double scale = std::ldexp(1.0, (int)(rng() % 40) - 10);
            l[i] = -scale * U(rng);
            u[i] = scale * U(rng);
            if (rng() % 8 == 0) u[i] = 0.0;
            const int where = (int)(rng() % 4);
            x[i] = where == 0 ? l[i] : where == 1 ? u[i] : l[i] + (u[i] - l[i]) * U(rng);
            x[i] = ga::sclamp(x[i], l[i], u[i]);
            g[i] = std::ldexp(U(rng) - 0.5, (int)(rng() % 80) - 40);
            if (rng() % 10 == 0) g[i] = 0.0;
        }
        const double delta = std::ldexp(0.5 + U(rng), (int)(rng() % 90) - 48);
        double gg = 0.0;
        for (int i = 0; i < N; ++i) gg += g[i] * g[i];
        const double gnorm = std::sqrt(gg);
        if (gnorm == 0.0) continue;
        double a = ga::smin(1.0, delta / gnorm);
        for (int k = 0; k <= 40; ++k) {
            double tt = 0.0;
            for (int i = 0; i < N; ++i) {
                const double t = ga::sclamp(x[i] - a * g[i], l[i], u[i]) - x[i];
                tt += t * t;
            }
            const bool pass = std::sqrt(tt) <= delta;
            if (k >= 2 && !pass) ++viol;
            if (k == 0 && !pass) ++k1_fail;  // alpha0 itself can fail (the test is live)
            a *= 0.5;
        }
    }
    std::printf("%ld %ld %ld\n", viol, k1_fail, n);
    return 0;
}
