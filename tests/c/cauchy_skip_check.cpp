// cauchy_skip_check.cpp — host check of the Cauchy backtracking pre-screen
// (tron.cuh cauchy_skip): the product's cauchy_point (with the skip) against
// the reference's loop (proj/src/tron.cpp:101-137, restated below without
// any skip) on random and adversarial instances, comparing the step bits.
// Built and run by tests/test_tron_prescreen.py with g++ -O2
// -ffp-contract=off (same IEEE double operations as the -fmad=false device
// build; the skip's proof does not depend on where it runs).
// usage: cauchy_skip_check <instances> <seed>   -> prints "mismatches skipped_trials trials"
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>

#include "tron.cuh"

namespace {

struct Mat {
    const double* p;
    double operator[](int k) const { return p[k]; }
};

// tron.cpp:101-137 as written (counts the trials it evaluates)
template <int N>
void reference_cauchy(const double* x, const double* g, const double* h, const double* l,
                      const double* u, double delta, double* s, long* trials) {
    auto dot = [](const double* a, const double* b) {
        double r = 0.0;
        for (int i = 0; i < N; ++i) r += a[i] * b[i];
        return r;
    };
    auto model = [&](const double* st) {
        double q = dot(g, st);
        for (int i = 0; i < N; ++i) {
            double hs = 0.0;
            for (int j = 0; j < N; ++j) hs += h[i * N + j] * st[j];
            q += 0.5 * st[i] * hs;
        }
        return q;
    };
    const double gnorm = std::sqrt(dot(g, g));
    if (gnorm == 0.0) {
        for (int i = 0; i < N; ++i) s[i] = 0.0;
        return;
    }
    auto step_at = [&](double alpha, double* out) {
        for (int i = 0; i < N; ++i) out[i] = ga::sclamp(x[i] - alpha * g[i], l[i], u[i]) - x[i];
    };
    auto ok = [&](const double* st) {
        ++*trials;
        return std::sqrt(dot(st, st)) <= delta && model(st) <= ga::kTronMu0 * dot(g, st);
    };
    double alpha = ga::smin(1.0, delta / gnorm);
    step_at(alpha, s);
    if (ok(s)) {
        double trial[N];
        for (int it = 0; it < 20; ++it) {
            const double next = alpha * 2.0;
            step_at(next, trial);
            if (!ok(trial)) break;
            alpha = next;
            std::memcpy(s, trial, sizeof trial);
        }
        return;
    }
    for (int it = 0; it < 40; ++it) {
        alpha *= 0.5;
        step_at(alpha, s);
        if (ok(s)) return;
    }
}

double scale(std::mt19937_64& r, double lo_exp, double hi_exp) {
    std::uniform_real_distribution<double> e(lo_exp, hi_exp);
    return std::pow(10.0, e(r));
}

template <int N>
long run(long count, std::mt19937_64& rng, long* skipped, long* trials) {
    std::uniform_real_distribution<double> U(-1.0, 1.0);
    std::uniform_int_distribution<int> pick(0, 9);
    long bad = 0;
    for (long c = 0; c < count; ++c) {
        double x[N], g[N], h[N * N], l[N], u[N];
        // penalty-dominated Hessians like the branch problems: a random
        // symmetric part plus a large diagonal / rank-one term
        const double hs = scale(rng, -3, 7), gs = scale(rng, -6, 6);
        double v[N];
        for (int i = 0; i < N; ++i) v[i] = U(rng);
        for (int i = 0; i < N; ++i)
            for (int j = 0; j <= i; ++j) {
                double e = hs * (0.3 * U(rng) + v[i] * v[j] * (pick(rng) < 5 ? 1.0 : 30.0));
                if (i == j) e = std::fabs(e) * (pick(rng) == 0 ? -0.1 : 1.0) + hs * 0.01;
                h[i * N + j] = e;
                h[j * N + i] = (pick(rng) == 0 && i != j) ? std::nextafter(e, 1e300) : e;  // slight asymmetry
            }
        for (int i = 0; i < N; ++i) {
            const double w = scale(rng, -3, 2);
            l[i] = -w * (0.5 + std::fabs(U(rng)));
            u[i] = w * (0.5 + std::fabs(U(rng)));
            const int k = pick(rng);
            x[i] = k == 0 ? l[i] : k == 1 ? u[i] : l[i] + (u[i] - l[i]) * (0.5 + 0.5 * U(rng));
            if (pick(rng) == 0) x[i] += 1e3 * w;  // large offsets: coarse ulp(x)
            if (x[i] > u[i]) u[i] = x[i] + w;
            const int z = pick(rng);
            g[i] = z == 0 ? 0.0 : gs * U(rng) * (z == 1 ? 1e-9 : 1.0);
        }
        double delta = scale(rng, -8, 4);
        if (pick(rng) < 3) {
            // boundary stress: alpha0 = 1 (delta >= |g|) and some component
            // reaching its bound exactly (to a few ulps) at a trial alpha 2^-k
            const int i = pick(rng) % N;
            const int k = 1 + pick(rng) * 2;
            x[i] = l[i] + (u[i] - l[i]) * 0.25;
            g[i] = std::ldexp(x[i] - l[i], k);
            for (int r = pick(rng) % 4; r > 0; --r) g[i] = std::nextafter(g[i], pick(rng) < 5 ? 0.0 : 1e300);
            double gn = 0.0;
            for (int j = 0; j < N; ++j) gn += g[j] * g[j];
            delta = 2.0 * std::sqrt(gn) + 1.0;
        }
        double s1[N], s2[N], qs = 0.0;
        bool qok = false;
        long t0 = 0;
        reference_cauchy<N>(x, g, h, l, u, delta, s2, &t0);
        ga::cauchy_point<N, false>(x, g, Mat{h}, l, u, delta, s1, &qs, &qok);
        if (std::memcmp(s1, s2, sizeof s1) != 0) ++bad;
        // skipped count as the product sees it (trial 0 failed)
        const double gn = std::sqrt(ga::vdot<N>(g, g));
        if (gn > 0.0) {
            const double a0 = ga::smin(1.0, delta / gn);
            *skipped += ga::cauchy_skip<N>(x, g, Mat{h}, l, u, a0);
        }
        *trials += t0;
    }
    return bad;
}

}  // namespace

int main(int argc, char** argv) {
    const long count = argc > 1 ? std::atol(argv[1]) : 200000;
    std::mt19937_64 rng(argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 1);
    long skipped = 0, trials = 0;
    long bad = run<6>(count, rng, &skipped, &trials);
    bad += run<4>(count, rng, &skipped, &trials);
    bad += run<2>(count / 4, rng, &skipped, &trials);
    std::printf("%ld %ld %ld\n", bad, skipped, trials);
    return bad == 0 ? 0 : 1;
}
