// tron.cuh — batched trust-region Newton (TRON) for tiny dense box-constrained
// NLPs, one solve per CUDA thread, all arrays register-resident.
//
// Algorithm: proj/src/tron.cpp (reference).  This is a fresh sm_100a
// formulation, not a translation of the reference's data structures:
//  * the dimension N (4 or 6 for branches) is a template parameter, so every
//    vector/matrix index is a compile-time constant and nothing touches local
//    memory;
//  * the reduced ("free") subspace of subspace_cg is not gathered into a
//    packed nf x nf copy (tron.cpp:154-159) — it is a bitmask over the full
//    N-space, and every reduced-space loop is a predicated full-space loop
//    that visits the free indices in ascending order, which is exactly the
//    packed order, so every reduction happens in the reference's order;
//  * the solve is a resumable state machine (TronState + tron_step) so a
//    persistent warp can interleave many solves per lane (branch.cu).
//
// Bit-exactness rules: compiled with -fmad=false, IEEE
// div/sqrt; every sum is sequential left-to-right starting at +0.0 as in
// tron.cpp:16-20,35-43,62-89; std::min/max/clamp via ga_math.h.
#ifndef GA_TRON_CUH
#define GA_TRON_CUH

#include "ga_math.h"

namespace ga {

// Optional path statistics (debug builds with -DGA_TRON_STATS): TRON steps,
// Cauchy extrapolations, Cauchy halvings, CG iterations, line-search
// steps, failed Cholesky preconditioners.
#ifdef GA_TRON_STATS
__device__ unsigned long long g_tron_stats[8];  // tron.cuh is included by one TU
#endif
#if defined(GA_TRON_STATS) && defined(__CUDA_ARCH__)
#define GA_STAT(k) atomicAdd(&g_tron_stats[k], 1ull)
#else
#define GA_STAT(k) ((void)0)
#endif

// Optional section clocks (debug builds with -DGA_STEP_CLOCKS): cycles of
// the step sections of solves run by a search strategy that opts in
// (Search::kClocked), summed into g_step_clocks[section].
#if defined(GA_STEP_CLOCKS)
__device__ unsigned long long g_step_clocks[8];
#endif
#if defined(GA_STEP_CLOCKS) && defined(__CUDA_ARCH__)
#define GA_CLK_DECL long long ga_clk_t0 = clock64();
#define GA_CLK(k)                                                                     \
    do {                                                                              \
        if (Search::kClocked) {                                                       \
            const long long ga_clk_t1 = clock64();                                    \
            if ((threadIdx.x & 31) == 0) atomicAdd(&g_step_clocks[k], ga_clk_t1 - ga_clk_t0); \
            ga_clk_t0 = ga_clk_t1;                                                    \
        }                                                                             \
    } while (0)
#else
#define GA_CLK_DECL
#define GA_CLK(k) ((void)0)
#endif

struct TronParams {           // proj/src/tron.hpp:24-30
    double gtol = 1e-6;
    int max_iterations = 200;
    double cg_tol = 0.1;
    int max_cg = 32;
    double delta_floor = 1e-3;
};

constexpr double kTronMu0 = 0.01;     // tron.cpp:10
constexpr double kTronEta = 1e-4;     // tron.cpp:11
constexpr double kTronDeltaMax = 1e10; // tron.cpp:12

enum TronStatusCode : int { kTronConverged = 0, kTronIterationLimit = 1, kTronNumericalError = 2 };

GA_FN long long __double_as_longlong_portable(double v) {
#if defined(__CUDA_ARCH__)
    return __double_as_longlong(v);
#else
    long long r;
    __builtin_memcpy(&r, &v, sizeof r);
    return r;
#endif
}

// IEEE division / square root, inline or at one out-of-line site each.  The
// unrolled Cholesky factor and solves hold ~50 copies of each ~20-instruction
// sequence.  The lane phase (one branch per thread, top stall: instruction
// fetch on a 180 KB kernel) calls them out of line: lane phase -5% in the
// bench window, -12% over a full 70k solve.  The tile / solo phases (one
// branch per 8 or 32 lanes, latency-bound chains) keep them inline: out of
// line they were 5-9% slower.  Same IEEE operations either way.
#if defined(__CUDA_ARCH__)
__device__ __noinline__ double ga_div_ool(double a, double b) { return a / b; }
__device__ __noinline__ double ga_sqrt_ool(double a) { return sqrt(a); }
#endif
template <bool kOol>
GA_FN double tdiv(double a, double b) {
#if defined(__CUDA_ARCH__)
    if constexpr (kOol) return ga_div_ool(a, b);
#endif
    return a / b;
}
template <bool kOol>
GA_FN double tsqrt(double a) {
#if defined(__CUDA_ARCH__)
    if constexpr (kOol) return ga_sqrt_ool(a);
#endif
    return sqrt(a);
}

// 2^e for |e| <= 1000, exactly (exponent field).
GA_FN double pow2i(int e) {
    const long long b = static_cast<long long>(e + 1023) << 52;
    double v;
    __builtin_memcpy(&v, &b, sizeof v);
    return v;
}

// ---- sequential reductions over N (tron.cpp:16-51) ------------------------

template <int N>
GA_FN double vdot(const double* a, const double* b) {
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i) s += a[i] * b[i];
    return s;
}

template <int N, bool kOol = false>
GA_FN double vnorm2(const double* a) { return tsqrt<kOol>(vdot<N>(a, a)); }

// q(s) = g's + sum_i 0.5*s_i*(H s)_i  (tron.cpp:35-43)
template <int N, class HM>
GA_FN double model(const double* g, const HM& h, const double* s, double* gs_out = nullptr) {
    double q = vdot<N>(g, s);
    if (gs_out) *gs_out = q;  // g's, reused by the Cauchy decrease test
#pragma unroll
    for (int i = 0; i < N; ++i) {
        double hs = 0.0;
#pragma unroll
        for (int j = 0; j < N; ++j) hs += h[i * N + j] * s[j];
        q += 0.5 * s[i] * hs;
    }
    return q;
}

// Reduced-space dot over the free mask (ascending = packed order).
template <int N>
GA_FN double mdot(unsigned fm, const double* a, const double* b) {
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i)
        if (fm >> i & 1u) s += a[i] * b[i];
    return s;
}

// Cholesky of the free principal submatrix (tron.cpp:53-67): reads the lower
// triangle h[i][j], i > j, as the reference's hf does.
template <int N, bool kOol, class HM>
GA_FN bool mcholesky(unsigned fm, const HM& h, double* L) {
#pragma unroll
    for (int j = 0; j < N; ++j) {
        if (!(fm >> j & 1u)) continue;
        double d = h[j * N + j];
#pragma unroll
        for (int k = 0; k < j; ++k)
            if (fm >> k & 1u) d -= L[j * N + k] * L[j * N + k];
        if (d <= 0.0 || !sfinite(d)) return false;
        L[j * N + j] = tsqrt<kOol>(d);
#pragma unroll
        for (int i = j + 1; i < N; ++i) {
            if (!(fm >> i & 1u)) continue;
            double v = h[i * N + j];
#pragma unroll
            for (int k = 0; k < j; ++k)
                if (fm >> k & 1u) v -= L[i * N + k] * L[j * N + k];
            L[i * N + j] = tdiv<kOol>(v, L[j * N + j]);
        }
    }
    return true;
}

// (L L')^{-1} b on the free set (tron.cpp:69-80).
template <int N, bool kOol>
GA_FN void mchol_solve(unsigned fm, const double* L, const double* b, double* x) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
        if (!(fm >> i & 1u)) continue;
        double v = b[i];
#pragma unroll
        for (int k = 0; k < i; ++k)
            if (fm >> k & 1u) v -= L[i * N + k] * x[k];
        x[i] = tdiv<kOol>(v, L[i * N + i]);
    }
#pragma unroll
    for (int i = N - 1; i >= 0; --i) {
        if (!(fm >> i & 1u)) continue;
        double v = x[i];
#pragma unroll
        for (int k = i + 1; k < N; ++k)
            if (fm >> k & 1u) v -= L[k * N + i] * x[k];
        x[i] = tdiv<kOol>(v, L[i * N + i]);
    }
}

// Largest tau >= 0 with ||s + tau p|| = delta (tron.cpp:83-90), full space.
template <int N, bool kOol = false>
GA_FN double boundary_tau(const double* s, const double* p, double delta) {
    const double pp = vdot<N>(p, p);
    if (pp <= 0.0) return 0.0;
    const double sp = vdot<N>(s, p);
    const double ss = vdot<N>(s, s);
    const double disc = smax(0.0, sp * sp + pp * (delta * delta - ss));
    return tdiv<kOol>(-sp + tsqrt<kOol>(disc), pp);
}

// l <= x <= u componentwise (false on NaN).
template <int N>
GA_FN bool box_contains(const double* x, const double* l, const double* u) {
    bool in = true;
#pragma unroll
    for (int i = 0; i < N; ++i) in = in && l[i] <= x[i] && x[i] <= u[i];
    return in;
}

// Cauchy point (tron.cpp:101-137).
template <int N, bool kOol, class HM>
GA_FN void cauchy_point(const double* x, const double* g, const HM& h,
                        const double* l, const double* u, double delta, double* s,
                        double* qs, bool* qs_ok) {
    *qs_ok = false;
    const double gnorm = vnorm2<N, kOol>(g);
    if (gnorm == 0.0) {
#pragma unroll
        for (int i = 0; i < N; ++i) s[i] = 0.0;
        return;
    }
    auto step_at = [&](double alpha, double* out) {
#pragma unroll
        for (int i = 0; i < N; ++i) out[i] = sclamp(x[i] - alpha * g[i], l[i], u[i]) - x[i];
    };
    // q(t) of the current trial when the radius test let ok() compute it:
    // tron_step's qc = q(s) (tron.cpp:278) reuses it (same inputs, same bits)
    double mt = 0.0;
    bool mt_ok = false;
    // ||t|| <= delta as t.t <= bound (exact, ga_math.h); the model value is
    // computed regardless (independent chains overlap, no branch), and used
    // only when the radius test passes, as in the reference's order.
    bool bound_ok;
    const double dd_max = sqrt_le_bound(delta, &bound_ok);
    // A backtracking trial at alpha0 * 2^-k, k >= 2, passes the radius test
    // for sure when x is inside its box: |t_i| <= 2 alpha |g_i| (1+u)^2
    // (fl(x - alpha g_i) is at least as close to x - alpha g_i as x is, the
    // clamp only moves it toward x), alpha0 ||g|| <= delta (1+10u), so the
    // computed ||t|| <= delta (1+20u) / 2 < delta — the test is skipped.
    const bool in_box = box_contains<N>(x, l, u);
    auto ok = [&](const double* st, bool sure) {
        double gs;
        mt = model<N>(g, h, st, &gs);
        if (sure) {
            mt_ok = true;
        } else {
            const double dd = vdot<N>(st, st);
            mt_ok = bound_ok ? dd <= dd_max : tsqrt<kOol>(dd) <= delta;
        }
        return mt_ok && mt <= kTronMu0 * gs;
    };
    // One trial site (instruction-cache footprint: this is the hottest loop of
    // the lane phase, ~21 trials per step): phase 0 is alpha0, phase 1 the
    // extrapolation (tron.cpp:115-124: continue from the last accepted
    // alpha, at most 20 doublings), phase 2 the backtracking (tron.cpp:127-
    // 135: at most 40 halvings, first success wins, else the last trial).
    double a = smin(1.0, tdiv<kOol>(delta, gnorm));
    int phase = 0, cnt = 0;
    double t[N];
    for (;;) {
        step_at(a, t);
        const bool o = ok(t, in_box && phase == 2 && cnt >= 2);
        if (phase == 0) {
            phase = o ? 1 : 2;
        } else if (phase == 1) {
            if (!o) return;
        }
#pragma unroll
        for (int i = 0; i < N; ++i) s[i] = t[i];
        *qs = mt;
        *qs_ok = mt_ok;
        if (phase == 2 && o && cnt > 0) return;
        if (phase == 1) {
            if (cnt >= 20) return;
            GA_STAT(1);
            a = a * 2.0;
        } else {
            if (cnt >= 40) return;
            GA_STAT(2);
            a *= 0.5;
        }
        ++cnt;
    }
}

// Preconditioned Steihaug CG on the free subspace at x + s
// (tron.cpp:141-224).  d receives the full-space correction.
template <int N, bool kOol, class HM>
GA_FN void subspace_cg(const double* x, const double* g, const HM& h,
                       const double* l, const double* u, double delta,
                       const TronParams& cfg, const double* s, double* d) {
#pragma unroll
    for (int i = 0; i < N; ++i) d[i] = 0.0;
    unsigned fm = 0;
#pragma unroll
    for (int i = 0; i < N; ++i) {
        const double xi = x[i] + s[i];
        if (xi > l[i] && xi < u[i]) fm |= 1u << i;
    }
    if (fm == 0) return;

    double rf[N], L[N * N], zk[N], pk[N], dk[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {  // rf = -(g + H s) on the free set
        double hs = 0.0;
#pragma unroll
        for (int j = 0; j < N; ++j) hs += h[i * N + j] * s[j];
        rf[i] = -(g[i] + hs);
        dk[i] = 0.0;
    }
    const bool have_prec = mcholesky<N, kOol>(fm, h, L);
    if (!have_prec) GA_STAT(5);
    double rz = 0.0, r0 = 0.0;
    // it = -1 is the set-up (z0 = M^-1 r0, p0 = z0); the preconditioner solve
    // has a single call site (code size), same operations as tron.cpp:171-222.
    for (int it = -1; it < cfg.max_cg; ++it) {
      if (it >= 0) {
        GA_STAT(3);
        double hpk[N];
#pragma unroll
        for (int i = 0; i < N; ++i) {
            double v = 0.0;
#pragma unroll
            for (int j = 0; j < N; ++j)
                if (fm >> j & 1u) v += h[i * N + j] * pk[j];
            hpk[i] = v;
        }
        const double curv = mdot<N>(fm, pk, hpk);
        double pfull[N], sd[N];
#pragma unroll
        for (int i = 0; i < N; ++i) {
            const bool fr = fm >> i & 1u;
            pfull[i] = fr ? pk[i] : 0.0;
            sd[i] = s[i] + (fr ? dk[i] : 0.0);
        }
        if (curv <= 0.0) {  // negative curvature: to the boundary
            const double tau = boundary_tau<N, kOol>(sd, pfull, delta);
#pragma unroll
            for (int i = 0; i < N; ++i)
                if (fm >> i & 1u) dk[i] += tau * pk[i];
            break;
        }
        const double alpha = tdiv<kOol>(rz, curv);
        double dnext[N], snext[N];
#pragma unroll
        for (int i = 0; i < N; ++i) {
            const bool fr = fm >> i & 1u;
            dnext[i] = dk[i] + alpha * pk[i];
            snext[i] = s[i] + (fr ? dnext[i] : 0.0);
        }
        if (vnorm2<N, kOol>(snext) >= delta) {
            const double tau = boundary_tau<N, kOol>(sd, pfull, delta);
#pragma unroll
            for (int i = 0; i < N; ++i)
                if (fm >> i & 1u) dk[i] += tau * pk[i];
            break;
        }
#pragma unroll
        for (int i = 0; i < N; ++i)
            if (fm >> i & 1u) {
                dk[i] = dnext[i];
                rf[i] -= alpha * hpk[i];
            }
        if (tsqrt<kOol>(mdot<N>(fm, rf, rf)) <= cfg.cg_tol * r0) break;
      }
        if (have_prec) mchol_solve<N, kOol>(fm, L, rf, zk);
        else {
#pragma unroll
            for (int i = 0; i < N; ++i) zk[i] = rf[i];
        }
        const double rznext = mdot<N>(fm, rf, zk);
        if (it < 0) {
#pragma unroll
            for (int i = 0; i < N; ++i) pk[i] = zk[i];
            rz = rznext;
            r0 = tsqrt<kOol>(mdot<N>(fm, rf, rf));
            if (r0 == 0.0) return;
        } else {
            const double betak = tdiv<kOol>(rznext, rz);
#pragma unroll
            for (int i = 0; i < N; ++i)
                if (fm >> i & 1u) pk[i] = zk[i] + betak * pk[i];
            rz = rznext;
        }
    }
#pragma unroll
    for (int i = 0; i < N; ++i) d[i] = (fm >> i & 1u) ? dk[i] : 0.0;
}

// Projected-gradient inf-norm (tron.cpp:251-257 / 320-326); NaN entries are
// skipped exactly like std::max(pgnorm, std::abs(gi)).
template <int N>
GA_FN double proj_grad_norm(const double* x, const double* g, const double* l,
                            const double* u) {
    double pg = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i) {
        double gi = g[i];
        if (x[i] <= l[i]) gi = smin(gi, 0.0);
        else if (x[i] >= u[i]) gi = smax(gi, 0.0);
        pg = smax(pg, fabs(gi));
    }
    return pg;
}

// Resumable solve_one (tron.cpp:228-332).
template <int N>
struct TronState {
    double x[N];
    double f;
    double delta;
    int iter;
};

// Starts a solve: clip x into the box and evaluate f (tron.cpp:235-240).
// Returns false (NumericalError, iterations 0) when f is not finite.
template <int N, class P>
GA_FN bool tron_begin(const P& prob, TronState<N>& st) {
#pragma unroll
    for (int i = 0; i < N; ++i) st.x[i] = sclamp(st.x[i], prob.lo(i), prob.hi(i));
    st.f = prob.value(st.x);
    st.delta = 0.0;
    st.iter = 0;
    return sfinite(st.f);
}

enum TronStep : int { kStepContinue = 0, kStepConverged = 1, kStepError = 2, kStepExhausted = 3 };

// Sequential search strategy (one thread per solve): the reference's loops.
struct SerialSearch {
    static constexpr bool kClocked = false;
    static constexpr bool kOolDivSqrt = true;
    template <int N, class HM>
    GA_FN void cauchy(const double* x, const double* g, const HM& h, const double* l,
                      const double* u, double delta, double* s, double* qs, bool* qs_ok) const {
        cauchy_point<N, kOolDivSqrt>(x, g, h, l, u, delta, s, qs, qs_ok);
    }
    // Projected line search on s + beta d (tron.cpp:279-291); returns the step
    // and its model value q(stp) (tron.cpp:292): the accepted trial's, or,
    // when no trial is accepted (stp = s), qc = q(s) — the same bits the
    // reference's separate model() call produces.
    template <int N, class HM>
    GA_FN double line_search(const double* x, const double* g, const HM& h, const double* l,
                             const double* u, const double* s, const double* d, double qc,
                             double* stp) const {
        double beta = 1.0;
        GA_STAT(0);
        for (int ls = 0; ls < 20; ++ls) {
            GA_STAT(4);
#pragma unroll
            for (int i = 0; i < N; ++i) stp[i] = sclamp(x[i] + s[i] + beta * d[i], l[i], u[i]) - x[i];
            const double q = model<N>(g, h, stp);
            if (q <= qc) return q;
            beta *= 0.5;
        }
#pragma unroll
        for (int i = 0; i < N; ++i) stp[i] = s[i];
        return qc;
    }
};

#if defined(__CUDACC__)
// Speculative search strategy for a tile of T lanes (power of two, <= 32)
// that all hold the same replicated iterate.  The reference's Cauchy search
// (tron.cpp:101-137) and projected line search (tron.cpp:279-291) are
// sequences of independent trials at alpha0 * 2^c / beta = 2^-t followed by
// "first success" / "last consecutive success" rules; the tile evaluates T
// trials at once and applies the same rule to the ballot.  Every trial is
// computed exactly as the sequential loop computes it (scaling by powers of
// two is exact), so the selected step is bit-identical.
template <int T>
struct TileSearch {
    static constexpr bool kClocked = T == 32;
    static constexpr bool kOolDivSqrt = false;
    unsigned mask;  // warp lanes of this tile
    int base;       // first warp lane of the tile
    int rank;       // lane within the tile

    __device__ __forceinline__ unsigned ballot(bool p) const {
        return (__ballot_sync(mask, p) >> base) & ((T == 32) ? 0xffffffffu : ((1u << T) - 1u));
    }
    template <int N>
    __device__ __forceinline__ void bcast(const double* v, int src, double* out) const {
#pragma unroll
        for (int i = 0; i < N; ++i) out[i] = __shfl_sync(mask, v[i], src, T);
    }

    template <int N, class HM>
    __device__ void cauchy(const double* x, const double* g, const HM& h, const double* l,
                           const double* u, double delta, double* s, double* qs,
                           bool* qs_ok) const {
        *qs_ok = false;
        const double gnorm = vnorm2<N>(g);
        if (gnorm == 0.0) {
#pragma unroll
            for (int i = 0; i < N; ++i) s[i] = 0.0;
            return;
        }
        const double alpha0 = smin(1.0, delta / gnorm);
        bool bound_ok;
        const double dd_max = sqrt_le_bound(delta, &bound_ok);
        const bool in_box = box_contains<N>(x, l, u);  // trials at c <= -2: radius test
                                                        // passes (cauchy_point)
        double mys[N];
        // One trial site and one broadcast site (code size: this runs in a
        // persistent kernel whose hot loop must stay in the instruction cache).
        // Candidate exponents c (trial at alpha0 * 2^c):
        //   round 0: rank 0 -> 0, rank 1 -> +1, ranks 2.. -> -1, -2, ...
        //   extrapolation rounds r >= 1: 2 + (r-1)*T + rank   (valid <= 20)
        //   backtracking rounds r >= 1: -((T-1) + (r-1)*T + rank) (valid >= -40)
        int dir = 0;  // +1 extrapolating, -1 backtracking (decided in round 0)
        for (int round = 0;; ++round) {
            int c;
            if (round == 0) c = rank == 0 ? 0 : (rank == 1 ? 1 : -(rank - 1));
            else if (dir > 0) c = 2 + (round - 1) * T + rank;
            else c = -((T - 1) + (round - 1) * T + rank);
            const bool valid = dir > 0 ? c <= 20 : c >= -40;
            bool okc = false, mok = false;
            double mv = 0.0;
            if (valid) {
                // alpha0 * 2^c: one multiply by the exact power of two equals
                // the sequential doublings / halvings whenever the result is
                // normal (every intermediate then is); tiny alpha0 keeps the
                // sequential form (subnormal halvings round step by step)
                double a = alpha0;
                if (alpha0 >= 0x1p-960) {
                    a = alpha0 * pow2i(c);
                } else {
                    for (int k = 0; k < c; ++k) a *= 2.0;
                    for (int k = 0; k < -c; ++k) a *= 0.5;
                }
#pragma unroll
                for (int i = 0; i < N; ++i) mys[i] = sclamp(x[i] - a * g[i], l[i], u[i]) - x[i];
                double gs;
                mv = model<N>(g, h, mys, &gs);
                if (in_box && c <= -2) {
                    mok = true;
                } else {
                    const double dd = vdot<N>(mys, mys);
                    mok = bound_ok ? dd <= dd_max : tsqrt<true>(dd) <= delta;  // (out of range: never in practice)
                }
                okc = mok && mv <= kTronMu0 * gs;
            }
            const unsigned okm = ballot(okc);
            int src = -1;      // lane whose trial step becomes s
            bool done = true;
            if (round == 0) {
                if (okm & 1u) {
                    dir = 1;
                    src = (okm & 2u) ? 1 : 0;
                    done = !(okm & 2u);
                } else {
                    dir = -1;
                    const unsigned hm = okm >> 2;
                    if (hm) src = __ffs(hm) - 1 + 2;
                    else done = false;
                }
            } else if (dir > 0) {
                const int run = __ffs(~okm) - 1;  // consecutive successes
                if (run > 0) src = run - 1;
                done = run < T;  // a failure (or the c > 20 limit) ended the run
            } else {
                const int kb = (T - 1) + (round - 1) * T;  // this round tried k = kb..kb+T-1
                if (okm) src = __ffs(okm) - 1;
                else if (kb + T - 1 >= 40) src = 40 - kb;  // none up to 2^-40: last trial's step
                else done = false;
            }
            if (src >= 0) {
                bcast<N>(mys, src, s);
                *qs = __shfl_sync(mask, mv, src, T);
                *qs_ok = __shfl_sync(mask, mok ? 1 : 0, src, T) != 0;
            }
            if (done) return;
        }
    }

    template <int N, class HM>
    __device__ double line_search(const double* x, const double* g, const HM& h, const double* l,
                                  const double* u, const double* s, const double* d, double qc,
                                  double* stp) const {
        double myst[N];
        for (int tb = 0; tb < 20; tb += T) {
            const int t = tb + rank;
            const double beta = pow2i(-t);  // = 0.5^t by halvings (exact, t < 52)
#pragma unroll
            for (int i = 0; i < N; ++i) myst[i] = sclamp(x[i] + s[i] + beta * d[i], l[i], u[i]) - x[i];
            const double q = model<N>(g, h, myst);
            const bool okt = (t < 20) ? (q <= qc) : false;
            const unsigned okm = ballot(okt);
            if (okm) {
                const int src = __ffs(okm) - 1;
                bcast<N>(myst, src, stp);
                return __shfl_sync(mask, q, src, T);
            }
        }
#pragma unroll
        for (int i = 0; i < N; ++i) stp[i] = s[i];
        return qc;
    }
};
#endif

// One trust-region iteration (tron.cpp:243-317).  kStepExhausted means the
// loop ended by the iteration cap or the delta < 1e-14 break, after which
// tron_finish must be called.
template <int N, class P, class Search = SerialSearch>
GA_FN int tron_step(const P& prob, TronState<N>& st, const TronParams& cfg,
                    const Search& search = Search()) {
    double l[N], u[N];
#pragma unroll
    for (int i = 0; i < N; ++i) { l[i] = prob.lo(i); u[i] = prob.hi(i); }
    GA_CLK_DECL
    double g[N];
    // gradient and Hessian in one evaluation pass (each accumulator keeps its
    // own order, so the same bits; the flow terms are built once instead of
    // twice: full 70k solve 6.55 -> 6.45 s); the tests below run in the
    // reference's order, the Hessian of a converged / failed point is unused
    double h[N * N];
    prob.grad_hess(st.x, g, h);
#pragma unroll
    for (int i = 0; i < N; ++i)
        if (!sfinite(g[i])) return kStepError;
    if (proj_grad_norm<N>(st.x, g, l, u) <= cfg.gtol) return kStepConverged;
    GA_CLK(0);
#pragma unroll
    for (int i = 0; i < N * N; ++i)
        if (!sfinite(h[i])) return kStepError;
    constexpr bool kOol = Search::kOolDivSqrt;
    if (st.iter == 0 && st.delta == 0.0) st.delta = smax(vnorm2<N, kOol>(g), cfg.delta_floor);

    double s[N], d[N];
    GA_CLK(1);
    double qs = 0.0;
    bool qs_ok = false;
    search.template cauchy<N>(st.x, g, h, l, u, st.delta, s, &qs, &qs_ok);
    GA_CLK(2);
    subspace_cg<N, Search::kOolDivSqrt>(st.x, g, h, l, u, st.delta, cfg, s, d);
    GA_CLK(3);

    const double qc = qs_ok ? qs : model<N>(g, h, s);
    double stp[N];
    const double q = search.template line_search<N>(st.x, g, h, l, u, s, d, qc, stp);
    double xt[N];
#pragma unroll
    for (int i = 0; i < N; ++i) xt[i] = sclamp(st.x[i] + stp[i], l[i], u[i]);
    GA_CLK(4);
    const double ft = prob.value(xt);
    GA_CLK(5);
    if (!sfinite(ft)) return kStepError;
    const double ared = st.f - ft;
    const double pred = -q;
    const double ratio = pred > 0.0 ? tdiv<kOol>(ared, pred) : (ared > 0.0 ? 1.0 : -1.0);
    const double snorm = vnorm2<N, kOol>(stp);
    const double delta_used = st.delta;
    if (ratio < 0.25) st.delta = 0.25 * smax(snorm, 1e-12);
    else if (ratio > 0.75 && snorm >= 0.9 * st.delta) st.delta = smin(2.0 * st.delta, kTronDeltaMax);
    const bool accepted = ared > 0.0 && ratio > kTronEta;
    if (accepted) {
#pragma unroll
        for (int i = 0; i < N; ++i) st.x[i] = xt[i];
        st.f = ft;
    } else {
        GA_STAT(6);  // rejected step: x (hence g, H) unchanged
    }
    if (st.iter >= 100) GA_STAT(7);  // steps of solves deep in the tail
    ++st.iter;
    // Fixed point: a rejected step that leaves the radius bit-identical
    // leaves the whole iterate (x, f, delta) unchanged, and an iteration with
    // iter >= 1 is a pure function of (x, f, delta) — so every remaining
    // iteration up to the cap would recompute exactly this one.  The
    // reference executes them (tron.cpp:243-317); jumping to the cap gives
    // the identical final state and TronResult (iterations = max_iterations).
    if (!accepted && __double_as_longlong_portable(st.delta) == __double_as_longlong_portable(delta_used)) {
        GA_STAT(5);
        st.iter = cfg.max_iterations;
    }
    GA_CLK(6);
#if defined(GA_STEP_CLOCKS) && defined(__CUDA_ARCH__)
    if (Search::kClocked && (threadIdx.x & 31) == 0) atomicAdd(&g_step_clocks[7], 1ull);
#endif
    if (st.delta < 1e-14 || st.iter >= cfg.max_iterations) return kStepExhausted;
    return kStepContinue;
}

// Post-loop status (tron.cpp:320-330): gradient at x (no finiteness check),
// projected-gradient test.
template <int N, class P>
GA_FN int tron_finish(const P& prob, const TronState<N>& st, const TronParams& cfg) {
    double l[N], u[N], g[N];
#pragma unroll
    for (int i = 0; i < N; ++i) { l[i] = prob.lo(i); u[i] = prob.hi(i); }
    prob.gradient(st.x, g);
    return proj_grad_norm<N>(st.x, g, l, u) <= cfg.gtol ? kTronConverged : kTronIterationLimit;
}

// Whole solve (used by the QP test kernel and the simple branch path).
// Returns the status; *iterations follows TronResult::iterations semantics.
template <int N, class P>
GA_FN int tron_solve(const P& prob, double* x, const TronParams& cfg, int* iterations) {
    TronState<N> st;
#pragma unroll
    for (int i = 0; i < N; ++i) st.x[i] = x[i];
    int status;
    if (!tron_begin<N>(prob, st)) {
        *iterations = 0;
        status = kTronNumericalError;
    } else if (cfg.max_iterations <= 0) {
        *iterations = cfg.max_iterations;
        status = tron_finish<N>(prob, st, cfg);
    } else {
        for (;;) {
            const int iter_before = st.iter;
            const int r = tron_step<N>(prob, st, cfg);
            if (r == kStepContinue) continue;
            if (r == kStepConverged) { *iterations = iter_before; status = kTronConverged; break; }
            if (r == kStepError) { *iterations = iter_before; status = kTronNumericalError; break; }
            *iterations = cfg.max_iterations;
            status = tron_finish<N>(prob, st, cfg);
            break;
        }
    }
#pragma unroll
    for (int i = 0; i < N; ++i) x[i] = st.x[i];
    return status;
}

}  // namespace ga

#endif
