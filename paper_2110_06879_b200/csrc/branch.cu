// branch.cu — the branch-NLP phase (north-star (b)): per branch, an
// augmented-Lagrangian loop on the line limits around a register-resident
// TRON solve of the 4- or 6-variable branch subproblem (Eq. 4 of the paper).
//
// Reference semantics: proj/src/kernels.cpp:17-192 (BranchProblem, eval,
// consensus values) and :211-292 (solve_branch_batch).
//
// Scheduling (the B200 design; the reference's is a static block partition
// over threads, proj/src/parallel.hpp:13-33): the TRON cost per branch is
// heavy-tailed (median 2-3 iterations, 10-40% at the 200 cap), so a
// thread-per-branch grid leaves whole warps waiting on one capped branch.
// Instead a persistent grid of warps drains two work queues (rate-limited
// 6-variable branches, unlimited 4-variable ones), each ordered by the
// branch's TRON iteration count in the previous sweep, longest first
// (LPT).  Each lane owns one branch at a time and advances it ONE trust-region
// iteration per loop trip; when its solve ends (converged / cap / error /
// AL round done) the lane finalizes the branch and immediately refills from
// the queue with a warp-aggregated atomic, so lanes stay busy until the queue
// is empty.  Per-lane problem data (48 doubles) lives in shared memory in a
// [field][lane] layout (conflict-free), the TRON iterate and all per-iteration
// vectors/matrices in registers.  Results do not depend on the schedule: each
// branch's arithmetic is identical wherever it runs.
//
// Bit-exactness notes:
//  * eval accumulation order is the reference's: rows 0-3 (flows), 4 (w_i),
//    6 (w_j), then the angle rows 5, 7, then limit ij, limit ji
//    (kernels.cpp:124-162);
//  * terms that are structurally zero in the reference's dense Quad4
//    arithmetic are skipped.  This is exact: every skipped term is a signed
//    zero added into an accumulator that starts at +0.0 and therefore can
//    never hold -0.0, so x + (+-0) == x bit-for-bit (and an intermediate
//    whose only difference is the sign of a zero only ever reaches such an
//    accumulator through products);
//  * the gradient and Hessian of one TRON iteration share one pinned sincos
//    (the reference recomputes it; same input, same bits).
#include <climits>

#include "device.hpp"
#include "ga_math.h"
#include "ga_sincos.h"
#include "tron.cuh"

namespace ga {

void tron_stats(unsigned long long out[8], bool reset) {
#ifdef GA_TRON_STATS
    cudaMemcpyFromSymbol(out, g_tron_stats, 8 * sizeof(unsigned long long));
    if (reset) {
        const unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        cudaMemcpyToSymbol(g_tron_stats, z, sizeof z);
    }
#else
    (void)reset;
    for (int k = 0; k < 8; ++k) out[k] = 0;
#endif
}

namespace {

constexpr double kTwoPi = 6.283185307179586;  // 2.0 * std::numbers::pi
constexpr double kLtBound = 1e8;              // kernels.cpp:16
constexpr int kMaxAl = 10;                    // kernels.cpp:219
constexpr double kAlTol = 1e-8;
constexpr double kAlShrink = 0.25;
constexpr double kRhoTildeMax = 1e7;

constexpr int kBranchBlock = 128;  // threads per block of the persistent kernel
constexpr int kCostBuckets = 256;  // LPT ordering buckets (cost >> 2, capped)

// ---- per-lane problem data in shared memory ------------------------------
// Field indices of the [field][lane] layout.
enum Field : int {
    F_YC = 0,     // 8 admittance coefficients gii bii gij bij gji bji gjj bjj
    F_TGT = 8,    // 8 bus-side targets (xbar rows)
    F_Y = 16,     // 8 multipliers y
    F_Z = 24,     // 8 artificial z
    F_RHO = 32,   // 8 penalties
    F_LTIJ = 40, F_LTJI = 41, F_RHOT = 42,
    F_VMIN_I = 43, F_VMAX_I = 44, F_VMIN_J = 45, F_VMAX_J = 46, F_R2 = 47,
    kFields = 48
};

template <int BS>
struct Slot {
    double* p;  // smem + threadIdx.x
    GA_FN double operator()(int f) const { return p[f * BS]; }
    GA_FN void set(int f, double v) const { p[f * BS] = v; }
};

// Flow quantities (value, gradient over vi,vj,thi,thj, Hessian) of the four
// branch flows in BranchRow order, built from the basis functions
// wi, wj, wr, wim (kernels.cpp:25-87).  Hessian entries that are structural
// zeros of the reference's Quad4 arithmetic are never read.
struct Flows {
    double v[4];
    double g[4][4];
    double h[4][16];
};

struct Basis {
    double vi, vj, c, s;
    double vivj, nvivj;
};

GA_FN Basis make_basis(double vi, double vj, double c, double s) {
    Basis b;
    b.vi = vi; b.vj = vj; b.c = c; b.s = s;
    b.vivj = vi * vj;
    b.nvivj = (-vi) * vj;
    return b;
}

// wr and wim gradient entries (kernels.cpp:40,50)
GA_FN double wr_g(const Basis& b, int i) {
    switch (i) {
        case 0: return b.vj * b.c;
        case 1: return b.vi * b.c;
        case 2: return b.nvivj * b.s;
        default: return b.vivj * b.s;
    }
}
GA_FN double wim_g(const Basis& b, int i) {
    switch (i) {
        case 0: return b.vj * b.s;
        case 1: return b.vi * b.s;
        case 2: return b.vivj * b.c;
        default: return b.nvivj * b.c;
    }
}
// wr / wim Hessian entry (i, j) (kernels.cpp:41-48, 51-58); (0,0),(1,1) are 0.
GA_FN double wr_h(const Basis& b, int i, int j) {
    const int a = i < j ? i : j, c = i < j ? j : i;
    if (a == 0 && c == 1) return b.c;
    if (a == 0 && c == 2) return (-b.vj) * b.s;
    if (a == 0 && c == 3) return b.vj * b.s;
    if (a == 1 && c == 2) return (-b.vi) * b.s;
    if (a == 1 && c == 3) return b.vi * b.s;
    if (a == 2 && c == 2) return b.nvivj * b.c;
    if (a == 3 && c == 3) return b.nvivj * b.c;
    return b.vivj * b.c;  // (2,3)
}
GA_FN double wim_h(const Basis& b, int i, int j) {
    const int a = i < j ? i : j, c = i < j ? j : i;
    if (a == 0 && c == 1) return b.s;
    if (a == 0 && c == 2) return b.vj * b.c;
    if (a == 0 && c == 3) return (-b.vj) * b.c;
    if (a == 1 && c == 2) return b.vi * b.c;
    if (a == 1 && c == 3) return (-b.vi) * b.c;
    if (a == 2 && c == 2) return b.nvivj * b.s;
    if (a == 3 && c == 3) return b.nvivj * b.s;
    return b.vivj * b.s;  // (2,3)
}

// Flow k uses A = wi (k < 2, index a = 0) or wj (k >= 2, a = 1) and the
// coefficients of flow_quads (kernels.cpp:80-87).
template <bool WG, bool WH, class Y>
GA_FN void make_flows(const Basis& b, const Y& yc, Flows& F) {
    // yc(k): gii bii gij bij gji bji gjj bjj
    const double ca[4] = {yc(0), -yc(1), yc(6), -yc(7)};
    const double cb[4] = {yc(2), -yc(3), yc(4), -yc(5)};
    const double cc[4] = {yc(3), yc(2), -yc(5), -yc(4)};
    const double wi_v = b.vi * b.vi, wj_v = b.vj * b.vj;
    const double wr_v = b.vivj * b.c, wim_v = b.vivj * b.s;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int a = k < 2 ? 0 : 1;
        const double av = a == 0 ? wi_v : wj_v;
        F.v[k] = ca[k] * av + cb[k] * wr_v + cc[k] * wim_v;
        if (WG || WH) {
            const double ag = a == 0 ? 2 * b.vi : 2 * b.vj;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                if (i == a) F.g[k][i] = ca[k] * ag + cb[k] * wr_g(b, i) + cc[k] * wim_g(b, i);
                else F.g[k][i] = cb[k] * wr_g(b, i) + cc[k] * wim_g(b, i);
            }
        }
        if (WH) {
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    if (i == a && j == a) F.h[k][i * 4 + j] = ca[k] * 2.0;
                    else if (i == 1 - a && j == 1 - a) F.h[k][i * 4 + j] = 0.0;  // never read
                    else F.h[k][i * 4 + j] = cb[k] * wr_h(b, i, j) + cc[k] * wim_h(b, i, j);
                }
        }
    }
}

// Structural-zero masks of the flow Hessians: (1,1) for flows 0-1, (0,0)
// for flows 2-3.
GA_FN bool flow_h_zero(int k, int i, int j) {
    const int na = k < 2 ? 1 : 0;
    return i == na && j == na;
}

template <int BS>
struct YcView {
    Slot<BS> s;
    GA_FN double operator()(int k) const { return s(F_YC + k); }
};

// The branch subproblem over a shared-memory slot (kernels.cpp:17-163).
template <int N, int BS>
struct BranchProb {
    static constexpr bool kLimited = N == 6;
    Slot<BS> s;
    mutable double cc_, ss_;  // sincos at the last gradient point

    GA_FN double lo(int i) const {
        switch (i) {
            case 0: return s(F_VMIN_I);
            case 1: return s(F_VMIN_J);
            case 2: case 3: return -kTwoPi;
            default: return -s(F_R2);
        }
    }
    GA_FN double hi(int i) const {
        switch (i) {
            case 0: return s(F_VMAX_I);
            case 1: return s(F_VMAX_J);
            case 2: case 3: return kTwoPi;
            default: return 0.0;
        }
    }

    // f, g, H of Eq. (4) at x (kernels.cpp:103-163).
    template <bool WF, bool WG, bool WH>
    GA_FN void eval(const double* x, double c, double sn, double* f, double* g, double* h) const {
        if (WF) *f = 0.0;
        if (WG) {
#pragma unroll
            for (int i = 0; i < N; ++i) g[i] = 0.0;
        }
        if (WH) {
#pragma unroll
            for (int i = 0; i < N * N; ++i) h[i] = 0.0;
        }
        const Basis b = make_basis(x[0], x[1], c, sn);
        Flows F;
        make_flows<WG, WH>(b, YcView<BS>{s}, F);

        // flows, rows 0..3
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const double rh = s(F_RHO + k), yv = s(F_Y + k);
            const double d = F.v[k] - s(F_TGT + k) + s(F_Z + k);
            const double w = yv + rh * d;
            if (WF) *f += yv * d + 0.5 * rh * d * d;
            if (WG) {
#pragma unroll
                for (int i = 0; i < 4; ++i) g[i] += w * F.g[k][i];
            }
            if (WH) {
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const double gg = rh * F.g[k][i] * F.g[k][j];
                        if (flow_h_zero(k, i, j)) h[i * N + j] += gg;
                        else h[i * N + j] += w * F.h[k][i * 4 + j] + gg;
                    }
            }
        }
        // w_i (row 4) then w_j (row 6): e = v^2, grad 2v on one index, hess 2.
#pragma unroll
        for (int t = 0; t < 2; ++t) {
            const int row = t == 0 ? 4 : 6;
            const int a = t;  // variable index of v
            const double v = x[a];
            const double ev = v * v;
            const double eg = 2 * v;
            const double rh = s(F_RHO + row), yv = s(F_Y + row);
            const double d = ev - s(F_TGT + row) + s(F_Z + row);
            const double w = yv + rh * d;
            if (WF) *f += yv * d + 0.5 * rh * d * d;
            if (WG) g[a] += w * eg;
            if (WH) h[a * N + a] += w * 2.0 + rh * eg * eg;
        }
        // angle rows 5 (thi, var 2) and 7 (thj, var 3) are linear
#pragma unroll
        for (int t = 0; t < 2; ++t) {
            const int row = t == 0 ? 5 : 7;
            const int i = 2 + t;
            const double rh = s(F_RHO + row), yv = s(F_Y + row);
            const double d = x[i] - s(F_TGT + row) + s(F_Z + row);
            if (WF) *f += yv * d + 0.5 * rh * d * d;
            if (WG) g[i] += yv + rh * d;
            if (WH) h[i * N + i] += rh;
        }
        if constexpr (kLimited) {
            const double rho_t = s(F_RHOT);
            // line-limit AL terms: res = p^2 + q^2 + s (kernels.cpp:146-162)
#pragma unroll
            for (int t = 0; t < 2; ++t) {
                const int kp = t == 0 ? 0 : 2, kq = kp + 1;
                const int srow = 4 + t;
                const double lt = s(t == 0 ? F_LTIJ : F_LTJI);
                const double pv = F.v[kp], qv = F.v[kq];
                const double res = pv * pv + qv * qv + x[srow];
                const double w = lt + rho_t * res;
                if (WF) *f += lt * res + 0.5 * rho_t * res * res;
                if (WG || WH) {
                    double gr[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) gr[i] = 2 * pv * F.g[kp][i] + 2 * qv * F.g[kq][i];
                    if (WG) {
#pragma unroll
                        for (int i = 0; i < 4; ++i) g[i] += w * gr[i];
                        g[srow] += w * 1.0;
                    }
                    if (WH) {
                        const double w2 = w * 2.0;
#pragma unroll
                        for (int i = 0; i < 4; ++i)
#pragma unroll
                            for (int j = 0; j < 4; ++j) {
                                double acc;
                                if (flow_h_zero(kp, i, j))
                                    acc = F.g[kp][i] * F.g[kp][j] + F.g[kq][i] * F.g[kq][j];
                                else
                                    acc = F.g[kp][i] * F.g[kp][j] + pv * F.h[kp][i * 4 + j] +
                                          F.g[kq][i] * F.g[kq][j] + qv * F.h[kq][i * 4 + j];
                                h[i * N + j] += w2 * acc;
                            }
                        // rho_t * gr gr' over all n with gr[srow] = 1, other slack 0
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
#pragma unroll
                            for (int j = 0; j < 4; ++j) h[i * N + j] += rho_t * gr[i] * gr[j];
                            h[i * N + srow] += rho_t * gr[i] * 1.0;
                        }
#pragma unroll
                        for (int j = 0; j < 4; ++j) h[srow * N + j] += rho_t * 1.0 * gr[j];
                        h[srow * N + srow] += rho_t * 1.0 * 1.0;
                    }
                }
            }
        }
    }

    GA_FN double value(const double* x) const {
        double c, sn, f;
        ga_sincos(x[2] - x[3], &sn, &c);
        eval<true, false, false>(x, c, sn, &f, nullptr, nullptr);
        return f;
    }
    GA_FN void gradient(const double* x, double* g) const {
        ga_sincos(x[2] - x[3], &ss_, &cc_);
        eval<false, true, false>(x, cc_, ss_, nullptr, g, nullptr);
    }
    // Called by TRON right after gradient() at the same x.
    GA_FN void hessian(const double* x, double* h) const {
        eval<false, false, true>(x, cc_, ss_, nullptr, nullptr, h);
    }
};

// branch_flows (netdata.cpp:33-45)
template <class Y>
GA_FN void branch_flows(const Y& yc, double vi, double vj, double thi, double thj, double* out) {
    double s, c;
    ga_sincos(thi - thj, &s, &c);
    const double wi = vi * vi, wj = vj * vj;
    const double wr = vi * vj * c, wim = vi * vj * s;
    out[0] = yc(0) * wi + yc(2) * wr + yc(3) * wim;     // pij
    out[1] = -yc(1) * wi - yc(3) * wr + yc(2) * wim;    // qij
    out[2] = yc(6) * wj + yc(4) * wr - yc(5) * wim;     // pji
    out[3] = -yc(7) * wj - yc(5) * wr - yc(4) * wim;    // qji
}

// Fills this lane's slot for branch b (kernels.cpp:229-241).
template <int BS>
__device__ __forceinline__ void load_slot(const DevNet& net, const DevState& st,
                                          const BranchCfg& cfg, int b, Slot<BS> s) {
    const int from = net.br_from[b], to = net.br_to[b];
#pragma unroll
    for (int k = 0; k < 8; ++k) s.set(F_YC + k, __ldg(&net.br_y[k * net.nl + b]));
    const int base = 2 * net.ng + 8 * b;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        s.set(F_TGT + k, st.xbar[base + k]);
        s.set(F_Y + k, st.y[base + k]);
        s.set(F_Z + k, st.z[base + k]);
        s.set(F_RHO + k, st.rho[base + k]);
    }
    s.set(F_LTIJ, st.lt_ij[b]);
    s.set(F_LTJI, st.lt_ji[b]);
    s.set(F_RHOT, st.rho_t[b]);
    s.set(F_VMIN_I, __ldg(&net.b_vmin[from]));
    s.set(F_VMAX_I, __ldg(&net.b_vmax[from]));
    s.set(F_VMIN_J, __ldg(&net.b_vmin[to]));
    s.set(F_VMAX_J, __ldg(&net.b_vmax[to]));
    const double rt = cfg.limit_tighten * __ldg(&net.br_rate[b]);
    s.set(F_R2, rt * rt);
}

struct Queue {
    const int* order;  // branch indices, longest expected first
    int count;
    int* counter;      // next index to hand out
};

// Drains one queue with per-lane refill (see file header).
template <int N, int BS>
__device__ __noinline__ void drain_queue(const DevNet& net, const DevState& st,
                                         const BranchCfg& cfg, const Queue q, int* cost,
                                         double* smem, unsigned long long* iters_out,
                                         int* fail_out) {
    constexpr unsigned kFull = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const Slot<BS> slot{smem + threadIdx.x};
    BranchProb<N, BS> p{slot};
    TronParams tp;
    tp.gtol = cfg.gtol;
    tp.max_iterations = cfg.max_iterations;
    tp.cg_tol = cfg.cg_tol;
    tp.max_cg = cfg.max_cg;
    tp.delta_floor = cfg.delta_floor;
    const double kInf = __longlong_as_double(0x7ff0000000000000LL);

    TronState<N> ts;
    int b = -1;
    bool exhausted = false;
    int al_it = 0, iters = 0;
    double prev_res = kInf;
    unsigned long long my_iters = 0;
    int my_fail = 0;

    // Branch done: restore on failure, write back (kernels.cpp:273-281).
    auto finalize = [&](bool failed) {
        double pt[6];
#pragma unroll
        for (int k = 0; k < N; ++k) pt[k] = failed ? st.bp[k * net.nl + b] : ts.x[k];
        st.lt_ij[b] = slot(F_LTIJ);
        st.lt_ji[b] = slot(F_LTJI);
        st.rho_t[b] = slot(F_RHOT);
        if (!failed) {
#pragma unroll
            for (int k = 0; k < N; ++k) st.bp[k * net.nl + b] = pt[k];
        }
        double fl[4];
        branch_flows(YcView<BS>{slot}, pt[0], pt[1], pt[2], pt[3], fl);
        const int base = 2 * net.ng + 8 * b;
        double2* xr = reinterpret_cast<double2*>(st.x + base);
        xr[0] = make_double2(fl[0], fl[1]);
        xr[1] = make_double2(fl[2], fl[3]);
        xr[2] = make_double2(pt[0] * pt[0], pt[2]);
        xr[3] = make_double2(pt[1] * pt[1], pt[3]);
        cost[b] = iters;
        my_iters += iters;
        my_fail += failed ? 1 : 0;
        b = -1;
    };
    // A TRON solve ended with `status`: AL bookkeeping (kernels.cpp:246-271);
    // either restarts TRON for the next AL round or finalizes the branch.
    auto after_solve = [&](int status) {
        for (;;) {
            if (status == kTronNumericalError) { finalize(true); return; }
            if constexpr (N == 4) {
                finalize(false);
                return;
            } else {
                double fl[4];
                branch_flows(YcView<BS>{slot}, ts.x[0], ts.x[1], ts.x[2], ts.x[3], fl);
                const double rij = fl[0] * fl[0] + fl[1] * fl[1] + ts.x[4];
                const double rji = fl[2] * fl[2] + fl[3] * fl[3] + ts.x[5];
                const double res = smax(fabs(rij), fabs(rji));
                if (res <= kAlTol) { finalize(false); return; }
                const double rho_t = slot(F_RHOT);
                slot.set(F_LTIJ, sclamp(slot(F_LTIJ) + rho_t * rij, -kLtBound, kLtBound));
                slot.set(F_LTJI, sclamp(slot(F_LTJI) + rho_t * rji, -kLtBound, kLtBound));
                if (res > kAlShrink * prev_res) slot.set(F_RHOT, smin(10.0 * rho_t, kRhoTildeMax));
                prev_res = res;
                if (++al_it >= kMaxAl) { finalize(false); return; }
                if (tron_begin<N>(p, ts)) return;  // next AL round runs in the loop
                status = kTronNumericalError;
            }
        }
    };

    for (;;) {
        // refill idle lanes: one atomic per warp
        const unsigned need = __ballot_sync(kFull, b < 0 && !exhausted);
        if (need) {
            const int leader = __ffs(need) - 1;
            int base = 0;
            if (lane == leader) base = atomicAdd(q.counter, __popc(need));
            base = __shfl_sync(kFull, base, leader);
            if (need >> lane & 1u) {
                const int idx = base + __popc(need & ((1u << lane) - 1u));
                if (idx < q.count) {
                    b = q.order[idx];
                    load_slot<BS>(net, st, cfg, b, slot);
#pragma unroll
                    for (int k = 0; k < N; ++k) ts.x[k] = st.bp[k * net.nl + b];
                    al_it = 0;
                    iters = 0;
                    prev_res = kInf;
                    if (!tron_begin<N>(p, ts)) after_solve(kTronNumericalError);
                } else {
                    exhausted = true;
                }
            }
        }
        if (__all_sync(kFull, b < 0 && exhausted)) break;
        if (b >= 0) {
            const int iter_before = ts.iter;
            const int r = tron_step<N>(p, ts, tp);
            if (r != kStepContinue) {
                int status;
                if (r == kStepConverged) {
                    iters += iter_before;
                    status = kTronConverged;
                } else if (r == kStepError) {
                    iters += iter_before;
                    status = kTronNumericalError;
                } else {
                    iters += tp.max_iterations;
                    status = tron_finish<N>(p, ts, tp);
                }
                after_solve(status);
            }
        }
    }
    *iters_out += my_iters;
    *fail_out += my_fail;
}

// Persistent kernel: even warps start on the 6-variable queue, odd warps on
// the 4-variable one; each then drains the other.
template <int BS>
__global__ void __launch_bounds__(BS) branch_persistent_kernel(DevNet net, DevState st,
                                                               BranchCfg cfg, Queue q6, Queue q4,
                                                               int* cost, DevScalars* sc) {
    extern __shared__ double smem[];
    unsigned long long it6 = 0, it4 = 0;
    int fails = 0;
    const int warp = (blockIdx.x * BS + threadIdx.x) >> 5;
    if ((warp & 1) == 0) {
        drain_queue<6, BS>(net, st, cfg, q6, cost, smem, &it6, &fails);
        drain_queue<4, BS>(net, st, cfg, q4, cost, smem, &it4, &fails);
    } else {
        drain_queue<4, BS>(net, st, cfg, q4, cost, smem, &it4, &fails);
        drain_queue<6, BS>(net, st, cfg, q6, cost, smem, &it6, &fails);
    }
    const unsigned full = 0xffffffffu;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        it6 += __shfl_down_sync(full, it6, o);
        it4 += __shfl_down_sync(full, it4, o);
        fails += __shfl_down_sync(full, fails, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (it6) atomicAdd(&sc->tron_iters6, it6);
        if (it4) atomicAdd(&sc->tron_iters4, it4);
        if (fails) atomicAdd(&sc->failures, (unsigned long long)fails);
    }
}

// ---- LPT ordering: counting sort of each class list by last cost, desc ---
__device__ __forceinline__ int cost_bucket(int c) {
    const int k = c >> 2;
    return kCostBuckets - 1 - (k < kCostBuckets - 1 ? k : kCostBuckets - 1);
}

__global__ void order_hist_kernel(const int* lim, int nlim, const int* unl, int nunl,
                                  const int* cost, int* hist /* [2][B] */) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < nlim) atomicAdd(&hist[cost_bucket(cost[lim[t]])], 1);
    else if (t < nlim + nunl) atomicAdd(&hist[kCostBuckets + cost_bucket(cost[unl[t - nlim]])], 1);
}

__global__ void order_scan_kernel(int* hist) {
    // two independent exclusive scans of 256 entries; one warp each
    const int cls = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (cls > 1) return;
    int* h = hist + cls * kCostBuckets;
    int carry = 0;
    for (int base = 0; base < kCostBuckets; base += 32) {
        const int v = h[base + lane];
        int incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int n = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += n;
        }
        h[base + lane] = carry + incl - v;
        carry += __shfl_sync(0xffffffffu, incl, 31);
    }
}

__global__ void order_scatter_kernel(const int* lim, int nlim, const int* unl, int nunl,
                                     const int* cost, int* hist, int* order6, int* order4) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < nlim) {
        const int b = lim[t];
        order6[atomicAdd(&hist[cost_bucket(cost[b])], 1)] = b;
    } else if (t < nlim + nunl) {
        const int b = unl[t - nlim];
        order4[atomicAdd(&hist[kCostBuckets + cost_bucket(cost[b])], 1)] = b;
    }
}

// Dense box QP for the TRON-core parity test (proj/tests/acceptance.cpp:458-520).
template <int N>
struct QpProb {
    const double *H, *G, *L, *U;
    GA_FN double lo(int i) const { return L[i]; }
    GA_FN double hi(int i) const { return U[i]; }
    GA_FN double value(const double* x) const {
        double f = 0.0;
        for (int i = 0; i < N; ++i) {
            double hx = 0.0;
            for (int j = 0; j < N; ++j) hx += H[i * N + j] * x[j];
            f += G[i] * x[i] + 0.5 * x[i] * hx;
        }
        return f;
    }
    GA_FN void gradient(const double* x, double* g) const {
        for (int i = 0; i < N; ++i) {
            double hx = 0.0;
            for (int j = 0; j < N; ++j) hx += H[i * N + j] * x[j];
            g[i] = G[i] + hx;
        }
    }
    GA_FN void hessian(const double*, double* h) const {
        for (int i = 0; i < N * N; ++i) h[i] = H[i];
    }
};

template <int N>
__global__ void tron_qp_kernel(int count, const double* H, const double* G, const double* L,
                               const double* U, double* X, int* status, int* iterations) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= count) return;
    QpProb<N> p{H + (size_t)k * N * N, G + (size_t)k * N, L + (size_t)k * N, U + (size_t)k * N};
    double x[N];
    for (int i = 0; i < N; ++i) x[i] = X[(size_t)k * N + i];
    TronParams tp;
    int its = 0;
    status[k] = tron_solve<N>(p, x, tp, &its);
    iterations[k] = its;
    for (int i = 0; i < N; ++i) X[(size_t)k * N + i] = x[i];
}

__global__ void sincos_probe_kernel(const double* x, double* s, double* c, int n) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n) ga_sincos(x[k], &s[k], &c[k]);
}

}  // namespace

// Workspace: [order6 nlim | order4 nunl | hist 2*B | counters 2]
size_t branch_workspace_ints(const DevNet& n) {
    return static_cast<size_t>(n.n_lim) + n.n_unl + 2 * kCostBuckets + 2;
}

void launch_branches(const DevNet& n, const DevState& s, const BranchCfg& cfg, DevScalars* sc,
                     cudaStream_t st) {
    if (n.nl <= 0) return;
    int* ws = s.branch_ws;
    int* order6 = ws;
    int* order4 = ws + n.n_lim;
    int* hist = order4 + n.n_unl;
    int* counters = hist + 2 * kCostBuckets;
    const int total = n.n_lim + n.n_unl;
    cudaMemsetAsync(hist, 0, (2 * kCostBuckets + 2) * sizeof(int), st);
    order_hist_kernel<<<(total + 255) / 256, 256, 0, st>>>(n.lim_list, n.n_lim, n.unl_list,
                                                           n.n_unl, s.br_cost, hist);
    order_scan_kernel<<<1, 64, 0, st>>>(hist);
    order_scatter_kernel<<<(total + 255) / 256, 256, 0, st>>>(n.lim_list, n.n_lim, n.unl_list,
                                                              n.n_unl, s.br_cost, hist, order6,
                                                              order4);
    static int blocks_per_sm = -1, sms = 0;
    const size_t smem = static_cast<size_t>(kFields) * kBranchBlock * sizeof(double);
    if (blocks_per_sm < 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaFuncSetAttribute(branch_persistent_kernel<kBranchBlock>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &blocks_per_sm, branch_persistent_kernel<kBranchBlock>, kBranchBlock, smem);
        if (blocks_per_sm < 1) blocks_per_sm = 1;
    }
    const int warps_needed = (total + 31) / 32;
    int blocks = sms * blocks_per_sm;
    const int max_blocks = (warps_needed * 32 + kBranchBlock - 1) / kBranchBlock;
    if (blocks > max_blocks) blocks = max_blocks;
    Queue q6{order6, n.n_lim, counters};
    Queue q4{order4, n.n_unl, counters + 1};
    branch_persistent_kernel<kBranchBlock><<<blocks, kBranchBlock, smem, st>>>(n, s, cfg, q6, q4,
                                                                              s.br_cost, sc);
}

void launch_tron_qp(int count, int n, const double* h, const double* g, const double* l,
                    const double* u, double* x, int* status, int* iterations, cudaStream_t st) {
    const int blocks = (count + 127) / 128;
    switch (n) {
        case 1: tron_qp_kernel<1><<<blocks, 128, 0, st>>>(count, h, g, l, u, x, status, iterations); break;
        case 2: tron_qp_kernel<2><<<blocks, 128, 0, st>>>(count, h, g, l, u, x, status, iterations); break;
        case 3: tron_qp_kernel<3><<<blocks, 128, 0, st>>>(count, h, g, l, u, x, status, iterations); break;
        case 4: tron_qp_kernel<4><<<blocks, 128, 0, st>>>(count, h, g, l, u, x, status, iterations); break;
        case 5: tron_qp_kernel<5><<<blocks, 128, 0, st>>>(count, h, g, l, u, x, status, iterations); break;
        case 6: tron_qp_kernel<6><<<blocks, 128, 0, st>>>(count, h, g, l, u, x, status, iterations); break;
        default: break;
    }
}

void launch_sincos_probe(const double* x, double* s, double* c, int n, cudaStream_t st) {
    if (n > 0) sincos_probe_kernel<<<(n + 255) / 256, 256, 0, st>>>(x, s, c, n);
}

}  // namespace ga
