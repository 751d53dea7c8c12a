// branch_problem.cuh — the branch subproblem of the two-level ADMM (Eq. 4 of
// the paper): f, gradient and Hessian over (vi, vj, thi, thj[, sij, sji]),
// evaluated from a per-branch shared-memory slot.
//
// Reference semantics: proj/src/kernels.cpp:17-192 (BranchProblem, Basis,
// Quad4, combine, flow_quads, eval, consensus values).  Bit-exactness notes:
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
#ifndef GA_BRANCH_PROBLEM_CUH
#define GA_BRANCH_PROBLEM_CUH

#include "device.hpp"
#include "ga_math.h"
#include "ga_sincos.h"
#include "tron.cuh"

namespace ga {
namespace bp {

constexpr double kTwoPi = 6.283185307179586;  // 2.0 * std::numbers::pi

// Field indices of the [field][slot] shared-memory layout.
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

// One branch's data: field f of slot s lives at smem[f * S + s].
template <int S>
struct Slot {
    double* p;  // smem + slot index
    __device__ __forceinline__ double operator()(int f) const { return p[f * S]; }
    __device__ __forceinline__ void set(int f, double v) const { p[f * S] = v; }
};

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

template <int S>
struct YcView {
    Slot<S> s;
    __device__ __forceinline__ double operator()(int k) const { return s(F_YC + k); }
};

// The branch subproblem over a shared-memory slot (kernels.cpp:17-163).
template <int N, int S>
struct BranchProb {
    static constexpr bool kLimited = N == 6;
    Slot<S> s;
    mutable double cc_, ss_;  // sincos at the last gradient point

    __device__ __forceinline__ double lo(int i) const {
        switch (i) {
            case 0: return s(F_VMIN_I);
            case 1: return s(F_VMIN_J);
            case 2: case 3: return -kTwoPi;
            default: return -s(F_R2);
        }
    }
    __device__ __forceinline__ double hi(int i) const {
        switch (i) {
            case 0: return s(F_VMAX_I);
            case 1: return s(F_VMAX_J);
            case 2: case 3: return kTwoPi;
            default: return 0.0;
        }
    }

    // f, g, H of Eq. (4) at x (kernels.cpp:103-163).
    template <bool WF, bool WG, bool WH>
    __device__ __forceinline__ void eval(const double* x, double c, double sn, double* f, double* g,
                                         double* h) const {
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
        make_flows<WG, WH>(b, YcView<S>{s}, F);

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

    __device__ __forceinline__ double value(const double* x) const {
        double c, sn, f;
        ga_sincos_ool(x[2] - x[3], &sn, &c);
        eval<true, false, false>(x, c, sn, &f, nullptr, nullptr);
        return f;
    }
    __device__ __forceinline__ void gradient(const double* x, double* g) const {
        ga_sincos_ool(x[2] - x[3], &ss_, &cc_);
        eval<false, true, false>(x, cc_, ss_, nullptr, g, nullptr);
    }
    // f's gradient and Hessian at x in one pass (TRON's step start)
    __device__ __forceinline__ void grad_hess(const double* x, double* g, double* h) const {
        ga_sincos_ool(x[2] - x[3], &ss_, &cc_);
        eval<false, true, true>(x, cc_, ss_, nullptr, g, h);
    }
};

// Admittance view over the global [8][nl] array (cold start).
struct YArr {
    const double* y;
    int nl, b;
    __device__ __forceinline__ double operator()(int k) const { return y[k * nl + b]; }
};

// branch_flows (netdata.cpp:33-45)
template <class Y>
GA_FN void branch_flows(const Y& yc, double vi, double vj, double thi, double thj, double* out) {
    double s, c;
    ga_sincos_ool(thi - thj, &s, &c);
    const double wi = vi * vi, wj = vj * vj;
    const double wr = vi * vj * c, wim = vi * vj * s;
    out[0] = yc(0) * wi + yc(2) * wr + yc(3) * wim;     // pij
    out[1] = -yc(1) * wi - yc(3) * wr + yc(2) * wim;    // qij
    out[2] = yc(6) * wj + yc(4) * wr - yc(5) * wim;     // pji
    out[3] = -yc(7) * wj - yc(5) * wr - yc(4) * wim;    // qji
}

// Storage position of branch row k (reference order pij, qij, pji, qji, wi,
// thi, wj, thj) given the branch's from-quad qf and to-quad qt (device.hpp).
__host__ __device__ __forceinline__ int branch_row_pos(int qf, int qt, int k) {
    return (((k >> 1) & 1) ? qt : qf) + (k & 1) + ((k >> 2) << 1);
}

// Fills a slot for branch b (kernels.cpp:229-241).
template <int S>
__device__ __forceinline__ void load_slot(const DevNet& net, const DevState& st,
                                          const BranchCfg& cfg, int b, Slot<S> s) {
    const int from = net.br_from[b], to = net.br_to[b];
#pragma unroll
    for (int k = 0; k < 8; ++k) s.set(F_YC + k, __ldg(&net.br_y[k * net.nl + b]));
    const int qf = __ldg(&net.qpos[2 * b]), qt = __ldg(&net.qpos[2 * b + 1]);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const int r = branch_row_pos(qf, qt, k);
        s.set(F_TGT + k, st.xbar[r]);
        s.set(F_Y + k, st.y[r]);
        s.set(F_Z + k, st.z[r]);
        s.set(F_RHO + k, st.rho[r]);
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

}  // namespace bp
}  // namespace ga

#endif
