// branch.cu — the branch-NLP phase (north-star (b)): per branch, an
// augmented-Lagrangian loop on the line limits around a register-resident
// TRON solve of the 4- or 6-variable branch subproblem (Eq. 4 of the paper).
//
// Reference semantics: proj/src/kernels.cpp:17-192 (BranchProblem, eval,
// consensus values) and :211-292 (solve_branch_batch).  Bit-exactness notes:
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

namespace {

constexpr double kTwoPi = 6.283185307179586;  // 2.0 * std::numbers::pi
constexpr double kLtBound = 1e8;              // kernels.cpp:16
constexpr int kMaxAl = 10;                    // kernels.cpp:219
constexpr double kAlTol = 1e-8;
constexpr double kAlShrink = 0.25;
constexpr double kRhoTildeMax = 1e7;

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
template <bool WG, bool WH>
GA_FN void make_flows(const Basis& b, const double* yc, Flows& F) {
    // yc: gii bii gij bij gji bji gjj bjj
    const double ca[4] = {yc[0], -yc[1], yc[6], -yc[7]};
    const double cb[4] = {yc[2], -yc[3], yc[4], -yc[5]};
    const double cc[4] = {yc[3], yc[2], -yc[5], -yc[4]};
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

// Row targets / multipliers / artificial values / penalties in BranchRow order.
struct RowData {
    double tgt[8], yv[8], zv[8], rh[8];
};

template <int N>
struct BranchProb {
    static constexpr bool kLimited = N == 6;
    double lo_[N], hi_[N];
    double yc[8];
    RowData r;
    double lt_ij, lt_ji, rho_t;
    mutable double cc_, ss_;  // sincos at the last gradient point

    GA_FN double lo(int i) const { return lo_[i]; }
    GA_FN double hi(int i) const { return hi_[i]; }

    // f, g, H of Eq. (4) at x (kernels.cpp:103-163).
    template <bool WF, bool WG, bool WH>
    GA_FN void eval(const double* x, double c, double s, double* f, double* g, double* h) const {
        if (WF) *f = 0.0;
        if (WG) {
#pragma unroll
            for (int i = 0; i < N; ++i) g[i] = 0.0;
        }
        if (WH) {
#pragma unroll
            for (int i = 0; i < N * N; ++i) h[i] = 0.0;
        }
        const Basis b = make_basis(x[0], x[1], c, s);
        Flows F;
        make_flows<WG, WH>(b, yc, F);

        // flows, rows 0..3
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const double d = F.v[k] - r.tgt[k] + r.zv[k];
            const double w = r.yv[k] + r.rh[k] * d;
            if (WF) *f += r.yv[k] * d + 0.5 * r.rh[k] * d * d;
            if (WG) {
#pragma unroll
                for (int i = 0; i < 4; ++i) g[i] += w * F.g[k][i];
            }
            if (WH) {
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const double gg = r.rh[k] * F.g[k][i] * F.g[k][j];
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
            const double d = ev - r.tgt[row] + r.zv[row];
            const double w = r.yv[row] + r.rh[row] * d;
            if (WF) *f += r.yv[row] * d + 0.5 * r.rh[row] * d * d;
            if (WG) g[a] += w * eg;
            if (WH) h[a * N + a] += w * 2.0 + r.rh[row] * eg * eg;
        }
        // angle rows 5 (thi, var 2) and 7 (thj, var 3) are linear
#pragma unroll
        for (int t = 0; t < 2; ++t) {
            const int row = t == 0 ? 5 : 7;
            const int i = 2 + t;
            const double d = x[i] - r.tgt[row] + r.zv[row];
            if (WF) *f += r.yv[row] * d + 0.5 * r.rh[row] * d * d;
            if (WG) g[i] += r.yv[row] + r.rh[row] * d;
            if (WH) h[i * N + i] += r.rh[row];
        }
        if (!kLimited) return;
        // line-limit AL terms: res = p^2 + q^2 + s (kernels.cpp:146-162)
#pragma unroll
        for (int t = 0; t < 2; ++t) {
            const int kp = t == 0 ? 0 : 2, kq = kp + 1;
            const int srow = 4 + t;
            const double lt = t == 0 ? lt_ij : lt_ji;
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

    GA_FN double value(const double* x) const {
        double c, s, f;
        ga_sincos(x[2] - x[3], &s, &c);
        eval<true, false, false>(x, c, s, &f, nullptr, nullptr);
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
GA_FN void branch_flows(const double* yc, double vi, double vj, double thi, double thj,
                        double* out) {
    double s, c;
    ga_sincos(thi - thj, &s, &c);
    const double wi = vi * vi, wj = vj * vj;
    const double wr = vi * vj * c, wim = vi * vj * s;
    out[0] = yc[0] * wi + yc[2] * wr + yc[3] * wim;     // pij
    out[1] = -yc[1] * wi - yc[3] * wr + yc[2] * wim;    // qij
    out[2] = yc[6] * wj + yc[4] * wr - yc[5] * wim;     // pji
    out[3] = -yc[7] * wj - yc[5] * wr - yc[4] * wim;    // qji
}

template <int N>
__device__ void load_problem(const DevNet& net, const DevState& st, const BranchCfg& cfg,
                             int b, BranchProb<N>& p) {
    const int from = net.br_from[b], to = net.br_to[b];
    p.lo_[0] = net.b_vmin[from];
    p.lo_[1] = net.b_vmin[to];
    p.lo_[2] = -kTwoPi;
    p.lo_[3] = -kTwoPi;
    p.hi_[0] = net.b_vmax[from];
    p.hi_[1] = net.b_vmax[to];
    p.hi_[2] = kTwoPi;
    p.hi_[3] = kTwoPi;
    if constexpr (N == 6) {
        const double rt = cfg.limit_tighten * net.br_rate[b];
        const double r2 = rt * rt;
        p.lo_[4] = -r2;
        p.lo_[5] = -r2;
        p.hi_[4] = 0.0;
        p.hi_[5] = 0.0;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) p.yc[k] = net.br_y[k * net.nl + b];
    const int base = 2 * net.ng + 8 * b;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        p.r.tgt[k] = st.xbar[base + k];
        p.r.yv[k] = st.y[base + k];
        p.r.zv[k] = st.z[base + k];
        p.r.rh[k] = st.rho[base + k];
    }
    p.lt_ij = st.lt_ij[b];
    p.lt_ji = st.lt_ji[b];
    p.rho_t = st.rho_t[b];
}

// One thread per branch (kernels.cpp:229-282).
template <int N>
__global__ void __launch_bounds__(128) branch_kernel(DevNet net, DevState st, BranchCfg cfg,
                                                     const int* __restrict__ list, int count,
                                                     DevScalars* sc) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long my_iters = 0;
    int my_fail = 0;
    if (idx < count) {
        const int b = list[idx];
        BranchProb<N> p;
        load_problem<N>(net, st, cfg, b, p);
        TronParams tp;
        tp.gtol = cfg.gtol;
        tp.max_iterations = cfg.max_iterations;
        tp.cg_tol = cfg.cg_tol;
        tp.max_cg = cfg.max_cg;
        tp.delta_floor = cfg.delta_floor;

        double prev[6], pt[6];
#pragma unroll
        for (int k = 0; k < 6; ++k) prev[k] = pt[k] = st.bp[k * net.nl + b];
        bool failed = false;
        if constexpr (N == 4) {
            int its = 0;
            const int status = tron_solve<4>(p, pt, tp, &its);
            failed = status == kTronNumericalError;
            my_iters += its;
        } else {
            double prev_res = __longlong_as_double(0x7ff0000000000000LL);  // +inf
            for (int it = 0; it < kMaxAl; ++it) {
                int its = 0;
                const int status = tron_solve<6>(p, pt, tp, &its);
                my_iters += its;
                if (status == kTronNumericalError) { failed = true; break; }
                double fl[4];
                branch_flows(p.yc, pt[0], pt[1], pt[2], pt[3], fl);
                const double rij = fl[0] * fl[0] + fl[1] * fl[1] + pt[4];
                const double rji = fl[2] * fl[2] + fl[3] * fl[3] + pt[5];
                const double res = smax(fabs(rij), fabs(rji));
                if (res <= kAlTol) break;
                p.lt_ij = sclamp(p.lt_ij + p.rho_t * rij, -kLtBound, kLtBound);
                p.lt_ji = sclamp(p.lt_ji + p.rho_t * rji, -kLtBound, kLtBound);
                if (res > kAlShrink * prev_res) p.rho_t = smin(10.0 * p.rho_t, kRhoTildeMax);
                prev_res = res;
            }
        }
        if (failed) {
#pragma unroll
            for (int k = 0; k < 6; ++k) pt[k] = prev[k];
            my_fail = 1;
        }
        st.lt_ij[b] = p.lt_ij;
        st.lt_ji[b] = p.lt_ji;
        st.rho_t[b] = p.rho_t;
#pragma unroll
        for (int k = 0; k < 6; ++k) st.bp[k * net.nl + b] = pt[k];
        double fl[4];
        branch_flows(p.yc, pt[0], pt[1], pt[2], pt[3], fl);
        const int base = 2 * net.ng + 8 * b;
        st.x[base + 0] = fl[0];
        st.x[base + 1] = fl[1];
        st.x[base + 2] = fl[2];
        st.x[base + 3] = fl[3];
        st.x[base + 4] = pt[0] * pt[0];
        st.x[base + 5] = pt[2];
        st.x[base + 6] = pt[1] * pt[1];
        st.x[base + 7] = pt[3];
    }
    // warp-aggregated counters
    const unsigned full = 0xffffffffu;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        my_iters += __shfl_down_sync(full, my_iters, o);
        my_fail += __shfl_down_sync(full, my_fail, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (my_iters) atomicAdd(N == 6 ? &sc->tron_iters6 : &sc->tron_iters4, my_iters);
        if (my_fail) atomicAdd(&sc->failures, (unsigned long long)my_fail);
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

void launch_branches(const DevNet& n, const DevState& s, const BranchCfg& cfg, DevScalars* sc,
                     cudaStream_t st) {
    constexpr int kBlock = 128;
    if (n.n_lim > 0)
        branch_kernel<6><<<(n.n_lim + kBlock - 1) / kBlock, kBlock, 0, st>>>(n, s, cfg, n.lim_list,
                                                                            n.n_lim, sc);
    if (n.n_unl > 0)
        branch_kernel<4><<<(n.n_unl + kBlock - 1) / kBlock, kBlock, 0, st>>>(n, s, cfg, n.unl_list,
                                                                            n.n_unl, sc);
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
