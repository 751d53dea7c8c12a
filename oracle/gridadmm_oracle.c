/* gridadmm_oracle.c — TEST INFRASTRUCTURE: plain-C restatement of the
 * reference's ADMM hot path (oracle only; never part of the product).
 *
 * Follows /root/reference/proj/src: decomp.cpp (layout, make_state,
 * primal_residual), kernels.cpp (branch problem, generator / branch / bus /
 * z / y / outer updates), tron.cpp (TRON), driver.cpp (cold start, Algorithm
 * 1 loop).  The branch evaluation is written in the "lean" form (terms that
 * are structurally zero in the reference's dense Quad4 arithmetic are not
 * formed; gradient/Hessian only when requested) — bit-identical to the
 * reference because every skipped term is a signed zero added to an
 * accumulator that cannot hold -0.0; tests/test_oracle.py pins this file to
 * the compiled reference bit-for-bit.  Each FL(k) records k FP64 operations
 * whose results are consumed: the lean op census used as the roofline
 * numerator of the branch kernel.  sin/cos come from the pinned ga_sincos.
 *
 * Build: oracle/Makefile (-O2 -ffp-contract=off).
 */
#include "gridadmm_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "../paper_2110_06879_b200/csrc/ga_sincos.h"

/* ---- census ------------------------------------------------------------ */
static unsigned long long g_census[6];
static int g_cls = 4;
#define FL(k)                                   \
    do {                                        \
        g_census[0] += (k);                     \
        g_census[g_cls == 6 ? 4 : 3] += (k);    \
    } while (0)

void oracle_census(unsigned long long* out, int reset) {
    memcpy(out, g_census, sizeof g_census);
    if (reset) memset(g_census, 0, sizeof g_census);
}

/* ---- libstdc++ semantics of std::min / max / clamp (ga_math.h) ---------- */
static double dmin(double a, double b) { return (b < a) ? b : a; }
static double dmax(double a, double b) { return (a < b) ? b : a; }
static double dclamp(double v, double lo, double hi) { return (v < lo) ? lo : ((hi < v) ? hi : v); }
static int dfinite(double v) { return v - v == 0.0; }

/* ======================= TRON (tron.cpp:16-332) ========================= */
#define MAXN 6
typedef struct branch_prob {
    int n, limited;
    double lo[MAXN], hi[MAXN];
    double y[8];  /* gii bii gij bij gji bji gjj bjj */
    double tgt[8], yv[8], zv[8], rh[8];
    double lt_ij, lt_ji, rho_t;
} branch_prob;

static double dot(int n, const double* a, const double* b) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += a[i] * b[i];
    FL(2 * n);
    return s;
}
static double norm2(int n, const double* a) { FL(1); return sqrt(dot(n, a, a)); }

static double model(int n, const double* g, const double* h, const double* s) {
    double q = dot(n, g, s);
    for (int i = 0; i < n; ++i) {
        double hs = 0.0;
        for (int j = 0; j < n; ++j) hs += h[i * n + j] * s[j];
        q += 0.5 * s[i] * hs;
    }
    FL(2 * n * n + 3 * n);
    return q;
}

static int cholesky(int n, const double* a, double* l) {
    for (int i = 0; i < n * n; ++i) l[i] = 0.0;
    for (int j = 0; j < n; ++j) {
        double d = a[j * n + j];
        for (int k = 0; k < j; ++k) d -= l[j * n + k] * l[j * n + k];
        FL(2 * j);
        if (d <= 0.0 || !dfinite(d)) return 0;
        l[j * n + j] = sqrt(d);
        FL(1);
        for (int i = j + 1; i < n; ++i) {
            double v = a[i * n + j];
            for (int k = 0; k < j; ++k) v -= l[i * n + k] * l[j * n + k];
            l[i * n + j] = v / l[j * n + j];
            FL(2 * j + 1);
        }
    }
    return 1;
}

static void chol_solve(int n, const double* l, const double* b, double* x) {
    for (int i = 0; i < n; ++i) {
        double v = b[i];
        for (int k = 0; k < i; ++k) v -= l[i * n + k] * x[k];
        x[i] = v / l[i * n + i];
        FL(2 * i + 1);
    }
    for (int i = n - 1; i >= 0; --i) {
        double v = x[i];
        for (int k = i + 1; k < n; ++k) v -= l[k * n + i] * x[k];
        x[i] = v / l[i * n + i];
        FL(2 * (n - 1 - i) + 1);
    }
}

static double boundary_tau(int n, const double* s, const double* p, double delta) {
    const double pp = dot(n, p, p);
    if (pp <= 0.0) return 0.0;
    const double sp = dot(n, s, p);
    const double ss = dot(n, s, s);
    const double disc = dmax(0.0, sp * sp + pp * (delta * delta - ss));
    FL(5 + 3);
    return (-sp + sqrt(disc)) / pp;
}

static void step_at(int n, const double* x, const double* g, const double* l, const double* u,
                    double alpha, double* out) {
    for (int i = 0; i < n; ++i) out[i] = dclamp(x[i] - alpha * g[i], l[i], u[i]) - x[i];
    FL(3 * n);
}

static int cauchy_ok(int n, const double* g, const double* h, const double* st, double delta) {
    if (!(norm2(n, st) <= delta)) return 0;
    const double m = model(n, g, h, st);
    const double gd = dot(n, g, st);
    FL(1);
    return m <= 0.01 * gd;
}

/* tron.cpp:101-137 */
static void cauchy_point(int n, const double* x, const double* g, const double* h, const double* l,
                         const double* u, double delta, double* s) {
    const double gnorm = norm2(n, g);
    if (gnorm == 0.0) {
        for (int i = 0; i < n; ++i) s[i] = 0.0;
        return;
    }
    double alpha = dmin(1.0, delta / gnorm);
    FL(1);
    step_at(n, x, g, l, u, alpha, s);
    if (cauchy_ok(n, g, h, s, delta)) {
        double trial[MAXN];
        for (int it = 0; it < 20; ++it) {
            const double next = alpha * 2.0;
            FL(1);
            step_at(n, x, g, l, u, next, trial);
            if (!cauchy_ok(n, g, h, trial, delta)) break;
            alpha = next;
            memcpy(s, trial, sizeof(double) * n);
        }
        return;
    }
    for (int it = 0; it < 40; ++it) {
        alpha *= 0.5;
        FL(1);
        step_at(n, x, g, l, u, alpha, s);
        if (cauchy_ok(n, g, h, s, delta)) return;
    }
}

/* tron.cpp:141-224: preconditioned Steihaug CG on the free subspace */
static void subspace_cg(int n, const double* x, const double* g, const double* h, const double* l,
                        const double* u, double delta, const double* s, double* d) {
    int fi[MAXN], nf = 0;
    for (int i = 0; i < n; ++i) d[i] = 0.0;
    for (int i = 0; i < n; ++i) {
        const double xi = x[i] + s[i];
        if (xi > l[i] && xi < u[i]) fi[nf++] = i;
    }
    FL(n);
    if (nf == 0) return;
    double hp[MAXN], rf[MAXN], hf[MAXN * MAXN], prec[MAXN * MAXN];
    for (int i = 0; i < n; ++i) {
        double v = 0.0;
        for (int j = 0; j < n; ++j) v += h[i * n + j] * s[j];
        hp[i] = v;
    }
    FL(2 * n * n);
    for (int a = 0; a < nf; ++a) {
        rf[a] = -(g[fi[a]] + hp[fi[a]]);
        for (int b = 0; b < nf; ++b) hf[a * nf + b] = h[fi[a] * n + fi[b]];
    }
    FL(nf);
    const int have_prec = cholesky(nf, hf, prec);
    double dk[MAXN] = {0}, zk[MAXN], pk[MAXN];
    if (have_prec) chol_solve(nf, prec, rf, zk);
    else memcpy(zk, rf, sizeof(double) * nf);
    memcpy(pk, zk, sizeof(double) * nf);
    double rz = dot(nf, rf, zk);
    const double r0 = norm2(nf, rf);
    if (r0 == 0.0) return;
    for (int it = 0; it < 32; ++it) {
        double hpk[MAXN], pfull[MAXN], sd[MAXN];
        for (int a = 0; a < nf; ++a) {
            double v = 0.0;
            for (int b = 0; b < nf; ++b) v += hf[a * nf + b] * pk[b];
            hpk[a] = v;
        }
        FL(2 * nf * nf);
        const double curv = dot(nf, pk, hpk);
        for (int i = 0; i < n; ++i) { pfull[i] = 0.0; sd[i] = s[i]; }
        for (int a = 0; a < nf; ++a) {
            pfull[fi[a]] = pk[a];
        }
        /* sd = sfull + expand(dk) (zero-padded add on non-free entries) */
        {
            double dfull[MAXN];
            for (int i = 0; i < n; ++i) dfull[i] = 0.0;
            for (int a = 0; a < nf; ++a) dfull[fi[a]] = dk[a];
            for (int i = 0; i < n; ++i) sd[i] = s[i] + dfull[i];
            FL(n);
        }
        if (curv <= 0.0) {
            const double tau = boundary_tau(n, sd, pfull, delta);
            for (int a = 0; a < nf; ++a) dk[a] += tau * pk[a];
            FL(2 * nf);
            break;
        }
        const double alpha = rz / curv;
        double dnext[MAXN], dnfull[MAXN], snext[MAXN];
        for (int a = 0; a < nf; ++a) dnext[a] = dk[a] + alpha * pk[a];
        for (int i = 0; i < n; ++i) dnfull[i] = 0.0;
        for (int a = 0; a < nf; ++a) dnfull[fi[a]] = dnext[a];
        for (int i = 0; i < n; ++i) snext[i] = s[i] + dnfull[i];
        FL(1 + 2 * nf + n);
        if (norm2(n, snext) >= delta) {
            const double tau = boundary_tau(n, sd, pfull, delta);
            for (int a = 0; a < nf; ++a) dk[a] += tau * pk[a];
            FL(2 * nf);
            break;
        }
        memcpy(dk, dnext, sizeof(double) * nf);
        for (int a = 0; a < nf; ++a) rf[a] -= alpha * hpk[a];
        FL(2 * nf);
        if (norm2(nf, rf) <= 0.1 * r0) { FL(1); break; }
        FL(1);
        double zn[MAXN];
        if (have_prec) chol_solve(nf, prec, rf, zn);
        else memcpy(zn, rf, sizeof(double) * nf);
        const double rzn = dot(nf, rf, zn);
        const double betak = rzn / rz;
        for (int a = 0; a < nf; ++a) pk[a] = zn[a] + betak * pk[a];
        FL(1 + 2 * nf);
        rz = rzn;
    }
    for (int i = 0; i < n; ++i) d[i] = 0.0;
    for (int a = 0; a < nf; ++a) d[fi[a]] = dk[a];
}

/* ===================== branch problem (kernels.cpp:17-192) ============== */
typedef struct flows {
    double v[4], g[4][4], h[4][16];
} flows;

static void make_flows(const double* y, double vi, double vj, double c, double s, int wg, int wh,
                       flows* F) {
    const double vivj = vi * vj, nvivj = (-vi) * vj;
    const double wi_v = vi * vi, wj_v = vj * vj, wr_v = vivj * c, wim_v = vivj * s;
    FL(6);
    const double wr_g[4] = {vj * c, vi * c, nvivj * s, vivj * s};
    const double wim_g[4] = {vj * s, vi * s, vivj * c, nvivj * c};
    if (wg || wh) FL(8);
    /* wr / wim Hessians (symmetric; (0,0),(1,1) structural zeros) */
    double wr_h[16], wim_h[16];
    if (wh) {
        const double e01 = c, e02 = (-vj) * s, e03 = vj * s, e12 = (-vi) * s, e13 = vi * s;
        const double e22 = nvivj * c, e23 = vivj * c;
        const double f01 = s, f02 = vj * c, f03 = (-vj) * c, f12 = vi * c, f13 = (-vi) * c;
        const double f22 = nvivj * s, f23 = vivj * s;
        FL(12);
        const double wr[16] = {0, e01, e02, e03, e01, 0, e12, e13, e02, e12, e22, e23, e03, e13, e23, e22};
        const double wi[16] = {0, f01, f02, f03, f01, 0, f12, f13, f02, f12, f22, f23, f03, f13, f23, f22};
        memcpy(wr_h, wr, sizeof wr);
        memcpy(wim_h, wi, sizeof wi);
    }
    const double ca[4] = {y[0], -y[1], y[6], -y[7]};
    const double cb[4] = {y[2], -y[3], y[4], -y[5]};
    const double cc[4] = {y[3], y[2], -y[5], -y[4]};
    for (int k = 0; k < 4; ++k) {
        const int a = k < 2 ? 0 : 1;
        F->v[k] = ca[k] * (a == 0 ? wi_v : wj_v) + cb[k] * wr_v + cc[k] * wim_v;
        FL(5);
        if (wg || wh) {
            const double ag = a == 0 ? 2 * vi : 2 * vj;
            FL(1);
            for (int i = 0; i < 4; ++i) {
                if (i == a) { F->g[k][i] = ca[k] * ag + cb[k] * wr_g[i] + cc[k] * wim_g[i]; FL(5); }
                else { F->g[k][i] = cb[k] * wr_g[i] + cc[k] * wim_g[i]; FL(3); }
            }
        }
        if (wh) {
            for (int i = 0; i < 4; ++i)
                for (int j = 0; j < 4; ++j) {
                    if (i == a && j == a) { F->h[k][i * 4 + j] = ca[k] * 2.0; FL(1); }
                    else if (i == 1 - a && j == 1 - a) F->h[k][i * 4 + j] = 0.0;
                    else { F->h[k][i * 4 + j] = cb[k] * wr_h[i * 4 + j] + cc[k] * wim_h[i * 4 + j]; FL(3); }
                }
        }
    }
}

static int flow_h_zero(int k, int i, int j) {
    const int na = k < 2 ? 1 : 0;
    return i == na && j == na;
}

/* f, g, H of Eq. (4), kernels.cpp:103-163 (lean form, same op order). */
static void branch_eval(const branch_prob* p, const double* x, double c, double s, double* f,
                        double* g, double* h) {
    const int n = p->n;
    if (f) *f = 0.0;
    if (g) for (int i = 0; i < n; ++i) g[i] = 0.0;
    if (h) for (int i = 0; i < n * n; ++i) h[i] = 0.0;
    flows F;
    make_flows(p->y, x[0], x[1], c, s, g != NULL, h != NULL, &F);
    for (int k = 0; k < 4; ++k) {
        const double d = F.v[k] - p->tgt[k] + p->zv[k];
        const double w = p->yv[k] + p->rh[k] * d;
        FL(4);
        if (f) { *f += p->yv[k] * d + 0.5 * p->rh[k] * d * d; FL(6); }
        if (g) { for (int i = 0; i < 4; ++i) g[i] += w * F.g[k][i]; FL(8); }
        if (h)
            for (int i = 0; i < 4; ++i)
                for (int j = 0; j < 4; ++j) {
                    const double gg = p->rh[k] * F.g[k][i] * F.g[k][j];
                    if (flow_h_zero(k, i, j)) { h[i * n + j] += gg; FL(3); }
                    else { h[i * n + j] += w * F.h[k][i * 4 + j] + gg; FL(5); }
                }
    }
    for (int t = 0; t < 2; ++t) {  /* w_i (row 4), w_j (row 6) */
        const int row = t == 0 ? 4 : 6, a = t;
        const double v = x[a], ev = v * v, eg = 2 * v;
        const double d = ev - p->tgt[row] + p->zv[row];
        const double w = p->yv[row] + p->rh[row] * d;
        FL(6);
        if (f) { *f += p->yv[row] * d + 0.5 * p->rh[row] * d * d; FL(6); }
        if (g) { g[a] += w * eg; FL(2); }
        if (h) { h[a * n + a] += w * 2.0 + p->rh[row] * eg * eg; FL(5); }
    }
    for (int t = 0; t < 2; ++t) {  /* angle rows 5, 7 */
        const int row = t == 0 ? 5 : 7, i = 2 + t;
        const double d = x[i] - p->tgt[row] + p->zv[row];
        FL(2);
        if (f) { *f += p->yv[row] * d + 0.5 * p->rh[row] * d * d; FL(6); }
        if (g) { g[i] += p->yv[row] + p->rh[row] * d; FL(3); }
        if (h) { h[i * n + i] += p->rh[row]; FL(1); }
    }
    if (!p->limited) return;
    for (int t = 0; t < 2; ++t) {  /* limit terms ij, ji */
        const int kp = t == 0 ? 0 : 2, kq = kp + 1, srow = 4 + t;
        const double lt = t == 0 ? p->lt_ij : p->lt_ji, rt = p->rho_t;
        const double pv = F.v[kp], qv = F.v[kq];
        const double res = pv * pv + qv * qv + x[srow];
        const double w = lt + rt * res;
        FL(6);
        if (f) { *f += lt * res + 0.5 * rt * res * res; FL(6); }
        if (g || h) {
            double gr[4];
            for (int i = 0; i < 4; ++i) gr[i] = 2 * pv * F.g[kp][i] + 2 * qv * F.g[kq][i];
            FL(20);
            if (g) {
                for (int i = 0; i < 4; ++i) g[i] += w * gr[i];
                g[srow] += w * 1.0;
                FL(10);
            }
            if (h) {
                const double w2 = w * 2.0;
                FL(1);
                for (int i = 0; i < 4; ++i)
                    for (int j = 0; j < 4; ++j) {
                        double acc;
                        if (flow_h_zero(kp, i, j)) { acc = F.g[kp][i] * F.g[kp][j] + F.g[kq][i] * F.g[kq][j]; FL(3); }
                        else {
                            acc = F.g[kp][i] * F.g[kp][j] + pv * F.h[kp][i * 4 + j] +
                                  F.g[kq][i] * F.g[kq][j] + qv * F.h[kq][i * 4 + j];
                            FL(7);
                        }
                        h[i * n + j] += w2 * acc;
                        FL(2);
                    }
                for (int i = 0; i < 4; ++i) {
                    for (int j = 0; j < 4; ++j) h[i * n + j] += rt * gr[i] * gr[j];
                    h[i * n + srow] += rt * gr[i] * 1.0;
                    FL(12 + 3);
                }
                for (int j = 0; j < 4; ++j) h[srow * n + j] += rt * 1.0 * gr[j];
                h[srow * n + srow] += rt * 1.0 * 1.0;
                FL(12 + 3);
            }
        }
    }
}

static double sc_c, sc_s;  /* sincos at the last gradient point */
static double bp_value(const branch_prob* p, const double* x) {
    double s, c, f;
    ga_sincos(x[2] - x[3], &s, &c);
    g_census[5]++;
    FL(1);
    branch_eval(p, x, c, s, &f, NULL, NULL);
    return f;
}
static void bp_gradient(const branch_prob* p, const double* x, double* g) {
    ga_sincos(x[2] - x[3], &sc_s, &sc_c);
    g_census[5]++;
    FL(1);
    branch_eval(p, x, sc_c, sc_s, NULL, g, NULL);
}
static void bp_hessian(const branch_prob* p, const double* x, double* h) {
    branch_eval(p, x, sc_c, sc_s, NULL, NULL, h);
}

static double proj_grad(int n, const double* x, const double* g, const double* l, const double* u) {
    double pg = 0.0;
    for (int i = 0; i < n; ++i) {
        double gi = g[i];
        if (x[i] <= l[i]) gi = dmin(gi, 0.0);
        else if (x[i] >= u[i]) gi = dmax(gi, 0.0);
        pg = dmax(pg, fabs(gi));
    }
    return pg;
}

enum { T_CONV = 0, T_LIMIT = 1, T_ERR = 2 };

/* solve_one, tron.cpp:228-332; returns status, *iters as TronResult. */
static int solve_one(const branch_prob* p, double* x, int* iters) {
    const int n = p->n;
    const double* l = p->lo;
    const double* u = p->hi;
    double g[MAXN], h[MAXN * MAXN], s[MAXN], d[MAXN], st[MAXN], xt[MAXN];
    for (int i = 0; i < n; ++i) x[i] = dclamp(x[i], l[i], u[i]);
    double f = bp_value(p, x);
    *iters = 0;
    if (!dfinite(f)) return T_ERR;
    double delta = 0.0;
    for (int iter = 0; iter < 200; ++iter) {
        g_census[g_cls == 6 ? 2 : 1]++;
        bp_gradient(p, x, g);
        for (int i = 0; i < n; ++i)
            if (!dfinite(g[i])) { *iters = iter; return T_ERR; }
        if (proj_grad(n, x, g, l, u) <= 1e-6) { *iters = iter; return T_CONV; }
        bp_hessian(p, x, h);
        for (int i = 0; i < n * n; ++i)
            if (!dfinite(h[i])) { *iters = iter; return T_ERR; }
        if (iter == 0 && delta == 0.0) delta = dmax(norm2(n, g), 1e-3);
        cauchy_point(n, x, g, h, l, u, delta, s);
        subspace_cg(n, x, g, h, l, u, delta, s, d);
        const double qc = model(n, g, h, s);
        double beta = 1.0;
        int used_d = 0;
        for (int ls = 0; ls < 20; ++ls) {
            for (int i = 0; i < n; ++i) st[i] = dclamp(x[i] + s[i] + beta * d[i], l[i], u[i]) - x[i];
            FL(4 * n);
            if (model(n, g, h, st) <= qc) { used_d = 1; break; }
            beta *= 0.5;
            FL(1);
        }
        const double* step = used_d ? st : s;
        const double q = model(n, g, h, step);
        for (int i = 0; i < n; ++i) xt[i] = dclamp(x[i] + step[i], l[i], u[i]);
        FL(n);
        const double ft = bp_value(p, xt);
        if (!dfinite(ft)) { *iters = iter; return T_ERR; }
        const double ared = f - ft, pred = -q;
        const double ratio = pred > 0.0 ? ared / pred : (ared > 0.0 ? 1.0 : -1.0);
        const double snorm = norm2(n, step);
        FL(3);
        if (ratio < 0.25) { delta = 0.25 * dmax(snorm, 1e-12); FL(1); }
        else if (ratio > 0.75 && snorm >= 0.9 * delta) { delta = dmin(2.0 * delta, 1e10); FL(2); }
        if (ared > 0.0 && ratio > 1e-4) {
            memcpy(x, xt, sizeof(double) * n);
            f = ft;
        }
        if (delta < 1e-14) break;
    }
    bp_gradient(p, x, g);
    *iters = 200;
    return proj_grad(n, x, g, l, u) <= 1e-6 ? T_CONV : T_LIMIT;
}

/* =================== ADMM phases (kernels.cpp:194-437) ================== */
typedef struct solver {
    const oracle_net* net;
    int m;
    double rho_pq, rho_va, beta0, eps, inner_tol, lam_max, beta_max;
    int max_outer, max_inner;
    /* bus CSR: groups w, theta, gen_p, gen_q, flow_p, flow_q (decomp.cpp:7-31) */
    int* grp;   /* 7 per bus */
    int* rows;  /* m */
} solver;

static void branch_flows(const double* y, double vi, double vj, double thi, double thj, double* o) {
    double s, c;
    ga_sincos(thi - thj, &s, &c);
    const double wi = vi * vi, wj = vj * vj, wr = vi * vj * c, wim = vi * vj * s;
    o[0] = y[0] * wi + y[2] * wr + y[3] * wim;
    o[1] = -y[1] * wi - y[3] * wr + y[2] * wim;
    o[2] = y[6] * wj + y[4] * wr - y[5] * wim;
    o[3] = -y[7] * wj - y[5] * wr - y[4] * wim;
}

static void setup(solver* S, const oracle_net* net, const double* cfg) {
    S->net = net;
    S->m = 2 * net->ng + 8 * net->nl;
    S->rho_pq = cfg[0]; S->rho_va = cfg[1]; S->beta0 = cfg[2]; S->eps = cfg[3];
    S->inner_tol = cfg[4]; S->max_outer = (int)cfg[5]; S->max_inner = (int)cfg[6];
    S->lam_max = cfg[8]; S->beta_max = cfg[9];
    const int nb = net->nb;
    int* cnt = calloc((size_t)6 * nb + 1, sizeof(int));
    for (int g = 0; g < net->ng; ++g) {
        const int b = (int)net->gen[8 * g];
        cnt[6 * b + 2]++; cnt[6 * b + 3]++;
    }
    for (int l = 0; l < net->nl; ++l) {
        const int f = net->ends[2 * l], t = net->ends[2 * l + 1];
        for (int k = 0; k < 6; ++k) { if (k != 2 && k != 3) { cnt[6 * f + k]++; cnt[6 * t + k]++; } }
    }
    S->grp = malloc(sizeof(int) * (7 * (size_t)nb + 1));
    S->rows = malloc(sizeof(int) * ((size_t)S->m + 1));
    int pos = 0;
    for (int i = 0; i < nb; ++i) {
        for (int k = 0; k < 6; ++k) { S->grp[7 * i + k] = pos; pos += cnt[6 * i + k]; }
        S->grp[7 * i + 6] = pos;
    }
    int* fill = calloc((size_t)6 * nb + 1, sizeof(int));
    #define PUSH(bus, k, row) S->rows[S->grp[7 * (bus) + (k)] + fill[6 * (bus) + (k)]++] = (row)
    for (int g = 0; g < net->ng; ++g) {
        const int b = (int)net->gen[8 * g];
        PUSH(b, 2, 2 * g); PUSH(b, 3, 2 * g + 1);
    }
    const int base = 2 * net->ng;
    for (int l = 0; l < net->nl; ++l) {
        const int f = net->ends[2 * l], t = net->ends[2 * l + 1], r0 = base + 8 * l;
        PUSH(f, 4, r0 + 0); PUSH(f, 5, r0 + 1); PUSH(f, 0, r0 + 4); PUSH(f, 1, r0 + 5);
        PUSH(t, 4, r0 + 2); PUSH(t, 5, r0 + 3); PUSH(t, 0, r0 + 6); PUSH(t, 1, r0 + 7);
    }
    #undef PUSH
    free(cnt);
    free(fill);
}

static void teardown(solver* S) { free(S->grp); free(S->rows); }

/* kernels.cpp:194-209 */
static void gen_update(const solver* S, gridadmm_state_view* v) {
    for (int g = 0; g < S->net->ng; ++g) {
        const double* G = S->net->gen + 8 * g;
        const int pr = 2 * g, qr = 2 * g + 1;
        const double p = (v->rho[pr] * (v->xbar[pr] - v->z[pr]) - v->y[pr] - G[6]) / (2.0 * G[5] + v->rho[pr]);
        v->x[pr] = dclamp(p, G[1], G[2]);
        const double q = (v->rho[qr] * (v->xbar[qr] - v->z[qr]) - v->y[qr]) / v->rho[qr];
        v->x[qr] = dclamp(q, G[3], G[4]);
    }
}

/* kernels.cpp:211-292; returns failures. */
static long branch_update(const solver* S, gridadmm_state_view* v) {
    const oracle_net* net = S->net;
    long fails = 0;
    const double kInf = 1.0 / 0.0;
    for (int b = 0; b < net->nl; ++b) {
        const double* B = net->branch + 14 * b;
        const int from = net->ends[2 * b], to = net->ends[2 * b + 1];
        branch_prob p;
        p.limited = B[5] > 0.0;
        p.n = p.limited ? 6 : 4;
        g_cls = p.n;
        p.lo[0] = net->bus[6 * from + 4]; p.hi[0] = net->bus[6 * from + 5];
        p.lo[1] = net->bus[6 * to + 4];   p.hi[1] = net->bus[6 * to + 5];
        p.lo[2] = p.lo[3] = -6.283185307179586;
        p.hi[2] = p.hi[3] = 6.283185307179586;
        if (p.limited) {
            const double rt = 0.99 * B[5], r2 = rt * rt;
            p.lo[4] = p.lo[5] = -r2;
            p.hi[4] = p.hi[5] = 0.0;
        }
        memcpy(p.y, B + 6, sizeof p.y);
        const int base = 2 * net->ng + 8 * b;
        for (int k = 0; k < 8; ++k) {
            p.tgt[k] = v->xbar[base + k];
            p.yv[k] = v->y[base + k];
            p.zv[k] = v->z[base + k];
            p.rh[k] = v->rho[base + k];
        }
        p.lt_ij = v->lt_ij[b];
        p.lt_ji = v->lt_ji[b];
        p.rho_t = v->rho_tilde[b];
        double* pt = v->branch_point + 6 * b;
        double prev[6];
        memcpy(prev, pt, sizeof prev);
        int status = T_CONV, its;
        if (!p.limited) {
            status = solve_one(&p, pt, &its);
        } else {
            double prev_res = kInf;
            for (int it = 0; it < 10; ++it) {
                const int r = solve_one(&p, pt, &its);
                if (r == T_ERR) { status = T_ERR; break; }
                double fl[4];
                branch_flows(p.y, pt[0], pt[1], pt[2], pt[3], fl);
                const double rij = fl[0] * fl[0] + fl[1] * fl[1] + pt[4];
                const double rji = fl[2] * fl[2] + fl[3] * fl[3] + pt[5];
                const double res = dmax(fabs(rij), fabs(rji));
                if (res <= 1e-8) break;
                p.lt_ij = dclamp(p.lt_ij + p.rho_t * rij, -1e8, 1e8);
                p.lt_ji = dclamp(p.lt_ji + p.rho_t * rji, -1e8, 1e8);
                if (res > 0.25 * prev_res) p.rho_t = dmin(10.0 * p.rho_t, 1e7);
                prev_res = res;
            }
        }
        if (status == T_ERR) { memcpy(pt, prev, sizeof prev); ++fails; }
        v->lt_ij[b] = p.lt_ij;
        v->lt_ji[b] = p.lt_ji;
        v->rho_tilde[b] = p.rho_t;
        double fl[4];
        branch_flows(p.y, pt[0], pt[1], pt[2], pt[3], fl);
        const double vals[8] = {fl[0], fl[1], fl[2], fl[3], pt[0] * pt[0], pt[2], pt[1] * pt[1], pt[3]};
        memcpy(v->x + base, vals, sizeof vals);
    }
    return fails;
}

/* kernels.cpp:294-413, dense as in the reference; returns -1 or the first
 * singular bus.  Writes max |xbar_new - xbar_old| to *dual_raw. */
static long bus_update(const solver* S, gridadmm_state_view* v, double* dual_raw) {
    const oracle_net* net = S->net;
    long singular = -1;
    double dual = 0.0;
    double* qd = NULL;
    double* cv = NULL;
    int cap = 0;
    for (int i = 0; i < net->nb; ++i) {
        const int* grp = S->grp + 7 * i;
        const int ndup = grp[6] - grp[2], nv = 2 + ndup;
        if (nv > cap) { cap = nv; qd = realloc(qd, sizeof(double) * cap); cv = realloc(cv, sizeof(double) * cap); }
        for (int j = 0; j < nv; ++j) { qd[j] = 0.0; cv[j] = 0.0; }
        for (int k = grp[0]; k < grp[1]; ++k) {
            const int r = S->rows[k];
            qd[0] += v->rho[r];
            cv[0] += v->rho[r] * (v->x[r] + v->z[r]) + v->y[r];
        }
        for (int k = grp[1]; k < grp[2]; ++k) {
            const int r = S->rows[k];
            qd[1] += v->rho[r];
            cv[1] += v->rho[r] * (v->x[r] + v->z[r]) + v->y[r];
        }
        for (int k = grp[2]; k < grp[6]; ++k) {
            const int r = S->rows[k], j = 2 + (k - grp[2]);
            qd[j] = v->rho[r];
            cv[j] = v->rho[r] * (v->x[r] + v->z[r]) + v->y[r];
        }
        if (qd[0] == 0.0) qd[0] = 1.0;
        if (qd[1] == 0.0) qd[1] = 1.0;
        const int ref = i == net->ref_bus, nc = ref ? 3 : 2;
        const double gs = net->bus[6 * i + 2], bs = net->bus[6 * i + 3];
        double* A = calloc((size_t)nc * nv, sizeof(double));
        A[0] = -gs;
        A[nv] = bs;
        if (ref) A[2 * nv + 1] = 1.0;
        int col = 2;
        for (int k = grp[2]; k < grp[3]; ++k, ++col) A[col] = 1.0;
        for (int k = grp[3]; k < grp[4]; ++k, ++col) A[nv + col] = 1.0;
        for (int k = grp[4]; k < grp[5]; ++k, ++col) A[col] = -1.0;
        for (int k = grp[5]; k < grp[6]; ++k, ++col) A[nv + col] = -1.0;
        const double bvec[3] = {net->bus[6 * i + 0], net->bus[6 * i + 1], 0.0};
        double Sm[9] = {0}, rhs[3] = {0};
        for (int r = 0; r < nc; ++r) {
            for (int s = 0; s < nc; ++s) {
                double acc = 0.0;
                for (int j = 0; j < nv; ++j) acc += A[r * nv + j] * A[s * nv + j] / qd[j];
                Sm[r * 3 + s] = acc;
            }
            double acc = 0.0;
            for (int j = 0; j < nv; ++j) acc += A[r * nv + j] * cv[j] / qd[j];
            rhs[r] = acc - bvec[r];
        }
        double mu[3] = {0};
        int piv[3] = {0, 1, 2}, sing = 0;
        for (int c = 0; c < nc && !sing; ++c) {
            int best = c;
            for (int r = c + 1; r < nc; ++r)
                if (fabs(Sm[piv[r] * 3 + c]) > fabs(Sm[piv[best] * 3 + c])) best = r;
            const int t = piv[c]; piv[c] = piv[best]; piv[best] = t;
            const double dd = Sm[piv[c] * 3 + c];
            if (fabs(dd) < 1e-14) { sing = 1; break; }
            for (int r = c + 1; r < nc; ++r) {
                const double fct = Sm[piv[r] * 3 + c] / dd;
                for (int s2 = c; s2 < nc; ++s2) Sm[piv[r] * 3 + s2] -= fct * Sm[piv[c] * 3 + s2];
                rhs[piv[r]] -= fct * rhs[piv[c]];
            }
        }
        if (sing) {
            if (singular < 0) singular = i;
            free(A);
            continue;
        }
        for (int c = nc - 1; c >= 0; --c) {
            double acc = rhs[piv[c]];
            for (int s2 = c + 1; s2 < nc; ++s2) acc -= Sm[piv[c] * 3 + s2] * mu[s2];
            mu[c] = acc / Sm[piv[c] * 3 + c];
        }
        double sol0 = 0, sol1 = 0;
        for (int j = 0; j < nv; ++j) {
            double acc = cv[j];
            for (int r = 0; r < nc; ++r) acc -= A[r * nv + j] * mu[r];
            const double sol = acc / qd[j];
            if (j == 0) sol0 = sol;
            else if (j == 1) sol1 = sol;
            else {
                const int r = S->rows[grp[2] + (j - 2)];
                dual = dmax(dual, fabs(sol - v->xbar[r]));
                v->xbar[r] = sol;
            }
        }
        v->bus_w[i] = sol0;
        v->bus_theta[i] = sol1;
        for (int k = grp[0]; k < grp[1]; ++k) {
            const int r = S->rows[k];
            dual = dmax(dual, fabs(sol0 - v->xbar[r]));
            v->xbar[r] = sol0;
        }
        for (int k = grp[1]; k < grp[2]; ++k) {
            const int r = S->rows[k];
            dual = dmax(dual, fabs(sol1 - v->xbar[r]));
            v->xbar[r] = sol1;
        }
        free(A);
    }
    free(qd);
    free(cv);
    if (dual_raw) *dual_raw = dual;
    return singular;
}

static void z_update(const solver* S, gridadmm_state_view* v) {
    for (int k = 0; k < S->m; ++k) {
        const double r = v->x[k] - v->xbar[k];
        v->z[k] = -(v->lambda[k] + v->y[k] + v->rho[k] * r) / (v->rho[k] + *v->beta);
    }
}

static void y_update(const solver* S, gridadmm_state_view* v) {
    for (int k = 0; k < S->m; ++k) v->y[k] += v->rho[k] * (v->x[k] - v->xbar[k] + v->z[k]);
}

static void outer_update(const solver* S, gridadmm_state_view* v, double z_inf, double prev) {
    for (int k = 0; k < S->m; ++k)
        v->lambda[k] = dclamp(v->lambda[k] + *v->beta * v->z[k], -S->lam_max, S->lam_max);
    if (prev >= 0.0 && z_inf > 0.25 * prev) *v->beta = dmin(*v->beta * 10.0, S->beta_max);
}

/* driver.cpp:26-63 */
void oracle_cold_start(const oracle_net* net, const double* cfg, gridadmm_state_view* v) {
    const int m = 2 * net->ng + 8 * net->nl;
    for (int k = 0; k < m; ++k) {
        v->x[k] = v->xbar[k] = v->z[k] = v->y[k] = v->lambda[k] = 0.0;
        v->rho[k] = (k < 2 * net->ng || (k - 2 * net->ng) % 8 < 4) ? cfg[0] : cfg[1];
    }
    *v->beta = cfg[2];
    for (int g = 0; g < net->ng; ++g) {
        const double* G = net->gen + 8 * g;
        v->x[2 * g] = v->xbar[2 * g] = 0.5 * (G[1] + G[2]);
        v->x[2 * g + 1] = v->xbar[2 * g + 1] = 0.5 * (G[3] + G[4]);
    }
    for (int i = 0; i < net->nb; ++i) {
        const double vv = 0.5 * (net->bus[6 * i + 4] + net->bus[6 * i + 5]);
        v->bus_w[i] = vv * vv;
        v->bus_theta[i] = 0.0;
    }
    for (int b = 0; b < net->nl; ++b) {
        const double* B = net->branch + 14 * b;
        const int f = net->ends[2 * b], t = net->ends[2 * b + 1];
        const double vi = 0.5 * (net->bus[6 * f + 4] + net->bus[6 * f + 5]);
        const double vj = 0.5 * (net->bus[6 * t + 4] + net->bus[6 * t + 5]);
        double* pt = v->branch_point + 6 * b;
        pt[0] = vi; pt[1] = vj; pt[2] = pt[3] = pt[4] = pt[5] = 0.0;
        double fl[4];
        branch_flows(B + 6, vi, vj, 0.0, 0.0, fl);
        const double vals[8] = {fl[0], fl[1], fl[2], fl[3], vi * vi, 0.0, vj * vj, 0.0};
        for (int k = 0; k < 8; ++k) v->x[2 * net->ng + 8 * b + k] = v->xbar[2 * net->ng + 8 * b + k] = vals[k];
        if (B[5] > 0.0) {
            const double rt = 0.99 * B[5];
            pt[4] = dclamp(-(fl[0] * fl[0] + fl[1] * fl[1]), -rt * rt, 0.0);
            pt[5] = dclamp(-(fl[2] * fl[2] + fl[3] * fl[3]), -rt * rt, 0.0);
        }
        v->lt_ij[b] = v->lt_ji[b] = 0.0;
        v->rho_tilde[b] = cfg[0];
    }
}

long oracle_phase(const oracle_net* net, int phase, const double* cfg, gridadmm_state_view* v,
                  double z_inf, double prev_z_inf) {
    solver S;
    setup(&S, net, cfg);
    long ret = 0;
    switch (phase) {
        case 0: gen_update(&S, v); break;
        case 1: ret = branch_update(&S, v); break;
        case 2: ret = bus_update(&S, v, NULL); break;
        case 3: z_update(&S, v); break;
        case 4: y_update(&S, v); break;
        case 5: outer_update(&S, v, z_inf, prev_z_inf); break;
        default: ret = -2;
    }
    teardown(&S);
    return ret;
}

/* driver.cpp:140-246 without solution extraction; series: 6 per record
 * (outer, inner, primal, dual, z_norm, 0); info: status, outer, inner,
 * failures, then 5 zeros (quality metrics are not part of the hot path). */
int oracle_solve(const oracle_net* net, const double* cfg, const gridadmm_state_view* init,
                 gridadmm_state_view* v, double* series, int cap, int* nseries, double* info) {
    solver S;
    setup(&S, net, cfg);
    const int m = S.m;
    if (init) {
        memcpy(v->x, init->x, sizeof(double) * m); memcpy(v->xbar, init->xbar, sizeof(double) * m);
        memcpy(v->z, init->z, sizeof(double) * m); memcpy(v->y, init->y, sizeof(double) * m);
        memcpy(v->lambda, init->lambda, sizeof(double) * m); memcpy(v->rho, init->rho, sizeof(double) * m);
        memcpy(v->bus_w, init->bus_w, sizeof(double) * net->nb);
        memcpy(v->bus_theta, init->bus_theta, sizeof(double) * net->nb);
        memcpy(v->branch_point, init->branch_point, sizeof(double) * 6 * net->nl);
        memcpy(v->lt_ij, init->lt_ij, sizeof(double) * net->nl);
        memcpy(v->lt_ji, init->lt_ji, sizeof(double) * net->nl);
        memcpy(v->rho_tilde, init->rho_tilde, sizeof(double) * net->nl);
        *v->beta = *init->beta;
    } else {
        oracle_cold_start(net, cfg, v);
    }
    const double inner_tol = S.inner_tol > 0.0 ? S.inner_tol : S.eps * sqrt((double)m);
    double* zprev = malloc(sizeof(double) * (m + 1));
    double rho_max = 0.0;
    for (int k = 0; k < m; ++k) rho_max = dmax(rho_max, v->rho[k]);
    double prev_z_inf = -1.0;
    int n = 0, status = 1, outer = 0, inner_total = 0;
    long fails = 0;
    for (outer = 1; outer <= S.max_outer; ++outer) {
        double z_inf = 0.0;
        for (int inner = 1; inner <= S.max_inner; ++inner) {
            gen_update(&S, v);
            fails += branch_update(&S, v);
            double dual_raw = 0.0;
            if (bus_update(&S, v, &dual_raw) >= 0) { free(zprev); teardown(&S); return -1; }
            memcpy(zprev, v->z, sizeof(double) * m);
            z_update(&S, v);
            y_update(&S, v);
            double primal = 0.0, drift = 0.0;
            z_inf = 0.0;
            for (int k = 0; k < m; ++k) {
                primal = dmax(primal, fabs(v->x[k] - v->xbar[k] + v->z[k]));
                z_inf = dmax(z_inf, fabs(v->z[k]));
                drift = dmax(drift, fabs(v->z[k] - zprev[k]));
            }
            const double dual = dual_raw * rho_max;
            ++inner_total;
            if (n < cap) {
                double* r = series + 6 * n;
                r[0] = outer; r[1] = inner; r[2] = primal; r[3] = dual; r[4] = z_inf; r[5] = 0.0;
            }
            ++n;
            if (!dfinite(primal) || !dfinite(dual) || primal > 1e8 || dual > 1e8) {
                status = 2;
                goto done;
            }
            if (dmax(primal, dual) <= inner_tol) break;
            if (primal <= inner_tol && z_inf <= S.eps && drift <= 0.01 * S.eps) break;
        }
        if (z_inf <= S.eps) { status = 0; break; }
        outer_update(&S, v, z_inf, prev_z_inf);
        prev_z_inf = z_inf;
    }
    if (outer > S.max_outer) outer = S.max_outer;
done:
    if (nseries) *nseries = n;
    if (info) {
        memset(info, 0, sizeof(double) * 9);
        info[0] = status; info[1] = outer; info[2] = inner_total; info[3] = (double)fails;
    }
    free(zprev);
    teardown(&S);
    return 0;
}
