// oracle/ref_harness.cpp — TEST INFRASTRUCTURE (parity checker only).
//
// Linked together with the UNMODIFIED reference sources
// (/root/reference/proj/src/*.cpp, compiled in place by oracle/Makefile) into
// oracle/_ref/libgridadmm_ref.so.  Exposes the reference's internal C++
// phase functions (proj/src/kernels.hpp:70-101, proj/src/driver.hpp:83-95)
// through a C ABI so the parity tests can replay one phase on a given state
// and compare the product's device result bit-for-bit.  Nothing here
// re-implements the algorithm; it only marshals the reference's own
// AdmmState (proj/src/decomp.hpp:64-78) to and from flat arrays.
#include <algorithm>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "decomp.hpp"
#include "driver.hpp"
#include "kernels.hpp"
#include "netdata.hpp"
#include "tron.hpp"

#include "gridadmm/gridadmm_ext.h"

using namespace gridadmm;

namespace {

thread_local std::string g_err;

void to_view(const AdmmState& s, const gridadmm_state_view* v) {
    auto cp = [](const std::vector<double>& src, double* dst) {
        if (dst) std::memcpy(dst, src.data(), src.size() * sizeof(double));
    };
    cp(s.x, v->x);
    cp(s.xbar, v->xbar);
    cp(s.z, v->z);
    cp(s.y, v->y);
    cp(s.lambda, v->lambda);
    cp(s.rho, v->rho);
    cp(s.bus_w, v->bus_w);
    cp(s.bus_theta, v->bus_theta);
    if (v->branch_point)
        for (size_t b = 0; b < s.branch_point.size(); ++b)
            for (int k = 0; k < 6; ++k) v->branch_point[6 * b + k] = s.branch_point[b][k];
    cp(s.lt_ij, v->lt_ij);
    cp(s.lt_ji, v->lt_ji);
    cp(s.rho_tilde, v->rho_tilde);
    if (v->beta) *v->beta = s.beta;
}

void from_view(AdmmState& s, const gridadmm_state_view* v) {
    auto cp = [](std::vector<double>& dst, const double* src) {
        if (src) std::memcpy(dst.data(), src, dst.size() * sizeof(double));
    };
    cp(s.x, v->x);
    cp(s.xbar, v->xbar);
    cp(s.z, v->z);
    cp(s.y, v->y);
    cp(s.lambda, v->lambda);
    cp(s.rho, v->rho);
    cp(s.bus_w, v->bus_w);
    cp(s.bus_theta, v->bus_theta);
    if (v->branch_point)
        for (size_t b = 0; b < s.branch_point.size(); ++b)
            for (int k = 0; k < 6; ++k) s.branch_point[b][k] = v->branch_point[6 * b + k];
    cp(s.lt_ij, v->lt_ij);
    cp(s.lt_ji, v->lt_ji);
    cp(s.rho_tilde, v->rho_tilde);
    if (v->beta) s.beta = *v->beta;
}

// cfg layout (doubles): rho_pq, rho_va, beta0, eps, inner_tol, max_outer,
// max_inner, workers, lambda_bound, beta_max
SolverConfig config_from(const double* c) {
    SolverConfig cfg;
    if (!c) return cfg;
    cfg.rho_pq = c[0];
    cfg.rho_va = c[1];
    cfg.beta0 = c[2];
    cfg.eps = c[3];
    cfg.inner_tol = c[4];
    cfg.max_outer = static_cast<int>(c[5]);
    cfg.max_inner = static_cast<int>(c[6]);
    cfg.workers = static_cast<int>(c[7]);
    cfg.lambda_max = c[8];
    cfg.lambda_min = -c[8];
    cfg.beta_max = c[9];
    return cfg;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

void* ref_net_load(const char* path) {
    try {
        return new PowerNetwork(load_case(path));
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

void ref_net_free(void* net) { delete static_cast<PowerNetwork*>(net); }

void ref_net_dims(const void* netp, int* nb, int* ng, int* nl, int* m) {
    const auto& net = *static_cast<const PowerNetwork*>(netp);
    *nb = static_cast<int>(net.buses.size());
    *ng = static_cast<int>(net.generators.size());
    *nl = static_cast<int>(net.branches.size());
    *m = build_layout(net).size();
}

// Parsed network in flat arrays (for checking the product parser).
// bus: 6 per bus (pd, qd, gs, bs, vmin, vmax) + ids; gen: 8 per gen (bus,
// pmin, pmax, qmin, qmax, c2, c1, c0); branch: 2 ints + 14 doubles
// (r, x, b, tap, shift, rate, gii, bii, gij, bij, gji, bji, gjj, bjj).
void ref_net_export(const void* netp, double* bus, int* bus_id, double* gen,
                    int* br_ends, double* br, int* ref_bus) {
    const auto& net = *static_cast<const PowerNetwork*>(netp);
    for (size_t i = 0; i < net.buses.size(); ++i) {
        const Bus& b = net.buses[i];
        const double v[6] = {b.pd, b.qd, b.gs, b.bs, b.vmin, b.vmax};
        std::memcpy(bus + 6 * i, v, sizeof v);
        bus_id[i] = b.id;
    }
    for (size_t g = 0; g < net.generators.size(); ++g) {
        const Generator& x = net.generators[g];
        const double v[8] = {static_cast<double>(x.bus), x.pmin, x.pmax, x.qmin,
                             x.qmax, x.c2, x.c1, x.c0};
        std::memcpy(gen + 8 * g, v, sizeof v);
    }
    for (size_t l = 0; l < net.branches.size(); ++l) {
        const Branch& x = net.branches[l];
        br_ends[2 * l] = x.from;
        br_ends[2 * l + 1] = x.to;
        const double v[14] = {x.r, x.x, x.b_charging, x.tap, x.shift, x.rate,
                              x.y.gii, x.y.bii, x.y.gij, x.y.bij,
                              x.y.gji, x.y.bji, x.y.gjj, x.y.bjj};
        std::memcpy(br + 14 * l, v, sizeof v);
    }
    *ref_bus = net.ref_bus;
}

// Bus row lists in the reference's CouplingLayout order (decomp.cpp:7-31):
// per bus, counts[6*i + {0..5}] = |gen_p|,|gen_q|,|flow_p|,|flow_q|,|w|,|theta|
// and rows concatenated in that group order into `rows` (length m).
void ref_layout_export(const void* netp, int* counts, int* rows) {
    const auto& net = *static_cast<const PowerNetwork*>(netp);
    const CouplingLayout layout = build_layout(net);
    int pos = 0;
    for (size_t i = 0; i < net.buses.size(); ++i) {
        const auto& r = layout.bus_rows(static_cast<int>(i));
        const std::vector<int>* groups[6] = {&r.gen_p, &r.gen_q, &r.flow_p,
                                             &r.flow_q, &r.w, &r.theta};
        for (int k = 0; k < 6; ++k) {
            counts[6 * i + k] = static_cast<int>(groups[k]->size());
            for (int row : *groups[k]) rows[pos++] = row;
        }
    }
}

int ref_cold_start(const void* netp, const double* cfgv,
                   const gridadmm_state_view* out) {
    const auto& net = *static_cast<const PowerNetwork*>(netp);
    const SolverConfig cfg = config_from(cfgv);
    const CouplingLayout layout = build_layout(net);
    to_view(cold_start(net, layout, cfg), out);
    return 0;
}

// Runs one phase on the given state in place.  Returns failures (branches),
// singular bus internal index or -1 (buses), 0 otherwise; -2 on error.
long ref_phase(const void* netp, int phase, const double* cfgv,
               gridadmm_state_view* io, double z_inf, double prev_z_inf) {
    const auto& net = *static_cast<const PowerNetwork*>(netp);
    const SolverConfig cfg = config_from(cfgv);
    const CouplingLayout layout = build_layout(net);
    AdmmState s = make_state(net, layout, cfg.rho_pq, cfg.rho_va, cfg.beta0);
    from_view(s, io);
    long ret = 0;
    try {
        switch (phase) {
            case GRIDADMM_PHASE_GENERATORS: solve_generators(s, net, layout); break;
            case GRIDADMM_PHASE_BRANCHES:
                ret = solve_branch_batch(s, net, layout, cfg.tron, cfg.workers,
                                         cfg.limit_tighten).failures;
                break;
            case GRIDADMM_PHASE_BUSES:
                ret = -1;
                solve_buses(s, net, layout, cfg.workers);
                break;
            case GRIDADMM_PHASE_Z: solve_z(s, layout); break;
            case GRIDADMM_PHASE_Y: update_y(s, layout); break;
            case GRIDADMM_PHASE_OUTER: {
                OuterSchedule sch;
                sch.lambda_min = cfg.lambda_min;
                sch.lambda_max = cfg.lambda_max;
                sch.beta_growth = cfg.beta_growth;
                sch.beta_shrink_trigger = cfg.beta_shrink_trigger;
                sch.beta_max = cfg.beta_max;
                update_outer(s, sch, z_inf, prev_z_inf);
                break;
            }
            default: g_err = "bad phase"; return -2;
        }
    } catch (const SingularBusError& e) {
        for (size_t i = 0; i < net.buses.size(); ++i)
            if (net.buses[i].id == e.bus) ret = static_cast<long>(i);
        g_err = e.what();
    }
    to_view(s, io);
    return ret;
}

// Full solve (proj/src/driver.cpp:140-246).  init may be NULL (cold start).
// series receives up to cap records of 6 doubles (outer, inner, primal,
// dual, z_norm, elapsed_s); info receives status, outer, inner, failures, objective,
// balance_inf, limit_violation, bound_violation, c_inf (9 doubles).
int ref_solve(const void* netp, const double* cfgv,
              const gridadmm_state_view* init, gridadmm_state_view* fin,
              double* series, int cap, int* nseries, double* info) {
    const auto& net = *static_cast<const PowerNetwork*>(netp);
    const SolverConfig cfg = config_from(cfgv);
    try {
        SolveReport rep;
        AdmmState final_state;
        if (init) {
            const CouplingLayout layout = build_layout(net);
            AdmmState s0 = make_state(net, layout, cfg.rho_pq, cfg.rho_va, cfg.beta0);
            from_view(s0, init);
            rep = solve(net, cfg, &s0, &final_state);
        } else {
            rep = solve(net, cfg, nullptr, &final_state);
        }
        if (fin) to_view(final_state, fin);
        const int n = static_cast<int>(rep.series.size());
        if (nseries) *nseries = n;
        for (int k = 0; k < std::min(n, cap); ++k) {
            const IterationRecord& r = rep.series[k];
            series[6 * k + 0] = r.outer;
            series[6 * k + 1] = r.inner;
            series[6 * k + 2] = r.primal_res;
            series[6 * k + 3] = r.dual_res;
            series[6 * k + 4] = r.z_norm;
            series[6 * k + 5] = r.elapsed_s;
        }
        if (info) {
            info[0] = static_cast<double>(rep.status);
            info[1] = rep.outer_iterations;
            info[2] = rep.inner_iterations;
            info[3] = rep.branch_solve_failures;
            info[4] = rep.quality.objective;
            info[5] = rep.quality.balance_inf;
            info[6] = rep.quality.limit_violation;
            info[7] = rep.quality.bound_violation;
            info[8] = rep.quality.c_inf;
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// Generic TRON on dense box QPs f = g'x + x'Hx/2 (acceptance criterion 3,
// proj/tests/acceptance.cpp:458-520): H is n*n per problem, g n, bounds n.
namespace {
class DenseQp final : public BoxNlp {
public:
    int n;
    const double *h, *g, *l, *u;
    int dim() const override { return n; }
    const double* lower() const override { return l; }
    const double* upper() const override { return u; }
    double value(const double* x) const override {
        double f = 0.0;
        for (int i = 0; i < n; ++i) {
            double hx = 0.0;
            for (int j = 0; j < n; ++j) hx += h[i * n + j] * x[j];
            f += g[i] * x[i] + 0.5 * x[i] * hx;
        }
        return f;
    }
    void gradient(const double* x, double* out) const override {
        for (int i = 0; i < n; ++i) {
            double hx = 0.0;
            for (int j = 0; j < n; ++j) hx += h[i * n + j] * x[j];
            out[i] = g[i] + hx;
        }
    }
    void hessian(const double*, double* out) const override {
        std::memcpy(out, h, sizeof(double) * n * n);
    }
};
}  // namespace

void ref_tron_qp(int count, int n, const double* h, const double* g,
                 const double* l, const double* u, double* x, int* status,
                 int* iterations) {
    TronSettings st;
    for (int k = 0; k < count; ++k) {
        DenseQp qp;
        qp.n = n;
        qp.h = h + static_cast<size_t>(k) * n * n;
        qp.g = g + static_cast<size_t>(k) * n;
        qp.l = l + static_cast<size_t>(k) * n;
        qp.u = u + static_cast<size_t>(k) * n;
        const TronResult r = solve_one(qp, x + static_cast<size_t>(k) * n, st);
        status[k] = static_cast<int>(r.status);
        iterations[k] = r.iterations;
    }
}

}  // extern "C"
