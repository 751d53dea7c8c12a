// capi.cpp — the C ABI (include/gridadmm/gridadmm.h, gridadmm_ext.h).
// Error/ownership contract of the reference proj/src/capi.cpp: exceptions
// never cross the boundary, gridadmm_last_error() is thread-local and never
// NULL, every *_free is NULL-safe, ITERATION_LIMIT / DIVERGED still return a
// report.  CUDA failures surface as GRIDADMM_ERR_INTERNAL with the CUDA
// error text (there is no CPU fallback).
#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "gridadmm/gridadmm.h"
#include "gridadmm/gridadmm_ext.h"
#include "solver.hpp"

namespace {

thread_local std::string g_last_error;

gridadmm_status fail(gridadmm_status code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

// (rho_pq, rho_va) presets: reference capi.cpp:25-39 / paper Table I.
const std::map<std::string, std::pair<double, double>>& presets() {
    static const std::map<std::string, std::pair<double, double>> t = {
        {"case2", {100.0, 10000.0}},          {"case9", {100.0, 10000.0}},
        {"case30", {100.0, 10000.0}},         {"case118", {100.0, 10000.0}},
        {"case1354pegase", {1e1, 1e3}},       {"case2869pegase", {1e1, 1e3}},
        {"case9241pegase", {5e1, 5e3}},       {"case13659pegase", {5e1, 5e3}},
        {"case_ACTIVSg25k", {3e3, 3e4}},      {"case_ACTIVSg70k", {3e4, 3e5}},
    };
    return t;
}

gridadmm_status status_of(ga::SolveStatus s) {
    switch (s) {
        case ga::SolveStatus::Converged: return GRIDADMM_OK;
        case ga::SolveStatus::IterationLimit: return GRIDADMM_ERR_ITERATION_LIMIT;
        case ga::SolveStatus::Diverged: return GRIDADMM_ERR_DIVERGED;
    }
    return GRIDADMM_ERR_INTERNAL;
}

}  // namespace

struct gridadmm_network {
    ga::Network net;
};
struct gridadmm_config {
    ga::SolverConfig solver;
    double ramp_frac = 0.02;
};
struct gridadmm_report {
    ga::SolveReport report;
    ga::Network net;
};
struct gridadmm_track {
    std::vector<ga::PeriodReport> periods;
    ga::Network net;
};
struct gridadmm_session {
    std::unique_ptr<ga::Engine> e;  // one Session or a MultiPart (config `partitions` > 1)
    ga::Session* s = nullptr;       // == e when single-part (kernel-level helpers)
};

namespace {

// Config key table (reference capi.cpp:97-128): name -> (get, set, integer, min)
struct Field {
    bool integer;
    double min;
    double (*get)(const gridadmm_config&);
    void (*set)(gridadmm_config&, double);
};

const std::map<std::string, Field>& fields() {
    static const std::map<std::string, Field> f = {
        {"rho_pq", {false, 1e-12, [](const gridadmm_config& c) { return c.solver.rho_pq; },
                    [](gridadmm_config& c, double v) { c.solver.rho_pq = v; }}},
        {"rho_va", {false, 1e-12, [](const gridadmm_config& c) { return c.solver.rho_va; },
                    [](gridadmm_config& c, double v) { c.solver.rho_va = v; }}},
        {"beta0", {false, 1e-12, [](const gridadmm_config& c) { return c.solver.beta0; },
                   [](gridadmm_config& c, double v) { c.solver.beta0 = v; }}},
        {"eps", {false, 1e-12, [](const gridadmm_config& c) { return c.solver.eps; },
                 [](gridadmm_config& c, double v) { c.solver.eps = v; }}},
        {"inner_tol", {false, 0.0, [](const gridadmm_config& c) { return c.solver.inner_tol; },
                       [](gridadmm_config& c, double v) { c.solver.inner_tol = v; }}},
        {"max_outer", {true, 1.0, [](const gridadmm_config& c) { return double(c.solver.max_outer); },
                       [](gridadmm_config& c, double v) { c.solver.max_outer = int(v); }}},
        {"max_inner", {true, 1.0, [](const gridadmm_config& c) { return double(c.solver.max_inner); },
                       [](gridadmm_config& c, double v) { c.solver.max_inner = int(v); }}},
        {"workers", {true, 1.0, [](const gridadmm_config& c) { return double(c.solver.workers); },
                     [](gridadmm_config& c, double v) { c.solver.workers = int(v); }}},
        {"lambda_bound", {false, 1.0, [](const gridadmm_config& c) { return c.solver.lambda_max; },
                          [](gridadmm_config& c, double v) { c.solver.lambda_max = v; }}},
        {"beta_max", {false, 1.0, [](const gridadmm_config& c) { return c.solver.beta_max; },
                      [](gridadmm_config& c, double v) { c.solver.beta_max = v; }}},
        {"ramp_frac", {false, 1e-12, [](const gridadmm_config& c) { return c.ramp_frac; },
                       [](gridadmm_config& c, double v) { c.ramp_frac = v; }}},
        {"device", {true, 0.0, [](const gridadmm_config& c) { return double(c.solver.device); },
                    [](gridadmm_config& c, double v) { c.solver.device = int(v); }}},
        // bus-graph partition (multi.cpp): parts, and GPUs they are spread over
        {"partitions", {true, 1.0, [](const gridadmm_config& c) { return double(c.solver.partitions); },
                        [](gridadmm_config& c, double v) { c.solver.partitions = int(v); }}},
        {"devices", {true, 1.0, [](const gridadmm_config& c) { return double(c.solver.devices); },
                     [](gridadmm_config& c, double v) { c.solver.devices = int(v); }}},
        // branch-phase scheduling (results do not depend on them): TRON steps a
        // branch may take in the lane phase / the 8-lane tile phase (0 = no solo phase)
        {"lane_budget", {true, 1.0, [](const gridadmm_config& c) { return double(c.solver.tron.lane_budget); },
                         [](gridadmm_config& c, double v) { c.solver.tron.lane_budget = int(v); }}},
        {"lane_cap", {true, 1.0, [](const gridadmm_config& c) { return double(c.solver.tron.lane_cap); },
                      [](gridadmm_config& c, double v) { c.solver.tron.lane_cap = int(v); }}},
        {"tile_budget", {true, 0.0, [](const gridadmm_config& c) { return double(c.solver.tron.tile_budget); },
                         [](gridadmm_config& c, double v) { c.solver.tron.tile_budget = int(v); }}},
    };
    return f;
}

template <class F>
gridadmm_status guarded(F&& fn) {
    try {
        return fn();
    } catch (const ga::ParseError& e) {
        return fail(GRIDADMM_ERR_PARSE, e.what());
    } catch (const ga::RampError& e) {
        return fail(GRIDADMM_ERR_INFEASIBLE_RAMP, e.what());
    } catch (const std::invalid_argument& e) {
        return fail(GRIDADMM_ERR_INVALID_ARG, e.what());
    } catch (const std::exception& e) {
        return fail(GRIDADMM_ERR_INTERNAL, e.what());
    } catch (...) {
        return fail(GRIDADMM_ERR_INTERNAL, "unknown error");
    }
}

}  // namespace

extern "C" {

const char* gridadmm_last_error(void) { return g_last_error.c_str(); }

gridadmm_status gridadmm_network_load(const char* path, gridadmm_network** out) {
    if (!path || !out) return fail(GRIDADMM_ERR_INVALID_ARG, "null argument to network_load");
    try {
        *out = new gridadmm_network{ga::load_matpower(path)};
        return GRIDADMM_OK;
    } catch (const ga::ParseError& e) {
        return fail(GRIDADMM_ERR_PARSE, e.what());
    } catch (const std::exception& e) {
        return fail(GRIDADMM_ERR_IO, e.what());
    }
}

void gridadmm_network_free(gridadmm_network* net) { delete net; }
int gridadmm_network_num_buses(const gridadmm_network* n) { return n ? n->net.nb() : 0; }
int gridadmm_network_num_generators(const gridadmm_network* n) { return n ? n->net.ng() : 0; }
int gridadmm_network_num_branches(const gridadmm_network* n) { return n ? n->net.nl() : 0; }
int gridadmm_network_num_rows(const gridadmm_network* n) { return n ? n->net.m() : 0; }

gridadmm_status gridadmm_network_export(const gridadmm_network* n, double* bus, int* bus_id,
                                        double* gen, int* ends, double* branch, int* ref_bus) {
    if (!n) return fail(GRIDADMM_ERR_INVALID_ARG, "null network");
    const ga::Network& net = n->net;
    for (int i = 0; i < net.nb(); ++i) {
        const ga::Bus& b = net.buses[i];
        if (bus) {
            const double v[6] = {b.pd, b.qd, b.gs, b.bs, b.vmin, b.vmax};
            std::memcpy(bus + 6 * i, v, sizeof v);
        }
        if (bus_id) bus_id[i] = b.id;
    }
    for (int g = 0; g < net.ng(); ++g) {
        const ga::Gen& x = net.gens[g];
        if (gen) {
            const double v[8] = {double(x.bus), x.pmin, x.pmax, x.qmin, x.qmax, x.c2, x.c1, x.c0};
            std::memcpy(gen + 8 * g, v, sizeof v);
        }
    }
    for (int l = 0; l < net.nl(); ++l) {
        const ga::Line& x = net.lines[l];
        if (ends) {
            ends[2 * l] = x.from;
            ends[2 * l + 1] = x.to;
        }
        if (branch) {
            const double v[6] = {x.r, x.x, x.b, x.tap, x.shift, x.rate};
            std::memcpy(branch + 14 * l, v, sizeof v);
            std::memcpy(branch + 14 * l + 6, x.y.c, sizeof x.y.c);
        }
    }
    if (ref_bus) *ref_bus = net.ref_bus;
    return GRIDADMM_OK;
}

gridadmm_status gridadmm_network_partition(const gridadmm_network* n, int k, int* part_of_bus) {
    if (!n || !part_of_bus || k < 1) return fail(GRIDADMM_ERR_INVALID_ARG, "bad argument to partition");
    const std::vector<int> part = ga::partition_buses(n->net, k);
    std::memcpy(part_of_bus, part.data(), part.size() * sizeof(int));
    return GRIDADMM_OK;
}

gridadmm_status gridadmm_network_set_branch_weights(gridadmm_network* n, const int* weights) {
    if (!n) return fail(GRIDADMM_ERR_INVALID_ARG, "null network");
    if (!weights) {
        n->net.branch_weight.clear();
        return GRIDADMM_OK;
    }
    const int nl = n->net.nl();
    for (int b = 0; b < nl; ++b)
        if (weights[b] < 0) return fail(GRIDADMM_ERR_INVALID_ARG, "negative branch weight");
    return guarded([&]() -> gridadmm_status {
        n->net.branch_weight.assign(weights, weights + nl);
        return GRIDADMM_OK;
    });
}

gridadmm_status gridadmm_network_exchange_rows(const gridadmm_network* n, int k, int p, int q,
                                               int* send_rows, int* n_send, int* recv_rows,
                                               int* n_recv) {
    if (!n || k < 1 || p < 0 || p >= k || q < 0 || q >= k || !n_send || !n_recv)
        return fail(GRIDADMM_ERR_INVALID_ARG, "bad argument to exchange_rows");
    return guarded([&]() -> gridadmm_status {
        const ga::PartPlan pl = ga::make_plan(n->net, ga::partition_buses(n->net, k), p, k);
        *n_send = static_cast<int>(pl.send_x[q].size());
        *n_recv = static_cast<int>(pl.recv_x[q].size());
        if (send_rows) std::memcpy(send_rows, pl.send_x[q].data(), pl.send_x[q].size() * sizeof(int));
        if (recv_rows) std::memcpy(recv_rows, pl.recv_x[q].data(), pl.recv_x[q].size() * sizeof(int));
        return GRIDADMM_OK;
    });
}

gridadmm_status gridadmm_network_layout(const gridadmm_network* n, int* counts, int* rows) {
    if (!n) return fail(GRIDADMM_ERR_INVALID_ARG, "null network");
    const ga::BusCsr csr = ga::build_bus_csr(n->net);
    // device CSR groups are [w, theta, gen_p, gen_q, flow_p, flow_q]; the
    // reference's BusRows order is (gen_p, gen_q, flow_p, flow_q, w, theta)
    static const int order[6] = {2, 3, 4, 5, 0, 1};
    int pos = 0;
    for (int i = 0; i < n->net.nb(); ++i) {
        for (int k = 0; k < 6; ++k) {
            const int g = order[k];
            const int a = csr.grp[7 * i + g], b = csr.grp[7 * i + g + 1];
            if (counts) counts[6 * i + k] = b - a;
            for (int j = a; j < b; ++j)
                if (rows) rows[pos++] = csr.rows[j];
        }
    }
    return GRIDADMM_OK;
}

gridadmm_config* gridadmm_config_new(void) { return new gridadmm_config{}; }
void gridadmm_config_free(gridadmm_config* cfg) { delete cfg; }

gridadmm_status gridadmm_config_set(gridadmm_config* cfg, const char* key, double value) {
    if (!cfg || !key) return fail(GRIDADMM_ERR_INVALID_ARG, "null argument to config_set");
    const auto it = fields().find(key);
    if (it == fields().end())
        return fail(GRIDADMM_ERR_INVALID_ARG, std::string("unknown config key: ") + key);
    const Field& f = it->second;
    if (!std::isfinite(value) || value < f.min || (f.integer && value != std::floor(value)))
        return fail(GRIDADMM_ERR_INVALID_ARG, std::string("invalid value for config key ") + key);
    f.set(*cfg, value);
    cfg->solver.lambda_min = -cfg->solver.lambda_max;
    return GRIDADMM_OK;
}

gridadmm_status gridadmm_config_get(const gridadmm_config* cfg, const char* key, double* out) {
    if (!cfg || !key || !out) return fail(GRIDADMM_ERR_INVALID_ARG, "null argument to config_get");
    const auto it = fields().find(key);
    if (it == fields().end())
        return fail(GRIDADMM_ERR_INVALID_ARG, std::string("unknown config key: ") + key);
    *out = it->second.get(*cfg);
    return GRIDADMM_OK;
}

gridadmm_status gridadmm_config_preset(gridadmm_config* cfg, const char* name) {
    if (!cfg || !name) return fail(GRIDADMM_ERR_INVALID_ARG, "null argument to config_preset");
    const auto it = presets().find(name);
    if (it == presets().end())
        return fail(GRIDADMM_ERR_INVALID_ARG, std::string("no penalty preset for case: ") + name);
    cfg->solver.rho_pq = it->second.first;
    cfg->solver.rho_va = it->second.second;
    return GRIDADMM_OK;
}

gridadmm_status gridadmm_solve(const gridadmm_network* net, const gridadmm_config* cfg,
                               gridadmm_report** out) {
    if (!net || !cfg || !out) return fail(GRIDADMM_ERR_INVALID_ARG, "null argument to solve");
    try {
        ga::trace_phase("gridadmm_solve entry");
        std::unique_ptr<ga::Engine> eng = ga::make_engine(net->net, cfg->solver);
        ga::trace_phase("engine ready");
        auto* rep = new gridadmm_report{ga::solve(*eng, cfg->solver, false), net->net};
        *out = rep;
        const gridadmm_status s = status_of(rep->report.status);
        if (s != GRIDADMM_OK)
            g_last_error = rep->report.diagnostic.empty() ? "solve did not converge"
                                                          : rep->report.diagnostic;
        return s;
    } catch (const std::exception& e) {
        return fail(GRIDADMM_ERR_INTERNAL, e.what());
    }
}

void gridadmm_report_free(gridadmm_report* rep) { delete rep; }

gridadmm_status gridadmm_report_metric(const gridadmm_report* rep, const char* key, double* out) {
    if (!rep || !key || !out) return fail(GRIDADMM_ERR_INVALID_ARG, "null argument to report_metric");
    const auto& r = rep->report;
    const std::map<std::string, double> m = {
        {"objective", r.quality.objective},
        {"balance_inf", r.quality.balance_inf},
        {"limit_violation", r.quality.limit_violation},
        {"bound_violation", r.quality.bound_violation},
        {"c_inf", r.quality.c_inf},
        {"outer_iterations", static_cast<double>(r.outer_iterations)},
        {"inner_iterations", static_cast<double>(r.inner_iterations)},
        {"branch_solve_failures", static_cast<double>(r.branch_solve_failures)},
    };
    const auto it = m.find(key);
    if (it == m.end()) return fail(GRIDADMM_ERR_INVALID_ARG, std::string("unknown metric key: ") + key);
    *out = it->second;
    return GRIDADMM_OK;
}

gridadmm_status gridadmm_report_dispatch(const gridadmm_report* rep, double* pg, double* qg) {
    if (!rep) return fail(GRIDADMM_ERR_INVALID_ARG, "null report in report_dispatch");
    const auto& sol = rep->report.solution;
    if (pg && !sol.pg.empty()) std::memcpy(pg, sol.pg.data(), sol.pg.size() * sizeof(double));
    if (qg && !sol.qg.empty()) std::memcpy(qg, sol.qg.data(), sol.qg.size() * sizeof(double));
    return GRIDADMM_OK;
}

gridadmm_status gridadmm_report_voltages(const gridadmm_report* rep, double* vm, double* va) {
    if (!rep) return fail(GRIDADMM_ERR_INVALID_ARG, "null report in report_voltages");
    const auto& sol = rep->report.solution;
    if (vm && !sol.vm.empty()) std::memcpy(vm, sol.vm.data(), sol.vm.size() * sizeof(double));
    if (va && !sol.va.empty()) std::memcpy(va, sol.va.data(), sol.va.size() * sizeof(double));
    return GRIDADMM_OK;
}

gridadmm_status gridadmm_report_write_solution(const gridadmm_report* rep, const char* path,
                                               double ref_objective) {
    if (!rep || !path) return fail(GRIDADMM_ERR_INVALID_ARG, "null argument to write_solution");
    try {
        ga::write_solution_json(path, rep->net, rep->report, ref_objective);
        return GRIDADMM_OK;
    } catch (const std::exception& e) {
        return fail(GRIDADMM_ERR_IO, e.what());
    }
}

gridadmm_status gridadmm_report_write_convergence(const gridadmm_report* rep, const char* path) {
    if (!rep || !path) return fail(GRIDADMM_ERR_INVALID_ARG, "null argument to write_convergence");
    try {
        ga::write_convergence_csv(path, rep->report.series);
        return GRIDADMM_OK;
    } catch (const std::exception& e) {
        return fail(GRIDADMM_ERR_IO, e.what());
    }
}

gridadmm_status gridadmm_track_run(const gridadmm_network* net, const gridadmm_config* cfg,
                                   const char* profile_path, gridadmm_track** out) {
    if (!net || !cfg || !profile_path || !out)
        return fail(GRIDADMM_ERR_INVALID_ARG, "null argument to track_run");
    return guarded([&]() -> gridadmm_status {
        ga::TrackingScenario sc = ga::load_profile_csv(profile_path, net->net);
        sc.ramp_fraction = cfg->ramp_frac;
        auto* trk = new gridadmm_track{ga::run_tracking(net->net, cfg->solver, sc), net->net};
        *out = trk;
        for (const auto& p : trk->periods) {
            const gridadmm_status s = status_of(p.report.status);
            if (s != GRIDADMM_OK) {
                g_last_error = "period " + std::to_string(p.period) + " did not converge";
                return s;
            }
        }
        return GRIDADMM_OK;
    });
}

void gridadmm_track_free(gridadmm_track* trk) { delete trk; }
int gridadmm_track_num_periods(const gridadmm_track* trk) {
    return trk ? static_cast<int>(trk->periods.size()) : 0;
}

gridadmm_status gridadmm_track_period_report(const gridadmm_track* trk, int period,
                                             gridadmm_report** out) {
    if (!trk || !out) return fail(GRIDADMM_ERR_INVALID_ARG, "null argument to period_report");
    if (period < 1 || period > static_cast<int>(trk->periods.size()))
        return fail(GRIDADMM_ERR_INVALID_ARG, "period out of range: " + std::to_string(period));
    *out = new gridadmm_report{trk->periods[period - 1].report, trk->net};
    return GRIDADMM_OK;
}

gridadmm_status gridadmm_track_write_periods(const gridadmm_track* trk, const char* path,
                                             const double* refs, int num_refs) {
    if (!trk || !path) return fail(GRIDADMM_ERR_INVALID_ARG, "null argument to write_periods");
    try {
        std::vector<double> r;
        if (refs && num_refs > 0) r.assign(refs, refs + num_refs);
        ga::write_periods_csv(path, trk->periods, r);
        return GRIDADMM_OK;
    } catch (const std::exception& e) {
        return fail(GRIDADMM_ERR_IO, e.what());
    }
}

// ---- extensions (gridadmm_ext.h) ----------------------------------------

gridadmm_status gridadmm_session_new(const gridadmm_network* net, const gridadmm_config* cfg,
                                     gridadmm_session** out) {
    if (!net || !cfg || !out) return fail(GRIDADMM_ERR_INVALID_ARG, "null argument to session_new");
    return guarded([&]() -> gridadmm_status {
        auto h = std::make_unique<gridadmm_session>();
        h->e = ga::make_engine(net->net, cfg->solver);
        h->s = dynamic_cast<ga::Session*>(h->e.get());
        h->e->cold_start();
        *out = h.release();
        return GRIDADMM_OK;
    });
}

void gridadmm_session_free(gridadmm_session* s) { delete s; }

gridadmm_status gridadmm_session_solve(gridadmm_session* s, const gridadmm_config* cfg, int warm,
                                       gridadmm_report** out) {
    if (!s || !cfg || !out) return fail(GRIDADMM_ERR_INVALID_ARG, "null argument to session_solve");
    try {
        auto* rep = new gridadmm_report{ga::solve(*s->e, cfg->solver, warm != 0), s->e->network()};
        *out = rep;
        const gridadmm_status st = status_of(rep->report.status);
        if (st != GRIDADMM_OK)
            g_last_error = rep->report.diagnostic.empty() ? "solve did not converge"
                                                          : rep->report.diagnostic;
        return st;
    } catch (const std::exception& e) {
        return fail(GRIDADMM_ERR_INTERNAL, e.what());
    }
}

gridadmm_status gridadmm_nccl_unique_id(unsigned char* out) {
    if (!out) return fail(GRIDADMM_ERR_INVALID_ARG, "null argument to nccl_unique_id");
    return guarded([&]() -> gridadmm_status {
        ga::nccl_unique_id(out);
        return GRIDADMM_OK;
    });
}

gridadmm_status gridadmm_session_new_dist(const gridadmm_network* net, const gridadmm_config* cfg,
                                          int rank, int world, const unsigned char* nccl_id,
                                          gridadmm_session** out) {
    if (!net || !cfg || !out || !nccl_id || world < 1 || rank < 0 || rank >= world)
        return fail(GRIDADMM_ERR_INVALID_ARG, "bad argument to session_new_dist");
    return guarded([&]() -> gridadmm_status {
        auto h = std::make_unique<gridadmm_session>();
        h->e = ga::make_dist_engine(net->net, cfg->solver, rank, world, nccl_id);
        h->e->cold_start();
        *out = h.release();
        return GRIDADMM_OK;
    });
}

gridadmm_status gridadmm_session_get_state(const gridadmm_session* s, const gridadmm_state_view* v) {
    if (!s || !v) return fail(GRIDADMM_ERR_INVALID_ARG, "null argument to session_get_state");
    return guarded([&]() -> gridadmm_status {
        ga::HostState h;
        s->e->download_state(h);
        auto cp = [](const std::vector<double>& src, double* dst) {
            if (dst && !src.empty()) std::memcpy(dst, src.data(), src.size() * sizeof(double));
        };
        cp(h.x, v->x); cp(h.xbar, v->xbar); cp(h.z, v->z); cp(h.y, v->y);
        cp(h.lambda, v->lambda); cp(h.rho, v->rho); cp(h.bus_w, v->bus_w);
        cp(h.bus_theta, v->bus_theta); cp(h.bp, v->branch_point); cp(h.lt_ij, v->lt_ij);
        cp(h.lt_ji, v->lt_ji); cp(h.rho_t, v->rho_tilde);
        if (v->beta) *v->beta = h.beta;
        return GRIDADMM_OK;
    });
}

gridadmm_status gridadmm_session_set_state(gridadmm_session* s, const gridadmm_state_view* v) {
    if (!s || !v) return fail(GRIDADMM_ERR_INVALID_ARG, "null argument to session_set_state");
    return guarded([&]() -> gridadmm_status {
        const ga::Network& n = s->e->network();
        const size_t m = n.m(), nb = n.nb(), nl = n.nl();
        ga::HostState h;
        auto cp = [](std::vector<double>& dst, const double* src, size_t count) {
            if (src) dst.assign(src, src + count);
        };
        cp(h.x, v->x, m); cp(h.xbar, v->xbar, m); cp(h.z, v->z, m); cp(h.y, v->y, m);
        cp(h.lambda, v->lambda, m); cp(h.rho, v->rho, m); cp(h.bus_w, v->bus_w, nb);
        cp(h.bus_theta, v->bus_theta, nb); cp(h.bp, v->branch_point, 6 * nl);
        cp(h.lt_ij, v->lt_ij, nl); cp(h.lt_ji, v->lt_ji, nl); cp(h.rho_t, v->rho_tilde, nl);
        h.beta = v->beta ? *v->beta : s->e->beta();
        s->e->upload_state(h);
        return GRIDADMM_OK;
    });
}

gridadmm_status gridadmm_session_phase(gridadmm_session* s, int phase, double* aux) {
    if (!s) return fail(GRIDADMM_ERR_INVALID_ARG, "null session");
    if (phase < 0 || phase > 5) return fail(GRIDADMM_ERR_INVALID_ARG, "unknown phase");
    if (!s->s) return fail(GRIDADMM_ERR_INVALID_ARG, "phase replay needs a single-part session");
    return guarded([&]() -> gridadmm_status {
        const double zi = (phase == 5 && aux) ? aux[0] : 0.0;
        const double pz = (phase == 5 && aux) ? aux[1] : -1.0;
        const long r = s->s->run_phase(phase, zi, pz);
        if (aux && (phase == 1 || phase == 2)) aux[0] = static_cast<double>(r);
        return GRIDADMM_OK;
    });
}

gridadmm_status gridadmm_session_iterate(gridadmm_session* s, int n, double* records, int* done,
                                         int* stop) {
    if (!s || n < 0) return fail(GRIDADMM_ERR_INVALID_ARG, "bad argument to session_iterate");
    return guarded([&]() -> gridadmm_status {
        const ga::SolverConfig& cfg = s->e->config();
        const double inner_tol = cfg.effective_inner_tol(s->e->m());
        const double rho_max = s->e->rho_max();
        int k = 0, why = 0;
        for (; k < n; ++k) {
            double nrm[4];
            const int fails = s->e->iterate(nrm, nullptr);
            const double primal = nrm[0], dual = nrm[1] * rho_max, z = nrm[2];
            if (records) {
                double* r = records + 5 * k;
                r[0] = primal; r[1] = dual; r[2] = z; r[3] = nrm[3]; r[4] = fails;
            }
            if (!std::isfinite(primal) || !std::isfinite(dual) || primal > cfg.divergence_threshold ||
                dual > cfg.divergence_threshold) { why = 2; ++k; break; }
            if (std::max(primal, dual) <= inner_tol ||
                (primal <= inner_tol && z <= cfg.eps && nrm[3] <= 0.01 * cfg.eps)) { why = 1; ++k; break; }
        }
        if (done) *done = k;
        if (stop) *stop = why;
        return GRIDADMM_OK;
    });
}

gridadmm_status gridadmm_session_timed_steps(gridadmm_session* s, int n, size_t flush_bytes,
                                             double* step_ms, double* records) {
    if (!s || n < 0) return fail(GRIDADMM_ERR_INVALID_ARG, "bad argument to session_timed_steps");
    return guarded([&]() -> gridadmm_status {
        s->e->timed_steps(n, flush_bytes, step_ms, records);
        return GRIDADMM_OK;
    });
}

gridadmm_status gridadmm_session_kernel_time(const gridadmm_session* s, int cls, double* ms,
                                             long long* launches) {
    if (!s || cls < 0 || cls > 5) return fail(GRIDADMM_ERR_INVALID_ARG, "bad argument to kernel_time");
    if (!s->s) return fail(GRIDADMM_ERR_INVALID_ARG, "kernel_time needs a single-part session");
    const ga::KernelClock c = s->s->kernel_clock(cls);
    if (ms) *ms = c.ms;
    if (launches) *launches = c.launches;
    return GRIDADMM_OK;
}

gridadmm_status gridadmm_session_counters(const gridadmm_session* s, long long* tron_iterations,
                                          long long* limited_iterations) {
    if (!s || !s->s) return fail(GRIDADMM_ERR_INVALID_ARG, "counters need a single-part session");
    return guarded([&]() -> gridadmm_status {
        if (tron_iterations) *tron_iterations = s->s->tron_iterations();
        if (limited_iterations) *limited_iterations = s->s->limited_tron_iterations();
        return GRIDADMM_OK;
    });
}

gridadmm_status gridadmm_session_step_counters(const gridadmm_session* s, long long* out) {
    if (!s || !out || !s->s) return fail(GRIDADMM_ERR_INVALID_ARG, "bad argument to step_counters");
    return guarded([&]() -> gridadmm_status {
        s->s->step_counters(out);
        return GRIDADMM_OK;
    });
}

gridadmm_status gridadmm_session_branch_costs(const gridadmm_session* s, int* costs) {
    if (!s || !costs || !s->s) return fail(GRIDADMM_ERR_INVALID_ARG, "bad argument to branch_costs");
    return guarded([&]() -> gridadmm_status {
        s->s->branch_costs(costs);
        return GRIDADMM_OK;
    });
}

gridadmm_status gridadmm_debug_tron_stats(unsigned long long* out, int reset) {
    if (!out) return fail(GRIDADMM_ERR_INVALID_ARG, "null argument to tron_stats");
    return guarded([&]() -> gridadmm_status {
        ga::tron_stats(out, reset != 0);
        return GRIDADMM_OK;
    });
}

int gridadmm_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}

// Parity probes of the TRON core and the pinned sincos (test-only entry
// points; same C conventions).
gridadmm_status gridadmm_probe_tron_qp(int count, int n, const double* h, const double* g,
                                       const double* l, const double* u, double* x, int* status,
                                       int* iterations, int tile) {
    if (count < 0 || n < 1 || n > 6 || (tile != 1 && tile != 4 && tile != 8 && tile != 32))
        return fail(GRIDADMM_ERR_INVALID_ARG, "bad qp batch");
    return guarded([&]() -> gridadmm_status {
        const size_t nn = static_cast<size_t>(count) * n;
        double *dh, *dg, *dl, *du, *dx;
        int *ds, *di;
        auto ck = [](cudaError_t e) { if (e != cudaSuccess) throw ga::CudaError(cudaGetErrorString(e)); };
        ck(cudaMalloc(&dh, std::max<size_t>(1, nn * n) * 8)); ck(cudaMalloc(&dg, std::max<size_t>(1, nn) * 8));
        ck(cudaMalloc(&dl, std::max<size_t>(1, nn) * 8)); ck(cudaMalloc(&du, std::max<size_t>(1, nn) * 8));
        ck(cudaMalloc(&dx, std::max<size_t>(1, nn) * 8));
        ck(cudaMalloc(&ds, std::max(1, count) * 4)); ck(cudaMalloc(&di, std::max(1, count) * 4));
        ck(cudaMemcpy(dh, h, nn * n * 8, cudaMemcpyHostToDevice));
        ck(cudaMemcpy(dg, g, nn * 8, cudaMemcpyHostToDevice));
        ck(cudaMemcpy(dl, l, nn * 8, cudaMemcpyHostToDevice));
        ck(cudaMemcpy(du, u, nn * 8, cudaMemcpyHostToDevice));
        ck(cudaMemcpy(dx, x, nn * 8, cudaMemcpyHostToDevice));
        ga::launch_tron_qp(count, n, dh, dg, dl, du, dx, ds, di, nullptr, tile);
        ck(cudaGetLastError());
        ck(cudaMemcpy(x, dx, nn * 8, cudaMemcpyDeviceToHost));
        ck(cudaMemcpy(status, ds, count * 4, cudaMemcpyDeviceToHost));
        ck(cudaMemcpy(iterations, di, count * 4, cudaMemcpyDeviceToHost));
        for (void* p : {(void*)dh, (void*)dg, (void*)dl, (void*)du, (void*)dx, (void*)ds, (void*)di}) cudaFree(p);
        return GRIDADMM_OK;
    });
}

gridadmm_status gridadmm_probe_fp64_peak(int device, double* tflops_mul_add, double* tflops_fma) {
    return guarded([&]() -> gridadmm_status {
        if (cudaSetDevice(device) != cudaSuccess) throw ga::CudaError("cudaSetDevice");
        double a = 0.0, b = 0.0;
        ga::measure_fp64_peak(&a, &b);
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) throw ga::CudaError(cudaGetErrorString(e));
        if (tflops_mul_add) *tflops_mul_add = a;
        if (tflops_fma) *tflops_fma = b;
        return GRIDADMM_OK;
    });
}

gridadmm_status gridadmm_probe_sincos(int n, const double* x, double* s, double* c) {
    if (n < 0) return fail(GRIDADMM_ERR_INVALID_ARG, "bad count");
    return guarded([&]() -> gridadmm_status {
        double *dx, *ds, *dc;
        auto ck = [](cudaError_t e) { if (e != cudaSuccess) throw ga::CudaError(cudaGetErrorString(e)); };
        const size_t b = std::max(1, n) * sizeof(double);
        ck(cudaMalloc(&dx, b)); ck(cudaMalloc(&ds, b)); ck(cudaMalloc(&dc, b));
        ck(cudaMemcpy(dx, x, n * sizeof(double), cudaMemcpyHostToDevice));
        ga::launch_sincos_probe(dx, ds, dc, n, nullptr);
        ck(cudaGetLastError());
        ck(cudaMemcpy(s, ds, n * sizeof(double), cudaMemcpyDeviceToHost));
        ck(cudaMemcpy(c, dc, n * sizeof(double), cudaMemcpyDeviceToHost));
        cudaFree(dx); cudaFree(ds); cudaFree(dc);
        return GRIDADMM_OK;
    });
}

}  // extern "C"
