// solve.cpp — Algorithm-1 loop control over a device-resident Session
// (proj/src/driver.cpp:65-246) and warm-start tracking
// (proj/src/tracking.cpp:30-85); file formats are in io.cpp.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <map>
#include <memory>
#include <sstream>

#include "ga_math.h"
#include "solver.hpp"

namespace ga {

namespace {

using Clock = std::chrono::steady_clock;

}  // namespace

void trace_phase(const char* what) {
    static const bool on = [] {
        const char* e = std::getenv("GRIDADMM_TRACE");
        return e && *e == '1';
    }();
    if (!on) return;
    static Clock::time_point last = Clock::now();
    const auto now = Clock::now();
    std::fprintf(stderr, "[gridadmm] %-28s +%9.3f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - last).count());
    last = now;
}

namespace {

double seconds_since(Clock::time_point t0) {
    return std::chrono::duration<double>(Clock::now() - t0).count();
}

// std::max over an initializer list: first maximal element by operator<.
double max_list(std::initializer_list<double> l) {
    const double* best = l.begin();
    for (const double* it = l.begin() + 1; it != l.end(); ++it)
        if (*best < *it) best = it;
    return *best;
}

}  // namespace

Solution extract_solution(const Network& net, const std::vector<double>& gen_rows,
                          const std::vector<double>& bus_w, const std::vector<double>& bus_theta) {
    Solution sol;
    const int ng = net.ng(), nb = net.nb(), nl = net.nl();
    sol.pg.resize(ng);
    sol.qg.resize(ng);
    for (int g = 0; g < ng; ++g) {
        sol.pg[g] = gen_rows[2 * g];
        sol.qg[g] = gen_rows[2 * g + 1];
    }
    sol.vm.resize(nb);
    sol.va.resize(nb);
    for (int i = 0; i < nb; ++i) {
        sol.vm[i] = std::sqrt(smax(0.0, bus_w[i]));
        sol.va[i] = bus_theta[i];
    }
    sol.flows.resize(4 * static_cast<size_t>(nl));
    for (int b = 0; b < nl; ++b) {
        const Line& l = net.lines[b];
        branch_flows_host(l.y, sol.vm[l.from], sol.vm[l.to], sol.va[l.from], sol.va[l.to],
                          &sol.flows[4 * static_cast<size_t>(b)]);
    }
    return sol;
}

// driver.cpp:89-138
QualityMetrics evaluate_solution(const Network& net, const Solution& sol) {
    QualityMetrics q;
    constexpr double kTwoPi = 6.283185307179586;
    const int nb = net.nb(), ng = net.ng(), nl = net.nl();
    std::vector<double> pbal(nb), qbal(nb);
    for (int i = 0; i < nb; ++i) {
        const Bus& bus = net.buses[i];
        const double w = sol.vm[i] * sol.vm[i];
        pbal[i] = -bus.pd - bus.gs * w;
        qbal[i] = -bus.qd + bus.bs * w;
    }
    for (int g = 0; g < ng; ++g) {
        const Gen& gen = net.gens[g];
        pbal[gen.bus] += sol.pg[g];
        qbal[gen.bus] += sol.qg[g];
        q.objective += gen.c2 * sol.pg[g] * sol.pg[g] + gen.c1 * sol.pg[g] + gen.c0;
    }
    for (int b = 0; b < nl; ++b) {
        const Line& l = net.lines[b];
        const double* f = &sol.flows[4 * static_cast<size_t>(b)];
        pbal[l.from] -= f[0];
        qbal[l.from] -= f[1];
        pbal[l.to] -= f[2];
        qbal[l.to] -= f[3];
        if (l.limited())
            q.limit_violation = max_list({q.limit_violation, std::hypot(f[0], f[1]) - l.rate,
                                          std::hypot(f[2], f[3]) - l.rate});
    }
    q.limit_violation = smax(0.0, q.limit_violation);
    auto inf_norm = [](const std::vector<double>& v) {
        double n = 0.0;
        for (double x : v) n = smax(n, std::abs(x));
        return n;
    };
    q.balance_inf = smax(inf_norm(pbal), inf_norm(qbal));
    for (int g = 0; g < ng; ++g) {
        const Gen& gen = net.gens[g];
        q.bound_violation = max_list({q.bound_violation, gen.pmin - sol.pg[g], sol.pg[g] - gen.pmax,
                                      gen.qmin - sol.qg[g], sol.qg[g] - gen.qmax});
    }
    for (int i = 0; i < nb; ++i) {
        const Bus& bus = net.buses[i];
        q.bound_violation = max_list({q.bound_violation, bus.vmin - sol.vm[i], sol.vm[i] - bus.vmax,
                                      std::abs(sol.va[i]) - kTwoPi});
    }
    q.bound_violation = smax(0.0, q.bound_violation);
    q.c_inf = max_list({q.balance_inf, q.limit_violation, q.bound_violation});
    return q;
}

// The two metric pieces the device leaves to the host (extract.cu): the
// objective, a sequential sum in generator order (driver.cpp:97-98), and the
// line-limit violation with glibc's hypot over the candidate branches (any
// other branch has hypot - rate < 0, driver.cpp:108-114).
void finish_metrics(const Network& net, const Solution& sol, std::vector<int>& cand,
                    double balance_inf, double bound_violation, QualityMetrics& q) {
    q = QualityMetrics{};
    for (int g = 0; g < net.ng(); ++g) {
        const Gen& gen = net.gens[g];
        q.objective += gen.c2 * sol.pg[g] * sol.pg[g] + gen.c1 * sol.pg[g] + gen.c0;
    }
    std::sort(cand.begin(), cand.end());
    for (int b : cand) {
        const Line& l = net.lines[b];
        const double* f = &sol.flows[4 * static_cast<size_t>(b)];
        q.limit_violation = max_list({q.limit_violation, std::hypot(f[0], f[1]) - l.rate,
                                      std::hypot(f[2], f[3]) - l.rate});
    }
    q.limit_violation = smax(0.0, q.limit_violation);
    q.balance_inf = balance_inf;
    q.bound_violation = bound_violation;
    q.c_inf = max_list({q.balance_inf, q.limit_violation, q.bound_violation});
}

namespace {

void finish_report(Engine& s, SolveReport& rep) {
    trace_phase("iteration loop");
    if (s.extract_on_device(rep.solution, rep.quality)) {
        trace_phase("device extract + metrics");
        return;
    }
    std::vector<double> gen_rows, w, th;
    s.download_solution_inputs(gen_rows, w, th);
    trace_phase("solution download");
    rep.solution = extract_solution(s.network(), gen_rows, w, th);
    rep.quality = evaluate_solution(s.network(), rep.solution);
    trace_phase("extract + evaluate");
}

}  // namespace

// driver.cpp:140-246.  warm == false -> cold start on the device state.
SolveReport solve(Engine& s, const SolverConfig& cfg, bool warm) {
    const auto t0 = Clock::now();
    trace_phase("solve entry");
    if (!warm) s.cold_start();
    trace_phase("cold start + upload");
    SolveReport report;
    const double inner_tol = cfg.effective_inner_tol(s.m());
    double prev_z_inf = -1.0;
    const double rho_max = s.rho_max();
    trace_phase("rho_max");
    double last_z_inf = 0.0;

    for (int outer = 1; outer <= cfg.max_outer; ++outer) {
        report.outer_iterations = outer;
        int stop = 0;
        if (s.inner_loop(cfg, outer, rho_max, inner_tol, seconds_since(t0), report, &stop,
                         &last_z_inf)) {
            if (stop == kLoopDiverged) {
                const IterationRecord& r = report.series.back();
                report.status = SolveStatus::Diverged;
                report.diagnostic = "residual norm exceeded divergence threshold at outer " +
                                    std::to_string(r.outer) + " inner " + std::to_string(r.inner);
                finish_report(s, report);
                return report;
            }
        } else {
            for (int inner = 1; inner <= cfg.max_inner; ++inner) {
                double nrm[4];
                report.branch_solve_failures += s.iterate(nrm, &report.phase_times);
                const double primal = nrm[0];
                const double dual = nrm[1] * rho_max;
                const double z_inf = nrm[2];
                last_z_inf = z_inf;
                ++report.inner_iterations;
                report.series.push_back({outer, inner, primal, dual, z_inf, seconds_since(t0)});
                if (!sfinite(primal) || !sfinite(dual) || primal > cfg.divergence_threshold ||
                    dual > cfg.divergence_threshold) {
                    report.status = SolveStatus::Diverged;
                    report.diagnostic = "residual norm exceeded divergence threshold at outer " +
                                        std::to_string(outer) + " inner " + std::to_string(inner);
                    finish_report(s, report);
                    return report;
                }
                if (smax(primal, dual) <= inner_tol) break;
                if (primal <= inner_tol && z_inf <= cfg.eps && nrm[3] <= 0.01 * cfg.eps) break;
            }
        }
        // ||z||_inf of the state after the inner loop == the last record's
        const double z_inf = last_z_inf;
        if (z_inf <= cfg.eps) {
            report.status = SolveStatus::Converged;
            break;
        }
        s.outer_update();
        if (prev_z_inf >= 0.0 && z_inf > cfg.beta_shrink_trigger * prev_z_inf)
            s.set_beta(smin(s.beta() * cfg.beta_growth, cfg.beta_max));
        prev_z_inf = z_inf;
    }
    finish_report(s, report);
    return report;
}

// ---- tracking (tracking.cpp:30-85) --------------------------------------
std::vector<PeriodReport> run_tracking(const Network& net, const SolverConfig& cfg,
                                       const TrackingScenario& sc) {
    if (sc.periods() == 0) throw std::invalid_argument("tracking scenario has no periods");
    for (const auto& row : sc.per_bus)
        if (!row.empty() && row.size() != net.buses.size())
            throw std::invalid_argument("per-bus multiplier row size mismatch");
    std::vector<PeriodReport> reports;
    reports.reserve(sc.periods());
    std::unique_ptr<Engine> eng = make_engine(net, cfg);
    Engine& session = *eng;
    std::vector<double> prev_pg;
    const int nb = net.nb(), ng = net.ng();
    std::vector<double> pd(nb), qd(nb), pmin(ng), pmax(ng);
    for (int t = 0; t < sc.periods(); ++t) {
        const bool per_bus = static_cast<size_t>(t) < sc.per_bus.size() && !sc.per_bus[t].empty();
        for (int i = 0; i < nb; ++i) {
            const double mult = per_bus ? sc.per_bus[t][i] : sc.multipliers[t];
            pd[i] = net.buses[i].pd * mult;
            qd[i] = net.buses[i].qd * mult;
        }
        const auto tp = Clock::now();
        session.set_loads(pd, qd);
        if (t > 0) {
            for (int g = 0; g < ng; ++g) {
                const Gen& gen = net.gens[g];
                const double rg = sc.ramp_fraction * gen.pmax;
                const double lo = smax(gen.pmin, prev_pg[g] - rg);
                const double hi = smin(gen.pmax, prev_pg[g] + rg);
                if (lo > hi) {
                    char buf[64];
                    std::snprintf(buf, sizeof buf, "[%f, %f]", lo, hi);
                    throw RampError(t + 1, g,
                                    "empty ramp window for generator " + std::to_string(g) +
                                        " in period " + std::to_string(t + 1) + ": " + buf);
                }
                pmin[g] = lo;
                pmax[g] = hi;
            }
            session.set_gen_p_bounds(pmin, pmax);
            session.clamp_gen_p();
            if (cfg.warm_beta_cap > 0.0) session.set_beta(smin(session.beta(), cfg.warm_beta_cap));
        }
        PeriodReport pr;
        pr.period = t + 1;
        pr.report = solve(session, cfg, t > 0);
        pr.time_s = seconds_since(tp);
        prev_pg = pr.report.solution.pg;
        reports.push_back(std::move(pr));
    }
    return reports;
}

}  // namespace ga
