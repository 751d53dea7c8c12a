// solve.cpp — Algorithm-1 loop control over a device-resident Session
// (proj/src/driver.cpp:65-246), warm-start tracking
// (proj/src/tracking.cpp:30-196) and the report writers
// (proj/src/outputs.cpp).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <map>
#include <memory>
#include <sstream>

#include <json.hpp>

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

namespace {

void finish_report(Engine& s, SolveReport& rep) {
    trace_phase("iteration loop");
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

// tracking.cpp:114-196
TrackingScenario load_profile_csv(const std::string& path, const Network& net) {
    std::ifstream in(path);
    if (!in) throw ParseError("cannot open profile file: " + path);
    std::string line;
    if (!std::getline(in, line)) throw ParseError("empty profile file: " + path);
    auto split = [](const std::string& s) {
        std::vector<std::string> out;
        std::stringstream ss(s);
        std::string f;
        while (std::getline(ss, f, ',')) {
            f.erase(0, f.find_first_not_of(" \t\r"));
            f.erase(f.find_last_not_of(" \t\r") + 1);
            out.push_back(f);
        }
        return out;
    };
    const auto header = split(line);
    bool per_bus_mode;
    if (header.size() == 2 && header[0] == "period" && header[1] == "multiplier") per_bus_mode = false;
    else if (header.size() == 3 && header[0] == "period" && header[1] == "bus" &&
             header[2] == "multiplier")
        per_bus_mode = true;
    else throw ParseError("unrecognized profile header: " + line);

    std::map<int, double> uniform;
    std::map<int, std::vector<double>> table;
    int lineno = 1;
    while (std::getline(in, line)) {
        ++lineno;
        const auto fields = split(line);
        if (fields.empty() || (fields.size() == 1 && fields[0].empty())) continue;
        try {
            if (!per_bus_mode) {
                if (fields.size() != 2) throw std::invalid_argument("field count");
                uniform[std::stoi(fields[0])] = std::stod(fields[1]);
            } else {
                if (fields.size() != 3) throw std::invalid_argument("field count");
                const int period = std::stoi(fields[0]);
                const int bus = std::stoi(fields[1]);
                const auto it = net.bus_index.find(bus);
                if (it == net.bus_index.end())
                    throw std::invalid_argument("unknown bus " + std::to_string(bus));
                auto& row = table[period];
                row.resize(net.buses.size(), 1.0);
                row[it->second] = std::stod(fields[2]);
            }
        } catch (const std::exception& e) {
            throw ParseError("profile line " + std::to_string(lineno) + ": " + e.what());
        }
    }
    std::map<int, double> keys;
    if (per_bus_mode)
        for (const auto& kv : table) keys[kv.first] = 1.0;
    else keys = uniform;
    if (keys.empty()) throw ParseError("profile has no data rows: " + path);
    const int periods = static_cast<int>(keys.size());
    for (int t = 1; t <= periods; ++t)
        if (!keys.count(t))
            throw ParseError("profile periods must be contiguous 1..T; missing " + std::to_string(t));
    TrackingScenario sc;
    sc.multipliers.assign(periods, 1.0);
    if (per_bus_mode) {
        sc.per_bus.resize(periods);
        for (auto& kv : table) sc.per_bus[kv.first - 1] = std::move(kv.second);
    } else {
        for (const auto& kv : uniform) sc.multipliers[kv.first - 1] = kv.second;
    }
    return sc;
}

// ---- outputs (outputs.cpp) ----------------------------------------------
namespace {

const char* status_name(SolveStatus s) {
    switch (s) {
        case SolveStatus::Converged: return "converged";
        case SolveStatus::IterationLimit: return "iteration_limit";
        case SolveStatus::Diverged: return "diverged";
    }
    return "unknown";
}

std::ofstream open_or_throw(const std::string& path) {
    std::ofstream out(path);
    if (!out) throw std::runtime_error("cannot write output file: " + path);
    return out;
}

std::string fmt17(double v) {
    char buf[32];
    std::snprintf(buf, sizeof buf, "%.17g", v);
    return buf;
}

}  // namespace

double report_gap(double objective, double reference) {
    if (!(reference > 0.0)) throw std::invalid_argument("reference objective must be positive");
    return std::abs(objective - reference) / reference;
}

void write_solution_json(const std::string& path, const Network& net, const SolveReport& r,
                         double ref_objective) {
    nlohmann::json j;
    j["status"] = status_name(r.status);
    j["outer_iterations"] = r.outer_iterations;
    j["inner_iterations"] = r.inner_iterations;
    j["branch_solve_failures"] = r.branch_solve_failures;
    if (!r.diagnostic.empty()) j["diagnostic"] = r.diagnostic;
    j["metrics"] = {{"objective", r.quality.objective},
                    {"balance_inf", r.quality.balance_inf},
                    {"limit_violation", r.quality.limit_violation},
                    {"bound_violation", r.quality.bound_violation},
                    {"c_inf", r.quality.c_inf}};
    if (ref_objective > 0.0) {
        j["metrics"]["reference_objective"] = ref_objective;
        j["metrics"]["gap"] = report_gap(r.quality.objective, ref_objective);
    }
    j["phase_times_s"] = {{"x", r.phase_times.x_s},
                          {"xbar", r.phase_times.xbar_s},
                          {"z", r.phase_times.z_s},
                          {"y", r.phase_times.y_s}};
    auto gens = nlohmann::json::array();
    for (size_t g = 0; g < r.solution.pg.size(); ++g)
        gens.push_back({{"bus", net.buses[net.gens[g].bus].id},
                        {"pg", r.solution.pg[g]},
                        {"qg", r.solution.qg[g]}});
    j["generators"] = gens;
    auto buses = nlohmann::json::array();
    for (size_t i = 0; i < r.solution.vm.size(); ++i)
        buses.push_back({{"bus", net.buses[i].id}, {"vm", r.solution.vm[i]}, {"va", r.solution.va[i]}});
    j["buses"] = buses;
    auto branches = nlohmann::json::array();
    for (size_t b = 0; b < net.lines.size(); ++b) {
        const Line& l = net.lines[b];
        const double* f = &r.solution.flows[4 * b];
        branches.push_back({{"from", net.buses[l.from].id},
                            {"to", net.buses[l.to].id},
                            {"pij", f[0]},
                            {"qij", f[1]},
                            {"pji", f[2]},
                            {"qji", f[3]}});
    }
    j["branches"] = branches;
    open_or_throw(path) << j.dump(2) << "\n";
}

void write_convergence_csv(const std::string& path, const std::vector<IterationRecord>& s) {
    std::ofstream out = open_or_throw(path);
    out << "outer,inner,primal_res,dual_res,z_norm,elapsed_s\n";
    for (const auto& r : s)
        out << r.outer << ',' << r.inner << ',' << fmt17(r.primal_res) << ',' << fmt17(r.dual_res)
            << ',' << fmt17(r.z_norm) << ',' << fmt17(r.elapsed_s) << '\n';
}

void write_periods_csv(const std::string& path, const std::vector<PeriodReport>& p,
                       const std::vector<double>& refs) {
    std::ofstream out = open_or_throw(path);
    out << "period,inner_iters,time_s,viol_inf,gap\n";
    for (size_t t = 0; t < p.size(); ++t) {
        out << p[t].period << ',' << p[t].report.inner_iterations << ',' << fmt17(p[t].time_s) << ','
            << fmt17(p[t].report.quality.c_inf) << ',';
        if (t < refs.size() && refs[t] > 0.0) out << fmt17(report_gap(p[t].report.quality.objective, refs[t]));
        else out << "nan";
        out << '\n';
    }
}

}  // namespace ga
