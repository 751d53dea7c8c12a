// io.cpp — the host-side file formats around the solver: the tracking
// profile reader (format of proj/src/tracking.cpp:114-196) and the three
// report writers (formats of proj/src/outputs.cpp:25-135).  Formats and
// error behaviour are the reference's contract (README.md:110-126); the
// code is organised around whole-buffer I/O so a 70k-bus solution is
// written with one syscall instead of ~10^6 stream insertions.
#include <cmath>
#include <cstdio>
#include <fstream>
#include <iterator>
#include <stdexcept>
#include <string>
#include <string_view>
#include <unordered_map>
#include <vector>

#include <json.hpp>

#include "solver.hpp"

namespace ga {

namespace {

// ---- profile reader ------------------------------------------------------

// The comma-separated fields of one line, each with surrounding blanks
// (space, tab, CR) removed.  An empty line yields no fields.
std::vector<std::string> csv_fields(std::string_view line) {
    std::vector<std::string> out;
    if (line.empty()) return out;
    constexpr std::string_view kBlank = " \t\r";
    size_t pos = 0;
    for (;;) {
        const size_t comma = line.find(',', pos);
        std::string_view f = line.substr(pos, comma == std::string_view::npos ? line.npos : comma - pos);
        const size_t a = f.find_first_not_of(kBlank);
        f = a == f.npos ? std::string_view{} : f.substr(a, f.find_last_not_of(kBlank) - a + 1);
        out.emplace_back(f);
        if (comma == std::string_view::npos) break;
        pos = comma + 1;
        if (pos == line.size()) break;  // a trailing comma adds no empty field
    }
    return out;
}

enum class ProfileKind { Uniform, PerBus };

ProfileKind profile_kind(const std::vector<std::string>& h, const std::string& raw) {
    if (h.size() == 2 && h[0] == "period" && h[1] == "multiplier") return ProfileKind::Uniform;
    if (h.size() == 3 && h[0] == "period" && h[1] == "bus" && h[2] == "multiplier")
        return ProfileKind::PerBus;
    throw ParseError("unrecognized profile header: " + raw);
}

}  // namespace

TrackingScenario load_profile_csv(const std::string& path, const Network& net) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw ParseError("cannot open profile file: " + path);
    const std::string text{std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>()};

    size_t pos = 0;
    auto next_line = [&](std::string_view& line) {
        if (pos >= text.size()) return false;
        const size_t nl = text.find('\n', pos);
        const size_t end = nl == std::string::npos ? text.size() : nl;
        line = std::string_view(text).substr(pos, end - pos);
        pos = end + 1;
        return true;
    };

    std::string_view line;
    if (!next_line(line)) throw ParseError("empty profile file: " + path);
    const ProfileKind kind = profile_kind(csv_fields(line), std::string(line));
    const size_t width = kind == ProfileKind::Uniform ? 2 : 3;

    // period -> its values: one multiplier (uniform) or one per bus in
    // network order, buses not listed keep 1.0; a repeated entry overwrites
    std::unordered_map<int, std::vector<double>> by_period;
    for (int lineno = 2; next_line(line); ++lineno) {
        const auto f = csv_fields(line);
        if (f.empty() || (f.size() == 1 && f[0].empty())) continue;
        try {
            if (f.size() != width) throw std::invalid_argument("field count");
            const int period = std::stoi(f[0]);
            if (kind == ProfileKind::Uniform) {
                by_period[period] = {std::stod(f[1])};
                continue;
            }
            const int bus_id = std::stoi(f[1]);
            const auto bus = net.bus_index.find(bus_id);
            if (bus == net.bus_index.end())
                throw std::invalid_argument("unknown bus " + std::to_string(bus_id));
            auto& row = by_period[period];
            if (row.empty()) row.assign(net.buses.size(), 1.0);
            row[bus->second] = std::stod(f[2]);
        } catch (const std::exception& e) {
            throw ParseError("profile line " + std::to_string(lineno) + ": " + e.what());
        }
    }
    if (by_period.empty()) throw ParseError("profile has no data rows: " + path);
    const int periods = static_cast<int>(by_period.size());
    for (int t = 1; t <= periods; ++t)
        if (!by_period.count(t))
            throw ParseError("profile periods must be contiguous 1..T; missing " + std::to_string(t));

    TrackingScenario sc;
    sc.multipliers.assign(periods, 1.0);
    if (kind == ProfileKind::PerBus) sc.per_bus.resize(periods);
    for (auto& [period, values] : by_period) {
        if (kind == ProfileKind::Uniform) sc.multipliers[period - 1] = values[0];
        else sc.per_bus[period - 1] = std::move(values);
    }
    return sc;
}

// ---- report writers ------------------------------------------------------

namespace {

// Text built in memory, written to `path` in one call.
class TextFile {
public:
    explicit TextFile(std::string path) : path_(std::move(path)) {}
    TextFile& str(std::string_view s) { buf_.append(s); return *this; }
    TextFile& ch(char c) { buf_.push_back(c); return *this; }
    TextFile& num(long v) { return str(std::to_string(v)); }
    // %.17g: every double printed so it reads back to the same bits
    TextFile& g17(double v) {
        char tmp[32];
        const int n = std::snprintf(tmp, sizeof tmp, "%.17g", v);
        buf_.append(tmp, static_cast<size_t>(n));
        return *this;
    }
    void commit() const {
        std::FILE* f = std::fopen(path_.c_str(), "wb");
        if (!f) throw std::runtime_error("cannot write output file: " + path_);
        const size_t n = std::fwrite(buf_.data(), 1, buf_.size(), f);
        const bool ok = n == buf_.size() && std::fclose(f) == 0;
        if (!ok) throw std::runtime_error("cannot write output file: " + path_);
    }

private:
    std::string path_;
    std::string buf_;
};

constexpr const char* kStatusText[] = {"converged", "iteration_limit", "diverged"};

}  // namespace

double report_gap(double objective, double reference) {
    if (!(reference > 0.0)) throw std::invalid_argument("reference objective must be positive");
    return std::abs(objective - reference) / reference;
}

void write_solution_json(const std::string& path, const Network& net, const SolveReport& r,
                         double ref_objective) {
    using nlohmann::json;
    const Solution& sol = r.solution;
    const QualityMetrics& q = r.quality;

    json metrics = json::object();
    for (const auto& [key, v] : {std::pair<const char*, double>{"objective", q.objective},
                                 {"balance_inf", q.balance_inf},
                                 {"limit_violation", q.limit_violation},
                                 {"bound_violation", q.bound_violation},
                                 {"c_inf", q.c_inf}})
        metrics[key] = v;
    if (ref_objective > 0.0) {
        metrics["reference_objective"] = ref_objective;
        metrics["gap"] = report_gap(q.objective, ref_objective);
    }
    json doc = {{"status", kStatusText[static_cast<int>(r.status)]},
                {"outer_iterations", r.outer_iterations},
                {"inner_iterations", r.inner_iterations},
                {"branch_solve_failures", r.branch_solve_failures},
                {"metrics", std::move(metrics)},
                {"phase_times_s", {{"x", r.phase_times.x_s},
                                   {"xbar", r.phase_times.xbar_s},
                                   {"z", r.phase_times.z_s},
                                   {"y", r.phase_times.y_s}}}};
    if (!r.diagnostic.empty()) doc["diagnostic"] = r.diagnostic;

    json& gens = doc["generators"] = json::array();
    for (size_t g = 0; g < sol.pg.size(); ++g)
        gens.push_back({{"bus", net.buses[net.gens[g].bus].id}, {"pg", sol.pg[g]}, {"qg", sol.qg[g]}});
    json& buses = doc["buses"] = json::array();
    for (size_t i = 0; i < sol.vm.size(); ++i)
        buses.push_back({{"bus", net.buses[i].id}, {"vm", sol.vm[i]}, {"va", sol.va[i]}});
    json& lines = doc["branches"] = json::array();
    static constexpr const char* kFlow[4] = {"pij", "qij", "pji", "qji"};
    for (size_t b = 0; b < net.lines.size(); ++b) {
        json e = {{"from", net.buses[net.lines[b].from].id}, {"to", net.buses[net.lines[b].to].id}};
        for (int k = 0; k < 4; ++k) e[kFlow[k]] = sol.flows[4 * b + k];
        lines.push_back(std::move(e));
    }
    TextFile(path).str(doc.dump(2)).ch('\n').commit();
}

void write_convergence_csv(const std::string& path, const std::vector<IterationRecord>& series) {
    TextFile out(path);
    out.str("outer,inner,primal_res,dual_res,z_norm,elapsed_s\n");
    for (const IterationRecord& it : series) {
        out.num(it.outer).ch(',').num(it.inner);
        for (double v : {it.primal_res, it.dual_res, it.z_norm, it.elapsed_s}) out.ch(',').g17(v);
        out.ch('\n');
    }
    out.commit();
}

void write_periods_csv(const std::string& path, const std::vector<PeriodReport>& periods,
                       const std::vector<double>& refs) {
    TextFile out(path);
    out.str("period,inner_iters,time_s,viol_inf,gap\n");
    for (size_t t = 0; t < periods.size(); ++t) {
        const PeriodReport& p = periods[t];
        out.num(p.period).ch(',').num(p.report.inner_iterations).ch(',').g17(p.time_s).ch(',');
        out.g17(p.report.quality.c_inf).ch(',');
        const bool have_ref = t < refs.size() && refs[t] > 0.0;
        if (have_ref) out.g17(report_gap(p.report.quality.objective, refs[t]));
        else out.str("nan");
        out.ch('\n');
    }
    out.commit();
}

}  // namespace ga
