// multi.cpp — the bus-graph-partitioned ADMM inside one
// process: `partitions` parts, each a Session that computes only its own
// generators / branches / buses / rows (partition.hpp), placed round-robin on
// `devices` GPUs.  Per inner iteration:
//   x phase on every part (concurrent streams / devices)
//   -> cut-branch far-end x rows copied solver part -> to-bus part
//      (a copy kernel on the destination device reading the source buffer;
//      across GPUs the read is a peer load over NVLink)
//   -> bus + z/y phase on every part
//   -> (xbar, z, y) of those rows copied back
//   -> residual norms max-reduced over parts (order-free, exact),
//      failures summed, first singular bus = min index.
// Every part holds full-size (replicated) arrays so row indices need no
// translation; only owned entries are computed.  Results are bit-identical
// to one Session (tests/test_gpu_parity.py::test_partitioned_*).
#include <algorithm>
#include <chrono>
#include <climits>
#include <cstring>

#include "ga_math.h"
#include "solver.hpp"

namespace ga {

namespace {

void check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

class MultiPart final : public Engine {
public:
    MultiPart(const Network& net, const SolverConfig& cfg) : net_(net), cfg_(cfg) {
        const int k = std::max(1, cfg.partitions);
        const int ndev = std::max(1, cfg.devices);
        part_of_bus_ = partition_buses(net, k);
        for (int p = 0; p < k; ++p) {
            SolverConfig c = cfg;
            c.device = cfg.device + (p % ndev);
            plans_.push_back(make_plan(net, part_of_bus_, p, k));
            parts_.push_back(std::make_unique<Session>(net, c, &plans_.back()));
        }
        // peer access between distinct devices (NVLink)
        for (int a = 0; a < ndev && a < k; ++a)
            for (int b = 0; b < ndev && b < k; ++b) {
                if (a == b) continue;
                int can = 0;
                cudaDeviceCanAccessPeer(&can, cfg.device + a, cfg.device + b);
                if (!can) throw CudaError("multi-device partition needs peer access between GPUs");
                cudaSetDevice(cfg.device + a);
                const cudaError_t e = cudaDeviceEnablePeerAccess(cfg.device + b, 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
                    check(e, "cudaDeviceEnablePeerAccess");
                cudaGetLastError();
            }
    }

    const Network& network() const override { return net_; }
    const SolverConfig& config() const override { return cfg_; }
    int m() const override { return net_.m(); }
    int parts() const override { return static_cast<int>(parts_.size()); }

    void cold_start() override {
        for (auto& s : parts_) on(*s).cold_start();
    }
    void upload_state(const HostState& s) override {
        for (auto& p : parts_) on(*p).upload_state(s);
    }
    // Merge by ownership: rows from their row owner, buses from their bus
    // owner, branch variables from the solver part.
    void download_state(HostState& out) const override {
        on(*parts_[0]).download_state(out);
        const int nl = net_.nl();
        for (size_t p = 1; p < parts_.size(); ++p) {
            HostState s;
            on(*parts_[p]).download_state(s);
            const PartPlan& pl = plans_[p];
            for (int r : pl.rows) {
                out.x[r] = s.x[r]; out.xbar[r] = s.xbar[r]; out.z[r] = s.z[r];
                out.y[r] = s.y[r]; out.lambda[r] = s.lambda[r]; out.rho[r] = s.rho[r];
            }
            for (int i : pl.buses) { out.bus_w[i] = s.bus_w[i]; out.bus_theta[i] = s.bus_theta[i]; }
            auto take_branch = [&](int b) {
                for (int k = 0; k < 6; ++k) out.bp[6 * static_cast<size_t>(b) + k] = s.bp[6 * static_cast<size_t>(b) + k];
                out.lt_ij[b] = s.lt_ij[b]; out.lt_ji[b] = s.lt_ji[b]; out.rho_t[b] = s.rho_t[b];
            };
            for (int b : pl.lim) take_branch(b);
            for (int b : pl.unl) take_branch(b);
            (void)nl;
        }
    }
    double beta() const override { return parts_[0]->beta(); }
    void set_beta(double b) override {
        for (auto& p : parts_) p->set_beta(b);
    }
    void set_loads(const std::vector<double>& pd, const std::vector<double>& qd) override {
        for (auto& p : parts_) on(*p).set_loads(pd, qd);
        for (size_t i = 0; i < pd.size(); ++i) {  // period network for the metrics
            net_.buses[i].pd = pd[i];
            net_.buses[i].qd = qd[i];
        }
    }
    void set_gen_p_bounds(const std::vector<double>& a, const std::vector<double>& b) override {
        for (auto& p : parts_) on(*p).set_gen_p_bounds(a, b);
        for (size_t g = 0; g < a.size(); ++g) {
            net_.gens[g].pmin = a[g];
            net_.gens[g].pmax = b[g];
        }
    }
    void clamp_gen_p() override {
        for (auto& p : parts_) on(*p).clamp_gen_p();
        for (auto& p : parts_) p->sync();
    }
    double rho_max() override {
        double r = 0.0;
        for (auto& p : parts_) r = smax(r, on(*p).rho_max());  // rho is replicated; all equal
        return r;
    }
    void outer_update() override {
        for (auto& p : parts_) on(*p).outer_update();
        for (auto& p : parts_) p->sync();
    }

    int iterate(double out[4], PhaseTimes* times) override {
        (void)times;
        const int k = parts();
        for (auto& p : parts_) p->enqueue_x_phase();
        for (auto& p : parts_) p->sync();
        // far-end x of cut branches: solver part p -> to-bus part q
        for (int p = 0; p < k; ++p)
            for (int q = 0; q < k; ++q) {
                if (p == q) continue;
                const int n = static_cast<int>(plans_[p].send_x[q].size());
                if (!n) continue;
                check(cudaSetDevice(parts_[q]->config().device), "cudaSetDevice");
                // q's recv list from p == p's send list to q (same rows, same order)
                launch_copy_rows(parts_[q]->d_recv_x(p), n, parts_[p]->dev_state().x,
                                 parts_[q]->dev_state().x, parts_[q]->stream());
            }
        for (auto& p : parts_) p->enqueue_xbar_zy_phase();
        IterScalars total;
        total.singular_bus = INT_MAX;
        for (auto& p : parts_) {
            const IterScalars s = p->read_scalars();
            total.primal = smax(total.primal, s.primal);
            total.dual_raw = smax(total.dual_raw, s.dual_raw);
            total.z_inf = smax(total.z_inf, s.z_inf);
            total.z_drift = smax(total.z_drift, s.z_drift);
            total.failures += s.failures;
            if (s.singular_bus >= 0) total.singular_bus = std::min(total.singular_bus, s.singular_bus);
        }
        // (xbar, z, y) of those rows back: to-bus part p -> solver part q
        for (int p = 0; p < k; ++p)
            for (int q = 0; q < k; ++q) {
                if (p == q) continue;
                const int n = static_cast<int>(plans_[p].recv_x[q].size());
                if (!n) continue;
                check(cudaSetDevice(parts_[q]->config().device), "cudaSetDevice");
                const DevState& a = parts_[p]->dev_state();
                const DevState& b = parts_[q]->dev_state();
                const int* rows = parts_[q]->d_send_x(p);  // == p's recv list from q
                launch_copy_rows(rows, n, a.xbar, b.xbar, parts_[q]->stream());
                launch_copy_rows(rows, n, a.z, b.z, parts_[q]->stream());
                launch_copy_rows(rows, n, a.y, b.y, parts_[q]->stream());
            }
        for (auto& p : parts_) p->sync();
        check(cudaGetLastError(), "exchange");
        if (total.singular_bus != INT_MAX) {
            const int id = net_.buses[total.singular_bus].id;
            throw SingularBusError(id, "isolated bus " + std::to_string(id) + ": singular balance system");
        }
        out[0] = total.primal;
        out[1] = total.dual_raw;
        out[2] = total.z_inf;
        out[3] = total.z_drift;
        return total.failures;
    }

    void download_solution_inputs(std::vector<double>& gen_rows, std::vector<double>& w,
                                  std::vector<double>& th) const override {
        on(*parts_[0]).download_solution_inputs(gen_rows, w, th);
        for (size_t p = 1; p < parts_.size(); ++p) {
            std::vector<double> g2, w2, t2;
            on(*parts_[p]).download_solution_inputs(g2, w2, t2);
            for (int g : plans_[p].gens) { gen_rows[2 * g] = g2[2 * g]; gen_rows[2 * g + 1] = g2[2 * g + 1]; }
            for (int i : plans_[p].buses) { w[i] = w2[i]; th[i] = t2[i]; }
        }
    }

    int timed_steps(int k, size_t, double* step_ms, double* records) override {
        // parts run on several streams: time each step host-side around the
        // fully synchronous iterate (every step ends with all streams synced)
        const double rmax = rho_max();
        for (int i = 0; i < k; ++i) {
            const auto t0 = std::chrono::steady_clock::now();
            double nrm[4];
            const int fails = iterate(nrm, nullptr);
            const double ms = std::chrono::duration<double, std::milli>(
                                  std::chrono::steady_clock::now() - t0).count();
            if (step_ms) step_ms[i] = ms;
            if (records) {
                double* r = records + 5 * i;
                r[0] = nrm[0]; r[1] = nrm[1] * rmax; r[2] = nrm[2]; r[3] = nrm[3]; r[4] = fails;
            }
        }
        return k;
    }

    const std::vector<int>& part_of_bus() const { return part_of_bus_; }

private:
    static Session& on(Session& s) {  // make the part's device current
        check(cudaSetDevice(s.config().device), "cudaSetDevice");
        return s;
    }

    Network net_;
    SolverConfig cfg_;
    std::vector<int> part_of_bus_;
    std::vector<PartPlan> plans_;
    std::vector<std::unique_ptr<Session>> parts_;
};

}  // namespace

std::unique_ptr<Engine> make_engine(const Network& net, const SolverConfig& cfg) {
    if (cfg.partitions > 1) return std::make_unique<MultiPart>(net, cfg);
    return std::make_unique<Session>(net, cfg);
}

}  // namespace ga
