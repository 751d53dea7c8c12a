// solver.hpp — host driver of the device-resident two-level ADMM
// (Algorithm 1; reference proj/src/driver.{hpp,cpp}) and warm-start
// tracking (proj/src/tracking.{hpp,cpp}).
//
// A Session owns one copy of the network and the full AdmmState in HBM on
// one CUDA device plus a private stream; every inner iteration is four
// kernel phases on that stream followed by one 56-byte D2H of the reduced
// norms (the only host<->device traffic of the loop).  The state never
// leaves the device between iterations, outer iterations or tracking
// periods.
#ifndef GA_SOLVER_HPP
#define GA_SOLVER_HPP

#include <memory>
#include <stdexcept>
#include <string>
#include <cstdio>
#include <vector>

#include "device.hpp"
#include "network.hpp"
#include "partition.hpp"

namespace ga {

struct SolverConfig {  // proj/src/driver.hpp:15-40
    double rho_pq = 10.0;
    double rho_va = 1000.0;
    double beta0 = 1e3;
    double beta_growth = 10.0;
    double beta_shrink_trigger = 0.25;
    double beta_max = 1e12;
    double eps = 1e-4;
    double inner_tol = 0.0;
    int max_outer = 20;
    int max_inner = 1000;
    double lambda_min = -1e12;
    double lambda_max = 1e12;
    double divergence_threshold = 1e8;
    double limit_tighten = 0.99;
    double warm_beta_cap = 1e6;
    BranchCfg tron;  // gtol, max_iterations, cg_tol, max_cg, delta_floor
    int workers = 1;  // accepted for API compatibility; unused on the GPU
    int device = 0;
    int partitions = 1;  // bus-graph parts (multi.cpp); 1 = single session
    int devices = 1;     // parts are placed round-robin on devices [device, device+devices)

    double effective_inner_tol(int m) const;
};

enum class SolveStatus { Converged = 0, IterationLimit = 1, Diverged = 2 };

struct IterationRecord {
    int outer = 0, inner = 0;
    double primal_res = 0, dual_res = 0, z_norm = 0, elapsed_s = 0;
};

struct Solution {
    std::vector<double> pg, qg, vm, va;
    std::vector<double> flows;  // 4 per branch: pij, qij, pji, qji
};

struct QualityMetrics {
    double balance_inf = 0, limit_violation = 0, bound_violation = 0, c_inf = 0, objective = 0;
};

struct PhaseTimes {
    double x_s = 0, xbar_s = 0, z_s = 0, y_s = 0;
};

struct SolveReport {
    SolveStatus status = SolveStatus::IterationLimit;
    std::vector<IterationRecord> series;
    int outer_iterations = 0;
    int inner_iterations = 0;
    int branch_solve_failures = 0;
    PhaseTimes phase_times;
    Solution solution;
    QualityMetrics quality;
    std::string diagnostic;
};

class SingularBusError : public std::runtime_error {
public:
    SingularBusError(int bus_id, const std::string& w) : std::runtime_error(w), bus(bus_id) {}
    int bus;
};

class CudaError : public std::runtime_error {
public:
    explicit CudaError(const std::string& w) : std::runtime_error(w) {}
};

// Host copy of one AdmmState (proj/src/decomp.hpp:64-78); bp is 6 per
// branch, branch-major as in the reference.
struct HostState {
    std::vector<double> x, xbar, z, y, lambda, rho, bus_w, bus_theta, bp, lt_ij, lt_ji, rho_t;
    double beta = 0.0;
};

struct KernelClock {
    double ms = 0.0;
    long long launches = 0;
};

struct IterScalars {
    double primal = 0, dual_raw = 0, z_inf = 0, z_drift = 0;
    int failures = 0;
    int singular_bus = -1;  // internal index of the first singular bus, -1 if none
};

// What the Algorithm-1 driver (solve, run_tracking) needs from a device
// backend: one Session (one GPU), or MultiPart (a bus-graph partition over
// several sessions with boundary exchange, multi.cpp).
class Engine {
public:
    virtual ~Engine() = default;
    virtual const Network& network() const = 0;
    virtual const SolverConfig& config() const = 0;
    virtual int m() const = 0;
    virtual void cold_start() = 0;
    virtual void upload_state(const HostState& s) = 0;
    virtual void download_state(HostState& s) const = 0;
    virtual double beta() const = 0;
    virtual void set_beta(double b) = 0;
    virtual void set_loads(const std::vector<double>& pd, const std::vector<double>& qd) = 0;
    virtual void set_gen_p_bounds(const std::vector<double>& pmin,
                                  const std::vector<double>& pmax) = 0;
    virtual void clamp_gen_p() = 0;
    // One inner iteration; out = primal, dual (raw), z_inf, z_drift; returns
    // branch failures; throws SingularBusError.
    virtual int iterate(double out[4], PhaseTimes* times) = 0;
    virtual void outer_update() = 0;
    virtual double rho_max() = 0;
    virtual void download_solution_inputs(std::vector<double>& gen_rows, std::vector<double>& w,
                                          std::vector<double>& th) const = 0;
    // Solution extraction + quality metrics on the device (extract.cu);
    // false when this engine leaves them to the host (multi-part engines).
    virtual bool extract_on_device(Solution& sol, QualityMetrics& q) { return false; }
    // The inner loop of one outer iteration as CUDA graphs of several
    // iterations with the stop tests on the device (no host round trip per
    // iteration).  Appends the records, counts and phase times to `rep`;
    // *stop = LoopStop, *last_z = ||z||_inf of the last iteration.  Returns
    // false when this engine runs the host loop instead.
    virtual bool inner_loop(const SolverConfig& cfg, int outer, double rho_max, double inner_tol,
                            double elapsed_s, SolveReport& rep, int* stop, double* last_z) {
        return false;
    }
    virtual int parts() const { return 1; }
    // k iterations each bracketed by CUDA events (see Session::timed_steps)
    virtual int timed_steps(int k, size_t flush_bytes, double* step_ms, double* records) = 0;
};

class Session : public Engine {
public:
    // plan == nullptr: the session owns the whole network; otherwise only the
    // plan's generators / branches / buses / rows (multi-part runs).
    Session(const Network& net, const SolverConfig& cfg, const PartPlan* plan = nullptr);
    ~Session() override;

    // Split inner iteration for multi-part drivers: x phase (generators +
    // branches), bus + z/y phase, then the D2H of this part's scalars.
    void enqueue_x_phase();
    void enqueue_xbar_zy_phase(bool copy_scalars = true);
    void enqueue_scalars_d2h();
    IterScalars read_scalars();
    DevScalars* dev_scalars() const { return sc_; }
    cudaStream_t stream() const { return stream_; }
    const DevState& dev_state() const { return ds_; }
    const PartPlan* plan() const { return plan_.parts > 1 ? &plan_ : nullptr; }
    // device copies of plan_.send_x[q] / recv_x[q]
    const int* d_send_x(int q) const { return d_send_[q]; }
    const int* d_recv_x(int q) const { return d_recv_[q]; }
    Session(const Session&) = delete;
    Session& operator=(const Session&) = delete;

    const Network& network() const override { return net_; }
    const SolverConfig& config() const override { return cfg_; }
    int m() const override { return dn_.m; }

    void cold_start() override;                      // driver.cpp:26-63 (host) -> upload
    void upload_state(const HostState& s) override;  // any empty vector is skipped
    void download_state(HostState& s) const override;
    double beta() const override { return beta_; }
    void set_beta(double b) override { beta_ = b; }

    // Tracking: per-period loads and generator p-bounds (tracking.cpp:14-26,50-63).
    void set_loads(const std::vector<double>& pd, const std::vector<double>& qd) override;
    void set_gen_p_bounds(const std::vector<double>& pmin,
                          const std::vector<double>& pmax) override;
    void clamp_gen_p() override;

    // One phase (phase-replay API).  Returns failures / singular bus / 0.
    long run_phase(int phase, double z_inf, double prev_z_inf);

    // One fused inner iteration: gen, branch, bus, z/y/norms, then one D2H of
    // the scalars.  Fills out[0..3] = primal_inf, dual_inf (raw, before
    // rho_max), z_inf, z_drift; returns branch failures; throws
    // SingularBusError.
    int iterate(double out[4], PhaseTimes* times) override { return iterate_ev(out, times, nullptr); }
    // One inner iteration's branch and bus kernels on stream_: the bus kernel
    // for the buses not adjacent to a branch still running after the lane
    // phase runs on side_ beside the tile / solo phases, the rest after them
    // (GRIDADMM_BUS_OVERLAP=0: one bus kernel after the branch phase).
    void enqueue_iteration(const BranchCfg& bc, LoopCtl* gate, cudaEvent_t mid,
                           cudaEvent_t before_bus);
    int iterate_ev(double out[4], PhaseTimes* times, cudaEvent_t end_event);

    // Benchmark helper: k iterations, each bracketed by CUDA events on the
    // session stream (launches through the D2H of its norms); an L2 flush of
    // flush_bytes runs between steps outside the brackets.  records gets 5
    // doubles per step (primal, dual, z, z_drift, failures).
    int timed_steps(int k, size_t flush_bytes, double* step_ms, double* records) override;
    void outer_update() override;              // lambda clamp on the device
    double rho_max() override;                 // max over rows, device reduction

    KernelClock kernel_clock(int cls) const { return clocks_[cls]; }
    long long tron_iterations() const;
    void branch_costs(int* out) const;
    // TRON iterations (reference semantics) and executed steps, 4-/6-var.
    void step_counters(long long out[4]) const;
    long long limited_tron_iterations() const;  // 6-variable branches only
    void sync() const;

    bool extract_on_device(Solution& sol, QualityMetrics& q) override;
    bool inner_loop(const SolverConfig& cfg, int outer, double rho_max, double inner_tol,
                    double elapsed_s, SolveReport& rep, int* stop, double* last_z) override;
    // Solution extraction inputs: x gen rows, bus_w, bus_theta.
    void download_solution_inputs(std::vector<double>& gen_rows, std::vector<double>& w,
                                  std::vector<double>& th) const override;

private:
    void use_device() const;
    void upload_network();
    void free_all();
    Network net_;
    SolverConfig cfg_;
    DevNet dn_;
    DevState ds_;
    DevExtract ext_;  // single-part sessions only
    RowLayout layout_;  // device storage order of the rows
    // graph path (inner_loop): control block, records, the captured batch
    LoopCtl* ctl_ = nullptr;
    LoopCtl* ctl_host_ = nullptr;  // pinned
    LoopRec* rec_ = nullptr;
    LoopRec* rec_host_ = nullptr;  // pinned
    int rec_cap_ = 0;
    cudaGraphExec_t graph_ = nullptr;
    static constexpr int kGraphIters = 16;
    DevScalars* sc_ = nullptr;       // device
    DevScalars* sc_host_ = nullptr;  // pinned mirror
    unsigned long long* red_ = nullptr;
    void* flush_buf_ = nullptr;
    size_t flush_size_ = 0;
    double beta_ = 0.0;
    cudaStream_t stream_ = nullptr;
    cudaStream_t side_ = nullptr;  // bus kernel (undeferred buses) beside the tile / solo phases
    cudaEvent_t fork_ = nullptr, join_ = nullptr;
    cudaEvent_t side_ev_[2] = {};  // bus kernel on side_ (timed iterations)
    bool side_timed_ = false;      // the last timed iteration split the bus kernel
    cudaEvent_t ev_[6] = {};
    KernelClock clocks_[6];  // gen, branch, bus(+z/y), zy (fused: 0), lane phase, tile phase
    std::FILE* prof_ = nullptr;  // GRIDADMM_PROFILE=<csv>: per-iteration kernel times
    long prof_it_ = 0;
    std::vector<void*> allocs_;
    PartPlan plan_;
    std::vector<int*> d_send_, d_recv_;
};

SolveReport solve(Engine& s, const SolverConfig& cfg, bool warm);

// One Session, or a MultiPart over cfg.partitions parts on cfg.devices
// devices when partitions > 1 (multi.cpp).
std::unique_ptr<Engine> make_engine(const Network& net, const SolverConfig& cfg);

// One process per GPU (dist.cpp): rank `rank` of `world` owns part rank of
// partition_buses(net, world); boundary rows and norms go over NCCL.
void nccl_unique_id(unsigned char out[128]);
std::unique_ptr<Engine> make_dist_engine(const Network& net, const SolverConfig& cfg, int rank,
                                         int world, const unsigned char* id);

Solution extract_solution(const Network& net, const std::vector<double>& gen_rows,
                          const std::vector<double>& bus_w, const std::vector<double>& bus_theta);
QualityMetrics evaluate_solution(const Network& net, const Solution& sol);
void finish_metrics(const Network& net, const Solution& sol, std::vector<int>& cand,
                    double balance_inf, double bound_violation, QualityMetrics& q);

// ---- tracking (tracking.hpp) --------------------------------------------
class RampError : public std::runtime_error {
public:
    RampError(int period, int gen, const std::string& w)
        : std::runtime_error(w), period(period), generator(gen) {}
    int period, generator;
};

struct TrackingScenario {
    std::vector<double> multipliers;
    std::vector<std::vector<double>> per_bus;
    double ramp_fraction = 0.02;
    int periods() const { return static_cast<int>(multipliers.size()); }
};

struct PeriodReport {
    int period = 0;
    SolveReport report;
    double time_s = 0.0;
};

std::vector<PeriodReport> run_tracking(const Network& net, const SolverConfig& cfg,
                                       const TrackingScenario& sc);
TrackingScenario load_profile_csv(const std::string& path, const Network& net);

// ---- outputs (outputs.hpp) ----------------------------------------------
double report_gap(double objective, double reference);
void write_solution_json(const std::string& path, const Network& net, const SolveReport& r,
                         double ref_objective);
void write_convergence_csv(const std::string& path, const std::vector<IterationRecord>& s);
void write_periods_csv(const std::string& path, const std::vector<PeriodReport>& p,
                       const std::vector<double>& refs);

// GRIDADMM_TRACE=1: host-side phase timings of a solve on stderr
// (engine setup, cold start, iteration loop, solution extraction).
void trace_phase(const char* what);

}  // namespace ga

#endif
