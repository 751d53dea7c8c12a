// device.hpp — HBM-resident layout of one network + ADMM state, and the
// extern "C"-style launchers the host driver calls (one per phase).
//
// Layout (all FP64 unless noted, SoA, 256-B aligned allocations):
//   rows   the m = 2G + 8L coupling rows of the reference's CouplingLayout
//          (proj/src/decomp.hpp:32-36) stored bus-major (network.hpp
//          RowLayout): bus i owns the contiguous positions
//          [seg, gen_end) generator (p, q) pairs in generator order,
//          [gen_end, qstart) padding to a multiple of 4,
//          [qstart, end) one quad (p, q, w, theta) per incident branch end in
//          branch order.  x, xbar, z, y, lambda, rho: 6 mpad-vectors; the
//          padding positions hold zeros forever.  gpos / qpos map
//          generators / branch ends to positions.
//   branch L: ends (int32 from/to), 8 admittance coefficients [k*L + b],
//          rate, point [k*L + b] (k < 6), lt_ij, lt_ji, rho_tilde.
//   bus    N: pd, qd, gs, bs, vmin, vmax, w, theta; segment bounds.
//   gen    G: pmin, pmax, qmin, qmax, c2, c1.
#ifndef GA_DEVICE_HPP
#define GA_DEVICE_HPP

#include <cstdint>

#include <cuda_runtime.h>
#include <functional>

// Device-side bounds checks of the queue, flag and row indices (debug build
// -DGA_CHECKS, `make checks`; compute-sanitizer is unavailable on the GPU
// pool): a violated check traps, so the launch fails with an error.
#if defined(GA_CHECKS) && defined(__CUDA_ARCH__)
#define GA_CHECK(c) \
    do {            \
        if (!(c)) __trap(); \
    } while (0)
#else
#define GA_CHECK(c) ((void)0)
#endif

namespace ga {

struct DevNet {
    int nb = 0, ng = 0, nl = 0, m = 0;
    int mpad = 0;  // storage positions of the row vectors (m rows + padding)
    int ref_bus = -1;
    // generators
    double *g_pmin = nullptr, *g_pmax = nullptr, *g_qmin = nullptr, *g_qmax = nullptr;
    double *g_c2 = nullptr, *g_c1 = nullptr;
    // the same generator data in storage order, indexed by position / 2 of
    // the generator's (p, q) pair (read by the bus kernel without indirection)
    double *pr_c1 = nullptr, *pr_c2 = nullptr, *pr_pmin = nullptr, *pr_pmax = nullptr;
    double *pr_qmin = nullptr, *pr_qmax = nullptr;
    // branches
    int *br_from = nullptr, *br_to = nullptr;
    double* br_y = nullptr;     // [8][nl]: gii bii gij bij gji bji gjj bjj
    double* br_rate = nullptr;  // [nl], 0 = unlimited
    int* lim_list = nullptr;    // indices of rate-limited branches
    int* unl_list = nullptr;    // indices of unlimited branches
    int n_lim = 0, n_unl = 0;
    // buses
    double *b_pd = nullptr, *b_qd = nullptr, *b_gs = nullptr, *b_bs = nullptr;
    double *b_vmin = nullptr, *b_vmax = nullptr;
    int* bus_seg = nullptr;   // [4*nb] start, gen_end, qstart, end of each bus's rows
    int* gpos = nullptr;      // [ng] position of generator g's p row (q row at +1)
    int* qpos = nullptr;      // [2*nl] from-quad and to-quad position of branch b
    int* quad_branch = nullptr;  // [mpad/4 + 1] 2 b + side of the quad at 4 q, else -1
    int* rid = nullptr;       // [mpad] reference row of each position, -1 = padding
    // ownership subset of a multi-part run (partition.hpp); nullptr = all.
    // lim_list / unl_list above already hold only the owned branches.
    int* own_gens = nullptr;
    int* own_buses = nullptr;
    int* own_rows = nullptr;
    int n_own_gens = 0, n_own_buses = 0, n_own_rows = 0;

    __host__ __device__ int gens_count() const { return own_gens ? n_own_gens : ng; }
    __host__ __device__ int buses_count() const { return own_buses ? n_own_buses : nb; }
    __host__ __device__ int rows_count() const { return own_rows ? n_own_rows : mpad; }
    __host__ __device__ int gen_at(int t) const { return own_gens ? own_gens[t] : t; }
    __host__ __device__ int bus_at(int t) const { return own_buses ? own_buses[t] : t; }
    __host__ __device__ int row_at(int t) const { return own_rows ? own_rows[t] : t; }
};

struct DevState {
    double *x = nullptr, *xbar = nullptr, *z = nullptr, *y = nullptr;
    double *lambda = nullptr, *rho = nullptr;
    double *bus_w = nullptr, *bus_theta = nullptr;
    double* bp = nullptr;  // [6][nl]
    double *lt_ij = nullptr, *lt_ji = nullptr, *rho_t = nullptr;
    // scheduling state of the branch phase (not part of the ADMM state):
    int* br_cost = nullptr;    // [nl] TRON iterations of each branch, last sweep
    int* branch_ws = nullptr;  // [branch_workspace_ints] overflow queues + counters
    // a branch solve handed from the lane phase to the tile phase mid-way
    double* mig_x = nullptr;         // [6][nl] TRON iterate
    double* mig_f = nullptr;         // [nl]
    double* mig_delta = nullptr;     // [nl]
    double* mig_prev_res = nullptr;  // [nl] AL residual of the previous round
    int* mig_iter = nullptr;         // [nl] TRON iteration within the solve
    int* mig_al = nullptr;           // [nl] completed AL rounds
    int* mig_cost = nullptr;         // [nl] TRON iterations so far (stats)
};

struct DevNet;
size_t branch_workspace_ints(const DevNet& n);

// Per-iteration scalars reduced on the device.  Maxima of non-negative
// doubles are kept as their IEEE bit patterns (order-preserving as uint64).
struct DevScalars {
    unsigned long long primal_inf;  // max |x - xbar + z|
    unsigned long long dual_inf;    // max |xbar - xbar_prev| (times rho_max on host)
    unsigned long long z_inf;       // max |z|
    unsigned long long z_drift;     // max |z - z_prev|
    unsigned long long failures;    // branch NumericalError count
    unsigned long long tron_iters4; // TRON iterations, unlimited (4-var) branches
    unsigned long long tron_iters6; // TRON iterations, rate-limited (6-var) branches
    int singular_bus;               // min singular bus index, INT_MAX if none
    int pad;
    unsigned long long exec4;       // trust-region steps actually executed (4-var)
    unsigned long long exec6;       // (6-var); < TRON iterations when fixed points are skipped
};

// Solution extraction + quality metrics of a finished solve (extract.cu).
struct ExtractScalars {
    unsigned long long balance_inf;      // max(|pbal|, |qbal|), bits
    unsigned long long bound_violation;  // max(0, generator / voltage bound excess), bits
    int n_cand;                          // branches on the line-limit candidate list
    int pad;
};
struct DevExtract {
    double* flows = nullptr;  // [4 * nl] AoS pij qij pji qji
    double* vm = nullptr;     // [nb]
    double* va = nullptr;     // [nb]
    int* cand = nullptr;      // [nl] line-limit candidates (unordered)
    double* gen_pq = nullptr; // [2 * ng] dispatch (pg, qg) in generator order
    ExtractScalars* sc = nullptr;
};

// Device-side inner-loop control (solve.cpp's graph path): the stop tests of
// driver.cpp:186-220 evaluated on the device after every iteration, so a
// CUDA graph of several iterations runs without a host round trip; kernels
// of iterations after a stop see `stop` and return at entry.
enum LoopStop : int { kLoopRunning = 0, kLoopInner = 1, kLoopLimit = 2, kLoopDiverged = 3,
                      kLoopSingular = 4 };
struct LoopCtl {
    // inputs, written by the host before each outer iteration
    double inner_tol, eps, diverge, rho_max, beta;
    int outer, max_inner;
    // state
    int inner;      // inner iterations done in this outer iteration
    int stop;       // LoopStop
    int singular;   // internal index of the singular bus (kLoopSingular)
    int pad;
    unsigned long long failures;  // branch failures in this outer iteration
    double last_z;                // ||z||_inf of the last iteration
    unsigned long long t_start, t_mark, t_bus, x_ns, xbar_ns;  // %globaltimer stamps / phase sums
};
struct LoopRec {  // one IterationRecord (driver.cpp:190) with a device timestamp
    int outer, inner;
    double primal, dual, z, drift;
    unsigned long long t_ns;
};

struct BranchCfg {
    double gtol = 1e-6;
    int max_iterations = 200;
    double cg_tol = 0.1;
    int max_cg = 32;
    double delta_floor = 1e-3;
    double limit_tighten = 0.99;
    int lane_budget = 4;  // lane-phase steps of a branch once the active set fits the tiles
    int lane_cap = 16;    // lane-phase steps while the active set exceeds the tile slots (swept)
    int tile_slots = 0;   // set by the launcher: tiles available per queue
    int tail_num = 2;     // whole-warp tiles when a queue <= tail_num/4 of the grid's warps
    int tile_budget = 0;  // steps in the tile phase before the solo phase takes over (0 = off;
                          // 70k solve with 8-lane tiles: 0 / 24 / 48 / 96 -> 6.23 / 6.28 / 6.28 / 6.27 s)
    const LoopCtl* gate = nullptr;  // graph path: skip the launch when gate->stop
};

// ---- launchers (kernels.cu / branch.cu) ----------------------------------
// Solution voltages / flows and the order-free quality maxima (extract.cu).
void launch_extract(const DevNet& n, const DevState& s, const DevExtract& e, cudaStream_t st);
void launch_generators(const DevNet& n, const DevState& s, cudaStream_t st);
// `mid` (optional) is recorded between the lane-phase and tile-phase kernels.
void launch_branches(const DevNet& n, const DevState& s, const BranchCfg& cfg,
                     DevScalars* sc, cudaStream_t st, cudaEvent_t mid = nullptr,
                     const std::function<void()>& after_lane = {});
// Per-bus flags set by the lane kernel for the end buses of every branch it
// hands on to the tile / solo phases (cleared by the caller per iteration).
unsigned char* bus_defer_flags(const DevNet& n, const DevState& s);
// One-time launch setup of the branch kernels (grid sizes, smem attribute);
// called before a stream capture, where such calls are not allowed.
void prepare_branch_launch();
// Overflow queue sizes (6-var, 4-var) of the last branch sweep (device ints).
const int* branch_overflow_counts(const DevNet& n, const DevState& s);
void launch_buses(const DevNet& n, const DevState& s, DevScalars* sc, cudaStream_t st);
// Bus QP fused with the generator projection, z, y and all four residual
// norms (the iteration path).  With a gate (graph path) beta is read from
// gate->beta and the launch is a no-op once gate->stop is set.
// sel: 0 every bus; 1 the buses whose flag in `defer` is clear; 2 the
// flagged ones.  Buses are independent and the norms order-free maxima, so
// 1 then 2 is the same as 0 (the split lets 1 run beside the tile phase).
void launch_bus_zy(const DevNet& n, const DevState& s, double beta, DevScalars* sc,
                   cudaStream_t st, LoopCtl* gate = nullptr,
                   const unsigned char* defer = nullptr, int sel = 0);
// Graph path: stamp the loop start and clear the scalars / the control
// kernel after each iteration (records, stop tests, scalar reset).
void launch_loop_start(LoopCtl* ctl, DevScalars* sc, cudaStream_t st);
void launch_loop_control(LoopCtl* ctl, LoopRec* rec, DevScalars* sc, cudaStream_t st);
// Separate z / y phases (phase-replay API).
void launch_z_only(const DevNet& n, const DevState& s, double beta, cudaStream_t st);
void launch_y_only(const DevNet& n, const DevState& s, cudaStream_t st);
void launch_outer(const DevNet& n, const DevState& s, double beta, double lam_min,
                  double lam_max, cudaStream_t st);
void launch_reset_scalars(DevScalars* sc, cudaStream_t st);
// make_state + cold_start on the device (driver.cpp:26-63, decomp.cpp:37-57).
void launch_cold_start(const DevNet& n, const DevState& s, double rho_pq, double rho_va,
                       double limit_tighten, cudaStream_t st);
// max(0, max_k v[k]) with NaN skipped (driver.cpp:179-183 rho_max), as bits.
void launch_rowmax(const double* v, int n, unsigned long long* dst, cudaStream_t st);
// Boundary exchange of multi-part runs (partition.hpp).
void launch_copy_rows(const int* rows, int count, const double* src, double* dst, cudaStream_t st);
void launch_gather_rows(const int* rows, int count, const double* v, double* buf, cudaStream_t st);
void launch_scatter_rows(const int* rows, int count, const double* buf, double* v, cudaStream_t st);
// Tracking carry-over: clamp x/xbar p-rows into [pmin, pmax] (tracking.cpp:65-70).
void launch_clamp_gen_p(const DevNet& n, const DevState& s, cudaStream_t st);
// Batched TRON on dense box QPs (parity test of the TRON core).
// tile = 1 (one thread per QP, serial search) or 8 (tile search).
void launch_tron_qp(int count, int n, const double* h, const double* g,
                    const double* l, const double* u, double* x, int* status,
                    int* iterations, cudaStream_t st, int tile);
// TRON path statistics (all zero unless built with -DGA_TRON_STATS).
void tron_stats(unsigned long long out[8], bool reset);
// FP64 pipe peak (TFLOP/s) for DMUL+DADD (no FMA) and DFMA issue.
void measure_fp64_peak(double* tflops_mul_add, double* tflops_fma);
// Pinned sincos on the device (parity probe).
void launch_sincos_probe(const double* x, double* s, double* c, int n, cudaStream_t st);

}  // namespace ga

#endif
