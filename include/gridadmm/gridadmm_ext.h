/* gridadmm_ext.h — B200 extensions to the gridadmm C ABI.
 *
 * The 23 functions of gridadmm.h are the drop-in boundary.  This header adds
 * what the reference exposes only as C++ (proj/src/kernels.hpp:70-101,
 * proj/src/driver.hpp:83-90): a device-resident solver session whose ADMM
 * state can be read/written in the reference's flat layout
 * (proj/src/decomp.hpp:64-78) and whose phases can be launched one at a
 * time.  Parity tests replay a reference state through one phase and compare
 * bit-for-bit; bench.py times inner iterations with the state resident in
 * HBM.  All functions are synchronous with respect to the host unless noted;
 * errors map to gridadmm_status exactly like gridadmm.h.
 */
#ifndef GRIDADMM_EXT_H
#define GRIDADMM_EXT_H

#include "gridadmm.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Host view of one AdmmState (proj/src/decomp.hpp:64-78).  Row vectors have
 * m = 2G + 8L entries in CouplingLayout order (proj/src/decomp.hpp:32-36);
 * branch_point is 6 doubles per branch (vi, vj, thi, thj, sij, sji).  Any
 * pointer may be NULL to skip that array on get/set. */
typedef struct gridadmm_state_view {
    double* x;
    double* xbar;
    double* z;
    double* y;
    double* lambda;
    double* rho;
    double* bus_w;        /* num_buses */
    double* bus_theta;    /* num_buses */
    double* branch_point; /* 6 * num_branches */
    double* lt_ij;        /* num_branches */
    double* lt_ji;        /* num_branches */
    double* rho_tilde;    /* num_branches */
    double* beta;         /* scalar */
} gridadmm_state_view;

typedef struct gridadmm_session gridadmm_session;

/* Phases of one inner iteration, proj/src/driver.cpp:155-176. */
typedef enum gridadmm_phase {
    GRIDADMM_PHASE_GENERATORS = 0, /* kernels.cpp:194-209 */
    GRIDADMM_PHASE_BRANCHES = 1,   /* kernels.cpp:211-292 */
    GRIDADMM_PHASE_BUSES = 2,      /* kernels.cpp:294-413 */
    GRIDADMM_PHASE_Z = 3,          /* kernels.cpp:415-422 */
    GRIDADMM_PHASE_Y = 4,          /* kernels.cpp:424-428 */
    GRIDADMM_PHASE_OUTER = 5       /* kernels.cpp:430-437 (uses z_inf args) */
} gridadmm_phase;

/* Number of m rows of the coupling layout (2G + 8L). */
int gridadmm_network_num_rows(const gridadmm_network* net);

/* Parsed network in flat arrays (host only, no device needed), for checking
 * the parser against the reference's (proj/src/netdata.cpp:124-237):
 * bus 6 per bus (pd, qd, gs, bs, vmin, vmax) + external ids; gen 8 per gen
 * (bus, pmin, pmax, qmin, qmax, c2, c1, c0); branch ends 2 per branch and 14
 * doubles (r, x, b, tap, shift, rate, gii, bii, gij, bij, gji, bji, gjj, bjj).
 * Any pointer may be NULL. */
gridadmm_status gridadmm_network_export(const gridadmm_network* net, double* bus,
                                        int* bus_id, double* gen, int* ends,
                                        double* branch, int* ref_bus);

/* Deterministic k-way bus-graph partition used when the config key
 * `partitions` is k > 1 (host only): part_of_bus[i] in [0, k).  Branch b is
 * solved by the part of its from-bus; per iteration a cut branch's four
 * to-side rows (pji, qji, wj, thj) are exchanged (x forward, xbar/z/y back). */
gridadmm_status gridadmm_network_partition(const gridadmm_network* net, int k,
                                           int* part_of_bus);

/* Per-branch work weights for the partition above (e.g. the TRON steps of
 * a previous sweep from gridadmm_session_branch_costs, so the heavy-tailed
 * branches spread over the parts): weights[b] >= 0 for every branch, or NULL
 * to restore the class weights.  Every rank of a multi-process run must set
 * the same weights before creating its session.  Results never depend on
 * the partition. */
gridadmm_status gridadmm_network_set_branch_weights(gridadmm_network* net, const int* weights);

/* Exchange plan of part p of the k-way partition (host only): the rows
 * whose x part p sends to peer q after the branch phase (and whose xbar, z,
 * y it gets back after the bus phase), and the rows whose x it receives from
 * q (and returns).  Branch-major, k = pji, qji, wj, thj per cut branch.  With
 * NULL row buffers only the counts are written. */
gridadmm_status gridadmm_network_exchange_rows(const gridadmm_network* net, int k, int p, int q,
                                               int* send_rows, int* n_send, int* recv_rows,
                                               int* n_recv);

/* Bus-owned row lists of the coupling layout (proj/src/decomp.cpp:7-31):
 * counts[6*i + k] = sizes of (gen_p, gen_q, flow_p, flow_q, w, theta) of bus
 * i, rows = the lists concatenated per bus in that group order (length m). */
gridadmm_status gridadmm_network_layout(const gridadmm_network* net, int* counts,
                                        int* rows);

/* Creates a device-resident session for (net, cfg) on the configured device
 * and loads the cold-start state (proj/src/driver.cpp:26-63). */
gridadmm_status gridadmm_session_new(const gridadmm_network* net,
                                     const gridadmm_config* cfg,
                                     gridadmm_session** out);
void gridadmm_session_free(gridadmm_session* s);

/* Multi-process bus-graph partition (one process per GPU, e.g. torchrun):
 * rank 0 creates a 128-byte NCCL unique id, shares it out of band, and every
 * rank opens its part on its configured `device`.  Rank r owns part r of
 * gridadmm_network_partition(net, world); per inner iteration boundary rows
 * and residual maxima go over NCCL (grouped send/recv, all-reduce), so every
 * rank sees the same residual series as a 1-GPU solve.  Supported on such
 * sessions: gridadmm_session_iterate (and _free); state getters return only
 * the entries this rank owns as current.  NCCL (libnccl.so.2) is loaded at
 * run time. */
gridadmm_status gridadmm_nccl_unique_id(unsigned char* out);
gridadmm_status gridadmm_session_new_dist(const gridadmm_network* net,
                                          const gridadmm_config* cfg, int rank,
                                          int world, const unsigned char* nccl_id,
                                          gridadmm_session** out);

/* Copies the device state to/from host arrays (synchronous). */
gridadmm_status gridadmm_session_get_state(const gridadmm_session* s,
                                           const gridadmm_state_view* v);
gridadmm_status gridadmm_session_set_state(gridadmm_session* s,
                                           const gridadmm_state_view* v);

/* The reference's solve(net, cfg, initial, final) (proj/src/driver.cpp:140-246)
 * on the session's device state: Algorithm 1 with cfg's stop rules, starting
 * from the current state (warm != 0, the `initial` argument) or from a fresh
 * cold start (warm == 0).  The state after the solve stays on the device
 * (the `final_state` argument: read it with gridadmm_session_get_state).
 * Status and report semantics are those of gridadmm_solve. */
gridadmm_status gridadmm_session_solve(gridadmm_session* s, const gridadmm_config* cfg,
                                       int warm, gridadmm_report** out);

/* Runs one phase on the device state.  For GRIDADMM_PHASE_BRANCHES,
 * *aux receives the number of branch solve failures; for BUSES, *aux is -1
 * or the internal index of the first singular bus; for OUTER, aux[0] is
 * z_inf and aux[1] prev_z_inf (inputs).  aux may be NULL otherwise. */
gridadmm_status gridadmm_session_phase(gridadmm_session* s, int phase,
                                       double* aux);

/* Runs up to n inner ADMM iterations of the current outer iteration with the
 * reference's inner-loop tests (proj/src/driver.cpp:155-220), appending one
 * record per iteration to records (5 doubles each: primal_res, dual_res,
 * z_norm, z_drift, branch_failures) when non-NULL.  *done receives the number
 * of iterations executed; *stop is 0 (ran n), 1 (inner converged / early
 * exit) or 2 (diverged). */
gridadmm_status gridadmm_session_iterate(gridadmm_session* s, int n,
                                         double* records, int* done,
                                         int* stop);

/* Benchmark form of iterate: runs exactly n inner iterations (no early
 * stop), each bracketed by CUDA events on the session stream from the first
 * launch through the D2H of that iteration's norms; when flush_bytes > 0 a
 * device buffer of that size is rewritten between iterations, outside the
 * brackets (L2 flush).  step_ms receives n device times, records 5 doubles
 * per iteration as in gridadmm_session_iterate. */
gridadmm_status gridadmm_session_timed_steps(gridadmm_session* s, int n,
                                             size_t flush_bytes,
                                             double* step_ms, double* records);

/* Total device time (ms) of the named kernel class since the session began,
 * measured with CUDA events on the session stream, and its launch count.
 * Classes: 0 gen, 1 branch (lane + tile phases), 2 bus (fused with z, y and
 * the residual norms), 3 zy (0 since the fusion), 4 branch lane phase,
 * 5 branch tile phase. */
gridadmm_status gridadmm_session_kernel_time(const gridadmm_session* s,
                                             int kernel_class, double* ms,
                                             long long* launches);

/* Cumulative TRON iterations of all branch solves since the session began
 * (the reference's count, tron.hpp:34-39) and the part of them spent on the
 * rate-limited (6-variable) branches. */
gridadmm_status gridadmm_session_counters(const gridadmm_session* s,
                                          long long* tron_iterations,
                                          long long* limited_iterations);

/* Cumulative counters: out[0], out[1] = TRON iterations with the reference's
 * accounting (TronResult::iterations; 4-var, 6-var branches), out[2],
 * out[3] = trust-region steps the device actually executed (fewer when a
 * solve reaches an exact fixed point and its remaining identical iterations
 * are skipped, see tron.cuh). */
gridadmm_status gridadmm_session_step_counters(const gridadmm_session* s, long long* out);

/* TRON iterations each branch took in the last branch sweep (num_branches
 * ints) — the LPT scheduling key, exposed for profiling. */
gridadmm_status gridadmm_session_branch_costs(const gridadmm_session* s, int* costs);

/* TRON path counters since the last reset (8 values: steps, Cauchy
 * extrapolations, Cauchy halvings, CG iterations, line-search steps, failed
 * preconditioners, -, -); all zero unless the library was built with
 * -DGA_TRON_STATS (`make stats`). */
gridadmm_status gridadmm_debug_tron_stats(unsigned long long* out, int reset);

/* Number of CUDA devices visible to the library. */
int gridadmm_device_count(void);

/* Parity probes (test entry points).  Batched TRON (the branch kernel's
 * trust-region core, proj/src/tron.cpp:228-332) on `count` dense box QPs
 * f = g'x + x'Hx/2 of dimension n <= 6 (H row-major n*n per problem); x is
 * the start point in, solution out; status uses TronStatus numbering
 * (0 converged, 1 iteration limit, 2 numerical error).  tile = 1 runs one
 * solve per thread (lane phase), tile = 4, 8 or 32 one solve per tile with the
 * speculative Cauchy/line search (tile phase).  And the pinned device sincos
 * (ga_sincos.h) on n arguments. */
gridadmm_status gridadmm_probe_tron_qp(int count, int n, const double* h,
                                       const double* g, const double* l,
                                       const double* u, double* x, int* status,
                                       int* iterations, int tile);
gridadmm_status gridadmm_probe_sincos(int n, const double* x, double* s,
                                      double* c);

/* FP64 pipe microbenchmark on `device` (the branch kernel's roofline
 * denominator): TFLOP/s issuing DMUL+DADD pairs (what -fmad=false code runs)
 * and issuing DFMA. */
gridadmm_status gridadmm_probe_fp64_peak(int device, double* tflops_mul_add,
                                         double* tflops_fma);

#ifdef __cplusplus
}
#endif

#endif /* GRIDADMM_EXT_H */
