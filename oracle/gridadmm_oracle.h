/* gridadmm_oracle.h — TEST INFRASTRUCTURE: plain-C restatement of the
 * reference's ADMM hot path (parity checker and CPU-baseline "port"; never
 * linked into the product).  Pinned bit-for-bit to the compiled reference
 * (oracle/_ref) by tests/test_oracle.py and to tests/golden fixtures.
 *
 * The network is passed in the flat export layout of
 * gridadmm_network_export (include/gridadmm/gridadmm_ext.h); the state in
 * gridadmm_state_view. */
#ifndef GRIDADMM_ORACLE_H
#define GRIDADMM_ORACLE_H

#include "../include/gridadmm/gridadmm_ext.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct oracle_net {
    int nb, ng, nl, ref_bus;
    const double* bus;     /* 6 per bus: pd qd gs bs vmin vmax */
    const double* gen;     /* 8 per gen: bus pmin pmax qmin qmax c2 c1 c0 */
    const int* ends;       /* 2 per branch: from to */
    const double* branch;  /* 14 per branch: r x b tap shift rate gii bii gij bij gji bji gjj bjj */
} oracle_net;

/* cfg: rho_pq rho_va beta0 eps inner_tol max_outer max_inner workers
 * lambda_bound beta_max (the harness order of oracle/ref_harness.cpp). */
void oracle_cold_start(const oracle_net* net, const double* cfg, gridadmm_state_view* out);
long oracle_phase(const oracle_net* net, int phase, const double* cfg, gridadmm_state_view* io,
                  double z_inf, double prev_z_inf);
int oracle_solve(const oracle_net* net, const double* cfg, const gridadmm_state_view* init,
                 gridadmm_state_view* fin, double* series, int cap, int* nseries, double* info);

/* Lean FP64 op census of the branch phase (ops whose results are consumed):
 * counters since the last reset: [0] flops, [1] TRON iterations (4-var),
 * [2] TRON iterations (6-var), [3] flops in 4-var solves, [4] flops in
 * 6-var solves, [5] sincos calls. */
void oracle_census(unsigned long long* out, int reset);

#ifdef __cplusplus
}
#endif

#endif
