// branch.cu — the branch-NLP phase (north-star (b)): per branch, an
// augmented-Lagrangian loop on the line limits around a TRON solve of the 4-
// or 6-variable branch subproblem (branch_problem.cuh).
//
// Reference semantics: proj/src/kernels.cpp:211-292 (solve_branch_batch);
// the reference schedules it as a static block partition over std::threads
// (proj/src/parallel.hpp:13-33).
//
// B200 schedule.  TRON cost per branch is heavy-tailed and changes over a
// solve: early, ~255k trust-region steps per sweep with ~5k branches past 4
// steps (the longest ~20); late, the same bulk plus a handful of rate-limited
// branches whose AL loop runs all 10 rounds (~1,000 steps in one chain).  So
// the phase runs in three kernels:
//
//  A. lane phase — a persistent grid where each lane owns one branch and
//     advances it one trust-region iteration per loop trip, refilling from the
//     work queue (warp-aggregated atomic) the moment its branch finishes.  A
//     branch stays up to `lane_cap` steps while more branches are active than
//     twice the tile slots (throughput mode), up to `lane_budget` after; then
//     its resumable state (TRON iterate, radius, iteration, AL round) is
//     saved and it is pushed to an overflow queue.
//  B. tile phase — the overflow branches are resumed by tiles of kTile lanes (or
//     whole warps when a queue is short).  All lanes of a tile hold the
//     replicated iterate; the Cauchy search and the projected line search
//     (the loops with many trials) are evaluated 8 (32) trials at a time
//     (TileSearch in tron.cuh).  After `tile_budget` steps a branch is handed
//     on again.
//  C. solo phase — one warp per branch, one block per SM, for the few very
//     long solves (their sequential chain bounds the late iterations).
//
// Results do not depend on the schedule: every branch executes the identical
// sequence of floating-point operations wherever and in whichever phase it
// runs (the migration saves/restores exact state), so parity is bit-exact.
#include <climits>
#include <cstdlib>

#include "branch_problem.cuh"
#include "device.hpp"
#include "ga_math.h"
#include "tron.cuh"

namespace ga {

void tron_stats(unsigned long long out[8], bool reset) {
#ifdef GA_STEP_CLOCKS
    cudaMemcpyFromSymbol(out, g_step_clocks, 8 * sizeof(unsigned long long));
    if (reset) {
        const unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        cudaMemcpyToSymbol(g_step_clocks, z, sizeof z);
    }
#elif defined(GA_TRON_STATS)
    cudaMemcpyFromSymbol(out, g_tron_stats, 8 * sizeof(unsigned long long));
    if (reset) {
        const unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        cudaMemcpyToSymbol(g_tron_stats, z, sizeof z);
    }
#else
    (void)reset;
    for (int k = 0; k < 8; ++k) out[k] = 0;
#endif
}

namespace {

using namespace bp;

constexpr double kLtBound = 1e8;  // kernels.cpp:16
constexpr int kMaxAl = 10;        // kernels.cpp:219
constexpr double kAlTol = 1e-8;
constexpr double kAlShrink = 0.25;
constexpr double kRhoTildeMax = 1e7;

#ifndef GA_LANE_BLOCK
#define GA_LANE_BLOCK 256
#endif
constexpr int kLaneBlock = GA_LANE_BLOCK;  // lane phase: one slot per thread (64 / 128 / 256 per block:
                                 // 7.05 / 7.05 / 6.99 s on the full 70k solve)
constexpr int kTileBlock = 128;  // tile phase: one slot per tile
#ifndef GA_TILE
#define GA_TILE 8
#endif
constexpr int kTile = GA_TILE;  // lanes per branch in the tile phase (full 70k solve, final
                                // build: 2 / 4 / 8 / 16 lanes -> 6.60 / 6.35 / 6.27 / 6.36 s)
constexpr int kCounters = 12;
constexpr int kSoloBlock = 32;  // solo phase: one warp per block, one branch per warp

// Workspace: [overflow6 n_lim | overflow4 n_unl | solo6 n_lim | solo4 n_unl | counters]
// counters: 0/1 lane-queue cursors (6/4), 2/3 overflow sizes, 4/5 tile cursors,
//           6/7 solo sizes, 8/9 solo cursors, 10/11 lane-phase branches done or handed on
struct Work {
    int* ovf6;
    int* ovf4;
    int* solo6;
    int* solo4;
    int* ctr;
    unsigned char* defer;  // [nb] bus adjacent to a branch handed on by the lane phase
};

Work work_of(const DevNet& n, const DevState& s) {
    Work w;
    w.ovf6 = s.branch_ws;
    w.ovf4 = w.ovf6 + n.n_lim;
    w.solo6 = w.ovf4 + n.n_unl;
    w.solo4 = w.solo6 + n.n_lim;
    w.ctr = w.solo4 + n.n_unl;
    w.defer = reinterpret_cast<unsigned char*>(w.ctr + kCounters);
    return w;
}

__device__ __forceinline__ unsigned sm_id() {
    unsigned id;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(id));
    return id;
}

__device__ __forceinline__ TronParams tron_params(const BranchCfg& cfg) {
    TronParams tp;
    tp.gtol = cfg.gtol;
    tp.max_iterations = cfg.max_iterations;
    tp.cg_tol = cfg.cg_tol;
    tp.max_cg = cfg.max_cg;
    tp.delta_floor = cfg.delta_floor;
    return tp;
}

enum AlAction : int { kAlContinue = 0, kAlDone = 1, kAlFailed = 2 };

// A TRON solve ended with `status`: AL bookkeeping of kernels.cpp:246-271.
// Either restarts TRON for the next AL round (kAlContinue) or ends the branch.
// `share` is the mask of the lanes that share `slot` (a tile) or 0 when the
// slot is the lane's own: every sharer reads the multipliers before any of
// them writes, so no lane can see an already-updated value.
template <int N, int S, class BP>
__device__ __forceinline__ int al_after_solve(int status, Slot<S> slot, const BP& p,
                                              TronState<N>& ts, int& al_it, double& prev_res,
                                              unsigned share) {
    for (;;) {
        if (status == kTronNumericalError) return kAlFailed;
        if constexpr (N == 4) {
            return kAlDone;
        } else {
            double fl[4];
            branch_flows(YcView<S>{slot}, ts.x[0], ts.x[1], ts.x[2], ts.x[3], fl);
            const double rij = fl[0] * fl[0] + fl[1] * fl[1] + ts.x[4];
            const double rji = fl[2] * fl[2] + fl[3] * fl[3] + ts.x[5];
            const double res = smax(fabs(rij), fabs(rji));
            if (res <= kAlTol) return kAlDone;
            const double rho_t = slot(F_RHOT);
            const double lt_ij = slot(F_LTIJ);
            const double lt_ji = slot(F_LTJI);
            if (share) __syncwarp(share);
            const double lij = sclamp(lt_ij + rho_t * rij, -kLtBound, kLtBound);
            const double lji = sclamp(lt_ji + rho_t * rji, -kLtBound, kLtBound);
            slot.set(F_LTIJ, lij);
            slot.set(F_LTJI, lji);
            if (res > kAlShrink * prev_res) slot.set(F_RHOT, smin(10.0 * rho_t, kRhoTildeMax));
            if (share) __syncwarp(share);
            prev_res = res;
            if (++al_it >= kMaxAl) return kAlDone;
            if (tron_begin<N>(p, ts)) return kAlContinue;
            status = kTronNumericalError;
        }
    }
}

// Branch finished: restore the previous point on failure, write back
// multipliers, point and the eight consensus rows (kernels.cpp:273-281).
template <int N, int S>
__device__ __forceinline__ void finalize_branch(const DevNet& net, const DevState& st, Slot<S> slot,
                                                const TronState<N>& ts, int b, bool failed,
                                                int iters) {
    double pt[N];
#pragma unroll
    for (int k = 0; k < N; ++k) pt[k] = failed ? st.bp[k * net.nl + b] : ts.x[k];
    st.lt_ij[b] = slot(F_LTIJ);
    st.lt_ji[b] = slot(F_LTJI);
    st.rho_t[b] = slot(F_RHOT);
    if (!failed) {
#pragma unroll
        for (int k = 0; k < N; ++k) st.bp[k * net.nl + b] = pt[k];
    }
    double fl[4];
    branch_flows(YcView<S>{slot}, pt[0], pt[1], pt[2], pt[3], fl);
    // the from-quad (pij, qij, wi, thi) and the to-quad (pji, qji, wj, thj)
    GA_CHECK(net.qpos[2 * b] >= 0 && net.qpos[2 * b] + 4 <= net.mpad);
    GA_CHECK(net.qpos[2 * b + 1] >= 0 && net.qpos[2 * b + 1] + 4 <= net.mpad);
    double2* xf = reinterpret_cast<double2*>(st.x + net.qpos[2 * b]);
    double2* xt = reinterpret_cast<double2*>(st.x + net.qpos[2 * b + 1]);
    xf[0] = make_double2(fl[0], fl[1]);
    xt[0] = make_double2(fl[2], fl[3]);
    xf[1] = make_double2(pt[0] * pt[0], pt[2]);
    xt[1] = make_double2(pt[1] * pt[1], pt[3]);
#if defined(GA_TRON_STATS) || defined(GA_BRANCH_STEPS)
    (void)iters;  // stats builds: br_cost = executed steps (+2^20 if the tile phase ran it)
#else
    st.br_cost[b] = iters;
#endif
}

// Solve-level status of a TRON step that did not continue; updates iters.
template <int N, int S, class Search, class BP>
__device__ __forceinline__ int solve_status(int r, int iter_before, const BP& p,
                                            const TronState<N>& ts, const TronParams& tp,
                                            int& iters) {
    if (r == kStepConverged) { iters += iter_before; return kTronConverged; }
    if (r == kStepError) { iters += iter_before; return kTronNumericalError; }
    iters += tp.max_iterations;
    return tron_finish<N>(p, ts, tp);
}

// ---- phase A: one lane per branch, bounded iterations ----------------------
template <int N>
__device__ __noinline__ void lane_phase(const DevNet& net, const DevState& st,
                                        const BranchCfg& cfg, const int* list, int count,
                                        int* cursor, int* ovf, int* ovf_count, double* smem,
                                        unsigned long long* iters_out, int* fail_out,
                                        unsigned long long* exec_dst, int* done_ctr,
                                        unsigned char* defer) {
    constexpr unsigned kFull = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    unsigned my_exec = 0;  // trust-region steps executed by this lane
    const Slot<kLaneBlock> slot{smem + threadIdx.x};
    BranchProb<N, kLaneBlock> p{slot};
    const TronParams tp = tron_params(cfg);
    const double kInf = __longlong_as_double(0x7ff0000000000000LL);

    TronState<N> ts;
    int b = -1;
    bool exhausted = false;
    int al_it = 0, iters = 0, steps = 0;
    double prev_res = kInf;
    unsigned long long my_iters = 0;
    int my_fail = 0;

    auto end_branch = [&](int act) {
        const bool failed = act == kAlFailed;
        finalize_branch<N>(net, st, slot, ts, b, failed, iters);
        my_iters += iters;
        my_fail += failed ? 1 : 0;
        atomicAdd(done_ctr, 1);
        b = -1;
    };
    for (;;) {
        const unsigned need = __ballot_sync(kFull, b < 0 && !exhausted);
        if (need) {
            const int leader = __ffs(need) - 1;
            int base = 0;
            if (lane == leader) base = atomicAdd(cursor, __popc(need));
            base = __shfl_sync(kFull, base, leader);
            if (need >> lane & 1u) {
                const int idx = base + __popc(need & ((1u << lane) - 1u));
                if (idx < count) {
                    b = list[idx];
                    GA_CHECK(b >= 0 && b < net.nl);
                    load_slot<kLaneBlock>(net, st, cfg, b, slot);
#pragma unroll
                    for (int k = 0; k < N; ++k) ts.x[k] = st.bp[k * net.nl + b];
                    al_it = 0;
                    iters = 0;
                    steps = 0;
                    prev_res = kInf;
                    if (!tron_begin<N>(p, ts)) {
                        const int act = al_after_solve<N>(kTronNumericalError, slot, p, ts, al_it,
                                                          prev_res, 0u);
                        end_branch(act);
                    }
                } else {
                    exhausted = true;
                }
            }
        }
        if (__all_sync(kFull, b < 0 && exhausted)) break;
        // Throughput mode while more branches are still active than the tile
        // phase has tiles for: a branch may take up to lane_cap steps here
        // (32 branches per warp beat 4 per warp when there is enough work).
        // Once the active set fits the tiles, branches past lane_budget move
        // to the tile phase, whose parallel searches have the shorter
        // per-step latency.
        int active = 0;
        if (lane == 0) active = count - *reinterpret_cast<volatile int*>(done_ctr);
        active = __shfl_sync(kFull, active, 0);
        const int budget = active <= cfg.tile_slots ? cfg.lane_budget : cfg.lane_cap;
        if (b >= 0) {
            const int iter_before = ts.iter;
            const int r = tron_step<N>(p, ts, tp);
            ++my_exec;
            if (r != kStepContinue) {
                const int status = solve_status<N, kLaneBlock, SerialSearch>(r, iter_before, p, ts,
                                                                            tp, iters);
                const int act = al_after_solve<N>(status, slot, p, ts, al_it, prev_res, 0u);
#if defined(GA_TRON_STATS) || defined(GA_BRANCH_STEPS)
                if (act != kAlContinue) st.br_cost[b] = steps + 1;
#endif
                if (act != kAlContinue) end_branch(act);
            }
            if (b >= 0 && ++steps >= budget) {
                // hand the solve to the tile phase with its exact state
#pragma unroll
                for (int k = 0; k < N; ++k) st.mig_x[k * net.nl + b] = ts.x[k];
                st.mig_f[b] = ts.f;
                st.mig_delta[b] = ts.delta;
                st.mig_iter[b] = ts.iter;
                st.mig_al[b] = al_it;
                st.mig_prev_res[b] = prev_res;
                st.mig_cost[b] = iters;
                st.lt_ij[b] = slot(F_LTIJ);
                st.lt_ji[b] = slot(F_LTJI);
                st.rho_t[b] = slot(F_RHOT);
#if defined(GA_TRON_STATS) || defined(GA_BRANCH_STEPS)
                st.br_cost[b] = steps;
#endif
                const int slot_o = atomicAdd(ovf_count, 1);
                GA_CHECK(slot_o >= 0 && slot_o < count);
                ovf[slot_o] = b;
                // its end buses wait for the tile / solo phases (bus kernel split)
                GA_CHECK(net.br_from[b] >= 0 && net.br_from[b] < net.nb);
                GA_CHECK(net.br_to[b] >= 0 && net.br_to[b] < net.nb);
                defer[net.br_from[b]] = 1;
                defer[net.br_to[b]] = 1;
                atomicAdd(done_ctr, 1);
                b = -1;
            }
        }
    }
    *iters_out += my_iters;
    *fail_out += my_fail;
    const unsigned warp_exec = __reduce_add_sync(kFull, my_exec);
    if (lane == 0 && warp_exec) atomicAdd(exec_dst, (unsigned long long)warp_exec);
}

#ifndef GA_LANE_MINB
#define GA_LANE_MINB 1
#endif
#ifndef GA_TILE_MINB
#define GA_TILE_MINB 1
#endif
__device__ __forceinline__ bool gate_closed(const BranchCfg& cfg) {
    return cfg.gate && *reinterpret_cast<const volatile int*>(&cfg.gate->stop);
}

__global__ void __launch_bounds__(kLaneBlock, GA_LANE_MINB) lane_kernel(DevNet net, DevState st, BranchCfg cfg,
                                                          Work w, DevScalars* sc) {
    if (gate_closed(cfg)) return;
    extern __shared__ double smem[];
    unsigned long long it6 = 0, it4 = 0;
    int fails = 0;
    // Even SMs start on the 6-variable queue, odd SMs on the 4-variable one,
    // so each SM's warps share one code path (instruction-cache locality).
    if ((sm_id() & 1u) == 0) {
        lane_phase<6>(net, st, cfg, net.lim_list, net.n_lim, &w.ctr[0], w.ovf6, &w.ctr[2], smem,
                      &it6, &fails, &sc->exec6, &w.ctr[10], w.defer);
        lane_phase<4>(net, st, cfg, net.unl_list, net.n_unl, &w.ctr[1], w.ovf4, &w.ctr[3], smem,
                      &it4, &fails, &sc->exec4, &w.ctr[11], w.defer);
    } else {
        lane_phase<4>(net, st, cfg, net.unl_list, net.n_unl, &w.ctr[1], w.ovf4, &w.ctr[3], smem,
                      &it4, &fails, &sc->exec4, &w.ctr[11], w.defer);
        lane_phase<6>(net, st, cfg, net.lim_list, net.n_lim, &w.ctr[0], w.ovf6, &w.ctr[2], smem,
                      &it6, &fails, &sc->exec6, &w.ctr[10], w.defer);
    }
    const unsigned full = 0xffffffffu;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        it6 += __shfl_down_sync(full, it6, o);
        it4 += __shfl_down_sync(full, it4, o);
        fails += __shfl_down_sync(full, fails, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (it6) atomicAdd(&sc->tron_iters6, it6);
        if (it4) atomicAdd(&sc->tron_iters4, it4);
        if (fails) atomicAdd(&sc->failures, (unsigned long long)fails);
    }
}

// ---- phase B: tiles of kTile lanes per overflow branch ---------------------
// Budget > 0: a branch still running after `budget` steps here is saved and
// pushed to the solo queue (solo / solo_count), resumed by the solo phase.
template <int N, int T>
__device__ __noinline__ void tile_phase(const DevNet& net, const DevState& st,
                                        const BranchCfg& cfg, const int* ovf, const int* ovf_count,
                                        int* cursor, double* smem, unsigned long long* iters_out,
                                        int* fail_out, unsigned long long* exec_dst, int budget,
                                        int* solo, int* solo_count) {
    constexpr int S = kTileBlock / kTile;  // slots allocated (one per kTile lanes)
    unsigned long long my_exec = 0;
    const int lane = threadIdx.x & 31;
    const int rank = lane & (T - 1);
    const int tbase = lane & ~(T - 1);
    const unsigned mask = (T == 32 ? 0xffffffffu : ((1u << T) - 1u)) << tbase;
    const TileSearch<T> search{mask, tbase, rank};
    // A warp only ever uses the slots of its own 32 / kTile tiles, whatever T:
    // warps of one block may run different T (tail mode is decided per
    // queue), and must not share a slot.
    const Slot<S> slot{smem + (threadIdx.x / T) * (T / kTile)};
    BranchProb<N, S> p{slot};
    const TronParams tp = tron_params(cfg);
    const int count = *ovf_count;
    unsigned long long my_iters = 0;
    int my_fail = 0;
    for (;;) {
        int idx = 0;
        if (rank == 0) idx = atomicAdd(cursor, 1);
        idx = __shfl_sync(mask, idx, 0, T);
        if (idx >= count) break;
        const int b = ovf[idx];
        GA_CHECK(b >= 0 && b < net.nl);
        load_slot<S>(net, st, cfg, b, slot);
        TronState<N> ts;
#pragma unroll
        for (int k = 0; k < N; ++k) ts.x[k] = st.mig_x[k * net.nl + b];
        ts.f = st.mig_f[b];
        ts.delta = st.mig_delta[b];
        ts.iter = st.mig_iter[b];
        int al_it = st.mig_al[b];
        double prev_res = st.mig_prev_res[b];
        int iters = st.mig_cost[b];
        __syncwarp(mask);
        int act = kAlContinue;
        unsigned branch_exec = 0;
        bool handed_off = false;
        while (act == kAlContinue) {
            if (budget > 0 && branch_exec >= (unsigned)budget) {
                // hand the solve to the solo phase with its exact state
                __syncwarp(mask);
                if (rank == 0) {
#pragma unroll
                    for (int k = 0; k < N; ++k) st.mig_x[k * net.nl + b] = ts.x[k];
                    st.mig_f[b] = ts.f;
                    st.mig_delta[b] = ts.delta;
                    st.mig_iter[b] = ts.iter;
                    st.mig_al[b] = al_it;
                    st.mig_prev_res[b] = prev_res;
                    st.mig_cost[b] = iters;
                    st.lt_ij[b] = slot(F_LTIJ);
                    st.lt_ji[b] = slot(F_LTJI);
                    st.rho_t[b] = slot(F_RHOT);
#if defined(GA_TRON_STATS) || defined(GA_BRANCH_STEPS)
                    st.br_cost[b] += (int)branch_exec;
#endif
                    const int slot_s = atomicAdd(solo_count, 1);
                    GA_CHECK(slot_s >= 0 && slot_s < count);
                    solo[slot_s] = b;
                }
                handed_off = true;
                break;
            }
            const int iter_before = ts.iter;
            const int r = tron_step<N>(p, ts, tp, search);
            ++my_exec;
            ++branch_exec;
            if (r == kStepContinue) continue;
            const int status = solve_status<N, S, TileSearch<T>>(r, iter_before, p, ts, tp, iters);
            act = al_after_solve<N>(status, slot, p, ts, al_it, prev_res, mask);
        }
        __syncwarp(mask);
        if (handed_off) continue;
        if (rank == 0) {
            finalize_branch<N>(net, st, slot, ts, b, act == kAlFailed, iters);
#if defined(GA_TRON_STATS) || defined(GA_BRANCH_STEPS)
            st.br_cost[b] += (int)branch_exec + (1 << 20);
#endif
            my_iters += iters;
            my_fail += act == kAlFailed ? 1 : 0;
        }
        __syncwarp(mask);
    }
    *iters_out += my_iters;
    *fail_out += my_fail;
    if (rank == 0 && my_exec) atomicAdd(exec_dst, my_exec);
}

__global__ void __launch_bounds__(kTileBlock, GA_TILE_MINB) tile_kernel(DevNet net, DevState st, BranchCfg cfg,
                                                          Work w, DevScalars* sc) {
    if (gate_closed(cfg)) return;
    __shared__ double smem[kFields * (kTileBlock / kTile)];
    unsigned long long it6 = 0, it4 = 0;
    int fails = 0;
    // Tail mode: when a queue holds no more branches than half the grid's
    // warps, each branch gets a whole warp (T = 32: no other tile diverging in
    // its warp, 32 search trials per round); otherwise kTile-lane tiles.
#ifndef GA_TILE_TAIL
#define GA_TILE_TAIL 1
#endif
    const int half_warps =
        GA_TILE_TAIL ? (int)(gridDim.x * (kTileBlock / 32) * cfg.tail_num / 4) : -1;
    // kTile-lane tiles hand branches that exceed cfg.tile_budget steps to the
    // solo phase (one warp per branch, one block per SM).
    auto run6 = [&] {
        if (w.ctr[2] <= half_warps)
            tile_phase<6, 32>(net, st, cfg, w.ovf6, &w.ctr[2], &w.ctr[4], smem, &it6, &fails, &sc->exec6,
                              0, nullptr, nullptr);
        else
            tile_phase<6, kTile>(net, st, cfg, w.ovf6, &w.ctr[2], &w.ctr[4], smem, &it6, &fails,
                                 &sc->exec6, cfg.tile_budget, w.solo6, &w.ctr[6]);
    };
    auto run4 = [&] {
        if (w.ctr[3] <= half_warps)
            tile_phase<4, 32>(net, st, cfg, w.ovf4, &w.ctr[3], &w.ctr[5], smem, &it4, &fails, &sc->exec4,
                              0, nullptr, nullptr);
        else
            tile_phase<4, kTile>(net, st, cfg, w.ovf4, &w.ctr[3], &w.ctr[5], smem, &it4, &fails,
                                 &sc->exec4, cfg.tile_budget, w.solo4, &w.ctr[7]);
    };
    if ((sm_id() & 1u) == 0) {
        run6();
        run4();
    } else {
        run4();
        run6();
    }
    if ((threadIdx.x & (kTile - 1)) == 0) {
        if (it6) atomicAdd(&sc->tron_iters6, it6);
        if (it4) atomicAdd(&sc->tron_iters4, it4);
        if (fails) atomicAdd(&sc->failures, (unsigned long long)fails);
    }
}

// ---- phase C: solo warps for the few branches with very long solves -------
// Late in a solve a handful of rate-limited branches run 10 AL rounds of up
// to 200 TRON iterations (~1000 executed steps) while every other branch is
// done in tens; the iteration then waits on their sequential chains.  Each
// such branch gets a whole warp (32 search trials per round, no other tile
// diverging in the warp) in a block of its own.
__global__ void __launch_bounds__(kSoloBlock) solo_kernel(DevNet net, DevState st, BranchCfg cfg,
                                                          Work w, DevScalars* sc) {
    if (gate_closed(cfg)) return;
    __shared__ double smem[kFields * (kTileBlock / kTile)];
    unsigned long long it6 = 0, it4 = 0;
    int fails = 0;
    tile_phase<6, 32>(net, st, cfg, w.solo6, &w.ctr[6], &w.ctr[8], smem, &it6, &fails, &sc->exec6, 0,
                      nullptr, nullptr);
    tile_phase<4, 32>(net, st, cfg, w.solo4, &w.ctr[7], &w.ctr[9], smem, &it4, &fails, &sc->exec4, 0,
                      nullptr, nullptr);
    if (threadIdx.x == 0) {
        if (it6) atomicAdd(&sc->tron_iters6, it6);
        if (it4) atomicAdd(&sc->tron_iters4, it4);
        if (fails) atomicAdd(&sc->failures, (unsigned long long)fails);
    }
}

// Dense box QP for the TRON-core parity test (proj/tests/acceptance.cpp:458-520).
template <int N>
struct QpProb {
    const double *H, *G, *L, *U;
    GA_FN double lo(int i) const { return L[i]; }
    GA_FN double hi(int i) const { return U[i]; }
    GA_FN double value(const double* x) const {
        double f = 0.0;
        for (int i = 0; i < N; ++i) {
            double hx = 0.0;
            for (int j = 0; j < N; ++j) hx += H[i * N + j] * x[j];
            f += G[i] * x[i] + 0.5 * x[i] * hx;
        }
        return f;
    }
    GA_FN void gradient(const double* x, double* g) const {
        for (int i = 0; i < N; ++i) {
            double hx = 0.0;
            for (int j = 0; j < N; ++j) hx += H[i * N + j] * x[j];
            g[i] = G[i] + hx;
        }
    }
    GA_FN void grad_hess(const double* x, double* g, double* h) const {
        gradient(x, g);
        for (int i = 0; i < N * N; ++i) h[i] = H[i];
    }
    GA_FN double hess_entry(const double*, int i, int j) const { return H[i * N + j]; }
};

// One QP per thread (SerialSearch) or per tile of T lanes (TileSearch) —
// both must reproduce the reference's solve_one bit-for-bit.
template <int N, int T>
__global__ void tron_qp_kernel(int count, const double* H, const double* G, const double* L,
                               const double* U, double* X, int* status, int* iterations) {
    const int gt = blockIdx.x * blockDim.x + threadIdx.x;
    const int k = gt / T;
    if (T == 1) {
        if (k >= count) return;
        QpProb<N> p{H + (size_t)k * N * N, G + (size_t)k * N, L + (size_t)k * N, U + (size_t)k * N};
        double x[N];
        for (int i = 0; i < N; ++i) x[i] = X[(size_t)k * N + i];
        TronParams tp;
        int its = 0;
        status[k] = tron_solve<N>(p, x, tp, &its);
        iterations[k] = its;
        for (int i = 0; i < N; ++i) X[(size_t)k * N + i] = x[i];
        return;
    }
    // tile path: whole tiles are in or out of range (count rounded per tile)
    const int lane = threadIdx.x & 31;
    const int rank = lane & (T - 1);
    const int tbase = lane & ~(T - 1);
    const unsigned mask = (T == 32 ? 0xffffffffu : ((1u << T) - 1u)) << tbase;
    if (k >= count) return;
    const TileSearch<T> search{mask, tbase, rank};
    QpProb<N> p{H + (size_t)k * N * N, G + (size_t)k * N, L + (size_t)k * N, U + (size_t)k * N};
    TronParams tp;
    TronState<N> ts;
    for (int i = 0; i < N; ++i) ts.x[i] = X[(size_t)k * N + i];
    int its = 0, st;
    if (!tron_begin<N>(p, ts)) {
        st = kTronNumericalError;
    } else {
        for (;;) {
            const int before = ts.iter;
            const int r = tron_step<N>(p, ts, tp, search);
            if (r == kStepContinue) continue;
            if (r == kStepConverged) { its = before; st = kTronConverged; break; }
            if (r == kStepError) { its = before; st = kTronNumericalError; break; }
            its = tp.max_iterations;
            st = tron_finish<N>(p, ts, tp);
            break;
        }
    }
    if (rank == 0) {
        status[k] = st;
        iterations[k] = its;
        for (int i = 0; i < N; ++i) X[(size_t)k * N + i] = ts.x[i];
    }
}

// ---- cold start on the device (driver.cpp:26-63, decomp.cpp:37-57) -------
// Same expressions as Session's host restatement; items: rows (z, y, lambda,
// rho), branches (8 x / xbar rows, point, multipliers), generators (2 rows),
// buses (w, theta).  Every x / xbar row is written by exactly one item.
__global__ void cold_start_kernel(DevNet n, DevState s, double rho_pq, double rho_va,
                                  double limit_tighten) {
    const long long total = (long long)n.mpad + n.nl + n.ng + n.nb;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        if (t < n.mpad) {
            const int p = (int)t;
            const int k = n.rid[p];  // reference row, -1 = padding (all zeros)
            const bool pq = k < 2 * n.ng || (k - 2 * n.ng) % 8 < 4;
            s.z[p] = 0.0;
            s.y[p] = 0.0;
            s.lambda[p] = 0.0;
            s.rho[p] = k < 0 ? 0.0 : (pq ? rho_pq : rho_va);
            if (k < 0) {
                s.x[p] = 0.0;
                s.xbar[p] = 0.0;
            }
        } else if (t < (long long)n.mpad + n.nl) {
            const int b = (int)(t - n.mpad);
            const int from = n.br_from[b], to = n.br_to[b];
            const double vi = 0.5 * (n.b_vmin[from] + n.b_vmax[from]);
            const double vj = 0.5 * (n.b_vmin[to] + n.b_vmax[to]);
            const YArr yc{n.br_y, n.nl, b};
            double f[4];
            bp::branch_flows(yc, vi, vj, 0.0, 0.0, f);
            const double vals[8] = {f[0], f[1], f[2], f[3], vi * vi, 0.0, vj * vj, 0.0};
            const int qf = n.qpos[2 * b], qt = n.qpos[2 * b + 1];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int r = bp::branch_row_pos(qf, qt, k);
                s.x[r] = vals[k];
                s.xbar[r] = vals[k];
            }
            double sij = 0.0, sji = 0.0;
            const double rate = n.br_rate[b];
            if (rate > 0.0) {
                const double rt = limit_tighten * rate;
                sij = sclamp(-(f[0] * f[0] + f[1] * f[1]), -rt * rt, 0.0);
                sji = sclamp(-(f[2] * f[2] + f[3] * f[3]), -rt * rt, 0.0);
            }
            const double pt[6] = {vi, vj, 0.0, 0.0, sij, sji};
#pragma unroll
            for (int k = 0; k < 6; ++k) s.bp[k * n.nl + b] = pt[k];
            s.lt_ij[b] = 0.0;
            s.lt_ji[b] = 0.0;
            s.rho_t[b] = rho_pq;
        } else if (t < (long long)n.mpad + n.nl + n.ng) {
            const int g = (int)(t - n.mpad - n.nl);
            const double p = 0.5 * (n.g_pmin[g] + n.g_pmax[g]);
            const double q = 0.5 * (n.g_qmin[g] + n.g_qmax[g]);
            const int r = n.gpos[g];
            s.x[r] = p;
            s.xbar[r] = p;
            s.x[r + 1] = q;
            s.xbar[r + 1] = q;
        } else {
            const int i = (int)(t - n.mpad - n.nl - n.ng);
            const double v = 0.5 * (n.b_vmin[i] + n.b_vmax[i]);
            s.bus_w[i] = v * v;
            s.bus_theta[i] = 0.0;
        }
    }
}

__global__ void sincos_probe_kernel(const double* x, double* s, double* c, int n) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n) ga_sincos(x[k], &s[k], &c[k]);
}

template <class K>
int persistent_blocks(K kernel, int block, size_t smem) {
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, block, smem);
    return sms * (per_sm > 0 ? per_sm : 1);
}

}  // namespace

size_t branch_workspace_ints(const DevNet& n) {
    return 2 * (static_cast<size_t>(n.n_lim) + n.n_unl) + kCounters + (static_cast<size_t>(n.nb) + 3) / 4;
}

unsigned char* bus_defer_flags(const DevNet& n, const DevState& s) { return work_of(n, s).defer; }

const int* branch_overflow_counts(const DevNet& n, const DevState& s) {
    return work_of(n, s).ctr + 2;
}

namespace {

constexpr size_t kLaneSmem = static_cast<size_t>(kFields) * kLaneBlock * sizeof(double);

struct Grids {
    int lane, tile, solo;
};

// persistent grid sizes (thread-safe one-time init; the pool's GPUs are identical)
const Grids& branch_grids() {
    static const Grids grids = [] {
        Grids gr;
        gr.lane = persistent_blocks(lane_kernel, kLaneBlock, kLaneSmem);
        gr.tile = persistent_blocks(tile_kernel, kTileBlock, 0);
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&gr.solo, cudaDevAttrMultiProcessorCount, dev);
        return gr;
    }();
    return grids;
}

}  // namespace

void prepare_branch_launch() { (void)branch_grids(); }

void launch_branches(const DevNet& n, const DevState& s, const BranchCfg& cfg, DevScalars* sc,
                     cudaStream_t st, cudaEvent_t mid, const std::function<void()>& after_lane) {
    if (n.nl <= 0) return;
    const Work w = work_of(n, s);
    cudaMemsetAsync(w.ctr, 0, kCounters * sizeof(int), st);
    const size_t lane_smem = kLaneSmem;
    const Grids& grids = branch_grids();
    const int lane_blocks = grids.lane, tile_blocks = grids.tile, solo_blocks = grids.solo;
    const int total = n.n_lim + n.n_unl;
    const int need = (total + kLaneBlock - 1) / kLaneBlock;
    BranchCfg lc = cfg;
    // the lane phase keeps branches (throughput mode) while the active set
    // exceeds twice the tile slots (swept 1/2/4: 2 best on both the bench
    // window and a truncated full solve; GRIDADMM_SLOT_MULT overrides)
    static const int slot_mult = [] {
        const char* e = std::getenv("GRIDADMM_SLOT_MULT");
        return e && std::atoi(e) > 0 ? std::atoi(e) : 2;
    }();
    lc.tile_slots = slot_mult * tile_blocks * (kTileBlock / kTile) / 2;  // per queue (two share)
    lane_kernel<<<lane_blocks < need ? lane_blocks : need, kLaneBlock, lane_smem, st>>>(n, s, lc,
                                                                                       w, sc);
    if (mid) cudaEventRecord(mid, st);
    if (after_lane) after_lane();
    tile_kernel<<<tile_blocks, kTileBlock, 0, st>>>(n, s, cfg, w, sc);
    if (cfg.tile_budget > 0) solo_kernel<<<solo_blocks, kSoloBlock, 0, st>>>(n, s, cfg, w, sc);
}

void launch_tron_qp(int count, int n, const double* h, const double* g, const double* l,
                    const double* u, double* x, int* status, int* iterations, cudaStream_t st,
                    int tile) {
    const int threads = count * tile;
    const int blocks = (threads + 127) / 128;
#define GA_QP(NN)                                                                                \
    case NN:                                                                                     \
        if (tile == 4)                                                                           \
            tron_qp_kernel<NN, 4><<<blocks, 128, 0, st>>>(count, h, g, l, u, x, status, iterations); \
        else if (tile == 8)                                                                      \
            tron_qp_kernel<NN, 8><<<blocks, 128, 0, st>>>(count, h, g, l, u, x, status, iterations); \
        else if (tile == 32)                                                                     \
            tron_qp_kernel<NN, 32><<<blocks, 128, 0, st>>>(count, h, g, l, u, x, status, iterations); \
        else                                                                                     \
            tron_qp_kernel<NN, 1><<<blocks, 128, 0, st>>>(count, h, g, l, u, x, status, iterations); \
        break;
    switch (n) {
        GA_QP(1) GA_QP(2) GA_QP(3) GA_QP(4) GA_QP(5) GA_QP(6)
        default: break;
    }
#undef GA_QP
}

void launch_cold_start(const DevNet& n, const DevState& s, double rho_pq, double rho_va,
                       double limit_tighten, cudaStream_t st) {
    const long long total = (long long)n.mpad + n.nl + n.ng + n.nb;
    if (total <= 0) return;
    long long blocks = (total + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    cold_start_kernel<<<(int)blocks, 256, 0, st>>>(n, s, rho_pq, rho_va, limit_tighten);
}

void launch_sincos_probe(const double* x, double* s, double* c, int n, cudaStream_t st) {
    if (n > 0) sincos_probe_kernel<<<(n + 255) / 256, 256, 0, st>>>(x, s, c, n);
}

}  // namespace ga
