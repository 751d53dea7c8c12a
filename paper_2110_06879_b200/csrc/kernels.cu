// kernels.cu — the HBM-bound phases of one inner ADMM iteration:
//   generator projection (north-star (a), kernels.cpp:194-209),
//   bus consensus QP      (north-star (c), kernels.cpp:294-413),
//   fused z / y / residual norms (north-star (d), kernels.cpp:415-428 +
//   decomp.cpp:59-72 + driver.cpp:179-186,213-215),
//   outer multiplier update (kernels.cpp:430-437),
//   tracking carry-over clamp (tracking.cpp:65-70).
// All arithmetic mirrors the reference's expression trees (compiled with
// -fmad=false); the infinity-norm reductions are order-free maxima, so a
// warp+grid reduction gives the reference's bits exactly.
#include <climits>

#include "device.hpp"
#include "ga_math.h"

namespace ga {

namespace {

constexpr int kBlock = 256;

__device__ __forceinline__ unsigned long long dbits(double v) {
    return static_cast<unsigned long long>(__double_as_longlong(v));
}

// Block-wide max of non-negative doubles, then one atomicMax per block on the
// IEEE bit pattern (monotone for non-negative values).
template <int NV>
__device__ __forceinline__ void block_max_atomic(double (&v)[NV], unsigned long long* const (&dst)[NV]) {
    __shared__ double red[NV][kBlock / 32];
    const unsigned full = 0xffffffffu;
#pragma unroll
    for (int q = 0; q < NV; ++q) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[q] = fmax(v[q], __shfl_down_sync(full, v[q], o));
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) {
#pragma unroll
        for (int q = 0; q < NV; ++q) red[q][wid] = v[q];
    }
    __syncthreads();
    if (wid == 0) {
#pragma unroll
        for (int q = 0; q < NV; ++q) {
            double t = lane < (int)(blockDim.x >> 5) ? red[q][lane] : 0.0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) t = fmax(t, __shfl_down_sync(full, t, o));
            if (lane == 0 && t > 0.0) atomicMax(dst[q], dbits(t));
        }
    }
}

// ---- generators (kernels.cpp:194-209) ----------------------------------
__global__ void __launch_bounds__(kBlock) gen_kernel(DevNet n, DevState s) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n.gens_count()) return;
    const int g = n.gen_at(t);
    // the p and q rows are adjacent (an even position): one 16-B load per array
    const int h = n.gpos[g] >> 1;
    const double2 xb = reinterpret_cast<const double2*>(s.xbar)[h];
    const double2 zz = reinterpret_cast<const double2*>(s.z)[h];
    const double2 yy = reinterpret_cast<const double2*>(s.y)[h];
    const double2 rr = reinterpret_cast<const double2*>(s.rho)[h];
    const double p = (rr.x * (xb.x - zz.x) - yy.x - n.g_c1[g]) / (2.0 * n.g_c2[g] + rr.x);
    const double q = (rr.y * (xb.y - zz.y) - yy.y) / rr.y;
    double2 out;
    out.x = sclamp(p, n.g_pmin[g], n.g_pmax[g]);
    out.y = sclamp(q, n.g_qmin[g], n.g_qmax[g]);
    reinterpret_cast<double2*>(s.x)[h] = out;
}

// The generator projection of one generator row (the expressions of
// gen_kernel above), evaluated where the bus kernel consumes the row.  The
// row's generator data are loaded first (GenRow) so the loads issue with the
// row's state loads rather than after them.
struct GenRow {
    double c1, c2, lo, hi;  // p row: c1, c2, pmin, pmax; q row: -, -, qmin, qmax
};
// pos: the storage position of a generator row (p rows at even positions)
__device__ __forceinline__ GenRow load_gen_row(const DevNet& n, int pos) {
    const int h = pos >> 1;
    GenRow r;
    if ((pos & 1) == 0) {
        r.c1 = __ldg(n.pr_c1 + h);
        r.c2 = __ldg(n.pr_c2 + h);
        r.lo = __ldg(n.pr_pmin + h);
        r.hi = __ldg(n.pr_pmax + h);
    } else {
        r.c1 = r.c2 = 0.0;
        r.lo = __ldg(n.pr_qmin + h);
        r.hi = __ldg(n.pr_qmax + h);
    }
    return r;
}
__device__ __forceinline__ double gen_row_x(int row, const GenRow& p, double xb, double z, double y,
                                            double rho) {
    if ((row & 1) == 0) return sclamp((rho * (xb - z) - y - p.c1) / (2.0 * p.c2 + rho), p.lo, p.hi);
    return sclamp((rho * (xb - z) - y) / rho, p.lo, p.hi);
}

// ---- buses (kernels.cpp:294-413) ----------------------------------------
// Per bus, variables: [0] w, [1] theta, then one duplicate per row in gen_p,
// gen_q, flow_p, flow_q order.  A's entries are implied by the group of each
// column.  Sums run over columns in the reference's order; columns whose A
// entry is an exact zero are skipped when every c is finite (the skipped
// term is a signed zero added to an accumulator that started at +0.0 —
// exact), otherwise the dense loop is used.
__device__ __forceinline__ double a_coef(int r, int grp, double gs, double bs, bool ref) {
    // grp: 0 = w, 1 = theta, 2 = gen_p, 3 = gen_q, 4 = flow_p, 5 = flow_q
    switch (r) {
        case 0: return grp == 0 ? -gs : grp == 2 ? 1.0 : grp == 4 ? -1.0 : 0.0;
        case 1: return grp == 0 ? bs : grp == 3 ? 1.0 : grp == 5 ? -1.0 : 0.0;
        default: return (ref && grp == 1) ? 1.0 : 0.0;
    }
}

// Gaussian elimination with partial pivoting on the NC x NC system
// (kernels.cpp:364-391) with register-resident rows: the reference permutes
// row indices (piv), here the rows themselves are swapped — the same values
// meet the same operations, so the result is identical.  S is row-major 3x3.
template <int NC>
__device__ __forceinline__ bool ge_solve(double* S, double* rhs, double* mu) {
    double A[NC][NC], b[NC];
#pragma unroll
    for (int r = 0; r < NC; ++r) {
#pragma unroll
        for (int c = 0; c < NC; ++c) A[r][c] = S[r * 3 + c];
        b[r] = rhs[r];
    }
#pragma unroll
    for (int col = 0; col < NC; ++col) {
        int best = col;
#pragma unroll
        for (int r = col + 1; r < NC; ++r)
            if (fabs(A[r][col]) > fabs(A[best][col])) best = r;
#pragma unroll
        for (int r = col + 1; r < NC; ++r) {
            if (best == r) {
#pragma unroll
                for (int c = 0; c < NC; ++c) {
                    const double t = A[col][c];
                    A[col][c] = A[r][c];
                    A[r][c] = t;
                }
                const double t = b[col];
                b[col] = b[r];
                b[r] = t;
            }
        }
        const double d = A[col][col];
        if (fabs(d) < 1e-14) return false;
#pragma unroll
        for (int r = col + 1; r < NC; ++r) {
            const double f = A[r][col] / d;
#pragma unroll
            for (int s2 = col; s2 < NC; ++s2) A[r][s2] -= f * A[col][s2];
            b[r] -= f * b[col];
        }
    }
#pragma unroll
    for (int col = NC - 1; col >= 0; --col) {
        double acc = b[col];
#pragma unroll
        for (int s2 = col + 1; s2 < NC; ++s2) acc -= A[col][s2] * mu[s2];
        mu[col] = acc / A[col][col];
    }
    return true;
}

// Block-staged bus kernel (the one launched), optionally fused with the z / y
// updates and all four residual norms.
//
// A warp-per-bus formulation (previous version) spent its time issuing lane
// 0's serial code (ncu: 4 active threads per warp, 59% issue-slot busy).  Here a block of
// kBB threads owns kBB consecutive buses and works in three phases:
//   1. gather: the block's rows (CSR, contiguous per bus) are spread over all
//      threads; each thread loads rho, x, z, y of a row and stages either
//      (rho, c) for the w / theta columns or the S / rhs terms (a*a/rho,
//      a*c/rho) of a duplicate column (kernels.cpp:311-361) in shared memory;
//   2. solve: thread = bus: the ordered sums, the NC x NC elimination and mu,
//      with every lane of the warp busy;
//   3. write: rows again spread over all threads: xbar = (c - A'mu)/rho
//      (kernels.cpp:394-399) and, fused, z (kernels.cpp:415-422), y
//      (kernels.cpp:424-428) and the primal / dual / z / drift maxima.
// Fusing z / y is exact: every row is consumed by exactly one bus
// (proj/tests/test_decomp.cpp:59-71) and z / y of a row depend only on that
// row, so the order "all buses, then all z, then all y" is not observable.
// The iteration form (kZY) also absorbs the generator projection
// (kernels.cpp:194-209): x of a generator row depends only on that row's
// previous xbar, z, y, rho, which nothing between the generator phase and
// the bus phase writes (the branch phase touches branch rows only), so it is
// computed here — in the gather, the solve's unstaged reads and the write,
// always from the same inputs, hence the same bits — and written once.
#ifndef GA_BUS_BLOCK
#define GA_BUS_BLOCK 128
#endif
constexpr int kBB = GA_BUS_BLOCK;  // buses per block
// Threads per block kBT = kTPB * kBB: the per-row phases (gather, write) use
// all of them, the per-bus solve the first kBB.  A block's time is its
// per-thread row work plus the solve, so two threads per bus cut it by ~30%
// (2868-shaped grid: 37.5 -> 26.7 us) — worth it while the grid fits in one
// wave; on the 70k shape (547 blocks) the halved residency costs more
// (73 -> 78 us), so launch_bus_* pick kTPB by grid size.
// staged rows per block (the rest are read from global); 8 / 12 rows per bus
// with 6-8 blocks per SM forced by __launch_bounds__ measured 23-43% slower
constexpr int kStage = 16 * kBB;

// largest slot with off[slot] <= p  (off[0] = 0 <= p < off[kBB])
__device__ __forceinline__ int find_slot(const int* off, int p) {
    int lo = 0, hi = kBB;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (off[mid] <= p) lo = mid;
        else hi = mid;
    }
    return lo;
}

// Column group of the local position k of a bus's segment (device.hpp):
// 0 w, 1 theta, 2 gen_p, 3 gen_q, 4 flow_p, 5 flow_q, 6 padding.  ge / qs:
// local end of the generator pairs / start of the quads.
__device__ __forceinline__ int group_of(int ge, int qs, int k) {
    if (k < ge) return 2 + (k & 1);
    if (k < qs) return 6;
    constexpr unsigned kQuadGroups = 4u | 5u << 4 | 0u << 8 | 1u << 12;  // p, q, w, theta
    return (kQuadGroups >> (4 * ((k - qs) & 3))) & 15u;
}

constexpr int kFlagNonfinite = 1, kFlagSingular = 2, kFlagRef = 4;

__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

template <bool kZY, int kTPB, int kSel = 0>
__global__ void __launch_bounds__(kTPB * kBB) bus_block_kernel(DevNet n, DevState s, double beta,
                                                       DevScalars* sc, LoopCtl* gate,
                                                       const unsigned char* defer = nullptr) {
    if (gate) {
        if (*reinterpret_cast<volatile int*>(&gate->stop)) return;
        beta = gate->beta;
        if (kSel != 1 && blockIdx.x == 0 && threadIdx.x == 0) gate->t_bus = global_ns();
    }
    __shared__ int s_off[kBB + 1];
    __shared__ int s_base[kBB];       // segment start (storage position) of each slot's bus
    __shared__ int s_gl[kBB][4];      // local gen end, quad start, count, flags
    __shared__ double s_res[kBB][5];  // mu0..2, w, theta
    __shared__ double s_a[kStage], s_b[kStage];
    __shared__ unsigned short s_pos[kStage];  // staged position -> slot << 3 | group
    constexpr int kBT = kTPB * kBB;
    __shared__ int s_wsum[kBT / 32];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int t = blockIdx.x * kBB + tid;
    const int nbus = n.buses_count();
    int i = -1, cnt = 0, ge = 0, qs = 0;
    {
        int start = 0;
        if (tid < kBB && t < nbus) i = n.bus_at(t);
        // a bus outside this launch's selection owns no rows here (cnt 0)
        GA_CHECK(i < n.nb);
        if (kSel != 0 && i >= 0 && (defer[i] != 0) != (kSel == 2)) i = -1;
        if (i >= 0) {
            const int* seg = n.bus_seg + 4 * i;
            start = __ldg(seg);
            ge = __ldg(seg + 1) - start;
            qs = __ldg(seg + 2) - start;
            cnt = __ldg(seg + 3) - start;
        }
        if (tid < kBB) {
            s_base[tid] = start;
            s_gl[tid][0] = ge;
            s_gl[tid][1] = qs;
            s_gl[tid][2] = cnt;
            s_gl[tid][3] = (i >= 0 && i == n.ref_bus) ? kFlagRef : 0;
        }
    }
    // block exclusive scan of the segment lengths
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    if (lane == 31) s_wsum[wid] = incl;
    __syncthreads();
    int woff = 0;
#pragma unroll
    for (int w = 0; w < kBB / 32; ++w) woff += w < wid ? s_wsum[w] : 0;
    const int my_off = woff + incl - cnt;
    if (tid < kBB) s_off[tid] = my_off;
    if (tid == kBB - 1) s_off[kBB] = woff + incl;
    for (int k = 0; k < cnt && my_off + k < kStage; ++k)  // position map of the staged rows
        s_pos[my_off + k] = static_cast<unsigned short>(tid << 3 | group_of(ge, qs, k));
    __syncthreads();
    const int total = s_off[kBB];
    const int staged = total < kStage ? total : kStage;
    // (slot, local position, group) of block position p
    auto locate = [&](int p, int* slot, int* k, int* g) {
        if (p < kStage) {
            const int v = s_pos[p];
            *slot = v >> 3;
            *k = p - s_off[*slot];
            *g = v & 7;
        } else {
            *slot = find_slot(s_off, p);
            *k = p - s_off[*slot];
            *g = group_of(s_gl[*slot][0], s_gl[*slot][1], *k);
        }
    };

    // 1. gather: kUnroll positions per thread per trip, loads issued together
    // (for one block of consecutive buses the positions are one contiguous
    // range of the row vectors: coalesced)
    constexpr int kUnroll = 4;
    for (int p0 = tid; p0 < staged; p0 += kBT * kUnroll) {
        int row[kUnroll], slot[kUnroll], g[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const int p = p0 + u * kBT;
            row[u] = -1;
            if (p < staged) {
                int k;
                locate(p, &slot[u], &k, &g[u]);
                if (g[u] != 6) row[u] = s_base[slot[u]] + k;
                GA_CHECK(row[u] < n.mpad && slot[u] >= 0 && slot[u] < kBB);
            }
        }
        double q[kUnroll], xv[kUnroll], zv[kUnroll], yv[kUnroll];
        GenRow gp[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            if (row[u] >= 0) {
                const bool gen = kZY && (g[u] == 2 || g[u] == 3);
                q[u] = __ldg(s.rho + row[u]);
                zv[u] = __ldg(s.z + row[u]);
                yv[u] = __ldg(s.y + row[u]);
                xv[u] = __ldg((gen ? s.xbar : s.x) + row[u]);  // gen rows: the previous xbar
                if (gen) gp[u] = load_gen_row(n, row[u]);
            }
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u)
            if (row[u] >= 0 && kZY && (g[u] == 2 || g[u] == 3))
                xv[u] = gen_row_x(g[u] == 2 ? 0 : 1, gp[u], xv[u], zv[u], yv[u], q[u]);
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            if (row[u] < 0) continue;
            const int p = p0 + u * kBT;
            const double c = q[u] * (xv[u] + zv[u]) + yv[u];
            if (g[u] < 2) {
                s_a[p] = q[u];
                s_b[p] = c;
            } else {
                if (!sfinite(c)) atomicOr(&s_gl[slot[u]][3], kFlagNonfinite);
                const double a = g[u] < 4 ? 1.0 : -1.0;  // gen columns +1, flow columns -1
                s_a[p] = a * a / q[u];
                s_b[p] = a * c / q[u];
            }
        }
    }
    __syncthreads();

    // 2. solve (thread = bus), kernels.cpp:303-391; every group is a strided
    // walk of the segment in the reference's push order
    if (i >= 0) {
        const int base = my_off;
        const int start = s_base[tid];
        const bool ref = (s_gl[tid][3] & kFlagRef) != 0;
        const int nc = ref ? 3 : 2;
        const double gs = n.b_gs[i], bs = n.b_bs[i];
        auto raw = [&](int k, double* q, double* c) {
            const int row = start + k;
            *q = s.rho[row];
            const int grp = group_of(ge, qs, k);
            const double xr = (kZY && (grp == 2 || grp == 3))
                                  ? gen_row_x(grp == 2 ? 0 : 1, load_gen_row(n, row),
                                              s.xbar[row], s.z[row], s.y[row], *q)
                                  : s.x[row];
            *c = *q * (xr + s.z[row]) + s.y[row];
        };
        auto staged_qc = [&](int k, double* q, double* c) {  // w / theta rows
            const int p = base + k;
            if (p < kStage) { *q = s_a[p]; *c = s_b[p]; }
            else raw(k, q, c);
        };
        double q0 = 0.0, c0 = 0.0, q1 = 0.0, c1 = 0.0, q, c;
        for (int k = qs + 2; k < cnt; k += 4) { staged_qc(k, &q, &c); q0 += q; c0 += c; }
        for (int k = qs + 3; k < cnt; k += 4) { staged_qc(k, &q, &c); q1 += q; c1 += c; }
        if (q0 == 0.0) q0 = 1.0;
        if (q1 == 0.0) q1 = 1.0;
        bool finite = sfinite(c0) && sfinite(c1) && !(s_gl[tid][3] & kFlagNonfinite);
        for (int k = (kStage - base > 0 ? kStage - base : 0); k < cnt && finite; ++k) {
            const int grp = group_of(ge, qs, k);
            if (grp < 2 || grp == 6) continue;
            raw(k, &q, &c);
            finite = sfinite(c);
        }
        const int ngb = ge / 2, nq = (cnt - qs) / 4;
        double S[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0}, rhs[3] = {0, 0, 0};
        const double bvec[3] = {n.b_pd[i], n.b_qd[i], 0.0};
        if (finite) {
            const double a00 = -gs, a10 = bs;
            double s00 = 0.0, s01 = 0.0, s11 = 0.0, s22 = 0.0, r0 = 0.0, r1 = 0.0, r2 = 0.0;
            s00 += a00 * a00 / q0;
            s01 += a00 * a10 / q0;
            s11 += a10 * a10 / q0;
            r0 += a00 * c0 / q0;
            r1 += a10 * c0 / q0;
            if (ref) {
                s22 += 1.0 * 1.0 / q1;
                r2 += 1.0 * c1 / q1;
            }
            auto term = [&](int k, double a, double* ts, double* tr) {
                const int p = base + k;
                if (p < kStage) { *ts = s_a[p]; *tr = s_b[p]; return; }
                raw(k, &q, &c);
                *ts = a * a / q;
                *tr = a * c / q;
            };
            double ts, tr;
            for (int k = 0; k < ge; k += 2) { term(k, 1.0, &ts, &tr); s00 += ts; r0 += tr; }
            for (int k = qs; k < cnt; k += 4) { term(k, -1.0, &ts, &tr); s00 += ts; r0 += tr; }
            for (int k = 1; k < ge; k += 2) { term(k, 1.0, &ts, &tr); s11 += ts; r1 += tr; }
            for (int k = qs + 1; k < cnt; k += 4) { term(k, -1.0, &ts, &tr); s11 += ts; r1 += tr; }
            S[0] = s00; S[1] = s01; S[3] = s01; S[4] = s11;
            S[8] = s22;
            rhs[0] = r0 - bvec[0];
            rhs[1] = r1 - bvec[1];
            rhs[2] = r2 - bvec[2];
        } else {
            // dense reference loop (kernels.cpp:350-361) over the columns
            // [w, theta, gen_p..., gen_q..., flow_p..., flow_q...], any value
            auto col = [&](int j, int* gg, double* qj, double* cj) {
                if (j == 0) { *gg = 0; *qj = q0; *cj = c0; return; }
                if (j == 1) { *gg = 1; *qj = q1; *cj = c1; return; }
                const int d = j - 2;
                int k;
                if (d < ngb) { *gg = 2; k = 2 * d; }
                else if (d < 2 * ngb) { *gg = 3; k = 2 * (d - ngb) + 1; }
                else if (d < 2 * ngb + nq) { *gg = 4; k = qs + 4 * (d - 2 * ngb); }
                else { *gg = 5; k = qs + 4 * (d - 2 * ngb - nq) + 1; }
                raw(k, qj, cj);
            };
            const int nv = 2 + 2 * ngb + 2 * nq;
            for (int r = 0; r < nc; ++r) {
                for (int t2 = 0; t2 < nc; ++t2) {
                    double acc = 0.0;
                    for (int j = 0; j < nv; ++j) {
                        int gg; double qj, cj;
                        col(j, &gg, &qj, &cj);
                        acc += a_coef(r, gg, gs, bs, ref) * a_coef(t2, gg, gs, bs, ref) / qj;
                    }
                    S[r * 3 + t2] = acc;
                }
                double acc = 0.0;
                for (int j = 0; j < nv; ++j) {
                    int gg; double qj, cj;
                    col(j, &gg, &qj, &cj);
                    acc += a_coef(r, gg, gs, bs, ref) * cj / qj;
                }
                rhs[r] = acc - bvec[r];
            }
        }
        double mu[3] = {0, 0, 0};
        const bool singular = ref ? !ge_solve<3>(S, rhs, mu) : !ge_solve<2>(S, rhs, mu);
        if (!singular) {
            double acc = c0;
            for (int r = 0; r < nc; ++r) acc -= a_coef(r, 0, gs, bs, ref) * mu[r];
            const double w = acc / q0;
            acc = c1;
            for (int r = 0; r < nc; ++r) acc -= a_coef(r, 1, gs, bs, ref) * mu[r];
            const double th = acc / q1;
            s.bus_w[i] = w;
            s.bus_theta[i] = th;
            s_res[tid][3] = w;
            s_res[tid][4] = th;
        } else {
            atomicMin(&sc->singular_bus, i);
            s_gl[tid][3] |= kFlagSingular;
        }
        s_res[tid][0] = mu[0];
        s_res[tid][1] = mu[1];
        s_res[tid][2] = mu[2];
    }
    __syncthreads();

    // 3. write xbar (+ z, y) and the norms; the old values read here were
    // not written before in this kernel (each row belongs to one block)
    double dual = 0.0, pr = 0.0, zi = 0.0, zd = 0.0;
    for (int p0 = tid; p0 < total; p0 += kBT * kUnroll) {
        int row[kUnroll], slot[kUnroll], g[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const int p = p0 + u * kBT;
            row[u] = -1;
            if (p < total) {
                int k;
                locate(p, &slot[u], &k, &g[u]);
                if (g[u] != 6) row[u] = s_base[slot[u]] + k;
                GA_CHECK(row[u] < n.mpad && slot[u] >= 0 && slot[u] < kBB);
            }
        }
        double old[kUnroll], q[kUnroll], xv[kUnroll], zv[kUnroll], yv[kUnroll], lam[kUnroll];
        GenRow gp[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            if (row[u] >= 0) {
                old[u] = __ldg(s.xbar + row[u]);
                q[u] = __ldg(s.rho + row[u]);
                zv[u] = __ldg(s.z + row[u]);
                yv[u] = __ldg(s.y + row[u]);
                xv[u] = __ldg(s.x + row[u]);  // generator rows: replaced below
                if (kZY && (g[u] == 2 || g[u] == 3)) gp[u] = load_gen_row(n, row[u]);
                if (kZY) lam[u] = __ldg(s.lambda + row[u]);
            }
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            if (row[u] >= 0 && kZY && (g[u] == 2 || g[u] == 3)) {
                xv[u] = gen_row_x(g[u] == 2 ? 0 : 1, gp[u], old[u], zv[u], yv[u], q[u]);
                s.x[row[u]] = xv[u];
            }
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            if (row[u] < 0) continue;
            const int flags = s_gl[slot[u]][3];
            double xb = old[u];
            if (!(flags & kFlagSingular)) {
                if (g[u] == 0) xb = s_res[slot[u]][3];
                else if (g[u] == 1) xb = s_res[slot[u]][4];
                else {
                    // a_coef(r, g >= 2) does not depend on gs / bs / ref
                    const int nc = (flags & kFlagRef) ? 3 : 2;
                    double acc = q[u] * (xv[u] + zv[u]) + yv[u];
                    for (int r = 0; r < nc; ++r)
                        acc -= a_coef(r, g[u], 0.0, 0.0, false) * s_res[slot[u]][r];
                    xb = acc / q[u];
                }
                dual = smax(dual, abs_or_zero(xb - old[u]));
                s.xbar[row[u]] = xb;
            }
            if (kZY) {
                const double r = xv[u] - xb;
                const double z = -(lam[u] + yv[u] + q[u] * r) / (q[u] + beta);
                const double res = xv[u] - xb + z;
                s.z[row[u]] = z;
                s.y[row[u]] = yv[u] + q[u] * res;
                pr = smax(pr, abs_or_zero(res));
                zi = smax(zi, abs_or_zero(z));
                zd = smax(zd, abs_or_zero(z - zv[u]));
            }
        }
    }
    if (kZY) {
        double vals[4] = {dual, pr, zi, zd};
        unsigned long long* const dst[4] = {&sc->dual_inf, &sc->primal_inf, &sc->z_inf, &sc->z_drift};
        block_max_atomic<4>(vals, dst);
    } else {
        double vals[1] = {dual};
        unsigned long long* const dst[1] = {&sc->dual_inf};
        block_max_atomic<1>(vals, dst);
    }
}

__global__ void z_only_kernel(DevNet n, DevState s, double beta) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n.rows_count()) return;
    const int k = n.row_at(t);
    const double r = s.x[k] - s.xbar[k];
    s.z[k] = -(s.lambda[k] + s.y[k] + s.rho[k] * r) / (s.rho[k] + beta);
}

__global__ void y_only_kernel(DevNet n, DevState s) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n.rows_count()) return;
    const int k = n.row_at(t);
    s.y[k] += s.rho[k] * (s.x[k] - s.xbar[k] + s.z[k]);
}

__global__ void outer_kernel(DevNet n, DevState s, double beta, double lmin, double lmax) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n.rows_count()) return;
    const int k = n.row_at(t);
    s.lambda[k] = sclamp(s.lambda[k] + beta * s.z[k], lmin, lmax);
}

__global__ void clamp_gen_p_kernel(DevNet n, DevState s) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n.gens_count()) return;
    const int g = n.gen_at(t);
    const int pr = n.gpos[g];
    s.x[pr] = sclamp(s.x[pr], n.g_pmin[g], n.g_pmax[g]);
    s.xbar[pr] = sclamp(s.xbar[pr], n.g_pmin[g], n.g_pmax[g]);
}

__global__ void __launch_bounds__(kBlock) rowmax_kernel(const double* v, int n,
                                                        unsigned long long* dst) {
    double mx = 0.0;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x)
        mx = smax(mx, v[k]);
    double vals[1] = {mx};
    unsigned long long* const d[1] = {dst};
    block_max_atomic<1>(vals, d);
}

__global__ void reset_scalars_kernel(DevScalars* sc) {
    sc->primal_inf = 0;
    sc->dual_inf = 0;
    sc->z_inf = 0;
    sc->z_drift = 0;
    sc->failures = 0;
    sc->singular_bus = INT_MAX;
}

inline int blocks_for(int n) { return (n + kBlock - 1) / kBlock; }

__device__ __forceinline__ double from_bits_dev(unsigned long long b) {
    return __longlong_as_double(static_cast<long long>(b));
}

__global__ void loop_start_kernel(LoopCtl* c, DevScalars* sc) {
    c->t_start = global_ns();
    c->t_mark = c->t_start;
    c->t_bus = c->t_start;
    sc->primal_inf = 0;
    sc->dual_inf = 0;
    sc->z_inf = 0;
    sc->z_drift = 0;
    sc->failures = 0;
    sc->singular_bus = INT_MAX;
}

// driver.cpp:179-220 after one iteration: the record, then the divergence
// and inner stop tests in the reference's order; clears the scalars for the
// next iteration.  One thread.
__global__ void loop_control_kernel(LoopCtl* c, LoopRec* rec, DevScalars* sc) {
    if (c->stop) return;
    const unsigned long long now = global_ns();
    if (sc->singular_bus != INT_MAX) {
        c->singular = sc->singular_bus;
        c->stop = kLoopSingular;
        return;
    }
    const double primal = from_bits_dev(sc->primal_inf);
    const double dual = from_bits_dev(sc->dual_inf) * c->rho_max;
    const double z = from_bits_dev(sc->z_inf);
    const double drift = from_bits_dev(sc->z_drift);
    const int inner = ++c->inner;
    LoopRec r;
    r.outer = c->outer;
    r.inner = inner;
    r.primal = primal;
    r.dual = dual;
    r.z = z;
    r.drift = drift;
    r.t_ns = now;
    rec[inner - 1] = r;
    c->failures += sc->failures;
    c->x_ns += c->t_bus - c->t_mark;
    c->xbar_ns += now - c->t_bus;
    c->t_mark = now;
    c->last_z = z;
    int stop = kLoopRunning;
    if (!sfinite(primal) || !sfinite(dual) || primal > c->diverge || dual > c->diverge)
        stop = kLoopDiverged;
    else if (smax(primal, dual) <= c->inner_tol)
        stop = kLoopInner;
    else if (primal <= c->inner_tol && z <= c->eps && drift <= 0.01 * c->eps)
        stop = kLoopInner;
    else if (inner >= c->max_inner)
        stop = kLoopLimit;
    c->stop = stop;
    sc->primal_inf = 0;
    sc->dual_inf = 0;
    sc->z_inf = 0;
    sc->z_drift = 0;
    sc->failures = 0;
    sc->singular_bus = INT_MAX;
}

// FP64 pipe microbenchmark: 8 independent chains per thread.  kFma = false
// issues DMUL + DADD (what -fmad=false code runs), true issues DFMA.
template <bool kFma>
__global__ void __launch_bounds__(kBlock) fp64_peak_kernel(double* out, int iters, double b,
                                                            double c) {
    double a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-9 + k;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            if (kFma) a[k] = fma(a[k], b, c);
            else a[k] = a[k] * b + c;
        }
    }
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += a[k];
    if (s == 12345.678) out[0] = s;  // keep the chains alive
}

}  // namespace

void measure_fp64_peak(double* tflops_mul_add, double* tflops_fma) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    double* out = nullptr;
    cudaMalloc(&out, sizeof(double));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int blocks = sms * 8, iters = 4096;
    const double flops = 2.0 * 8.0 * iters * blocks * (double)kBlock;
    for (int pass = 0; pass < 2; ++pass) {
        float best = 1e30f;
        for (int rep = 0; rep < 5; ++rep) {
            cudaEventRecord(a);
            if (pass == 0) fp64_peak_kernel<false><<<blocks, kBlock>>>(out, iters, 0.999999, 1e-7);
            else fp64_peak_kernel<true><<<blocks, kBlock>>>(out, iters, 0.999999, 1e-7);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms = 0.0f;
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
        }
        const double tf = flops / (best * 1e-3) / 1e12;
        if (pass == 0) *tflops_mul_add = tf;
        else *tflops_fma = tf;
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(out);
}



void launch_generators(const DevNet& n, const DevState& s, cudaStream_t st) {
    const int c = n.gens_count();
    if (c > 0) gen_kernel<<<blocks_for(c), kBlock, 0, st>>>(n, s);
}

namespace {
// two threads per bus while the grid fits in one wave at two blocks per SM
bool bus_two_threads(int blocks) {
    static const int sms = [] {
        int dev = 0, v = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        return v;
    }();
    return blocks <= 2 * sms;
}
}  // namespace

void launch_buses(const DevNet& n, const DevState& s, DevScalars* sc, cudaStream_t st) {
    const int c = n.buses_count();
    if (c <= 0) return;
    const int blocks = (c + kBB - 1) / kBB;
    if (bus_two_threads(blocks))
        bus_block_kernel<false, 2><<<blocks, 2 * kBB, 0, st>>>(n, s, 0.0, sc, nullptr);
    else
        bus_block_kernel<false, 1><<<blocks, kBB, 0, st>>>(n, s, 0.0, sc, nullptr);
}

void launch_bus_zy(const DevNet& n, const DevState& s, double beta, DevScalars* sc,
                   cudaStream_t st, LoopCtl* gate, const unsigned char* defer, int sel) {
    const int c = n.buses_count();
    if (c <= 0) return;
    const int blocks = (c + kBB - 1) / kBB;
#define GA_BUS_SEL(TPB)                                                                          \
    switch (sel) {                                                                               \
        case 1: bus_block_kernel<true, TPB, 1><<<blocks, TPB * kBB, 0, st>>>(n, s, beta, sc, gate, defer); break; \
        case 2: bus_block_kernel<true, TPB, 2><<<blocks, TPB * kBB, 0, st>>>(n, s, beta, sc, gate, defer); break; \
        default: bus_block_kernel<true, TPB, 0><<<blocks, TPB * kBB, 0, st>>>(n, s, beta, sc, gate, nullptr); \
    }
    // (two threads per bus for the sel-2 launch alone, whose blocks hold a
    // few flagged buses each: 33.4 vs 27.8 us, profiles/ab/r02_bus_overlap_b_tpb2.jsonl)
    if (bus_two_threads(blocks)) {
        GA_BUS_SEL(2)
    } else {
        GA_BUS_SEL(1)
    }
#undef GA_BUS_SEL
}

void launch_z_only(const DevNet& n, const DevState& s, double beta, cudaStream_t st) {
    const int c = n.rows_count();
    if (c > 0) z_only_kernel<<<blocks_for(c), kBlock, 0, st>>>(n, s, beta);
}

void launch_y_only(const DevNet& n, const DevState& s, cudaStream_t st) {
    const int c = n.rows_count();
    if (c > 0) y_only_kernel<<<blocks_for(c), kBlock, 0, st>>>(n, s);
}

void launch_outer(const DevNet& n, const DevState& s, double beta, double lmin, double lmax,
                  cudaStream_t st) {
    const int c = n.rows_count();
    if (c > 0) outer_kernel<<<blocks_for(c), kBlock, 0, st>>>(n, s, beta, lmin, lmax);
}

void launch_clamp_gen_p(const DevNet& n, const DevState& s, cudaStream_t st) {
    const int c = n.gens_count();
    if (c > 0) clamp_gen_p_kernel<<<blocks_for(c), kBlock, 0, st>>>(n, s);
}

// dst[rows[t]] = src[rows[t]] for t < count (device-to-device, same device
// or peer-mapped): boundary exchange of the in-process multi-part transport.
__global__ void copy_rows_kernel(const int* rows, int count, const double* src, double* dst) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < count) dst[rows[t]] = src[rows[t]];
}

void launch_copy_rows(const int* rows, int count, const double* src, double* dst,
                      cudaStream_t st) {
    if (count > 0) copy_rows_kernel<<<blocks_for(count), kBlock, 0, st>>>(rows, count, src, dst);
}

// buf[t] = v[rows[t]] / v[rows[t]] = buf[t]: pack / unpack for NCCL.
__global__ void gather_rows_kernel(const int* rows, int count, const double* v, double* buf) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < count) buf[t] = v[rows[t]];
}
__global__ void scatter_rows_kernel(const int* rows, int count, const double* buf, double* v) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < count) v[rows[t]] = buf[t];
}

void launch_gather_rows(const int* rows, int count, const double* v, double* buf,
                        cudaStream_t st) {
    if (count > 0) gather_rows_kernel<<<blocks_for(count), kBlock, 0, st>>>(rows, count, v, buf);
}
void launch_scatter_rows(const int* rows, int count, const double* buf, double* v,
                         cudaStream_t st) {
    if (count > 0) scatter_rows_kernel<<<blocks_for(count), kBlock, 0, st>>>(rows, count, buf, v);
}

void launch_rowmax(const double* v, int n, unsigned long long* dst, cudaStream_t st) {
    cudaMemsetAsync(dst, 0, sizeof(unsigned long long), st);
    if (n > 0) rowmax_kernel<<<64, kBlock, 0, st>>>(v, n, dst);
}

void launch_loop_start(LoopCtl* ctl, DevScalars* sc, cudaStream_t st) {
    loop_start_kernel<<<1, 1, 0, st>>>(ctl, sc);
}

void launch_loop_control(LoopCtl* ctl, LoopRec* rec, DevScalars* sc, cudaStream_t st) {
    loop_control_kernel<<<1, 1, 0, st>>>(ctl, rec, sc);
}

void launch_reset_scalars(DevScalars* sc, cudaStream_t st) {
    reset_scalars_kernel<<<1, 1, 0, st>>>(sc);
}

}  // namespace ga
