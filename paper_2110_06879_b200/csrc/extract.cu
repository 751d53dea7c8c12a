// extract.cu — solution extraction and quality metrics on the device
// (reference proj/src/driver.cpp:65-138).
//
// Two kernels after the last iteration of a solve:
//  * ext_branch_kernel, one thread per branch: the solution voltages of the
//    two ends (vm = sqrt(max(0, w)), va = theta, driver.cpp:77-78) and the
//    four flows through the pinned sincos (netdata.cpp:33-45), written as the
//    report's AoS flow array; rate-limited branches whose apparent-power
//    flow may reach the rate go on a candidate list (below);
//  * ext_bus_kernel, one thread per bus and per generator: vm / va, the
//    power-balance residuals pbal / qbal accumulated in the reference's
//    order (driver.cpp:93-117: load and shunt, then generators in index
//    order, then branch ends in branch order — exactly the bus's segment of
//    the row storage, device.hpp), the voltage / generator bound violations,
//    and the dispatch in generator order.
// The infinity norms and bound maxima are order-free maxima (NaN skipped as
// std::max does), reduced as IEEE bit patterns of max(0, v): bit-identical
// to the reference.  Two pieces stay on the host, both exact: the objective
// (a sequential sum over generators, driver.cpp:97-98) and the line-limit
// violation, which the reference computes with glibc's hypot — the device
// only lists the branches whose flow magnitude is within 1e-12 relative of
// the rate (device hypot is within a few ulp of glibc's), and the host
// evaluates glibc hypot on exactly those; any other branch has
// hypot - rate < 0 and cannot raise max(0, ...).
#include "branch_problem.cuh"
#include "device.hpp"
#include "ga_math.h"

namespace ga {

namespace {

constexpr int kExtBlock = 256;
constexpr double kTwoPi = 6.283185307179586;  // 2.0 * std::numbers::pi
constexpr double kCandRel = 1e-12;

__device__ __forceinline__ double vmag(double w) { return sqrt(smax(0.0, w)); }

// max over the block of non-negative doubles (fmax skips NaN), one atomicMax
// of the bit pattern per block
__device__ __forceinline__ void block_max_bits(double v, unsigned long long* dst) {
    __shared__ double red[kExtBlock / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_down_sync(0xffffffffu, v, o));
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) red[wid] = v;
    __syncthreads();
    if (wid == 0) {
        double t = lane < (int)(blockDim.x >> 5) ? red[lane] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t = fmax(t, __shfl_down_sync(0xffffffffu, t, o));
        if (lane == 0 && t > 0.0) atomicMax(dst, static_cast<unsigned long long>(__double_as_longlong(t)));
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kExtBlock) ext_branch_kernel(DevNet n, DevState s, DevExtract e) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= n.nl) return;
    const int from = n.br_from[b], to = n.br_to[b];
    double f[4];
    bp::branch_flows(bp::YArr{n.br_y, n.nl, b}, vmag(s.bus_w[from]), vmag(s.bus_w[to]),
                     s.bus_theta[from], s.bus_theta[to], f);
    double2* out = reinterpret_cast<double2*>(e.flows) + 2 * static_cast<size_t>(b);
    out[0] = make_double2(f[0], f[1]);
    out[1] = make_double2(f[2], f[3]);
    const double rate = n.br_rate[b];
    if (rate > 0.0) {
        const double h = fmax(hypot(f[0], f[1]), hypot(f[2], f[3]));
        if (!(h < rate * (1.0 - kCandRel))) e.cand[atomicAdd(&e.sc->n_cand, 1)] = b;  // NaN included
    }
}

__global__ void __launch_bounds__(kExtBlock) ext_bus_kernel(DevNet n, DevState s, DevExtract e) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    double bal = 0.0, bound = 0.0;
    if (t < n.nb) {
        const int i = t;
        const double vm = vmag(s.bus_w[i]);
        const double va = s.bus_theta[i];
        e.vm[i] = vm;
        e.va[i] = va;
        const double w = vm * vm;
        double pb = -n.b_pd[i] - n.b_gs[i] * w;
        double qb = -n.b_qd[i] + n.b_bs[i] * w;
        // the bus's segment (device.hpp): generator (p, q) pairs in generator
        // order, then one quad per incident branch end in branch order
        const int* seg = n.bus_seg + 4 * i;
        for (int k = seg[0]; k < seg[1]; k += 2) pb += s.x[k];
        for (int k = seg[0] + 1; k < seg[1]; k += 2) qb += s.x[k];
        for (int k = seg[2]; k < seg[3]; k += 4) {  // pij / pji, branch order
            const int qb2 = n.quad_branch[k >> 2];  // 2 b + side
            pb -= e.flows[4 * static_cast<size_t>(qb2 >> 1) + 2 * (qb2 & 1)];
        }
        for (int k = seg[2]; k < seg[3]; k += 4) {  // qij / qji
            const int qb2 = n.quad_branch[k >> 2];
            qb -= e.flows[4 * static_cast<size_t>(qb2 >> 1) + 2 * (qb2 & 1) + 1];
        }
        bal = fmax(fabs(pb), fabs(qb));
        bound = fmax(fmax(n.b_vmin[i] - vm, vm - n.b_vmax[i]), fabs(va) - kTwoPi);
    }
    if (t < n.ng) {
        const int g = t;
        const double pg = s.x[n.gpos[g]], qg = s.x[n.gpos[g] + 1];
        e.gen_pq[2 * g] = pg;
        e.gen_pq[2 * g + 1] = qg;
        const double gv = fmax(fmax(n.g_pmin[g] - pg, pg - n.g_pmax[g]),
                               fmax(n.g_qmin[g] - qg, qg - n.g_qmax[g]));
        bound = fmax(bound, gv);
    }
    block_max_bits(fmax(bal, 0.0), &e.sc->balance_inf);
    block_max_bits(fmax(bound, 0.0), &e.sc->bound_violation);
}

}  // namespace

void launch_extract(const DevNet& n, const DevState& s, const DevExtract& e, cudaStream_t st) {
    cudaMemsetAsync(e.sc, 0, sizeof(ExtractScalars), st);
    if (n.nl > 0) ext_branch_kernel<<<(n.nl + kExtBlock - 1) / kExtBlock, kExtBlock, 0, st>>>(n, s, e);
    const int cnt = n.nb > n.ng ? n.nb : n.ng;
    if (cnt > 0) ext_bus_kernel<<<(cnt + kExtBlock - 1) / kExtBlock, kExtBlock, 0, st>>>(n, s, e);
}

}  // namespace ga
