// session.cpp — device residency of one network + AdmmState and the phase
// sequence of one inner iteration (proj/src/driver.cpp:155-186).
#include <algorithm>
#include <deque>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "ga_math.h"
#include "solver.hpp"

namespace ga {

namespace {

void check(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

// Process-wide pinned slots for the per-iteration scalar readback: a pinned
// allocation per session costs milliseconds, a slot costs nothing.
std::mutex g_pinned_mu;
std::vector<void*> g_pinned_free;
constexpr size_t kPinnedSlot = 256;

void* pinned_slot_acquire() {
    std::lock_guard<std::mutex> lk(g_pinned_mu);
    if (g_pinned_free.empty()) {
        char* blk = nullptr;
        check(cudaMallocHost(&blk, 64 * kPinnedSlot), "cudaMallocHost");
        for (int k = 0; k < 64; ++k) g_pinned_free.push_back(blk + k * kPinnedSlot);
    }
    void* p = g_pinned_free.back();
    g_pinned_free.pop_back();
    return p;
}

void pinned_slot_release(void* p) {
    std::lock_guard<std::mutex> lk(g_pinned_mu);
    g_pinned_free.push_back(p);
}

// The device's default memory pool keeps freed arenas (no release threshold),
// so a new session / solve / tracking period reuses mapped memory instead of
// paying cudaMalloc + cudaFree of ~100 MB.
void retain_pool(int device) {
    static std::mutex mu;
    static std::vector<int> done;
    std::lock_guard<std::mutex> lk(mu);
    for (int d : done)
        if (d == device) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        unsigned long long thr = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    done.push_back(device);
}

double from_bits(unsigned long long b) {
    double v;
    std::memcpy(&v, &b, sizeof v);
    return v;
}

}  // namespace

double SolverConfig::effective_inner_tol(int m) const {
    return inner_tol > 0.0 ? inner_tol : eps * std::sqrt(static_cast<double>(m));
}

Session::Session(const Network& net, const SolverConfig& cfg, const PartPlan* plan)
    : net_(net), cfg_(cfg) {
    if (plan) plan_ = *plan;
    trace_phase("session: network copy");
    check(cudaSetDevice(cfg.device), "cudaSetDevice");
    {
        // the side stream's bus kernel yields the SMs to the tile / solo
        // phases, whose chains bound the iteration (GRIDADMM_BUS_PRIO=0: equal)
        static const bool prio = [] {
            const char* e = std::getenv("GRIDADMM_BUS_PRIO");
            return !e || std::atoi(e) != 0;
        }();
        int least = 0, greatest = 0;
        if (prio) cudaDeviceGetStreamPriorityRange(&least, &greatest);
        check(cudaStreamCreateWithPriority(&stream_, cudaStreamNonBlocking, greatest), "cudaStreamCreate");
        check(cudaStreamCreateWithPriority(&side_, cudaStreamNonBlocking, least), "cudaStreamCreate");
    }
    check(cudaEventCreateWithFlags(&fork_, cudaEventDisableTiming), "cudaEventCreate");
    check(cudaEventCreateWithFlags(&join_, cudaEventDisableTiming), "cudaEventCreate");
    for (auto& e : side_ev_) check(cudaEventCreate(&e), "cudaEventCreate");
    for (auto& e : ev_) check(cudaEventCreate(&e), "cudaEventCreate");
    if (const char* pf = std::getenv("GRIDADMM_PROFILE")) {
        prof_ = std::fopen(pf, "a");
        if (prof_) std::fprintf(prof_, "iter,gen_ms,lane_ms,tile_ms,bus_zy_ms,bus_side_ms,ovf6,ovf4,beta\n");
    }
    trace_phase("session: stream/events");
    try {
        upload_network();  // also places sc_ and red_ in the arena
        trace_phase("session: upload network");
        sc_host_ = static_cast<DevScalars*>(pinned_slot_acquire());
    } catch (...) {
        free_all();
        throw;
    }
    beta_ = cfg.beta0;
}

Session::~Session() { free_all(); }

void Session::free_all() {
    cudaSetDevice(cfg_.device);  // no throw: runs in the destructor
    if (stream_) cudaStreamSynchronize(stream_);
    for (void* p : allocs_) cudaFreeAsync(p, stream_);  // back to the device pool
    if (!allocs_.empty() && stream_) cudaStreamSynchronize(stream_);
    allocs_.clear();
    if (sc_host_) pinned_slot_release(sc_host_);
    if (ctl_host_) pinned_slot_release(ctl_host_);
    ctl_host_ = nullptr;
    if (rec_host_) cudaFreeHost(rec_host_);
    rec_host_ = nullptr;
    if (graph_) cudaGraphExecDestroy(graph_);
    graph_ = nullptr;
    ctl_ = nullptr;
    rec_ = nullptr;
    rec_cap_ = 0;
    if (flush_buf_) cudaFree(flush_buf_);
    flush_buf_ = nullptr;
    sc_ = nullptr;
    red_ = nullptr;
    sc_host_ = nullptr;
    for (auto& e : ev_)
        if (e) cudaEventDestroy(e);
    if (prof_) std::fclose(prof_);
    prof_ = nullptr;
    for (auto& e : side_ev_)
        if (e) cudaEventDestroy(e);
    if (fork_) cudaEventDestroy(fork_);
    if (join_) cudaEventDestroy(join_);
    fork_ = join_ = nullptr;
    if (side_) cudaStreamDestroy(side_);
    side_ = nullptr;
    if (stream_) cudaStreamDestroy(stream_);
    stream_ = nullptr;
}

void Session::enqueue_iteration(const BranchCfg& bc, LoopCtl* gate, cudaEvent_t mid,
                                cudaEvent_t before_bus) {
    static const bool overlap = [] {
        const char* e = std::getenv("GRIDADMM_BUS_OVERLAP");
        return !e || std::atoi(e) != 0;
    }();
    side_timed_ = false;
    if (!overlap || dn_.nl <= 0 || plan_.parts > 1) {
        launch_branches(dn_, ds_, bc, sc_, stream_, mid);
        if (before_bus) cudaEventRecord(before_bus, stream_);
        launch_bus_zy(dn_, ds_, beta_, sc_, stream_, gate);
        return;
    }
    unsigned char* defer = bus_defer_flags(dn_, ds_);
    check(cudaMemsetAsync(defer, 0, static_cast<size_t>(dn_.nb), stream_), "defer reset");
    launch_branches(dn_, ds_, bc, sc_, stream_, mid, [&] {
        cudaEventRecord(fork_, stream_);
        cudaStreamWaitEvent(side_, fork_, 0);
        if (before_bus) cudaEventRecord(side_ev_[0], side_);
        launch_bus_zy(dn_, ds_, beta_, sc_, side_, gate, defer, 1);
        if (before_bus) cudaEventRecord(side_ev_[1], side_);
        cudaEventRecord(join_, side_);
    });
    cudaStreamWaitEvent(stream_, join_, 0);
    if (before_bus) cudaEventRecord(before_bus, stream_);
    launch_bus_zy(dn_, ds_, beta_, sc_, stream_, gate, defer, 2);
    side_timed_ = before_bus != nullptr;
}

void Session::upload_network() {
    const int nb = net_.nb(), ng = net_.ng(), nl = net_.nl(), m = net_.m();
    dn_.nb = nb;
    dn_.ng = ng;
    dn_.nl = nl;
    dn_.m = m;
    dn_.ref_bus = net_.ref_bus;
    // One device arena for the whole network + state (one cudaMalloc instead
    // of ~40); the host arrays are copied after the arena exists.
    struct Req {
        void** slot;
        size_t bytes;
    };
    struct Put {
        void** slot;
        const void* src;
        size_t bytes;
    };
    std::vector<Req> reqs;
    std::vector<Put> puts;
    auto alloc = [&](auto*& p, size_t count) {
        using T = std::remove_reference_t<decltype(*p)>;
        reqs.push_back({reinterpret_cast<void**>(&p), std::max<size_t>(count, 1) * sizeof(T)});
    };
    auto put = [&](auto*& dst, const auto& host) {
        if (!host.empty())
            puts.push_back({reinterpret_cast<void**>(&dst), host.data(), host.size() * sizeof(host[0])});
    };
    std::vector<std::vector<int>> keep;  // host copies that must outlive the uploads
    std::deque<std::vector<double>> keepd;
    auto put_copy = [&](int*& dst, std::vector<int>&& v) {
        keep.push_back(std::move(v));
        put(dst, keep.back());
    };
    // generators
    std::vector<double> pmin(ng), pmax(ng), qmin(ng), qmax(ng), c2(ng), c1(ng);
    for (int g = 0; g < ng; ++g) {
        const Gen& x = net_.gens[g];
        pmin[g] = x.pmin; pmax[g] = x.pmax; qmin[g] = x.qmin; qmax[g] = x.qmax;
        c2[g] = x.c2; c1[g] = x.c1;
    }
    alloc(dn_.g_pmin, ng); put(dn_.g_pmin, pmin);
    alloc(dn_.g_pmax, ng); put(dn_.g_pmax, pmax);
    alloc(dn_.g_qmin, ng); put(dn_.g_qmin, qmin);
    alloc(dn_.g_qmax, ng); put(dn_.g_qmax, qmax);
    alloc(dn_.g_c2, ng); put(dn_.g_c2, c2);
    alloc(dn_.g_c1, ng); put(dn_.g_c1, c1);
    // branches
    std::vector<int> from(nl), to(nl), lim, unl;
    std::vector<double> yc(8 * static_cast<size_t>(nl)), rate(nl);
    for (int b = 0; b < nl; ++b) {
        const Line& l = net_.lines[b];
        from[b] = l.from;
        to[b] = l.to;
        rate[b] = l.rate;
        for (int k = 0; k < 8; ++k) yc[static_cast<size_t>(k) * nl + b] = l.y.c[k];
        (l.limited() ? lim : unl).push_back(b);
    }
    if (plan_.parts > 1) {  // this part solves only its own branches
        lim = plan_.lim;
        unl = plan_.unl;
    }
    alloc(dn_.br_from, nl); put(dn_.br_from, from);
    alloc(dn_.br_to, nl); put(dn_.br_to, to);
    alloc(dn_.br_y, 8 * static_cast<size_t>(nl)); put(dn_.br_y, yc);
    alloc(dn_.br_rate, nl); put(dn_.br_rate, rate);
    alloc(dn_.lim_list, lim.size()); put(dn_.lim_list, lim);
    alloc(dn_.unl_list, unl.size()); put(dn_.unl_list, unl);
    dn_.n_lim = static_cast<int>(lim.size());
    dn_.n_unl = static_cast<int>(unl.size());
    // buses
    std::vector<double> pd(nb), qd(nb), gs(nb), bs(nb), vmin(nb), vmax(nb);
    for (int i = 0; i < nb; ++i) {
        const Bus& b = net_.buses[i];
        pd[i] = b.pd; qd[i] = b.qd; gs[i] = b.gs; bs[i] = b.bs; vmin[i] = b.vmin; vmax[i] = b.vmax;
    }
    alloc(dn_.b_pd, nb); put(dn_.b_pd, pd);
    alloc(dn_.b_qd, nb); put(dn_.b_qd, qd);
    alloc(dn_.b_gs, nb); put(dn_.b_gs, gs);
    alloc(dn_.b_bs, nb); put(dn_.b_bs, bs);
    alloc(dn_.b_vmin, nb); put(dn_.b_vmin, vmin);
    alloc(dn_.b_vmax, nb); put(dn_.b_vmax, vmax);
    trace_phase("upload: host SoA");
    layout_ = build_row_layout(net_);
    trace_phase("upload: row layout");
    const int mpad = layout_.mpad;
    dn_.mpad = mpad;
    {
        std::vector<int> seg(4 * static_cast<size_t>(nb));
        std::vector<int> ngen(nb, 0);
        for (int g = 0; g < ng; ++g) ++ngen[net_.gens[g].bus];
        for (int i = 0; i < nb; ++i) {
            seg[4 * i] = layout_.seg[3 * i];
            seg[4 * i + 1] = layout_.seg[3 * i] + 2 * ngen[i];
            seg[4 * i + 2] = layout_.seg[3 * i + 1];
            seg[4 * i + 3] = layout_.seg[3 * i + 2];
        }
        alloc(dn_.bus_seg, seg.size()); put_copy(dn_.bus_seg, std::move(seg));
    }
    alloc(dn_.gpos, layout_.gpos.size()); put(dn_.gpos, layout_.gpos);
    {
        const size_t np = static_cast<size_t>(mpad) / 2 + 1;
        std::vector<double>* pr[6];
        for (auto& p : pr) {
            keepd.emplace_back(np, 0.0);
            p = &keepd.back();
        }
        for (int g = 0; g < ng; ++g) {
            const size_t h = static_cast<size_t>(layout_.gpos[g]) / 2;
            (*pr[0])[h] = c1[g]; (*pr[1])[h] = c2[g]; (*pr[2])[h] = pmin[g];
            (*pr[3])[h] = pmax[g]; (*pr[4])[h] = qmin[g]; (*pr[5])[h] = qmax[g];
        }
        double** dst[6] = {&dn_.pr_c1, &dn_.pr_c2, &dn_.pr_pmin, &dn_.pr_pmax, &dn_.pr_qmin,
                           &dn_.pr_qmax};
        for (int k = 0; k < 6; ++k) {
            alloc(*dst[k], np);
            put(*dst[k], *pr[k]);
        }
    }
    alloc(dn_.qpos, layout_.qpos.size()); put(dn_.qpos, layout_.qpos);
    alloc(dn_.quad_branch, layout_.quad_branch.size()); put(dn_.quad_branch, layout_.quad_branch);
    alloc(dn_.rid, layout_.rid.size()); put(dn_.rid, layout_.rid);
    // state
    alloc(ds_.x, mpad); alloc(ds_.xbar, mpad); alloc(ds_.z, mpad); alloc(ds_.y, mpad);
    alloc(ds_.lambda, mpad); alloc(ds_.rho, mpad);
    alloc(ds_.bus_w, nb); alloc(ds_.bus_theta, nb);
    alloc(ds_.bp, 6 * static_cast<size_t>(nl));
    alloc(ds_.lt_ij, nl); alloc(ds_.lt_ji, nl); alloc(ds_.rho_t, nl);
    alloc(ds_.br_cost, nl);
    alloc(ds_.branch_ws, branch_workspace_ints(dn_));
    alloc(ds_.mig_x, 6 * static_cast<size_t>(nl));
    alloc(ds_.mig_f, nl);
    alloc(ds_.mig_delta, nl);
    alloc(ds_.mig_prev_res, nl);
    alloc(ds_.mig_iter, nl);
    alloc(ds_.mig_al, nl);
    alloc(ds_.mig_cost, nl);
    if (plan_.parts > 1) {
        alloc(dn_.own_gens, plan_.gens.size()); put(dn_.own_gens, plan_.gens);
        alloc(dn_.own_buses, plan_.buses.size()); put(dn_.own_buses, plan_.buses);
        // plan rows are reference row ids; the device works on positions
        auto to_pos = [&](const std::vector<int>& rows) {
            std::vector<int> p(rows.size());
            for (size_t k = 0; k < rows.size(); ++k) p[k] = layout_.pos[rows[k]];
            return p;
        };
        alloc(dn_.own_rows, plan_.rows.size()); put_copy(dn_.own_rows, to_pos(plan_.rows));
        dn_.n_own_gens = static_cast<int>(plan_.gens.size());
        dn_.n_own_buses = static_cast<int>(plan_.buses.size());
        dn_.n_own_rows = static_cast<int>(plan_.rows.size());
        d_send_.assign(plan_.parts, nullptr);
        d_recv_.assign(plan_.parts, nullptr);
        for (int q = 0; q < plan_.parts; ++q) {
            alloc(d_send_[q], plan_.send_x[q].size()); put_copy(d_send_[q], to_pos(plan_.send_x[q]));
            alloc(d_recv_[q], plan_.recv_x[q].size()); put_copy(d_recv_[q], to_pos(plan_.recv_x[q]));
        }
    }
    if (plan_.parts <= 1) {
        alloc(ext_.flows, 4 * static_cast<size_t>(nl));
        alloc(ext_.vm, nb);
        alloc(ext_.va, nb);
        alloc(ext_.cand, nl);
        alloc(ext_.gen_pq, 2 * static_cast<size_t>(ng));
        alloc(ext_.sc, 1);
    }
    alloc(sc_, 1);
    alloc(red_, 1);
    size_t total = 0;
    for (const Req& r : reqs) total += (r.bytes + 255) & ~size_t(255);
    void* arena = nullptr;
    retain_pool(cfg_.device);
    check(cudaMallocAsync(&arena, total, stream_), "cudaMallocAsync arena");
    allocs_.push_back(arena);
    size_t off = 0;
    for (const Req& r : reqs) {
        *r.slot = static_cast<char*>(arena) + off;
        off += (r.bytes + 255) & ~size_t(255);
    }
    trace_phase("upload: arena");
    for (const Put& p : puts)
        check(cudaMemcpyAsync(*p.slot, p.src, p.bytes, cudaMemcpyHostToDevice, stream_), "H2D");
    check(cudaMemsetAsync(ds_.br_cost, 0, std::max(nl, 1) * sizeof(int), stream_), "cudaMemset cost");
    check(cudaMemsetAsync(sc_, 0, sizeof(DevScalars), stream_), "cudaMemset scalars");
    check(cudaStreamSynchronize(stream_), "sync");
}

// make_state + cold_start (decomp.cpp:37-57, driver.cpp:26-63) on the device:
// one kernel over rows / branches / generators / buses (branch.cu), the same
// expressions as the reference, so no state upload is needed.
void Session::cold_start() {
    check(cudaSetDevice(cfg_.device), "cudaSetDevice");
    launch_cold_start(dn_, ds_, cfg_.rho_pq, cfg_.rho_va, cfg_.limit_tighten, stream_);
    check(cudaGetLastError(), "cold start launch");
    check(cudaStreamSynchronize(stream_), "sync");
    beta_ = cfg_.beta0;
}

void Session::upload_state(const HostState& s) {
    use_device();
    const size_t nl = static_cast<size_t>(dn_.nl);
    auto put = [&](double* dst, const std::vector<double>& v) {
        if (!v.empty())
            check(cudaMemcpyAsync(dst, v.data(), v.size() * sizeof(double), cudaMemcpyHostToDevice,
                                  stream_),
                  "upload_state");
    };
    // row vectors: reference row order (host) -> storage positions (device)
    std::vector<std::vector<double>> rowbuf;
    auto put_rows = [&](double* dst, const std::vector<double>& v) {
        if (v.empty()) return;
        if (v.size() != layout_.pos.size()) throw std::invalid_argument("state row vector size");
        rowbuf.emplace_back(static_cast<size_t>(dn_.mpad), 0.0);
        std::vector<double>& p = rowbuf.back();
        for (size_t r = 0; r < v.size(); ++r) p[layout_.pos[r]] = v[r];
        put(dst, p);
    };
    rowbuf.reserve(6);
    put_rows(ds_.x, s.x); put_rows(ds_.xbar, s.xbar); put_rows(ds_.z, s.z); put_rows(ds_.y, s.y);
    put_rows(ds_.lambda, s.lambda); put_rows(ds_.rho, s.rho);
    put(ds_.bus_w, s.bus_w); put(ds_.bus_theta, s.bus_theta);
    if (!s.bp.empty()) {  // branch-major (host) -> component-major (device)
        std::vector<double> t(6 * nl);
        for (size_t b = 0; b < nl; ++b)
            for (int k = 0; k < 6; ++k) t[k * nl + b] = s.bp[6 * b + k];
        check(cudaMemcpyAsync(ds_.bp, t.data(), t.size() * sizeof(double), cudaMemcpyHostToDevice,
                              stream_),
              "upload bp");
        check(cudaStreamSynchronize(stream_), "sync");
    }
    put(ds_.lt_ij, s.lt_ij); put(ds_.lt_ji, s.lt_ji); put(ds_.rho_t, s.rho_t);
    beta_ = s.beta;
    check(cudaStreamSynchronize(stream_), "sync");
}

void Session::download_state(HostState& s) const {
    use_device();
    const int m = dn_.m, nb = dn_.nb;
    const size_t nl = static_cast<size_t>(dn_.nl);
    auto get = [&](std::vector<double>& v, const double* src, size_t n) {
        v.resize(n);
        if (n) check(cudaMemcpyAsync(v.data(), src, n * sizeof(double), cudaMemcpyDeviceToHost, stream_),
                     "download_state");
    };
    std::vector<double> rows[6];
    const double* srcs[6] = {ds_.x, ds_.xbar, ds_.z, ds_.y, ds_.lambda, ds_.rho};
    for (int k = 0; k < 6; ++k) get(rows[k], srcs[k], static_cast<size_t>(dn_.mpad));
    get(s.bus_w, ds_.bus_w, nb); get(s.bus_theta, ds_.bus_theta, nb);
    std::vector<double> t;
    get(t, ds_.bp, 6 * nl);
    get(s.lt_ij, ds_.lt_ij, nl); get(s.lt_ji, ds_.lt_ji, nl); get(s.rho_t, ds_.rho_t, nl);
    check(cudaStreamSynchronize(stream_), "sync");
    std::vector<double>* dst[6] = {&s.x, &s.xbar, &s.z, &s.y, &s.lambda, &s.rho};
    for (int k = 0; k < 6; ++k) {  // storage positions -> reference row order
        dst[k]->resize(m);
        for (int r = 0; r < m; ++r) (*dst[k])[r] = rows[k][layout_.pos[r]];
    }
    s.bp.resize(6 * nl);
    for (size_t b = 0; b < nl; ++b)
        for (int k = 0; k < 6; ++k) s.bp[6 * b + k] = t[k * nl + b];
    s.beta = beta_;
}

void Session::download_solution_inputs(std::vector<double>& gen_rows, std::vector<double>& w,
                                       std::vector<double>& th) const {
    use_device();
    gen_rows.resize(2 * static_cast<size_t>(dn_.ng));
    w.resize(dn_.nb);
    th.resize(dn_.nb);
    std::vector<double> xall(static_cast<size_t>(dn_.mpad));
    if (!xall.empty())
        check(cudaMemcpyAsync(xall.data(), ds_.x, xall.size() * sizeof(double),
                              cudaMemcpyDeviceToHost, stream_), "D2H");
    if (dn_.nb) {
        check(cudaMemcpyAsync(w.data(), ds_.bus_w, w.size() * sizeof(double), cudaMemcpyDeviceToHost,
                              stream_), "D2H");
        check(cudaMemcpyAsync(th.data(), ds_.bus_theta, th.size() * sizeof(double),
                              cudaMemcpyDeviceToHost, stream_), "D2H");
    }
    check(cudaStreamSynchronize(stream_), "sync");
    for (int g = 0; g < dn_.ng; ++g) {  // generator rows in reference order
        gen_rows[2 * static_cast<size_t>(g)] = xall[layout_.gpos[g]];
        gen_rows[2 * static_cast<size_t>(g) + 1] = xall[layout_.gpos[g] + 1];
    }
}

BranchCfg branch_cfg(const SolverConfig& c);

// The graph path of Algorithm 1's inner loop (driver.cpp:155-220).  One
// captured batch = kGraphIters iterations, each: branch kernels, the fused
// bus kernel, the control kernel; every kernel is gated on ctl->stop, so the
// iterations after a stop are empty launches and the state is exactly that
// of the stopping iteration.  The host reads the control block and the new
// records once per batch instead of the norms once per iteration.
bool Session::inner_loop(const SolverConfig& cfg, int outer, double rho_max, double inner_tol,
                         double elapsed_s, SolveReport& rep, int* stop, double* last_z) {
    if (plan_.parts > 1 || prof_ || dn_.nl <= 0) return false;
    use_device();
    if (!ctl_) {
        check(cudaMallocAsync(reinterpret_cast<void**>(&ctl_), sizeof(LoopCtl), stream_), "ctl alloc");
        allocs_.push_back(ctl_);
        ctl_host_ = static_cast<LoopCtl*>(pinned_slot_acquire());
        check(cudaMallocHost(reinterpret_cast<void**>(&rec_host_), kGraphIters * sizeof(LoopRec)),
              "cudaMallocHost records");
    }
    if (rec_cap_ < cfg.max_inner) {
        check(cudaMallocAsync(reinterpret_cast<void**>(&rec_), cfg.max_inner * sizeof(LoopRec), stream_),
              "records alloc");
        allocs_.push_back(rec_);
        rec_cap_ = cfg.max_inner;
        if (graph_) cudaGraphExecDestroy(graph_);  // the control kernels hold the old pointer
        graph_ = nullptr;
    }
    if (!graph_) {
        BranchCfg bc = branch_cfg(cfg_);
        bc.gate = ctl_;
        cudaGraph_t g = nullptr;
        prepare_branch_launch();
        check(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal), "capture begin");
        for (int k = 0; k < kGraphIters; ++k) {
            enqueue_iteration(bc, ctl_, nullptr, nullptr);
            launch_loop_control(ctl_, rec_, sc_, stream_);
        }
        check(cudaStreamEndCapture(stream_, &g), "capture end");
        check(cudaGraphInstantiate(&graph_, g, 0), "graph instantiate");
        cudaGraphDestroy(g);
    }
    LoopCtl& h = *ctl_host_;
    std::memset(&h, 0, sizeof h);
    h.inner_tol = inner_tol;
    h.eps = cfg.eps;
    h.diverge = cfg.divergence_threshold;
    h.rho_max = rho_max;
    h.beta = beta_;
    h.outer = outer;
    h.max_inner = cfg.max_inner;
    check(cudaMemcpyAsync(ctl_, &h, sizeof h, cudaMemcpyHostToDevice, stream_), "ctl upload");
    launch_loop_start(ctl_, sc_, stream_);
    check(cudaGetLastError(), "loop start");
    int done = 0;
    unsigned long long t_start = 0;
    for (;;) {
        check(cudaGraphLaunch(graph_, stream_), "graph launch");
        const int window = std::min(kGraphIters, cfg.max_inner - done);
        check(cudaMemcpyAsync(ctl_host_, ctl_, sizeof(LoopCtl), cudaMemcpyDeviceToHost, stream_), "D2H");
        if (window > 0)
            check(cudaMemcpyAsync(rec_host_, rec_ + done, window * sizeof(LoopRec),
                                  cudaMemcpyDeviceToHost, stream_), "D2H");
        check(cudaStreamSynchronize(stream_), "graph sync");
        if (!t_start) t_start = h.t_start;
        const int n = h.inner;
        for (int i = done; i < n; ++i) {
            const LoopRec& r = rec_host_[i - done];
            rep.series.push_back({r.outer, r.inner, r.primal, r.dual, r.z,
                                  elapsed_s + 1e-9 * static_cast<double>(r.t_ns - t_start)});
        }
        done = n;
        if (h.stop != kLoopRunning) break;
    }
    if (h.stop == kLoopSingular) {
        const int id = net_.buses[h.singular].id;
        throw SingularBusError(id, "isolated bus " + std::to_string(id) + ": singular balance system");
    }
    rep.inner_iterations += done;
    rep.branch_solve_failures += static_cast<int>(h.failures);
    rep.phase_times.x_s += 1e-9 * static_cast<double>(h.x_ns);
    rep.phase_times.xbar_s += 1e-9 * static_cast<double>(h.xbar_ns);
    *stop = h.stop;
    *last_z = h.last_z;
    return true;
}

bool Session::extract_on_device(Solution& sol, QualityMetrics& q) {
    if (plan_.parts > 1 || !ext_.sc) return false;
    use_device();
    const int ng = dn_.ng, nb = dn_.nb, nl = dn_.nl;
    launch_extract(dn_, ds_, ext_, stream_);
    check(cudaGetLastError(), "extract launch");
    std::vector<double> gen_rows(2 * static_cast<size_t>(ng));
    sol.vm.resize(nb);
    sol.va.resize(nb);
    sol.flows.resize(4 * static_cast<size_t>(nl));
    ExtractScalars es{};
    auto d2h = [&](void* dst, const void* src, size_t bytes) {
        if (bytes) check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, stream_), "D2H");
    };
    d2h(gen_rows.data(), ext_.gen_pq, gen_rows.size() * sizeof(double));
    d2h(sol.vm.data(), ext_.vm, nb * sizeof(double));
    d2h(sol.va.data(), ext_.va, nb * sizeof(double));
    d2h(sol.flows.data(), ext_.flows, sol.flows.size() * sizeof(double));
    d2h(&es, ext_.sc, sizeof es);
    check(cudaStreamSynchronize(stream_), "extract sync");
    std::vector<int> cand(es.n_cand);
    d2h(cand.data(), ext_.cand, cand.size() * sizeof(int));
    check(cudaStreamSynchronize(stream_), "extract sync");
    sol.pg.resize(ng);
    sol.qg.resize(ng);
    for (int g = 0; g < ng; ++g) {
        sol.pg[g] = gen_rows[2 * static_cast<size_t>(g)];
        sol.qg[g] = gen_rows[2 * static_cast<size_t>(g) + 1];
    }
    finish_metrics(net_, sol, cand, from_bits(es.balance_inf), from_bits(es.bound_violation), q);
    return true;
}

void Session::set_loads(const std::vector<double>& pd, const std::vector<double>& qd) {
    use_device();
    check(cudaMemcpyAsync(dn_.b_pd, pd.data(), pd.size() * sizeof(double), cudaMemcpyHostToDevice,
                          stream_), "set_loads");
    check(cudaMemcpyAsync(dn_.b_qd, qd.data(), qd.size() * sizeof(double), cudaMemcpyHostToDevice,
                          stream_), "set_loads");
    check(cudaStreamSynchronize(stream_), "sync");
    // the host copy is the period network the quality metrics are evaluated
    // on (tracking.cpp:47 scaled_network -> driver.cpp:89 evaluate_solution)
    for (size_t i = 0; i < pd.size() && i < net_.buses.size(); ++i) {
        net_.buses[i].pd = pd[i];
        net_.buses[i].qd = qd[i];
    }
}

void Session::set_gen_p_bounds(const std::vector<double>& pmin, const std::vector<double>& pmax) {
    use_device();
    check(cudaMemcpyAsync(dn_.g_pmin, pmin.data(), pmin.size() * sizeof(double),
                          cudaMemcpyHostToDevice, stream_), "set_gen_p_bounds");
    check(cudaMemcpyAsync(dn_.g_pmax, pmax.data(), pmax.size() * sizeof(double),
                          cudaMemcpyHostToDevice, stream_), "set_gen_p_bounds");
    {  // and the storage-order copy the bus kernel reads
        const size_t np = static_cast<size_t>(dn_.mpad) / 2 + 1;
        std::vector<double> lo(np, 0.0), hi(np, 0.0);
        for (size_t g = 0; g < pmin.size(); ++g) {
            const size_t h = static_cast<size_t>(layout_.gpos[g]) / 2;
            lo[h] = pmin[g];
            hi[h] = pmax[g];
        }
        check(cudaMemcpyAsync(dn_.pr_pmin, lo.data(), np * sizeof(double), cudaMemcpyHostToDevice,
                              stream_), "set_gen_p_bounds");
        check(cudaMemcpyAsync(dn_.pr_pmax, hi.data(), np * sizeof(double), cudaMemcpyHostToDevice,
                              stream_), "set_gen_p_bounds");
        check(cudaStreamSynchronize(stream_), "sync");
    }
    check(cudaStreamSynchronize(stream_), "sync");
    for (size_t g = 0; g < pmin.size() && g < net_.gens.size(); ++g) {  // ramp window
        net_.gens[g].pmin = pmin[g];
        net_.gens[g].pmax = pmax[g];
    }
}

void Session::clamp_gen_p() {
    use_device();
    launch_clamp_gen_p(dn_, ds_, stream_);
    check(cudaGetLastError(), "clamp_gen_p");
}

BranchCfg branch_cfg(const SolverConfig& c) {
    BranchCfg b = c.tron;
    b.limit_tighten = c.limit_tighten;
    // Scheduling knob only (results are schedule-independent): TRON steps a
    // branch may take in the lane phase before moving to the tile phase.
    static const int budget = [] {
        const char* e = std::getenv("GRIDADMM_LANE_BUDGET");
        return e ? std::atoi(e) : -1;
    }();
    if (budget >= 1) b.lane_budget = budget;
    static const int tile_budget = [] {
        const char* e = std::getenv("GRIDADMM_TILE_BUDGET");
        return e ? std::atoi(e) : -1;
    }();
    if (tile_budget >= 0) b.tile_budget = tile_budget;
    static const int tail_num = [] {
        const char* e = std::getenv("GRIDADMM_TAIL_NUM");
        return e ? std::atoi(e) : -1;
    }();
    if (tail_num >= 0) b.tail_num = tail_num;
    static const int lane_cap = [] {
        const char* e = std::getenv("GRIDADMM_LANE_CAP");
        return e ? std::atoi(e) : -1;
    }();
    if (lane_cap >= 1) b.lane_cap = lane_cap;
    if (b.lane_cap < b.lane_budget) b.lane_cap = b.lane_budget;
    return b;
}

long Session::run_phase(int phase, double z_inf, double prev_z_inf) {
    use_device();
    long ret = 0;
    launch_reset_scalars(sc_, stream_);
    switch (phase) {
        case 0: launch_generators(dn_, ds_, stream_); break;
        case 1: launch_branches(dn_, ds_, branch_cfg(cfg_), sc_, stream_); break;
        case 2: launch_buses(dn_, ds_, sc_, stream_); break;
        case 3: launch_z_only(dn_, ds_, beta_, stream_); break;
        case 4: launch_y_only(dn_, ds_, stream_); break;
        case 5:
            launch_outer(dn_, ds_, beta_, cfg_.lambda_min, cfg_.lambda_max, stream_);
            // beta schedule (kernels.cpp:436-437)
            if (prev_z_inf >= 0.0 && z_inf > cfg_.beta_shrink_trigger * prev_z_inf)
                beta_ = smin(beta_ * cfg_.beta_growth, cfg_.beta_max);
            break;
        default: throw std::invalid_argument("unknown phase");
    }
    check(cudaGetLastError(), "phase launch");
    check(cudaMemcpyAsync(sc_host_, sc_, sizeof(DevScalars), cudaMemcpyDeviceToHost, stream_), "D2H");
    check(cudaStreamSynchronize(stream_), "phase sync");
    if (phase == 1) ret = static_cast<long>(sc_host_->failures);
    if (phase == 2) ret = sc_host_->singular_bus == INT32_MAX ? -1 : sc_host_->singular_bus;
    return ret;
}

int Session::timed_steps(int k, size_t flush_bytes, double* step_ms, double* records) {
    use_device();
    if (flush_bytes > flush_size_) {
        if (flush_buf_) cudaFree(flush_buf_);
        flush_buf_ = nullptr;
        check(cudaMalloc(&flush_buf_, flush_bytes), "cudaMalloc flush");
        flush_size_ = flush_bytes;
    }
    cudaEvent_t a, b;
    check(cudaEventCreate(&a), "event");
    check(cudaEventCreate(&b), "event");
    const double rmax = rho_max();
    int done = 0;
    for (; done < k; ++done) {
        if (flush_bytes) check(cudaMemsetAsync(flush_buf_, done & 0xff, flush_bytes, stream_), "flush");
        cudaEventRecord(a, stream_);
        double nrm[4];
        const int fails = iterate_ev(nrm, nullptr, b);
        float ms = 0.0f;
        cudaEventElapsedTime(&ms, a, b);
        if (step_ms) step_ms[done] = ms;
        if (records) {
            double* r = records + 5 * done;
            r[0] = nrm[0]; r[1] = nrm[1] * rmax; r[2] = nrm[2]; r[3] = nrm[3]; r[4] = fails;
        }
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return done;
}

int Session::iterate_ev(double out[4], PhaseTimes* times, cudaEvent_t end_event) {
    check(cudaSetDevice(cfg_.device), "cudaSetDevice");
    launch_reset_scalars(sc_, stream_);
    cudaEventRecord(ev_[0], stream_);
    // the generator projection runs inside the bus kernel (kernels.cu)
    cudaEventRecord(ev_[1], stream_);
    enqueue_iteration(branch_cfg(cfg_), nullptr, ev_[5], ev_[2]);
    cudaEventRecord(ev_[3], stream_);
    cudaEventRecord(ev_[4], stream_);
    check(cudaGetLastError(), "iteration launch");
    check(cudaMemcpyAsync(sc_host_, sc_, sizeof(DevScalars), cudaMemcpyDeviceToHost, stream_), "D2H");
    int ovf[2] = {0, 0};
    if (prof_ && dn_.nl)
        check(cudaMemcpyAsync(ovf, branch_overflow_counts(dn_, ds_), sizeof ovf,
                              cudaMemcpyDeviceToHost, stream_), "D2H");
    if (end_event) cudaEventRecord(end_event, stream_);
    check(cudaStreamSynchronize(stream_), "iteration sync");
    float ms[4] = {0, 0, 0, 0}, lane = 0.0f, tile = 0.0f;
    for (int k = 0; k < 4; ++k) {
        cudaEventElapsedTime(&ms[k], ev_[k], ev_[k + 1]);
        clocks_[k].ms += ms[k];
        clocks_[k].launches += 1;
    }
    const float bus_after = ms[2];  // the bus launch on the critical path
    float side_ms = 0.0f;
    if (side_timed_) {  // bus kernel = the part beside the tile phase + the rest
        cudaEventElapsedTime(&side_ms, side_ev_[0], side_ev_[1]);
        clocks_[2].ms += side_ms;
        ms[2] += side_ms;
    }
    if (dn_.nl) {
        cudaEventElapsedTime(&lane, ev_[1], ev_[5]);
        cudaEventElapsedTime(&tile, ev_[5], ev_[2]);
    }
    clocks_[4].ms += lane;
    clocks_[4].launches += 1;
    clocks_[5].ms += tile;
    clocks_[5].launches += 1;
    if (prof_)
        std::fprintf(prof_, "%ld,%.4f,%.4f,%.4f,%.4f,%.4f,%d,%d,%.6g\n", ++prof_it_, ms[0], lane,
                     tile, bus_after, side_ms, ovf[0], ovf[1], beta_);
    if (times) {
        times->x_s += (ms[0] + ms[1]) * 1e-3;
        times->xbar_s += ms[2] * 1e-3;
        times->z_s += ms[3] * 1e-3;  // z and y are fused into the bus kernel
    }
    const DevScalars& h = *sc_host_;
    if (h.singular_bus != INT32_MAX) {
        const int i = h.singular_bus;
        const int id = net_.buses[i].id;
        throw SingularBusError(id, "isolated bus " + std::to_string(id) + ": singular balance system");
    }
    out[0] = from_bits(h.primal_inf);
    out[1] = from_bits(h.dual_inf);
    out[2] = from_bits(h.z_inf);
    out[3] = from_bits(h.z_drift);
    return static_cast<int>(h.failures);
}

void Session::enqueue_x_phase() {
    check(cudaSetDevice(cfg_.device), "cudaSetDevice");
    launch_reset_scalars(sc_, stream_);
    launch_branches(dn_, ds_, branch_cfg(cfg_), sc_, stream_);  // generators: in the bus kernel
    check(cudaGetLastError(), "x phase launch");
}

void Session::enqueue_xbar_zy_phase(bool copy_scalars) {
    check(cudaSetDevice(cfg_.device), "cudaSetDevice");
    launch_bus_zy(dn_, ds_, beta_, sc_, stream_);
    check(cudaGetLastError(), "xbar/zy phase launch");
    if (copy_scalars) enqueue_scalars_d2h();
}

void Session::enqueue_scalars_d2h() {
    use_device();
    check(cudaMemcpyAsync(sc_host_, sc_, sizeof(DevScalars), cudaMemcpyDeviceToHost, stream_), "D2H");
}

IterScalars Session::read_scalars() {
    use_device();
    check(cudaStreamSynchronize(stream_), "iteration sync");
    const DevScalars& h = *sc_host_;
    IterScalars r;
    r.primal = from_bits(h.primal_inf);
    r.dual_raw = from_bits(h.dual_inf);
    r.z_inf = from_bits(h.z_inf);
    r.z_drift = from_bits(h.z_drift);
    r.failures = static_cast<int>(h.failures);
    r.singular_bus = h.singular_bus == INT32_MAX ? -1 : h.singular_bus;
    return r;
}

void Session::outer_update() {
    check(cudaSetDevice(cfg_.device), "cudaSetDevice");
    launch_outer(dn_, ds_, beta_, cfg_.lambda_min, cfg_.lambda_max, stream_);
    check(cudaGetLastError(), "outer launch");
}

double Session::rho_max() {
    use_device();
    launch_rowmax(ds_.rho, dn_.mpad, red_, stream_);
    unsigned long long bits = 0;
    check(cudaMemcpyAsync(&bits, red_, sizeof bits, cudaMemcpyDeviceToHost, stream_), "D2H");
    check(cudaStreamSynchronize(stream_), "sync");
    return from_bits(bits);
}

long long Session::tron_iterations() const {
    use_device();
    DevScalars h;
    check(cudaMemcpy(&h, sc_, sizeof h, cudaMemcpyDeviceToHost), "D2H");
    return static_cast<long long>(h.tron_iters4);
}

long long Session::limited_tron_iterations() const {
    use_device();
    DevScalars h;
    check(cudaMemcpy(&h, sc_, sizeof h, cudaMemcpyDeviceToHost), "D2H");
    return static_cast<long long>(h.tron_iters6);
}

void Session::step_counters(long long out[4]) const {
    use_device();
    DevScalars h;
    check(cudaMemcpy(&h, sc_, sizeof h, cudaMemcpyDeviceToHost), "D2H");
    out[0] = static_cast<long long>(h.tron_iters4);
    out[1] = static_cast<long long>(h.tron_iters6);
    out[2] = static_cast<long long>(h.exec4);
    out[3] = static_cast<long long>(h.exec6);
}

void Session::branch_costs(int* out) const {
    use_device();
    if (dn_.nl)
        check(cudaMemcpy(out, ds_.br_cost, dn_.nl * sizeof(int), cudaMemcpyDeviceToHost), "D2H");
}

void Session::sync() const {
    use_device();
    check(cudaStreamSynchronize(stream_), "sync");
}

// Every method that touches device memory or the stream makes the session's
// GPU current first: sessions on different GPUs may share a host thread.
void Session::use_device() const { check(cudaSetDevice(cfg_.device), "cudaSetDevice"); }

}  // namespace ga
