// dist.cpp — the bus-graph-partitioned ADMM across processes (one process per
// GPU, e.g. under torchrun): rank r owns part r of partition_buses(net, world)
// and exchanges boundary rows with NCCL over NVLink/NVSwitch.  Per inner
// iteration (same data flow as multi.cpp):
//   x phase -> pack far-end x rows of cut branches per peer -> grouped
//   ncclSend/ncclRecv -> unpack -> bus + z/y phase -> ncclAllReduce of the
//   residual maxima (uint64 bit patterns, MAX: exact), failures (SUM) and the
//   first singular bus (MIN) in place in the device scalars -> pack (xbar, z,
//   y) of the rows this rank owns for peers' branches -> grouped send/recv
//   -> unpack -> one D2H of the reduced scalars.
// NCCL is loaded with dlopen at session creation (libnccl.so.2 — the one the
// process already has, e.g. PyTorch's), so single-GPU users need no NCCL.
#include <dlfcn.h>

#include <climits>
#include <cstring>

#include "gridadmm/gridadmm_ext.h"
#include "solver.hpp"

namespace ga {

namespace {

// Minimal NCCL ABI (nccl.h, stable since 2.x).
using ncclComm_t = struct ncclComm*;
struct ncclUniqueId { char internal[128]; };
enum ncclDataType_t { ncclInt32 = 2, ncclUint64 = 5, ncclFloat64 = 8 };
enum ncclRedOp_t { ncclSum = 0, ncclMax = 2, ncclMin = 3 };
using ncclResult_t = int;

struct Nccl {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*);
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
    ncclResult_t (*CommDestroy)(ncclComm_t);
    ncclResult_t (*GroupStart)();
    ncclResult_t (*GroupEnd)();
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t);
    const char* (*GetErrorString)(ncclResult_t);
};

const Nccl& nccl() {
    static Nccl n = [] {
        Nccl r{};
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) throw CudaError(std::string("cannot load libnccl.so.2: ") + dlerror());
        auto sym = [&](const char* name) {
            void* p = dlsym(h, name);
            if (!p) throw CudaError(std::string("NCCL symbol missing: ") + name);
            return p;
        };
        r.GetUniqueId = reinterpret_cast<decltype(r.GetUniqueId)>(sym("ncclGetUniqueId"));
        r.CommInitRank = reinterpret_cast<decltype(r.CommInitRank)>(sym("ncclCommInitRank"));
        r.CommDestroy = reinterpret_cast<decltype(r.CommDestroy)>(sym("ncclCommDestroy"));
        r.GroupStart = reinterpret_cast<decltype(r.GroupStart)>(sym("ncclGroupStart"));
        r.GroupEnd = reinterpret_cast<decltype(r.GroupEnd)>(sym("ncclGroupEnd"));
        r.Send = reinterpret_cast<decltype(r.Send)>(sym("ncclSend"));
        r.Recv = reinterpret_cast<decltype(r.Recv)>(sym("ncclRecv"));
        r.AllReduce = reinterpret_cast<decltype(r.AllReduce)>(sym("ncclAllReduce"));
        r.GetErrorString = reinterpret_cast<decltype(r.GetErrorString)>(sym("ncclGetErrorString"));
        return r;
    }();
    return n;
}

void nc(ncclResult_t r, const char* what) {
    if (r != 0) throw CudaError(std::string(what) + ": " + nccl().GetErrorString(r));
}
void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

class DistPart final : public Engine {
public:
    DistPart(const Network& net, const SolverConfig& cfg, int rank, int world,
             const unsigned char* id)
        : net_(net), cfg_(cfg), rank_(rank), world_(world) {
        part_ = partition_buses(net, world);
        plan_ = make_plan(net, part_, rank, world);
        sess_ = std::make_unique<Session>(net, cfg, world > 1 ? &plan_ : nullptr);
        ncclUniqueId uid;
        std::memcpy(uid.internal, id, sizeof uid.internal);
        ck(cudaSetDevice(cfg.device), "cudaSetDevice");
        nc(nccl().CommInitRank(&comm_, world, uid, rank), "ncclCommInitRank");
        size_t mx = 0;
        for (int q = 0; q < world; ++q)
            mx = std::max(mx, std::max(plan_.send_x[q].size(), plan_.recv_x[q].size()));
        cap_ = 3 * std::max<size_t>(mx, 1);
        sbuf_.assign(world, nullptr);
        rbuf_.assign(world, nullptr);
        for (int q = 0; q < world; ++q) {
            ck(cudaMalloc(&sbuf_[q], cap_ * sizeof(double)), "cudaMalloc");
            ck(cudaMalloc(&rbuf_[q], cap_ * sizeof(double)), "cudaMalloc");
        }
    }
    ~DistPart() override {
        if (comm_) nccl().CommDestroy(comm_);
        for (double* p : sbuf_) cudaFree(p);
        for (double* p : rbuf_) cudaFree(p);
    }

    const Network& network() const override { return sess_->network(); }  // period network
    const SolverConfig& config() const override { return cfg_; }
    int m() const override { return net_.m(); }
    int parts() const override { return world_; }
    void cold_start() override { sess_->cold_start(); }
    void upload_state(const HostState& s) override { sess_->upload_state(s); }
    void download_state(HostState& s) const override { sess_->download_state(s); }
    double beta() const override { return sess_->beta(); }
    void set_beta(double b) override { sess_->set_beta(b); }
    void set_loads(const std::vector<double>& pd, const std::vector<double>& qd) override {
        sess_->set_loads(pd, qd);
    }
    void set_gen_p_bounds(const std::vector<double>& a, const std::vector<double>& b) override {
        sess_->set_gen_p_bounds(a, b);
    }
    void clamp_gen_p() override { sess_->clamp_gen_p(); }
    void outer_update() override { sess_->outer_update(); sess_->sync(); }
    double rho_max() override { return sess_->rho_max(); }  // rho replicated on every rank
    void download_solution_inputs(std::vector<double>& g, std::vector<double>& w,
                                  std::vector<double>& th) const override {
        sess_->download_solution_inputs(g, w, th);  // owned entries only are current
    }

    // Each step bracketed by CUDA events on this rank's stream (launches,
    // NCCL exchanges and the D2H of the reduced norms); optional L2 flush
    // between steps outside the brackets.
    int timed_steps(int k, size_t flush_bytes, double* step_ms, double* records) override {
        void* flush = nullptr;
        if (flush_bytes) ck(cudaMalloc(&flush, flush_bytes), "cudaMalloc flush");
        cudaEvent_t a, b;
        ck(cudaEventCreate(&a), "event");
        ck(cudaEventCreate(&b), "event");
        const double rmax = rho_max();
        for (int i = 0; i < k; ++i) {
            if (flush) ck(cudaMemsetAsync(flush, i & 0xff, flush_bytes, sess_->stream()), "flush");
            cudaEventRecord(a, sess_->stream());
            double nrm[4];
            const int fails = iterate_impl(nrm, b);
            float ms = 0.0f;
            cudaEventElapsedTime(&ms, a, b);
            if (step_ms) step_ms[i] = ms;
            if (records) {
                double* r = records + 5 * i;
                r[0] = nrm[0]; r[1] = nrm[1] * rmax; r[2] = nrm[2]; r[3] = nrm[3]; r[4] = fails;
            }
        }
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        if (flush) cudaFree(flush);
        return k;
    }

    int iterate(double out[4], PhaseTimes* times) override {
        (void)times;
        return iterate_impl(out, nullptr);
    }

    int iterate_impl(double out[4], cudaEvent_t end_event) {
        cudaStream_t st = sess_->stream();
        const DevState& s = sess_->dev_state();
        sess_->enqueue_x_phase();
        if (world_ > 1) {
            // x of cut branches' to-side rows -> to-bus owner
            for (int q = 0; q < world_; ++q)
                if (q != rank_)
                    launch_gather_rows(sess_->d_send_x(q), int(plan_.send_x[q].size()), s.x,
                                       sbuf_[q], st);
            nc(nccl().GroupStart(), "ncclGroupStart");
            for (int q = 0; q < world_; ++q) {
                if (q == rank_) continue;
                if (!plan_.send_x[q].empty())
                    nc(nccl().Send(sbuf_[q], plan_.send_x[q].size(), ncclFloat64, q, comm_, st), "ncclSend");
                if (!plan_.recv_x[q].empty())
                    nc(nccl().Recv(rbuf_[q], plan_.recv_x[q].size(), ncclFloat64, q, comm_, st), "ncclRecv");
            }
            nc(nccl().GroupEnd(), "ncclGroupEnd");
            for (int q = 0; q < world_; ++q)
                if (q != rank_)
                    launch_scatter_rows(sess_->d_recv_x(q), int(plan_.recv_x[q].size()), rbuf_[q],
                                        s.x, st);
        }
        sess_->enqueue_xbar_zy_phase(false);
        if (world_ > 1) {
            DevScalars* sc = sess_->dev_scalars();
            // maxima of non-negative doubles as uint64 bit patterns: exact
            nc(nccl().AllReduce(&sc->primal_inf, &sc->primal_inf, 4, ncclUint64, ncclMax, comm_, st),
               "ncclAllReduce max");
            nc(nccl().AllReduce(&sc->failures, &sc->failures, 1, ncclUint64, ncclSum, comm_, st),
               "ncclAllReduce sum");
            nc(nccl().AllReduce(&sc->singular_bus, &sc->singular_bus, 1, ncclInt32, ncclMin, comm_, st),
               "ncclAllReduce min");
            // (xbar, z, y) of the rows this rank owns for peers' branches
            for (int q = 0; q < world_; ++q) {
                if (q == rank_) continue;
                const int n = int(plan_.recv_x[q].size());
                launch_gather_rows(sess_->d_recv_x(q), n, s.xbar, sbuf_[q], st);
                launch_gather_rows(sess_->d_recv_x(q), n, s.z, sbuf_[q] + n, st);
                launch_gather_rows(sess_->d_recv_x(q), n, s.y, sbuf_[q] + 2 * n, st);
            }
            nc(nccl().GroupStart(), "ncclGroupStart");
            for (int q = 0; q < world_; ++q) {
                if (q == rank_) continue;
                if (!plan_.recv_x[q].empty())
                    nc(nccl().Send(sbuf_[q], 3 * plan_.recv_x[q].size(), ncclFloat64, q, comm_, st), "ncclSend");
                if (!plan_.send_x[q].empty())
                    nc(nccl().Recv(rbuf_[q], 3 * plan_.send_x[q].size(), ncclFloat64, q, comm_, st), "ncclRecv");
            }
            nc(nccl().GroupEnd(), "ncclGroupEnd");
            for (int q = 0; q < world_; ++q) {
                if (q == rank_) continue;
                const int n = int(plan_.send_x[q].size());
                launch_scatter_rows(sess_->d_send_x(q), n, rbuf_[q], s.xbar, st);
                launch_scatter_rows(sess_->d_send_x(q), n, rbuf_[q] + n, s.z, st);
                launch_scatter_rows(sess_->d_send_x(q), n, rbuf_[q] + 2 * n, s.y, st);
            }
        }
        sess_->enqueue_scalars_d2h();
        if (end_event) cudaEventRecord(end_event, st);
        const IterScalars r = sess_->read_scalars();
        ck(cudaGetLastError(), "dist iteration");
        if (r.singular_bus >= 0) {
            const int id = net_.buses[r.singular_bus].id;
            throw SingularBusError(id, "isolated bus " + std::to_string(id) + ": singular balance system");
        }
        out[0] = r.primal;
        out[1] = r.dual_raw;
        out[2] = r.z_inf;
        out[3] = r.z_drift;
        return r.failures;
    }

private:
    Network net_;
    SolverConfig cfg_;
    int rank_, world_;
    std::vector<int> part_;
    PartPlan plan_;
    std::unique_ptr<Session> sess_;
    ncclComm_t comm_ = nullptr;
    size_t cap_ = 0;
    std::vector<double*> sbuf_, rbuf_;
};

}  // namespace

void nccl_unique_id(unsigned char out[128]) {
    ncclUniqueId id;
    nc(nccl().GetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(out, id.internal, 128);
}

std::unique_ptr<Engine> make_dist_engine(const Network& net, const SolverConfig& cfg, int rank,
                                         int world, const unsigned char* id) {
    return std::make_unique<DistPart>(net, cfg, rank, world, id);
}

}  // namespace ga
