// qsim_comm.cu -- the two transports of qsim_comm.h: NCCL (+ CUDA IPC) and the in-process
// loopback used to test the multi-GPU schedules on one device.
#include <nccl.h>

#include <chrono>
#include <condition_variable>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>

#include "qsim_comm.h"

namespace qc {

namespace {

constexpr char kLoopMagic[16] = "QSIM-LOOPBACK-1";

// fold the world copies s[r * count + i] (rank order) into out[i]
__global__ void fold_kernel(const double *s, int world, size_t count, int op, double *out) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
        double a = s[i];
        for (int r = 1; r < world; ++r) {
            const double b = s[(size_t)r * count + i];
            a = op == 0 ? a + b : fmin(a, b);
        }
        out[i] = a;
    }
}

// ------------------------------------------------------------------------------------- NCCL
class NcclComm final : public Comm {
  public:
    NcclComm(int world, int rank) : world_(world), rank_(rank) {}
    ~NcclComm() override {
        if (d_bar_) cudaFree(d_bar_);
        if (d_tmp_) cudaFree(d_tmp_);
        if (comm_) ncclCommDestroy(comm_);
    }
    bool init(const void *id128) {
        ncclUniqueId id;
        std::memcpy(&id, id128, sizeof(id));
        if (!nk(ncclCommInitRank(&comm_, world_, id, rank_), "ncclCommInitRank")) return false;
        if (cudaMalloc(&d_bar_, sizeof(double)) != cudaSuccess || cudaMemset(d_bar_, 0, sizeof(double)) != cudaSuccess) {
            err_ = "cudaMalloc (barrier scratch)";
            return false;
        }
        return true;
    }
    int rank() const override { return rank_; }
    int world() const override { return world_; }
    const char *kind() const override { return "nccl"; }
    bool allreduce(double *buf, size_t count, Op op, cudaStream_t st) override {
        return nk(ncclAllReduce(buf, buf, count, ncclDouble, op == Op::Sum ? ncclSum : ncclMin, comm_, st),
                  "ncclAllReduce");
    }
    bool allgather(const void *send, void *recv, size_t bytes, cudaStream_t st) override {
        return nk(ncclAllGather(send, recv, bytes, ncclUint8, comm_, st), "ncclAllGather");
    }
    bool barrier(cudaStream_t st) override { return allreduce(d_bar_, 1, Op::Sum, st); }
    bool exchange(const std::vector<XPair> &pairs, cudaStream_t st) override {
        if (!nk(ncclGroupStart(), "ncclGroupStart")) return false;
        for (const XPair &x : pairs) {
            if (!nk(ncclSend(x.send, x.bytes, ncclUint8, x.peer, comm_, st), "ncclSend")) return false;
            if (!nk(ncclRecv(x.recv, x.bytes, ncclUint8, x.peer, comm_, st), "ncclRecv")) return false;
        }
        return nk(ncclGroupEnd(), "ncclGroupEnd");
    }
    bool share(void *mine, size_t, void **out, cudaStream_t st) override {
        const size_t hs = sizeof(cudaIpcMemHandle_t);
        std::vector<unsigned char> all(hs * world_);
        cudaIpcMemHandle_t h;
        long long ok = cudaIpcGetMemHandle(&h, mine) == cudaSuccess;
        if (!ok) cudaGetLastError();
        if (!tmp(hs * (world_ + 1))) return false;
        if (cudaMemcpyAsync(d_tmp_ + hs * rank_, &h, hs, cudaMemcpyHostToDevice, st) != cudaSuccess) return false;
        if (!allgather(d_tmp_ + hs * rank_, d_tmp_, hs, st)) return false;
        if (cudaMemcpyAsync(all.data(), d_tmp_, all.size(), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess) {
            err_ = "IPC handle exchange";
            return false;
        }
        for (int r = 0; r < world_; ++r) out[r] = nullptr;
        out[rank_] = mine;
        for (int r = 0; r < world_ && ok; ++r) {
            if (r == rank_) continue;
            cudaIpcMemHandle_t hr;
            std::memcpy(&hr, all.data() + hs * r, hs);
            if (cudaIpcOpenMemHandle(&out[r], hr, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
                cudaGetLastError();
                out[r] = nullptr;
                ok = 0;
            }
        }
        long long all_ok = 0;
        if (!agree_min(ok, &all_ok, st)) return false;
        if (!all_ok) {  // some rank could not map: nobody uses the mappings
            unshare(out);
            err_ = "cudaIpcOpenMemHandle failed on some rank";
            return false;
        }
        return true;
    }
    void unshare(void **mapped) override {
        for (int r = 0; r < world_; ++r)
            if (r != rank_ && mapped[r]) {
                cudaIpcCloseMemHandle(mapped[r]);
                mapped[r] = nullptr;
            }
    }
    bool agree_min(long long v, long long *out, cudaStream_t st) override {
        if (!tmp(sizeof(long long))) return false;
        if (cudaMemcpyAsync(d_tmp_, &v, sizeof(v), cudaMemcpyHostToDevice, st) != cudaSuccess) return false;
        if (!nk(ncclAllReduce(d_tmp_, d_tmp_, 1, ncclInt64, ncclMin, comm_, st), "ncclAllReduce(min)")) return false;
        if (cudaMemcpyAsync(out, d_tmp_, sizeof(v), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess) {
            err_ = "agree_min copy";
            return false;
        }
        return true;
    }

  private:
    bool nk(ncclResult_t r, const char *what) {
        if (r == ncclSuccess) return true;
        err_ = std::string(what) + ": " + ncclGetErrorString(r);
        return false;
    }
    bool tmp(size_t bytes) {
        if (tmp_cap_ >= bytes) return true;
        if (d_tmp_) cudaFree(d_tmp_);
        d_tmp_ = nullptr;
        tmp_cap_ = 0;
        if (cudaMalloc(&d_tmp_, bytes) != cudaSuccess) {
            err_ = "cudaMalloc (comm scratch)";
            return false;
        }
        tmp_cap_ = bytes;
        return true;
    }
    int world_, rank_;
    ncclComm_t comm_ = nullptr;
    double *d_bar_ = nullptr;
    unsigned char *d_tmp_ = nullptr;
    size_t tmp_cap_ = 0;
};

// --------------------------------------------------------------------------------- loopback
struct LoopGroup {
    int world = 0;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    unsigned long long gen = 0;
    bool broken = false;
    std::vector<const void *> ptr;
    std::vector<long long> val;
    std::vector<cudaEvent_t> ev;
    std::vector<int> dev;  // each rank's device
    int attached = 0, detached = 0;
};

std::mutex g_mu;
std::map<unsigned long long, std::shared_ptr<LoopGroup>> g_groups;
unsigned long long g_next = 1;

class LoopComm final : public Comm {
  public:
    LoopComm(std::shared_ptr<LoopGroup> g, unsigned long long key, int rank) : g_(std::move(g)), key_(key), rank_(rank) {}
    ~LoopComm() override {
        if (d_s_) cudaFree(d_s_);
        std::lock_guard<std::mutex> lk(g_mu);
        if (++g_->detached == g_->world) g_groups.erase(key_);
        if (ev_) cudaEventDestroy(ev_);
    }
    bool init() {
        if (cudaEventCreateWithFlags(&ev_, cudaEventDisableTiming) != cudaSuccess) {
            err_ = "cudaEventCreate";
            return false;
        }
        int d = 0;
        cudaGetDevice(&d);
        std::lock_guard<std::mutex> lk(g_->mu);
        g_->ev[rank_] = ev_;
        g_->dev[rank_] = d;
        return true;
    }
    bool shared_device() const override {
        for (int r = 1; r < g_->world; ++r)
            if (g_->dev[r] != g_->dev[0]) return false;
        return true;
    }
    int rank() const override { return rank_; }
    int world() const override { return g_->world; }
    const char *kind() const override { return "loopback"; }
    bool barrier(cudaStream_t st) override {
        if (cudaEventRecord(ev_, st) != cudaSuccess) return cerr("cudaEventRecord");
        if (!host_barrier()) return false;
        for (int r = 0; r < g_->world; ++r)
            if (r != rank_ && cudaStreamWaitEvent(st, g_->ev[r], 0) != cudaSuccess) return cerr("cudaStreamWaitEvent");
        return host_barrier();  // nobody re-records its event before every rank has enqueued its waits
    }
    bool allreduce(double *buf, size_t count, Op op, cudaStream_t st) override {
        const int G = g_->world;
        if (!scratch(sizeof(double) * count * G)) return false;
        g_->ptr[rank_] = buf;
        if (!barrier(st)) return false;
        for (int r = 0; r < G; ++r)
            if (cudaMemcpyAsync(d_s_ + (size_t)r * count, g_->ptr[r], sizeof(double) * count, cudaMemcpyDeviceToDevice,
                                st) != cudaSuccess)
                return cerr("cudaMemcpyAsync (allreduce)");
        if (!barrier(st)) return false;  // every rank has read every buffer before any is overwritten
        const int grid = (int)std::min<size_t>((count + 255) / 256, 1024);
        fold_kernel<<<grid, 256, 0, st>>>(d_s_, G, count, op == Op::Sum ? 0 : 1, buf);
        return cudaGetLastError() == cudaSuccess || cerr("fold_kernel");
    }
    bool allgather(const void *send, void *recv, size_t bytes, cudaStream_t st) override {
        g_->ptr[rank_] = send;
        if (!barrier(st)) return false;
        for (int r = 0; r < g_->world; ++r) {
            char *dst = (char *)recv + bytes * r;
            if (dst == g_->ptr[r]) continue;
            if (cudaMemcpyAsync(dst, g_->ptr[r], bytes, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
                return cerr("cudaMemcpyAsync (allgather)");
        }
        return barrier(st);
    }
    bool exchange(const std::vector<XPair> &pairs, cudaStream_t st) override {
        g_->ptr[rank_] = &pairs;
        if (!barrier(st)) return false;
        for (const XPair &x : pairs) {
            const auto *pv = static_cast<const std::vector<XPair> *>(g_->ptr[x.peer]);
            const void *src = nullptr;
            for (const XPair &y : *pv)
                if (y.peer == rank_) src = y.send;
            if (!src) {
                err_ = "loopback exchange: peer has no matching send";
                return false;
            }
            if (cudaMemcpyAsync(x.recv, src, x.bytes, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
                return cerr("cudaMemcpyAsync (exchange)");
        }
        return barrier(st);
    }
    bool share(void *mine, size_t, void **out, cudaStream_t st) override {
        g_->ptr[rank_] = mine;
        if (!host_barrier()) return false;
        long long ok = 1;
        for (int r = 0; r < g_->world; ++r) {
            out[r] = const_cast<void *>(g_->ptr[r]);
            if (g_->dev[r] != g_->dev[rank_]) {  // another GPU of this process: direct peer access
                cudaError_t e = cudaDeviceEnablePeerAccess(g_->dev[r], 0);
                if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
                else if (e != cudaSuccess) {
                    cudaGetLastError();
                    ok = 0;
                }
            }
        }
        if (!host_barrier()) return false;
        long long all = 0;
        if (!agree_min(ok, &all, st)) return false;
        if (!all) err_ = "peer access between the loopback ranks' devices is not possible";
        return all != 0;
    }
    void unshare(void **) override {}
    bool agree_min(long long v, long long *out, cudaStream_t) override {
        g_->val[rank_] = v;
        if (!host_barrier()) return false;
        long long m = v;
        for (int r = 0; r < g_->world; ++r) m = std::min(m, g_->val[r]);
        *out = m;
        return host_barrier();
    }

  private:
    bool cerr(const char *what) {
        err_ = std::string(what) + ": " + cudaGetErrorString(cudaGetLastError());
        return false;
    }
    // generation barrier over the group's threads; a rank that never arrives breaks the group
    // after the timeout (every waiting rank then fails instead of hanging)
    bool host_barrier() {
        std::unique_lock<std::mutex> lk(g_->mu);
        if (g_->broken) {
            err_ = "loopback group broken";
            return false;
        }
        const unsigned long long gen0 = g_->gen;
        if (++g_->arrived == g_->world) {
            g_->arrived = 0;
            ++g_->gen;
            g_->cv.notify_all();
            return true;
        }
        if (!g_->cv.wait_for(lk, std::chrono::seconds(600), [&] { return g_->gen != gen0 || g_->broken; })) {
            g_->broken = true;
            g_->cv.notify_all();
        }
        if (g_->broken) {
            err_ = "loopback barrier timed out (a rank stopped calling)";
            return false;
        }
        return true;
    }
    bool scratch(size_t bytes) {
        if (s_cap_ >= bytes) return true;
        if (d_s_) cudaFree(d_s_);
        d_s_ = nullptr;
        s_cap_ = 0;
        if (cudaMalloc(&d_s_, bytes) != cudaSuccess) return cerr("cudaMalloc (loopback scratch)");
        s_cap_ = bytes;
        return true;
    }
    std::shared_ptr<LoopGroup> g_;
    unsigned long long key_;
    int rank_;
    cudaEvent_t ev_ = nullptr;
    double *d_s_ = nullptr;
    size_t s_cap_ = 0;
};

}  // namespace

bool is_loopback_id(const void *id128) { return id128 && std::memcmp(id128, kLoopMagic, sizeof(kLoopMagic)) == 0; }

int make_loopback_id(int world, void *out128) {
    auto g = std::make_shared<LoopGroup>();
    g->world = world;
    g->ptr.assign(world, nullptr);
    g->val.assign(world, 0);
    g->ev.assign(world, nullptr);
    g->dev.assign(world, 0);
    unsigned long long key;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        key = g_next++;
        g_groups[key] = g;
    }
    std::memset(out128, 0, 128);
    std::memcpy(out128, kLoopMagic, sizeof(kLoopMagic));
    std::memcpy((char *)out128 + 16, &key, sizeof(key));
    std::memcpy((char *)out128 + 24, &world, sizeof(world));
    return 0;
}

Comm *make_comm(const void *id128, int world, int rank, std::string *err) {
    if (is_loopback_id(id128)) {
        unsigned long long key;
        int w;
        std::memcpy(&key, (const char *)id128 + 16, sizeof(key));
        std::memcpy(&w, (const char *)id128 + 24, sizeof(w));
        std::shared_ptr<LoopGroup> g;
        {
            std::lock_guard<std::mutex> lk(g_mu);
            auto it = g_groups.find(key);
            if (it != g_groups.end()) g = it->second;
            if (g && (w != world || g->attached >= world)) g.reset();
            if (g) ++g->attached;
        }
        if (!g) {
            *err = "unknown, used or mismatched loopback id";
            return nullptr;
        }
        auto *c = new LoopComm(g, key, rank);
        if (!c->init()) {
            *err = c->error();
            delete c;
            return nullptr;
        }
        return c;
    }
    auto *c = new NcclComm(world, rank);
    if (!c->init(id128)) {
        *err = c->error();
        delete c;
        return nullptr;
    }
    return c;
}

}  // namespace qc
