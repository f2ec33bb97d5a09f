// qsim_comm.h -- the cross-rank operations of the multi-GPU engine, behind one
// interface with two transports:
//
//   NcclComm  one process per GPU, NCCL over NVLink / NVSwitch; peer state buffers mapped with
//             CUDA IPC (the production path, P:104-108 partitioning).
//   LoopComm  "loopback" transport: the G ranks are threads of ONE process, on one device (the
//             one-GPU test mode) or one device each (a single-process multi-GPU run, e.g. for
//             ncu, which cannot follow a multi-process NCCL job), each with its own stream and
//             shard buffers.  Collectives are stream-ordered
//             with CUDA events plus a host barrier; peer "mappings" are the peers' raw pointers.
//             The engine, the pass kernels (the MV instances with their peer stores), the
//             split-swap group ranges and the permutation / flip bookkeeping are exactly those
//             of the NCCL path, so a one-GPU box exercises every multi-GPU swap schedule.
//
// Every call is collective: all ranks make the same calls in the same order.  All device work is
// enqueued on the caller's stream; host-returning helpers (agree_*) synchronise.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include <string>
#include <vector>

namespace qc {

enum class Op { Sum, Min };

// one send/receive pair of an all-to-all exchange: `send` goes to `peer`, which sends back into `recv`
struct XPair {
    int peer;
    const void *send;
    void *recv;
    size_t bytes;
};

class Comm {
  public:
    virtual ~Comm() {}
    virtual int rank() const = 0;
    virtual int world() const = 0;
    virtual const char *kind() const = 0;
    // in-place all-reduce of `count` doubles
    virtual bool allreduce(double *buf, size_t count, Op op, cudaStream_t st) = 0;
    // recv[r * bytes ..] = rank r's send (device buffers)
    virtual bool allgather(const void *send, void *recv, size_t bytes, cudaStream_t st) = 0;
    // stream-ordered barrier: work enqueued on any rank's stream after it starts only after every
    // rank's work enqueued before it has finished (and its peer stores are visible)
    virtual bool barrier(cudaStream_t st) = 0;
    // grouped point-to-point exchange (every XPair's peer makes the mirrored call)
    virtual bool exchange(const std::vector<XPair> &pairs, cudaStream_t st) = 0;
    // map every rank's device buffer `mine` (bytes) into this process: out[r] (out[rank] = mine).
    // Returns false (and leaves nothing mapped) if any rank could not map; collective.
    virtual bool share(void *mine, size_t bytes, void **out, cudaStream_t st) = 0;
    virtual void unshare(void **mapped) = 0;
    // host-side agreement, synchronous: minimum of v over ranks
    virtual bool agree_min(long long v, long long *out, cudaStream_t st) = 0;
    // true when every rank drives the same device (loopback on one GPU): kernels that wait on
    // each other must then fit on the device together
    virtual bool shared_device() const { return false; }
    const std::string &error() const { return err_; }

  protected:
    std::string err_;
};

// 128-byte group ids: an ncclUniqueId (qsim_nccl_unique_id) or a loopback id (qsim_loopback_id)
bool is_loopback_id(const void *id128);
int make_loopback_id(int world, void *out128);
Comm *make_comm(const void *id128, int world, int rank, std::string *err);

}  // namespace qc
