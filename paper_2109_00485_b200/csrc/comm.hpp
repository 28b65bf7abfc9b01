// Communicators of the multi-GPU hot path. One rank per GPU; the
// solver needs three stream-ordered collectives:
//   * allgather of the f32 X row segments before the SpMM,
//   * reduce-scatter of the partial f32 Y panels after it,
//   * allreduce (sum) of the small fp64 Gram / norm partials.
// They replace the simulated message steps of dist.hpp:256-371 and
// distributed_gram_allreduce (dist.hpp:375-391).
//
// Two backends behind one interface:
//   * NcclComm  — one process per GPU, NCCL over NVLink / NVSwitch;
//   * LocalComm — ranks are host threads of one process sharing a group
//     object; any device assignment, including several ranks on one GPU. The
//     collectives are device copies / rank-ordered sum kernels between the
//     ranks' buffers, fenced with events and a host barrier. This is how the
//     N > 1 path is exercised on a single B200.
// Every reduction sums in ascending rank order, so all ranks hold bitwise
// identical results (the determinism dist.hpp:277-371 documents).
#pragma once

#include <cuda_runtime.h>

#include <condition_variable>
#include <memory>
#include <mutex>
#include <vector>

#include "common.hpp"

namespace be {

// One point-to-point transfer of a grouped exchange (Comm::p2p).
struct P2POp {
    int peer;
    bool send;       // send `bytes` from ptr to peer, or receive them into ptr
    void* ptr;
    std::size_t bytes;
};

struct Comm {
    int rank = 0, world = 1, device = 0;
    virtual ~Comm() = default;
    // buf (count doubles, device) <- sum over ranks, in place
    virtual void allreduce_f64(double* buf, std::size_t count, cudaStream_t s) = 0;
    // recv (world * count floats) <- concatenation of every rank's send
    // (count floats). In place when send == recv + rank * count.
    virtual void allgather_f32(const float* send, float* recv, std::size_t count, cudaStream_t s) = 0;
    // recv (count floats) <- sum over ranks of send[rank * count ...]
    // (send holds world * count floats). In place when recv == send + rank * count.
    virtual void reduce_scatter_f32(const float* send, float* recv, std::size_t count, cudaStream_t s) = 0;
    // A grouped set of sends and receives, stream-ordered on s: every send to a
    // peer matches, in order, one receive of that peer from this rank (ncclSend /
    // ncclRecv inside one group). The segment-wise SpMM exchange.
    virtual void p2p(const std::vector<P2POp>& ops, cudaStream_t s) = 0;
    virtual const char* backend() const = 0;
    // Wait for stream s while watching the group (NCCL: ncclCommGetAsyncError; a failed
    // or vanished peer leaves the collective pending forever): an asynchronous error, or
    // no progress within BE_COMM_TIMEOUT_S seconds (default 600), aborts the
    // communicator and throws ProtocolDeadlock -- the reference's "a rank is missing from
    // the collective" (dist.hpp:256-263, 273-282).
    virtual void sync(cudaStream_t s);
    std::int64_t calls = 0;       // collectives issued
    std::int64_t bytes_moved = 0; // bytes this rank received (flat model, like SimComm::volume_doubles)
};

// Shared state of an in-process rank group.
struct LocalGroup {
    explicit LocalGroup(int w);
    int world;
    // generation barrier
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    std::uint64_t generation = 0;
    bool aborted = false;
    double timeout_s = 600.0;  // BE_COMM_TIMEOUT_S
    // throws ProtocolDeadlock (dist.hpp:256-263: "a rank is missing from the
    // collective") when the group was aborted or a peer never arrives
    void barrier();
    void abort();
    // per-rank slots published for the current collective
    struct Slot {
        const void* send = nullptr;
        void* recv = nullptr;
        int device = 0;
        cudaEvent_t ready = nullptr;  // send data complete on the owner's stream
        cudaEvent_t done = nullptr;   // the owner finished reading peers' data
        std::vector<P2POp> sends;     // (p2p) this rank's published sends
    };
    std::vector<Slot> slots;
};

std::unique_ptr<Comm> make_nccl_comm(int device, const unsigned char id[128], int rank, int world);
void nccl_unique_id(unsigned char id[128]);
std::unique_ptr<Comm> make_local_comm(int device, LocalGroup* group, int rank);

}  // namespace be

struct be_comm {
    std::unique_ptr<be::Comm> impl;
};
struct be_comm_group {
    std::unique_ptr<be::LocalGroup> impl;
};
