// comm.hpp — the exchange steps of the multi-GPU engine behind one interface.
//
// The reference fans its phases out over threads (parallel_for,
// parallel.cpp:11-43) and concatenates results in partition order
// (engine.cpp:41-63, 116-134; filter.cpp:15-33). Across GPUs those
// concatenations become collectives: counts are all-reduced, candidate and
// local-skyline rows are all-gathered (ragged), filtered rows are routed to
// their partition owners by an all-to-all. Two backends implement them:
//
//   NcclComm      one rank per GPU over NVLink/NVSwitch (ncclSend/ncclRecv
//                 groups for the ragged exchanges, ncclAllReduce for counts);
//                 built from a unique id (one process per GPU) or by
//                 ncclCommInitAll (one process driving every GPU).
//   LoopbackComm  ranks that are host threads of one process, possibly on
//                 the same device: every exchange is a set of
//                 cudaMemcpyAsync between the ranks' buffers, ordered by
//                 CUDA events and host barriers. No kernel ever waits on
//                 another rank, so ranks sharing one GPU cannot deadlock;
//                 this is how the multi-rank engine runs on one B200.
//
// Every call is collective: all ranks of the group call it in the same
// order with matching sizes. Device buffers; work is enqueued on `st`.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <condition_variable>
#include <cstddef>
#include <cstdint>
#include <memory>
#include <mutex>
#include <vector>

namespace sky {

class Comm {
   public:
    Comm(int rank, int world) : rank_(rank), world_(world) {}
    virtual ~Comm() = default;
    int rank() const { return rank_; }
    int world() const { return world_; }

    // in-place sums over ranks
    virtual void allreduce_sum_u32(uint32_t* buf, size_t count, cudaStream_t st) = 0;
    virtual void allreduce_sum_u64(uint64_t* buf, size_t count, cudaStream_t st) = 0;
    // float sums; used to assemble a table from disjoint per-rank rows (every
    // other rank contributes +0.0, and x + 0 == x for the finite x >= 0 here)
    virtual void allreduce_sum_f32(float* buf, size_t count, cudaStream_t st) = 0;
    // ragged all-gather: rank q contributes bytes[q] bytes (from `send`),
    // which land at recv + displ[q] on every rank (send may alias that slot)
    virtual void allgatherv(const void* send, void* recv, const size_t* bytes, const size_t* displ,
                            cudaStream_t st) = 0;
    // all-to-all: sbytes[q] bytes from send + sdispl[q] go to rank q; rbytes[q]
    // bytes from rank q land at recv + rdispl[q]
    virtual void alltoallv(const void* send, const size_t* sbytes, const size_t* sdispl, void* recv,
                           const size_t* rbytes, const size_t* rdispl, cudaStream_t st) = 0;
    // unblock every rank after a failure on one of them (best effort)
    virtual void abort() {}
    virtual const char* backend() const = 0;

    // equal-size all-gather (rank q's `bytes` at recv + q * bytes)
    void allgather(const void* send, void* recv, size_t bytes, cudaStream_t st);

   protected:
    int rank_, world_;
};

// ---------------------------------------------------------------- loopback
// Shared state of one loopback group (W ranks = W host threads).
class LoopbackGroup {
   public:
    explicit LoopbackGroup(int world);
    ~LoopbackGroup();
    int world() const { return world_; }
    // barrier over the W ranks; throws if the group was aborted
    void barrier();
    void abort();
    bool aborted() const { return aborted_.load(); }

    struct Slot {
        const void* send = nullptr;
        const size_t* sbytes = nullptr;  // alltoallv: per destination
        const size_t* sdispl = nullptr;
        size_t bytes = 0;                // allgatherv: own contribution
        cudaEvent_t ready = nullptr;     // send data complete on the owner's stream
        cudaEvent_t done = nullptr;      // the owner finished reading its peers
        int device = 0;
        // host staging for reductions (raw words of the reduced type)
        std::vector<unsigned char> red;
    };
    std::vector<Slot> slots;

   private:
    int world_;
    std::mutex mu_;
    std::condition_variable cv_;
    int waiting_ = 0;
    uint64_t generation_ = 0;
    std::atomic<bool> aborted_{false};
};

class LoopbackComm final : public Comm {
   public:
    // `group` shared by the W ranks; events are created on `device`
    LoopbackComm(std::shared_ptr<LoopbackGroup> group, int rank, int device);
    ~LoopbackComm() override;
    void allreduce_sum_u32(uint32_t* buf, size_t count, cudaStream_t st) override;
    void allreduce_sum_u64(uint64_t* buf, size_t count, cudaStream_t st) override;
    void allreduce_sum_f32(float* buf, size_t count, cudaStream_t st) override;
    void allgatherv(const void* send, void* recv, const size_t* bytes, const size_t* displ,
                    cudaStream_t st) override;
    void alltoallv(const void* send, const size_t* sbytes, const size_t* sdispl, void* recv, const size_t* rbytes,
                   const size_t* rdispl, cudaStream_t st) override;
    void abort() override { g_->abort(); }
    const char* backend() const override { return "loopback"; }

   private:
    template <class T>
    void allreduce(T* buf, size_t count, cudaStream_t st);
    void publish_ready(cudaStream_t st);
    void finish(cudaStream_t st);
    std::shared_ptr<LoopbackGroup> g_;
    int device_;
    void* pinned_ = nullptr;  // reduction staging
    size_t pinned_cap_ = 0;
};

// -------------------------------------------------------------------- NCCL
// Opaque so that only comm.cpp includes nccl.h.
std::unique_ptr<Comm> make_nccl_comm(int device, int rank, int world, const void* unique_id);
// One communicator per device of `devices` (ncclCommInitAll), rank = index.
std::vector<std::unique_ptr<Comm>> make_nccl_comms(const std::vector<int>& devices);
size_t nccl_unique_id_bytes();
void nccl_unique_id(void* out);

}  // namespace sky
