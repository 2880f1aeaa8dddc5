// comm.cpp — NCCL and loopback backends of the engine's exchange steps
// (comm.hpp).
#include "comm.hpp"

#include <nccl.h>

#include <cstring>
#include <string>

#include "common.cuh"

namespace sky {

#define SKY_NCCL_CALL(call)                                                                  \
    do {                                                                                     \
        ncclResult_t r_ = (call);                                                            \
        if (r_ != ncclSuccess)                                                               \
            throw ::sky::Error(SKY_E_NCCL, std::string(#call) + ": " + ncclGetErrorString(r_)); \
    } while (0)

void Comm::allgather(const void* send, void* recv, size_t bytes, cudaStream_t st) {
    std::vector<size_t> b(world_, bytes), dpl(world_);
    for (int q = 0; q < world_; ++q) dpl[q] = (size_t)q * bytes;
    allgatherv(send, recv, b.data(), dpl.data(), st);
}

// =============================================================== loopback
LoopbackGroup::LoopbackGroup(int world) : slots(world), world_(world) {}
LoopbackGroup::~LoopbackGroup() = default;

void LoopbackGroup::barrier() {
    std::unique_lock<std::mutex> lk(mu_);
    if (aborted_) throw Error(SKY_E_INTERNAL, "multi-rank run aborted by another rank");
    const uint64_t gen = generation_;
    if (++waiting_ == world_) {
        waiting_ = 0;
        ++generation_;
        cv_.notify_all();
        return;
    }
    cv_.wait(lk, [&] { return generation_ != gen || aborted_.load(); });
    if (generation_ == gen) throw Error(SKY_E_INTERNAL, "multi-rank run aborted by another rank");
}

void LoopbackGroup::abort() {
    std::lock_guard<std::mutex> lk(mu_);
    aborted_ = true;
    cv_.notify_all();
}

LoopbackComm::LoopbackComm(std::shared_ptr<LoopbackGroup> group, int rank, int device)
    : Comm(rank, group->world()), g_(std::move(group)), device_(device) {
    auto& s = g_->slots[rank];
    s.device = device;
    SKY_CUDA(cudaEventCreateWithFlags(&s.ready, cudaEventDisableTiming));
    SKY_CUDA(cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming));
}

LoopbackComm::~LoopbackComm() {
    auto& s = g_->slots[rank_];
    if (s.ready) cudaEventDestroy(s.ready);
    if (s.done) cudaEventDestroy(s.done);
    s.ready = s.done = nullptr;
    if (pinned_) cudaFreeHost(pinned_);
}

// my send data is complete once my stream reaches this point
void LoopbackComm::publish_ready(cudaStream_t st) {
    SKY_CUDA(cudaEventRecord(g_->slots[rank_].ready, st));
    g_->barrier();  // every rank's slot (pointers, sizes, ready event) is set
}

// Copies into my buffers are queued on my stream; my send buffer must stay
// untouched until every peer's copies out of it completed: my stream waits
// for the peers' `done` events before any later work.
void LoopbackComm::finish(cudaStream_t st) {
    SKY_CUDA(cudaEventRecord(g_->slots[rank_].done, st));
    g_->barrier();  // every rank recorded `done` after its reads
    for (int q = 0; q < world_; ++q)
        if (q != rank_) SKY_CUDA(cudaStreamWaitEvent(st, g_->slots[q].done, 0));
    g_->barrier();  // nobody reuses its events or slot before all waits are queued
}

void LoopbackComm::allgatherv(const void* send, void* recv, const size_t* bytes, const size_t* displ,
                              cudaStream_t st) {
    auto& me = g_->slots[rank_];
    me.send = send;
    me.bytes = bytes[rank_];
    publish_ready(st);
    for (int q = 0; q < world_; ++q) {
        const auto& s = g_->slots[q];
        if (!bytes[q]) continue;
        char* dst = static_cast<char*>(recv) + displ[q];
        if (q == rank_) {
            if (dst != send) SKY_CUDA(cudaMemcpyAsync(dst, send, bytes[q], cudaMemcpyDefault, st));
            continue;
        }
        SKY_CUDA(cudaStreamWaitEvent(st, s.ready, 0));
        SKY_CUDA(cudaMemcpyAsync(dst, s.send, bytes[q], cudaMemcpyDefault, st));
    }
    finish(st);
}

void LoopbackComm::alltoallv(const void* send, const size_t* sbytes, const size_t* sdispl, void* recv,
                             const size_t* rbytes, const size_t* rdispl, cudaStream_t st) {
    auto& me = g_->slots[rank_];
    me.send = send;
    me.sbytes = sbytes;
    me.sdispl = sdispl;
    publish_ready(st);
    for (int q = 0; q < world_; ++q) {
        const auto& s = g_->slots[q];
        const size_t nb = s.sbytes[rank_];
        if (nb != rbytes[q])
            throw Error(SKY_E_INTERNAL, "loopback all-to-all: sender and receiver disagree on a size");
        if (!nb) continue;
        char* dst = static_cast<char*>(recv) + rdispl[q];
        const char* src = static_cast<const char*>(s.send) + s.sdispl[rank_];
        if (q != rank_) SKY_CUDA(cudaStreamWaitEvent(st, s.ready, 0));
        SKY_CUDA(cudaMemcpyAsync(dst, src, nb, cudaMemcpyDefault, st));
    }
    finish(st);
}

// Reductions go through the host: each rank stages its words, the sums are
// formed after a barrier, and copied back (test-scale sizes: counts).
template <class T>
void LoopbackComm::allreduce(T* buf, size_t count, cudaStream_t st) {
    const size_t bytes = count * sizeof(T);
    if (pinned_cap_ < bytes) {
        if (pinned_) cudaFreeHost(pinned_);
        pinned_ = nullptr;
        SKY_CUDA(cudaMallocHost(&pinned_, bytes));
        pinned_cap_ = bytes;
    }
    T* h = static_cast<T*>(pinned_);
    SKY_CUDA(cudaMemcpyAsync(h, buf, bytes, cudaMemcpyDeviceToHost, st));
    SKY_CUDA(cudaStreamSynchronize(st));
    auto& me = g_->slots[rank_];
    me.red.resize(bytes);
    std::memcpy(me.red.data(), h, bytes);
    g_->barrier();
    for (size_t k = 0; k < count; ++k) {
        T s = 0;  // rank order: the same sum on every rank
        for (int q = 0; q < world_; ++q) s += reinterpret_cast<const T*>(g_->slots[q].red.data())[k];
        h[k] = s;
    }
    g_->barrier();  // everyone read every slot
    SKY_CUDA(cudaMemcpyAsync(buf, h, bytes, cudaMemcpyHostToDevice, st));
    SKY_CUDA(cudaStreamSynchronize(st));  // the staging is reused by the next call
}

void LoopbackComm::allreduce_sum_u32(uint32_t* buf, size_t count, cudaStream_t st) { allreduce(buf, count, st); }
void LoopbackComm::allreduce_sum_u64(uint64_t* buf, size_t count, cudaStream_t st) { allreduce(buf, count, st); }
void LoopbackComm::allreduce_sum_f32(float* buf, size_t count, cudaStream_t st) { allreduce(buf, count, st); }

// =================================================================== NCCL
namespace {

class NcclComm final : public Comm {
   public:
    NcclComm(ncclComm_t c, int rank, int world) : Comm(rank, world), c_(c) {}
    ~NcclComm() override {
        if (c_) ncclCommDestroy(c_);
    }
    void allreduce_sum_u32(uint32_t* buf, size_t count, cudaStream_t st) override {
        if (count) SKY_NCCL_CALL(ncclAllReduce(buf, buf, count, ncclUint32, ncclSum, c_, st));
    }
    void allreduce_sum_u64(uint64_t* buf, size_t count, cudaStream_t st) override {
        if (count) SKY_NCCL_CALL(ncclAllReduce(buf, buf, count, ncclUint64, ncclSum, c_, st));
    }
    void allreduce_sum_f32(float* buf, size_t count, cudaStream_t st) override {
        if (count) SKY_NCCL_CALL(ncclAllReduce(buf, buf, count, ncclFloat32, ncclSum, c_, st));
    }
    // point-to-point over NVLink: every rank sends its block to each peer
    void allgatherv(const void* send, void* recv, const size_t* bytes, const size_t* displ,
                    cudaStream_t st) override {
        char* r = static_cast<char*>(recv);
        if (bytes[rank_] && r + displ[rank_] != send)
            SKY_CUDA(cudaMemcpyAsync(r + displ[rank_], send, bytes[rank_], cudaMemcpyDeviceToDevice, st));
        SKY_NCCL_CALL(ncclGroupStart());
        for (int q = 0; q < world_; ++q) {
            if (q == rank_) continue;
            if (bytes[rank_]) SKY_NCCL_CALL(ncclSend(send, bytes[rank_], ncclUint8, q, c_, st));
            if (bytes[q]) SKY_NCCL_CALL(ncclRecv(r + displ[q], bytes[q], ncclUint8, q, c_, st));
        }
        SKY_NCCL_CALL(ncclGroupEnd());
    }
    void alltoallv(const void* send, const size_t* sbytes, const size_t* sdispl, void* recv, const size_t* rbytes,
                   const size_t* rdispl, cudaStream_t st) override {
        const char* s = static_cast<const char*>(send);
        char* r = static_cast<char*>(recv);
        if (sbytes[rank_])
            SKY_CUDA(cudaMemcpyAsync(r + rdispl[rank_], s + sdispl[rank_], sbytes[rank_], cudaMemcpyDeviceToDevice,
                                     st));
        SKY_NCCL_CALL(ncclGroupStart());
        for (int q = 0; q < world_; ++q) {
            if (q == rank_) continue;
            if (sbytes[q]) SKY_NCCL_CALL(ncclSend(s + sdispl[q], sbytes[q], ncclUint8, q, c_, st));
            if (rbytes[q]) SKY_NCCL_CALL(ncclRecv(r + rdispl[q], rbytes[q], ncclUint8, q, c_, st));
        }
        SKY_NCCL_CALL(ncclGroupEnd());
    }
    void abort() override {
        if (c_) ncclCommAbort(c_);
        c_ = nullptr;
    }
    const char* backend() const override { return "nccl"; }

   private:
    ncclComm_t c_;
};

}  // namespace

std::unique_ptr<Comm> make_nccl_comm(int device, int rank, int world, const void* unique_id) {
    SKY_CUDA(cudaSetDevice(device));
    ncclUniqueId id;
    std::memcpy(&id, unique_id, sizeof(id));
    ncclComm_t c = nullptr;
    SKY_NCCL_CALL(ncclCommInitRank(&c, world, id, rank));
    return std::make_unique<NcclComm>(c, rank, world);
}

std::vector<std::unique_ptr<Comm>> make_nccl_comms(const std::vector<int>& devices) {
    const int W = (int)devices.size();
    std::vector<ncclComm_t> cs(W, nullptr);
    SKY_NCCL_CALL(ncclCommInitAll(cs.data(), W, devices.data()));
    std::vector<std::unique_ptr<Comm>> out;
    for (int r = 0; r < W; ++r) out.push_back(std::make_unique<NcclComm>(cs[r], r, W));
    return out;
}

size_t nccl_unique_id_bytes() { return sizeof(ncclUniqueId); }

void nccl_unique_id(void* out) {
    ncclUniqueId id;
    SKY_NCCL_CALL(ncclGetUniqueId(&id));
    std::memcpy(out, &id, sizeof(id));
}

}  // namespace sky
