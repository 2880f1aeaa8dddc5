// common.cuh — shared types, error plumbing and the device arena.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/skyline_b200.h"

namespace sky {

// Error carried from the engine to the C ABI; `code` is a sky_status.
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define SKY_CUDA(call)                                                                  \
    do {                                                                                \
        cudaError_t e_ = (call);                                                        \
        if (e_ != cudaSuccess)                                                          \
            throw ::sky::Error(SKY_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

#define SKY_LAUNCH_CHECK() SKY_CUDA(cudaGetLastError())

constexpr uint32_t kNone = 0xFFFFFFFFu;
constexpr uint64_t kMaxPartitions = uint64_t{1} << 22;  // partition.cpp:13

// Device error bits raised by the prep pass (mapped to sky_status on host).
enum : uint32_t {
    kErrNonFinite = 1u,     // make_dataset (core.cpp:32-36): finite and >= 0
    kErrAboveOne = 2u,      // normalized dataset with x > 1 (core.cpp:38-41)
    kErrGridRange = 4u,     // cell_of: x outside [0,1] (partition.cpp:26-29)
};

// One relsky work item: candidates [cb, ce) are tested against every
// comparator range listed in ranges[lb, le) (each range sorted by skey).
struct Item {
    uint32_t cb, ce, lb, le;
};

// Grow-only device buffers keyed by slot; reused across runs so the timed
// loop never allocates. A slot that grows during a run keeps its old buffer
// alive until the next run starts (retire()), so a pointer taken earlier in
// the run stays valid whatever later code asks of the same slot.
class Arena {
   public:
    ~Arena() { release(); }
    void* get(int slot, size_t bytes) {
        if (slot >= (int)bufs_.size()) bufs_.resize(slot + 1);
        Buf& b = bufs_[slot];
        if (b.cap < bytes) {
            if (b.ptr) retired_.push_back(b.ptr);
            b.ptr = nullptr;
            size_t cap = bytes + bytes / 4 + 256;
            SKY_CUDA(cudaMalloc(&b.ptr, cap));
            b.cap = cap;
        }
        return b.ptr;
    }
    // free the buffers replaced during the previous run (its work has drained)
    void retire() {
        for (void* p : retired_) cudaFree(p);
        retired_.clear();
    }
    template <class T>
    T* as(int slot, size_t n) {
        return static_cast<T*>(get(slot, n * sizeof(T) + 16));
    }
    void release() {
        retire();
        for (Buf& b : bufs_)
            if (b.ptr) cudaFree(b.ptr);
        bufs_.clear();
    }

   private:
    struct Buf {
        void* ptr = nullptr;
        size_t cap = 0;
    };
    std::vector<Buf> bufs_;
    std::vector<void*> retired_;
};

// Pinned host staging buffers keyed by slot.
class PinnedArena {
   public:
    ~PinnedArena() {
        for (Buf& b : bufs_)
            if (b.ptr) cudaFreeHost(b.ptr);
    }
    void* get(int slot, size_t bytes) {
        if (slot >= (int)bufs_.size()) bufs_.resize(slot + 1);
        Buf& b = bufs_[slot];
        if (b.cap < bytes) {
            if (b.ptr) cudaFreeHost(b.ptr);
            b.ptr = nullptr;
            size_t cap = bytes + bytes / 4 + 256;
            SKY_CUDA(cudaMallocHost(&b.ptr, cap));
            b.cap = cap;
        }
        return b.ptr;
    }
    template <class T>
    T* as(int slot, size_t n) {
        return static_cast<T*>(get(slot, n * sizeof(T) + 16));
    }

   private:
    struct Buf {
        void* ptr = nullptr;
        size_t cap = 0;
    };
    std::vector<Buf> bufs_;
};

inline uint32_t ceil_div(uint64_t a, uint64_t b) { return static_cast<uint32_t>((a + b - 1) / b); }
inline int bits_for(uint64_t v) {  // bits needed to represent values < v
    int b = 0;
    while ((uint64_t{1} << b) < v) ++b;
    return b;
}

}  // namespace sky
