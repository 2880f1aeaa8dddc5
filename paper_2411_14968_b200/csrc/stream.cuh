// stream.cuh — persistent row-tile streaming for the HBM-bound passes.
//
// Rows are float32, row-major n x d. A CTA walks tiles of stream_tile_rows(d) rows
// (tile t, t + gridDim.x, ...); each tile is one contiguous span, copied
// global -> shared memory by the bulk-copy engine (cp.async.bulk, completion
// counted on an mbarrier), kStreamStages tiles in flight per CTA, so the SMs
// keep enough bytes in flight to stream at HBM rate while they compute on the
// current tile. A CTA has kStreamThreads threads; thread i takes rows
// i, i + kStreamThreads, ... of a tile (the per-tile wait, barrier and copy
// issue are shared by the tile rows / kStreamThreads rows per thread).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace sky {

constexpr uint32_t kStreamThreads = 256;  // threads per CTA
constexpr uint32_t kStreamStages = 2;     // tiles in flight per CTA
// rows per tile: two per thread while a stage stays <= 32 KB
__host__ __device__ constexpr uint32_t stream_tile_rows(uint32_t d) {
    return d <= 16 ? 2 * kStreamThreads : kStreamThreads;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// global -> shared bulk copy (16-byte aligned addresses, size % 16 == 0)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// Shared memory of the ring: kStreamStages stages of (tile rows * d
// floats [+ tile rows u64 of the optional per-row aux array]), then the
// barriers.
__host__ __device__ inline size_t stream_stage_bytes(uint32_t d, bool aux) {
    const size_t tr = stream_tile_rows(d);
    return tr * d * sizeof(float) + (aux ? tr * sizeof(uint64_t) : 0);
}
__host__ __device__ inline size_t stream_smem_bytes(uint32_t d, bool aux = false) {
    return (size_t)kStreamStages * stream_stage_bytes(d, aux) + kStreamStages * sizeof(uint64_t) + 16;
}

// Walk this CTA's tiles (stream_tile_rows(d) rows each). `body(tile, row0, nrows, aux_tile)` runs on every
// thread with the tile's rows in shared memory (row r of the tile at
// tile + r * d) and, if `aux` is given, aux[row0 .. row0 + nrows) at
// aux_tile; it must not call __syncthreads. `smem` is 16-byte aligned,
// stream_smem_bytes(d, aux != nullptr) long; pts and aux 16-byte aligned.
template <class Body>
__device__ __forceinline__ void stream_row_tiles(const float* __restrict__ pts, uint32_t n, uint32_t d, char* smem,
                                                 Body&& body, const uint64_t* __restrict__ aux = nullptr) {
    const size_t stage_bytes = stream_stage_bytes(d, aux != nullptr);
    const uint32_t TR = stream_tile_rows(d);
    const size_t row_bytes = (size_t)TR * d * sizeof(float);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kStreamStages * stage_bytes);
    const uint32_t tiles = (n + TR - 1) / TR;
    const uint32_t tid = threadIdx.x;
    if (tid == 0) {
        for (uint32_t s = 0; s < kStreamStages; ++s) mbar_init(bars + s, 1);
        mbar_fence_init();
    }
    __syncthreads();
    // the bulk copies take the 16-byte multiples of a tile; the few words of
    // an odd-sized last tile past them are loaded by the threads
    auto issue = [&](uint32_t t, uint32_t s) {
        const uint32_t r0 = t * TR;
        const uint32_t nr = min(TR, n - r0);
        const uint32_t bytes = (nr * d * (uint32_t)sizeof(float)) & ~15u;
        const uint32_t abytes = aux ? (nr * (uint32_t)sizeof(uint64_t)) & ~15u : 0u;
        char* st = smem + s * stage_bytes;
        mbar_arrive_expect_tx(bars + s, bytes + abytes);
        if (bytes) bulk_g2s(st, pts + (size_t)r0 * d, bytes, bars + s);
        if (abytes) bulk_g2s(st + row_bytes, aux + r0, abytes, bars + s);
    };
    if (tid == 0)
        for (uint32_t s = 0; s < kStreamStages; ++s) {
            const uint32_t t = blockIdx.x + s * gridDim.x;
            if (t < tiles) issue(t, s);
        }
    for (uint32_t it = 0;; ++it) {
        const uint32_t t = blockIdx.x + it * gridDim.x;
        if (t >= tiles) break;
        const uint32_t s = it % kStreamStages;
        mbar_wait(bars + s, (it / kStreamStages) & 1u);
        char* st = smem + s * stage_bytes;
        float* tile = reinterpret_cast<float*>(st);
        uint64_t* atile = aux ? reinterpret_cast<uint64_t*>(st + row_bytes) : nullptr;
        const uint32_t r0 = t * TR;
        const uint32_t nr = min(TR, n - r0);
        const uint32_t nf = nr * d, done = (nf * (uint32_t)sizeof(float) & ~15u) / (uint32_t)sizeof(float);
        const uint32_t adone = (nr * (uint32_t)sizeof(uint64_t) & ~15u) / (uint32_t)sizeof(uint64_t);
        if (done != nf || (aux && adone != nr)) {  // last tile only (uniform branch)
            for (uint32_t k = done + tid; k < nf; k += blockDim.x) tile[k] = pts[(size_t)r0 * d + k];
            if (aux)
                for (uint32_t k = adone + tid; k < nr; k += blockDim.x) atile[k] = aux[r0 + k];
            __syncthreads();
        }
        body(tile, r0, nr, atile);
        __syncthreads();  // stage s is free again
        const uint32_t tn = t + kStreamStages * gridDim.x;
        if (tid == 0 && tn < tiles) issue(tn, s);
    }
}

}  // namespace sky
