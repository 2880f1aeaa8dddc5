// small.cu — the fused tail of a stream-path run whose prefilter leaves few
// rows (C3: 965 of 10M, C5: 1 of 2M).
//
// After the representative prefilter (filter.cpp:147-159) the survivors S are
// packed (partition, truncated sum key, row) keys appended in arbitrary
// order. The general tail sorts them, lays them out per partition, runs the
// local skylines (engine.cpp:41-63) and the merge (engine.cpp:116-134), with
// host round trips to size each step. With at most kSmallCap survivors every
// result follows from one pass over the pairs of S, because
//   * the local skyline of partition p is {i in S_p : no j in S_p dominates i}
//     (core.hpp:89-96), so its size is a count per partition;
//   * every merge kind returns Sky(U) for the union U of the local skylines,
//     and Sky(U) = Sky(S): a row dominated within S is dominated by a row of
//     U (dominance is transitive and S is finite), and rows outside U are
//     dominated within S;
//   * the ascending ids are the final rows ordered by their rank among S.
// So the tail is two launches sized by the capacity (its flag words are
// cleared by the prefilter pass before it, else by one memset), every count
// staying on the device, and one round trip at the end:
//
//   k_small_pairs   tiles of 128 x 32 pairs (i, j) of S over resident CTAs: row
//                   i is locally dead when a row j of its partition dominates
//                   it, dead when any row j does; rank_i += #{j : row_j <
//                   row_i}. Only j with key_j <= key_i are tested (the sum key
//                   is monotone under dominance).
//   k_small_finish  one CTA: local skyline sizes per partition and their
//                   offsets (the union's layout), |U|, and the final rows
//                   written in rank order to mapped pinned host memory,
//                   with the run's counter words and the offsets (so the
//                   host reads everything after one synchronize).
//
// Both kernels read the device count and return at once when it exceeds the
// capacity; the host then continues with the general tail on the same
// survivors (nothing here writes them).
#include <cstdint>

#include "dom.cuh"
#include "kernels.cuh"

namespace sky {

namespace {

#define SKY_DISPATCH_DOM(D, ...)                                \
    switch (D) {                                                \
        case 2: { constexpr int DT = 2; __VA_ARGS__; break; }   \
        case 3: { constexpr int DT = 3; __VA_ARGS__; break; }   \
        case 4: { constexpr int DT = 4; __VA_ARGS__; break; }   \
        case 5: { constexpr int DT = 5; __VA_ARGS__; break; }   \
        case 6: { constexpr int DT = 6; __VA_ARGS__; break; }   \
        case 8: { constexpr int DT = 8; __VA_ARGS__; break; }   \
        case 10: { constexpr int DT = 10; __VA_ARGS__; break; } \
        case 12: { constexpr int DT = 12; __VA_ARGS__; break; } \
        case 16: { constexpr int DT = 16; __VA_ARGS__; break; } \
        default: throw Error(SKY_E_INTERNAL, "small tail needs D <= 16"); \
    }

constexpr uint32_t kPairRows = 128;       // rows i of a pair tile (one per thread)
constexpr uint32_t kPairCols = 32;        // rows j of a pair tile (staged in shared memory)
constexpr uint32_t kPairCtasPerSm = 4;
constexpr uint32_t kFinishThreads = 1024;

struct Unpacked {
    uint32_t row, pid, key;
};

// packed = ((pid << 32 | skey) >> key_shift) << row_bits | row
__device__ __forceinline__ Unpacked unpack(uint64_t k, const SmallTail& t) {
    const uint32_t pid_shift = t.row_bits + 32 - t.key_shift;  // <= 64
    const uint32_t kbits = 32 - t.key_shift;                   // <= 32
    Unpacked u;
    u.row = (uint32_t)(k & ((1ull << t.row_bits) - 1));
    u.pid = pid_shift < 64 ? (uint32_t)(k >> pid_shift) : 0u;
    u.key = (uint32_t)((k >> t.row_bits) & ((1ull << kbits) - 1));
    return u;
}

template <int D>
__device__ __forceinline__ void load_row(const SmallTail& t, uint32_t row, float4* x) {
    constexpr int V = Dims2<D>::V;
    const float* p = t.pts + (size_t)row * t.d;
#pragma unroll
    for (int v = 0; v < V; ++v) {
        float c[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) c[q] = (uint32_t)(4 * v + q) < t.d ? __ldg(p + 4 * v + q) : 0.0f;
        x[v] = make_float4(c[0], c[1], c[2], c[3]);
    }
}

__device__ __forceinline__ unsigned long long warp_total(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

template <int D>
__global__ void __launch_bounds__(kPairRows) k_small_pairs(SmallTail t) {
    constexpr int V = Dims2<D>::V;
    const uint32_t ns = *t.count;
    if (ns > t.cap) return;
    __shared__ float4 s_x[kPairCols * V];
    __shared__ uint32_t s_p[kPairCols], s_k[kPairCols], s_r[kPairCols];
    uint32_t* ld = t.flags;
    uint32_t* gd = t.flags + t.cap;
    uint32_t* rk = t.flags + 2 * t.cap;
    const uint32_t ni = (ns + kPairRows - 1) / kPairRows, nj = (ns + kPairCols - 1) / kPairCols;
    unsigned long long nt = 0;
    // CTA-uniform walk over the (row tile, column tile) pairs
    for (uint32_t tile = blockIdx.x; tile < ni * nj; tile += gridDim.x) {
        const uint32_t i0 = (tile % ni) * kPairRows, j0 = (tile / ni) * kPairCols;
        const uint32_t jn = min(ns - j0, kPairCols);
        __syncthreads();  // the previous tile's columns are consumed
        if (threadIdx.x < jn) {
            const Unpacked u = unpack(t.surv[j0 + threadIdx.x], t);
            s_p[threadIdx.x] = u.pid;
            s_k[threadIdx.x] = u.key;
            s_r[threadIdx.x] = u.row;
            load_row<D>(t, u.row, s_x + threadIdx.x * V);
        }
        __syncthreads();
        const uint32_t i = i0 + threadIdx.x;
        if (i >= ns) continue;
        const Unpacked me = unpack(t.surv[i], t);
        float4 xi[V];
        load_row<D>(t, me.row, xi);
        bool dead = false, ldead = false;
        uint32_t rank = 0;
        for (uint32_t q = 0; q < jn; ++q) {
            rank += s_r[q] < me.row ? 1u : 0u;
            const bool same = s_p[q] == me.pid;
            // once dead, only a dominator of the own partition still matters
            if (s_k[q] > me.key || ldead || (dead && !same)) continue;
            ++nt;
            if (dom_f4<D>(s_x + q * V, xi)) {
                dead = true;
                ldead = same;
            }
        }
        if (ldead) ld[i] = 1;
        if (dead) gd[i] = 1;
        if (rank) atomicAdd(rk + i, rank);
    }
    if (t.tests) {
        nt = warp_total(nt);
        if ((threadIdx.x & 31) == 0 && nt) atomicAdd(t.tests, nt);
    }
}

// block-wide exclusive scan of one value per thread; *total = the sum
__device__ __forceinline__ uint32_t block_scan(uint32_t v, uint32_t* s_warp, uint32_t* total) {
    const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    uint32_t inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if ((int)lane >= o) inc += y;
    }
    if (lane == 31) s_warp[wid] = inc;
    __syncthreads();
    uint32_t before = 0, all = 0;
    for (uint32_t w = 0; w < nw; ++w) {
        const uint32_t c = s_warp[w];
        before += w < wid ? c : 0u;
        all += c;
    }
    __syncthreads();  // s_warp is reused by the next call
    *total = all;
    return before + inc - v;
}

// the host's copy of the run's counter words and union offsets, written
// into mapped pinned memory (no copies after the kernel)
__device__ __forceinline__ void publish_counters(const SmallTail& t) {
    for (uint32_t k = threadIdx.x; k < kSmallMiscWords; k += blockDim.x) t.hmisc[k] = t.misc[k];
    if (t.hoffu)
        for (uint32_t p = threadIdx.x; p <= t.P; p += blockDim.x) t.hoffu[p] = t.offu[p];
}

__global__ void __launch_bounds__(kFinishThreads) k_small_finish(SmallTail t) {
    const uint32_t ns = *t.count;
    if (ns > t.cap) {
        publish_counters(t);  // the general tail goes on from these
        return;
    }
    extern __shared__ uint32_t s_pos[];  // cap words: final row by rank, or ~0
    __shared__ uint32_t s_warp[kFinishThreads / 32];
    const uint32_t* ld = t.flags;
    const uint32_t* gd = t.flags + t.cap;
    const uint32_t* rk = t.flags + 2 * t.cap;
    for (uint32_t p = threadIdx.x; p < t.P; p += blockDim.x) t.cnt[p] = 0;
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < ns; i += blockDim.x) {
        const Unpacked u = unpack(t.surv[i], t);
        s_pos[rk[i]] = gd[i] ? 0xFFFFFFFFu : u.row;  // ranks are a permutation of [0, ns)
        if (!ld[i]) atomicAdd(t.cnt + u.pid, 1u);
    }
    __syncthreads();
    // final rows in rank (= ascending row) order
    uint32_t run = 0;
    for (uint32_t b = 0; b < ns; b += blockDim.x) {
        const uint32_t i = b + threadIdx.x;
        const uint32_t r = i < ns ? s_pos[i] : 0xFFFFFFFFu;
        uint32_t tot;
        const uint32_t at = run + block_scan(r != 0xFFFFFFFFu ? 1u : 0u, s_warp, &tot);
        if (r != 0xFFFFFFFFu) t.hid[at] = r;
        run += tot;
    }
    // union offsets: exclusive scan of the local skyline sizes
    uint32_t u = 0;
    for (uint32_t b = 0; b < t.P; b += blockDim.x) {
        const uint32_t p = b + threadIdx.x;
        const uint32_t c = p < t.P ? t.cnt[p] : 0u;
        uint32_t tot;
        const uint32_t at = u + block_scan(c, s_warp, &tot);
        if (p < t.P) t.offu[p] = at;
        u += tot;
    }
    if (threadIdx.x == 0) {
        t.offu[t.P] = u;
        *t.u_count = u;
        *t.total = run;
    }
    __syncthreads();
    publish_counters(t);
}

}  // namespace

void launch_small_tail(int D, const SmallTail& t, cudaStream_t st) {
    if (!t.flags_zeroed) SKY_CUDA(cudaMemsetAsync(t.flags, 0, (size_t)3 * t.cap * sizeof(uint32_t), st));
    const uint32_t grid = kPairCtasPerSm * (uint32_t)device_sm_count();
    SKY_DISPATCH_DOM(D, (k_small_pairs<DT><<<grid, kPairRows, 0, st>>>(t)));
    const size_t smem = (size_t)t.cap * sizeof(uint32_t);
    k_small_finish<<<1, kFinishThreads, smem, st>>>(t);
    SKY_LAUNCH_CHECK();
}

}  // namespace sky
