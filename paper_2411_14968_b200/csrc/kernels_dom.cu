// kernels_dom.cu — the packed-code dominance core for sm_100a.
//
// Every point carries, besides its float coordinates, a monotone code per
// dimension (q(x) = number of per-dimension quantile thresholds <= x, reduced
// to b bits), packed into exactly two 32-bit words: word w holds dimensions
// [w*L, (w+1)*L), L = ceil(D/2), each in a lane of 32/L bits whose top bit is
// a guard (b = min(7, 32/L - 1): 7 bits up to D=8, 5 at D=10, 4 at D=12, 3 at
// D=16). For a candidate t the words carry all guard bits set (t' = q(t)|G);
// for a comparator s, t' - s keeps lane j's guard set iff q(t_j) >= q(s_j),
// and no lane ever borrows from its neighbour. A clear guard proves
// s_j > t_j, so s cannot dominate t; only pairs with every guard set go to the
// exact float test of core.hpp:89-96. Per pair: 2 IMAD.IADD (FMA pipe) + one
// LOP3 and one predicate-accumulating ISETP (ALU pipe), instead of D FP32
// compares on the ALU pipe.
//
// Work distribution: persistent warps pull host-planned items (<= 256
// candidates x comparator ranges) from an atomic counter in launch order.
#include <algorithm>

#include "kernels.cuh"

namespace sky {

namespace {

template <int D>
struct Dims2 {
    static constexpr int V = (D + 3) / 4;  // float4 per row == code words
};

__device__ __forceinline__ unsigned long long warp_sum(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Two-word code layout for D dimensions (see the file comment).
// Bit 31 of both words is never part of a lane; in word 0 it is the "alive"
// guard: set in t' while the candidate is alive, cleared when it is dominated
// (or the slot is empty), so a dead slot can never pass the coarse test.
template <int D>
struct CodeLayout {
    static constexpr int L = (D + 1) / 2;                     // lanes per word
    static constexpr int LW = 31 / L;                          // lane width in bits
    static constexpr int B = (LW - 1) < 7 ? (LW - 1) : 7;      // code bits
    static constexpr uint32_t G = [] {                         // lane guard bits
        uint32_t g = 0;
        for (int i = 0; i < L; ++i) g |= 1u << (i * LW + LW - 1);
        return g;
    }();
    static constexpr uint32_t ALIVE = 0x80000000u;
};

constexpr int kSample = 4096;
constexpr int kThr = kCodeLevels - 1;  // 127 thresholds per dimension

// One CTA per dimension: sort a strided sample of the column and keep 127
// quantiles as thresholds.
template <int D>
__global__ void __launch_bounds__(512) k_thresholds(DevSet s, float* thr) {
    constexpr int D4 = Dims2<D>::V * 4;
    __shared__ float v[kSample];
    const int j = blockIdx.x;
    const uint32_t S = s.n < (uint32_t)kSample ? s.n : (uint32_t)kSample;
    for (int i = threadIdx.x; i < kSample; i += blockDim.x) {
        float x = __int_as_float(0x7f800000);  // +inf padding
        if ((uint32_t)i < S) {
            const uint64_t row = (uint64_t)i * s.n / S;
            x = s.xyz[row * D4 + j];
        }
        v[i] = x;
    }
    __syncthreads();
    // bitonic sort of kSample floats
    for (int k = 2; k <= kSample; k <<= 1) {
        for (int jj = k >> 1; jj > 0; jj >>= 1) {
            for (int i = threadIdx.x; i < kSample; i += blockDim.x) {
                const int p = i ^ jj;
                if (p > i) {
                    const float a = v[i], b = v[p];
                    const bool up = (i & k) == 0;
                    if ((a > b) == up) {
                        v[i] = b;
                        v[p] = a;
                    }
                }
            }
            __syncthreads();
        }
    }
    for (int k = threadIdx.x; k < kThr; k += blockDim.x) {
        uint32_t idx = S ? (uint32_t)(((uint64_t)(k + 1) * S) / kCodeLevels) : 0;
        if (idx >= S) idx = S ? S - 1 : 0;
        thr[j * kThr + k] = S ? v[idx] : 0.0f;
    }
}

template <int D>
__global__ void __launch_bounds__(256) k_encode(DevSet s, const float* __restrict__ thr) {
    constexpr int V = Dims2<D>::V;
    __shared__ float t[D * kThr];
    for (int i = threadIdx.x; i < D * kThr; i += blockDim.x) t[i] = thr[i];
    __syncthreads();
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= s.n) return;
    const float4* x4 = reinterpret_cast<const float4*>(s.xyz) + (size_t)i * V;
    float x[4 * V];
#pragma unroll
    for (int v = 0; v < V; ++v) {
        const float4 q = x4[v];
        x[4 * v] = q.x;
        x[4 * v + 1] = q.y;
        x[4 * v + 2] = q.z;
        x[4 * v + 3] = q.w;
    }
    constexpr int L = CodeLayout<D>::L, LW = CodeLayout<D>::LW, B = CodeLayout<D>::B;
    uint32_t w[2] = {0, 0};
#pragma unroll
    for (int j = 0; j < D; ++j) {
        // upper_bound over the 127 sorted thresholds of dimension j
        const float* tj = t + j * kThr;
        int lo = 0, hi = kThr;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (tj[mid] <= x[j]) lo = mid + 1; else hi = mid;
        }
        w[j / L] |= ((uint32_t)lo >> (7 - B)) << (LW * (j % L));
    }
    s.qc[i] = make_uint2(w[0], w[1]);
}

// q(s_j) <= q(t_j) on every lane of both words, and t alive (t' carries the
// lane guards in both words and the alive guard in word 0)
template <uint32_t G>
__device__ __forceinline__ bool coarse_pass(const uint32_t (&t)[2], const uint2& s) {
    constexpr uint32_t GA = G | 0x80000000u;  // t'[1] always carries bit 31
    return ((t[0] - s.x) & (t[1] - s.y) & GA) == GA;
}

constexpr int RS3_WARPS = 8;
constexpr int RS3_THREADS = RS3_WARPS * 32;

template <int D>
__device__ __forceinline__ bool dominates_exact(const float4* __restrict__ s, const float4* __restrict__ t) {
    constexpr int V = Dims2<D>::V;
    bool gt = false, lt = false;
#pragma unroll
    for (int v = 0; v < V; ++v) {
        const float4 a = s[v], b = t[v];
        gt |= (a.x > b.x) | (a.y > b.y) | (a.z > b.z) | (a.w > b.w);
        lt |= (a.x < b.x) | (a.y < b.y) | (a.z < b.z) | (a.w < b.w);
    }
    return !gt && lt;
}

// Comparator range end: plain, or (flag bit) the current length of a
// device-side window counter (windowed SFS).
__device__ __forceinline__ uint32_t range_end(const Relsky2Args& a, uint2 rg) {
    return (rg.y & 0x80000000u) ? rg.x + a.wcount[rg.y & 0x7FFFFFFFu] : rg.y;
}

// Warp-autonomous dominance core: every warp fetches its own item
// (<= 32*K candidates, lane l owns candidates cb + 32k + l), streams the
// comparator ranges 32 at a time through its private shared-memory slot
// (codes, keys and coordinates of the next batch are prefetched into
// registers while the current one is tested), stops a range when a ballot
// shows the sorted keys passed the warp's bound and leaves the item once every
// candidate is dominated. Exact checks read both points from shared memory.
// No CTA barriers.
template <int D, int K>
struct Relsky3Smem {
    static constexpr int V = Dims2<D>::V;
    float4 cand[K][V][32];  // [k][v][lane]: conflict-free per-lane reads
    float4 comp[32][V];     // current comparator batch (broadcast reads)
    uint2 code[32];
};

template <int D, int K>
__global__ void __launch_bounds__(RS3_THREADS, 2) k_relsky3(Relsky2Args a) {
    constexpr int W = Dims2<D>::V;
    constexpr uint32_t G = CodeLayout<D>::G;
    constexpr uint32_t FULL = 0xffffffffu;
    extern __shared__ float4 smem_raw[];
    using S = Relsky3Smem<D, K>;

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    S& sm = reinterpret_cast<S*>(smem_raw)[warp];
    unsigned long long ntests = 0, nhits = 0;

    for (;;) {
        uint32_t item = 0;
        if (lane == 0) item = atomicAdd(a.counter, 1u);
        item = __shfl_sync(FULL, item, 0);
        if (item >= a.n_items) break;
        const Item it = a.items[item];

        uint32_t T[K][2];
        uint32_t alive = 0, my_max = 0;
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const uint32_t c = it.cb + k * 32 + lane;
            // empty / dead slot: lane guards set (no borrow can reach bit 31),
            // alive guard clear -> never passes
            T[k][0] = G;
            T[k][1] = G | 0x80000000u;
            if (c < it.ce && !a.dead[c]) {
                alive |= 1u << k;
                const uint2 q = a.cqc[c];
                T[k][0] = q.x | G | CodeLayout<D>::ALIVE;
                T[k][1] = q.y | G | 0x80000000u;
                my_max = max(my_max, a.cskey[c]);
                const float4* x = reinterpret_cast<const float4*>(a.cxyz) + (size_t)c * W;
#pragma unroll
                for (int v = 0; v < W; ++v) sm.cand[k][v][lane] = x[v];
            }
        }
        const uint32_t initial = alive;
        const uint32_t bound = a.bounded ? __reduce_max_sync(FULL, my_max) : 0xFFFFFFFFu;
        bool live = __any_sync(FULL, alive != 0);

        for (uint32_t r = it.lb; live && r < it.le; ++r) {
            const uint2 rg = a.ranges[r];
            const uint32_t sb = rg.x, se = range_end(a, rg);
            // prefetch the first batch
            uint32_t idx = sb + lane;
            uint2 nq = make_uint2(0, 0);
            uint32_t nk = 0xFFFFFFFFu;
            float4 nx[W];
            if (idx < se) {
                nq = a.sqc[idx];
                nk = a.sskey[idx];
                const float4* x = reinterpret_cast<const float4*>(a.sxyz) + (size_t)idx * W;
#pragma unroll
                for (int v = 0; v < W; ++v) nx[v] = x[v];
            }
            for (uint32_t base = sb; base < se; base += 32) {
                const uint32_t inb = __ballot_sync(FULL, nk <= bound);  // prefix (keys sorted)
                const uint32_t lim = __popc(inb);
                __syncwarp();
                sm.code[lane] = nq;
#pragma unroll
                for (int v = 0; v < W; ++v) sm.comp[lane][v] = nx[v];
                __syncwarp();
                idx = base + 32 + lane;
                if (lim == 32 && idx < se) {
                    nq = a.sqc[idx];
                    nk = a.sskey[idx];
                    const float4* x = reinterpret_cast<const float4*>(a.sxyz) + (size_t)idx * W;
#pragma unroll
                    for (int v = 0; v < W; ++v) nx[v] = x[v];
                } else {
                    nk = 0xFFFFFFFFu;
                }
                for (uint32_t i = 0; i < lim; ++i) {
                    const uint2 q = sm.code[i];
                    bool none = true;
#pragma unroll
                    for (int k = 0; k < K; ++k) none &= !coarse_pass<G>(T[k], q);
                    if (!none) {
                        // exact test (core.hpp:89-96) where the codes could not rule s out
#pragma unroll
                        for (int k = 0; k < K; ++k) {
                            if (coarse_pass<G>(T[k], q)) {
                                ++nhits;
                                bool gt = false, lt = false;
#pragma unroll
                                for (int v = 0; v < W; ++v) {
                                    const float4 sa = sm.comp[i][v], tb = sm.cand[k][v][lane];
                                    gt |= (sa.x > tb.x) | (sa.y > tb.y) | (sa.z > tb.z) | (sa.w > tb.w);
                                    lt |= (sa.x < tb.x) | (sa.y < tb.y) | (sa.z < tb.z) | (sa.w < tb.w);
                                }
                                if (!gt && lt) {
                                    alive &= ~(1u << k);
                                    T[k][0] &= ~CodeLayout<D>::ALIVE;
                                    ntests += i + 1;
                                }
                            }
                        }
                    }
                }
                ntests += (unsigned long long)__popc(alive) * lim;
                live = __any_sync(FULL, alive != 0);
                if (!live || lim < 32) break;  // all dominated, or past the key bound
            }
        }
        uint32_t killed = initial & ~alive;
        while (killed) {
            const int k = __ffs(killed) - 1;
            killed &= killed - 1;
            a.dead[it.cb + k * 32 + lane] = 1;
        }
    }
    if (a.tests) {
        ntests = warp_sum(ntests);
        if (lane == 0 && ntests) atomicAdd(a.tests, ntests);
    }
    if (a.coarse_hits) {
        nhits = warp_sum(nhits);
        if (lane == 0 && nhits) atomicAdd(a.coarse_hits, nhits);
    }
}

#define SKY_DISPATCH_D16(D, ...)                                \
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
        default: throw Error(SKY_E_INTERNAL, "packed-code kernel needs D <= 16"); \
    }

template <int D, int K>
void launch_k(const Relsky2Args& a, int sm_count, cudaStream_t st) {
    static int per_sm = 0;
    const size_t smem = sizeof(Relsky3Smem<D, K>) * RS3_WARPS;
    if (!per_sm) {
        SKY_CUDA(cudaFuncSetAttribute(k_relsky3<D, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        SKY_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_relsky3<D, K>, RS3_THREADS, smem));
        if (per_sm < 1) per_sm = 1;
    }
    const uint64_t warps = std::min<uint64_t>(a.n_items, (uint64_t)per_sm * sm_count * RS3_WARPS);
    const uint32_t grid = (uint32_t)((warps + RS3_WARPS - 1) / RS3_WARPS);
    k_relsky3<D, K><<<grid, RS3_THREADS, smem, st>>>(a);
    SKY_LAUNCH_CHECK();
}

}  // namespace

void launch_thresholds(int D, const DevSet& s, float* thr, cudaStream_t st) {
    if (!s.n) return;
    SKY_DISPATCH_D16(D, (k_thresholds<DT><<<DT, 512, 0, st>>>(s, thr)));
    SKY_LAUNCH_CHECK();
}

void launch_encode(int D, const DevSet& s, const float* thr, cudaStream_t st) {
    if (!s.n) return;
    SKY_DISPATCH_D16(D, (k_encode<DT><<<ceil_div(s.n, 256), 256, 0, st>>>(s, thr)));
    SKY_LAUNCH_CHECK();
}

void launch_relsky2(int D, int tile, const Relsky2Args& a, int sm_count, cudaStream_t st) {
    if (!a.n_items) return;
    if (tile <= 4 * 32) {
        SKY_DISPATCH_D16(D, (launch_k<DT, 4>(a, sm_count, st)));
    } else if (tile <= 8 * 32) {
        SKY_DISPATCH_D16(D, (launch_k<DT, 8>(a, sm_count, st)));
    } else {
        throw Error(SKY_E_INTERNAL, "relsky item larger than one warp's candidates");
    }
}

}  // namespace sky
