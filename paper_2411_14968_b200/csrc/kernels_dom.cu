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
// Work distribution: persistent CTAs pull host-planned items (candidate tile
// x comparator ranges) from an atomic counter in launch order; comparator
// tiles are staged in shared memory and broadcast; every warp stops a range
// at its own coordinate-sum-key bound (a warp-uniform binary search per tile)
// and as soon as all its candidates are dominated.
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
template <int D>
struct CodeLayout {
    static constexpr int L = (D + 1) / 2;                     // lanes per word
    static constexpr int LW = 32 / L;                          // lane width in bits
    static constexpr int B = (LW - 1) < 7 ? (LW - 1) : 7;      // code bits
    static constexpr uint32_t G = [] {                         // guard bits
        uint32_t g = 0;
        for (int i = 0; i < L; ++i) g |= 1u << (i * LW + LW - 1);
        return g;
    }();
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

// q(s_j) <= q(t_j) on every lane of both words (t' carries the guard bits)
template <uint32_t G>
__device__ __forceinline__ bool coarse_pass(const uint32_t (&t)[2], const uint2& s) {
    return ((t[0] - s.x) & (t[1] - s.y) & G) == G;
}

constexpr int RS2_THREADS = 128;
constexpr int RS2_TILE = 128;  // comparators per shared-memory tile

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

template <int D, int K>
__global__ void __launch_bounds__(RS2_THREADS) k_relsky2(Relsky2Args a, int tile) {
    constexpr int W = Dims2<D>::V;
    constexpr uint32_t G = CodeLayout<D>::G;
    __shared__ float4 s_xyz[RS2_TILE * W];
    __shared__ uint2 s_code[RS2_TILE];
    __shared__ uint32_t s_key[RS2_TILE];
    __shared__ uint32_t s_red[RS2_THREADS / 32];
    __shared__ uint32_t s_item, s_end;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int per_warp = (tile + 3) / 4;
    unsigned long long ntests = 0, nhits = 0;

    for (;;) {
        if (tid == 0) s_item = atomicAdd(a.counter, 1u);
        __syncthreads();
        const uint32_t item = s_item;
        if (item >= a.n_items) break;
        const Item it = a.items[item];

        // ---- candidates: warp w owns [w*per_warp, (w+1)*per_warp) of the tile
        uint32_t T[K][2];
        uint32_t alive = 0, my_max = 0;
        const uint32_t wbase = it.cb + warp * per_warp;
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const uint32_t off = k * 32 + lane;
            const uint32_t c = wbase + off;
            T[k][0] = T[k][1] = 0;
            if ((int)off < per_warp && c < it.ce && !a.dead[c]) {
                alive |= 1u << k;
                const uint2 q = a.cqc[c];
                T[k][0] = q.x | G;
                T[k][1] = q.y | G;
                my_max = max(my_max, a.cskey[c]);
            }
        }
        const uint32_t initial = alive;
        uint32_t warp_max = __reduce_max_sync(0xffffffffu, my_max);
        if (lane == 0) s_red[warp] = warp_max;
        __syncthreads();
        uint32_t cta_max = 0;
#pragma unroll
        for (int w = 0; w < RS2_THREADS / 32; ++w) cta_max = max(cta_max, s_red[w]);
        if (!a.bounded) warp_max = cta_max = 0xFFFFFFFFu;
        bool warp_alive = __any_sync(0xffffffffu, alive != 0);

        if (__syncthreads_or(alive != 0)) {
            for (uint32_t r = it.lb; r < it.le; ++r) {
                const uint2 rg = a.ranges[r];
                uint32_t sb = rg.x, se = rg.y;
                if (a.bounded) {
                    if (tid == 0) {
                        uint32_t lo = sb, hi = se;
                        while (lo < hi) {
                            const uint32_t mid = (lo + hi) >> 1;
                            if (a.sskey[mid] <= cta_max) lo = mid + 1; else hi = mid;
                        }
                        s_end = lo;
                    }
                    __syncthreads();
                    se = s_end;
                }
                bool warp_live = warp_alive;
                for (uint32_t base = sb; base < se; base += RS2_TILE) {
                    const uint32_t len = min((uint32_t)RS2_TILE, se - base);
                    __syncthreads();
                    {
                        const float4* src = reinterpret_cast<const float4*>(a.sxyz) + (size_t)base * W;
                        for (uint32_t i = tid; i < len * W; i += RS2_THREADS) s_xyz[i] = src[i];
                        for (uint32_t i = tid; i < len; i += RS2_THREADS) {
                            s_code[i] = a.sqc[base + i];
                            s_key[i] = a.sskey[base + i];
                        }
                    }
                    __syncthreads();
                    if (warp_live) {
                        // comparators of this tile inside the warp's key bound
                        uint32_t lo = 0, hi = len;
                        while (lo < hi) {
                            const uint32_t mid = (lo + hi) >> 1;
                            if (s_key[mid] <= warp_max) lo = mid + 1; else hi = mid;
                        }
                        const uint32_t lim = lo;
                        uint32_t i = 0;
                        const uint2* __restrict__ sc = s_code;
                        for (; i < lim; ++i) {
                            const uint2 q = sc[i];
                            // all guard bits set <=> (t' - s) | ~M == 0xFFFFFFFF in every word
                            bool none = true;
#pragma unroll
                            for (int k = 0; k < K; ++k) none &= !coarse_pass<G>(T[k], q);
                            if (!none) {
                                // exact test (core.hpp:89-96) for the pairs the codes could not rule out
                                const float4* sx = s_xyz + i * W;
#pragma unroll
                                for (int k = 0; k < K; ++k) {
                                    if ((alive >> k) & 1u) {
                                        if (coarse_pass<G>(T[k], q)) {
                                            ++nhits;
                                            const uint32_t c = wbase + k * 32 + lane;
                                            const float4* tx = reinterpret_cast<const float4*>(a.cxyz) + (size_t)c * W;
                                            if (dominates_exact<D>(sx, tx)) {
                                                alive &= ~(1u << k);
                                                ntests += i + 1;
                                            }
                                        }
                                    }
                                }
                            }
                            if ((i & 15) == 15 && !__any_sync(0xffffffffu, alive != 0)) {
                                ++i;
                                break;
                            }
                        }
                        ntests += (unsigned long long)__popc(alive) * i;
                        if (i < len) warp_live = false;  // key bound reached (sorted range)
                        warp_alive = __any_sync(0xffffffffu, alive != 0);
                        if (!warp_alive) warp_live = false;
                    }
                    if (!__syncthreads_or(warp_live)) break;
                }
                if (!__syncthreads_or(warp_alive)) break;
            }
        }
        uint32_t killed = initial & ~alive;
        while (killed) {
            const int k = __ffs(killed) - 1;
            killed &= killed - 1;
            a.dead[wbase + k * 32 + lane] = 1;
        }
        __syncthreads();  // s_item / s_red reuse
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
void launch_k(const Relsky2Args& a, int tile, int sm_count, cudaStream_t st) {
    static int per_sm = 0;
    if (!per_sm) {
        SKY_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_relsky2<D, K>, RS2_THREADS, 0));
        if (per_sm < 1) per_sm = 1;
    }
    const uint32_t grid = (uint32_t)std::min<uint64_t>(a.n_items, (uint64_t)per_sm * sm_count);
    k_relsky2<D, K><<<grid, RS2_THREADS, 0, st>>>(a, tile);
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
    if (tile <= 4 * 32 * 4) {
        SKY_DISPATCH_D16(D, (launch_k<DT, 4>(a, tile, sm_count, st)));
    } else {
        SKY_DISPATCH_D16(D, (launch_k<DT, 8>(a, tile, sm_count, st)));
    }
}

}  // namespace sky
