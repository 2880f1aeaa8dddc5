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
// Work distribution: persistent CTAs pull host-planned items (<= 256
// candidates x comparator ranges) from an atomic counter in launch order.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>

#include "dom.cuh"
#include "kernels.cuh"
#include "stream.cuh"

namespace sky {

namespace {

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

// Top B bits of upper_bound(thr[0..127), x) = #{thr <= x} over the sorted
// thresholds of one dimension: a branchless search that stops once the
// remaining steps could only change the dropped low bits (B loads, no
// divergence).
template <int B>
__device__ __forceinline__ uint32_t quant_code(const float* tj, float x) {
    int lo = 0;
#pragma unroll
    for (int step = 64; step >= (1 << (7 - B)); step >>= 1) lo += (tj[lo + step - 1] <= x) ? step : 0;
    return (uint32_t)lo >> (7 - B);
}

// One CTA per dimension: block radix sort of a strided sample of the column
// (2048 rows), keep 127 quantiles as thresholds.
constexpr int kThrThreads = 512, kThrItems = 4;
template <int D>
__global__ void __launch_bounds__(kThrThreads) k_thresholds(const float* __restrict__ src, uint32_t stride, uint32_t ncols,
                                                           uint32_t n_host, float* thr, const uint32_t* n_dev,
                                                           const uint32_t* gate = nullptr, uint32_t gate_min = 0) {
    // gate: skip when a device count says the thresholds will not be used
    if (gate && *gate < gate_min) return;
    constexpr int SMP = kThrThreads * kThrItems;
    using Sort = cub::BlockRadixSort<float, kThrThreads, kThrItems>;
    __shared__ typename Sort::TempStorage tmp;
    __shared__ float v[SMP];
    const int j = blockIdx.x;
    const uint32_t n = n_dev ? min(*n_dev, n_host) : n_host;
    const uint32_t S = n < (uint32_t)SMP ? n : (uint32_t)SMP;
    float keys[kThrItems];
#pragma unroll
    for (int k = 0; k < kThrItems; ++k) {
        const uint32_t i = threadIdx.x * kThrItems + k;
        keys[k] = __int_as_float(0x7f800000);  // +inf padding sorts last
        if (i < S) keys[k] = (uint32_t)j < ncols ? src[((uint64_t)i * n / S) * stride + j] : 0.0f;
    }
    Sort(tmp).Sort(keys);
#pragma unroll
    for (int k = 0; k < kThrItems; ++k) v[threadIdx.x * kThrItems + k] = keys[k];
    __syncthreads();
    for (int k = threadIdx.x; k < kThr; k += blockDim.x) {
        uint32_t idx = S ? (uint32_t)(((uint64_t)(k + 1) * S) / kCodeLevels) : 0;
        if (idx >= S) idx = S ? S - 1 : 0;
        thr[j * kThr + k] = S ? v[idx] : 0.0f;
    }
}

template <int D>
__global__ void __launch_bounds__(256) k_encode(DevSet s, const float* __restrict__ thr, const uint32_t* n_dev) {
    constexpr int V = Dims2<D>::V;
    __shared__ float t[D * kThr];
    for (int i = threadIdx.x; i < D * kThr; i += blockDim.x) t[i] = thr[i];
    __syncthreads();
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (n_dev ? *n_dev : s.n)) return;
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
        w[j / L] |= quant_code<B>(t + j * kThr, x[j]) << (LW * (j % L));
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


// Guard bits that survived the subtraction (GA <=> pass): 2 IADD + 1 LOP3.
// Since h <= GA as an integer with equality only on a pass, "any of N tests
// passes" is max(h_1..h_N) == GA: a 3-input max (VIMNMX3) folds two tests
// per instruction.
template <uint32_t G>
__device__ __forceinline__ uint32_t coarse_hit(const uint32_t (&t)[2], const uint2& s) {
    constexpr uint32_t GA = G | 0x80000000u;
    return (t[0] - s.x) & (t[1] - s.y) & GA;
}

template <int N>
__device__ __forceinline__ uint32_t max_fold(const uint32_t (&h)[N]) {
    uint32_t m = h[0];
#pragma unroll
    for (int j = 1; j + 1 < N; j += 2) m = max(m, max(h[j], h[j + 1]));
    if (N % 2 == 0 && N > 1) m = max(m, h[N - 1]);
    return m;
}

template <uint32_t G, int K>
__device__ __forceinline__ bool any_coarse_pass(const uint32_t (&T)[K][2], const uint2& q) {
    uint32_t h[K];
#pragma unroll
    for (int k = 0; k < K; ++k) h[k] = coarse_hit<G>(T[k], q);
    return max_fold<K>(h) == (G | 0x80000000u);
}

constexpr int RS3_WARPS = 8;
constexpr int RS3_THREADS = RS3_WARPS * 32;
#ifndef RS3_MINB
#define RS3_MINB 2
#endif

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

// Dominance core. A CTA of RS3_WARPS warps takes one item: <= 32*K candidates
// (lane l of every warp holds candidates cb + 32k + l as packed codes in
// registers) against a list of comparator ranges, each sorted by sum key.
// The warps split the comparator stream: warp w handles batches w, w+8, ...
// of 32 comparators (codes, keys and coordinates of its next batch are
// prefetched into registers while the current one is tested) and stops a
// range once a ballot shows the sorted keys passed the item's bound. A kill
// is published in a shared-memory mask that every warp folds into its alive
// bits before each batch, so no warp keeps testing a dominated candidate.
// Exact checks read both points from shared memory.
template <int D, int K>
struct Relsky3Smem {
    static constexpr int V = Dims2<D>::V;
    float4 cand[K][V][32];             // [k][v][lane]: conflict-free per-lane reads
    float4 comp[RS3_WARPS][32][V];     // each warp's current batch (broadcast reads)
    uint2 code[RS3_WARPS][32];
    uint32_t deadmask[32];             // bit k of word l: candidate (k, l) dominated
    uint32_t item, bound;
};

template <int D, int K>
__global__ void __launch_bounds__(RS3_THREADS, RS3_MINB) k_relsky3(Relsky2Args a) {
    constexpr int W = Dims2<D>::V;
    constexpr uint32_t G = CodeLayout<D>::G;
    constexpr uint32_t FULL = 0xffffffffu;
    extern __shared__ float4 smem_raw[];
    using S = Relsky3Smem<D, K>;
    S& sm = *reinterpret_cast<S*>(smem_raw);

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned long long ntests = 0, nhits = 0;

    for (;;) {
        if (threadIdx.x == 0) sm.item = atomicAdd(a.counter, 1u);
        if (threadIdx.x < 32) sm.deadmask[threadIdx.x] = 0;
        __syncthreads();
        const uint32_t item = sm.item;
        if (item >= (a.n_items_dev ? *a.n_items_dev : a.n_items)) break;
        const Item it = a.items[item];

        uint32_t T[K][2];
        uint32_t alive = 0, my_max = 0;
        // three rounds of independent loads (positions, dead flags, codes +
        // keys) instead of K dependent chains
        uint32_t cpos[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const uint32_t slot = it.cb + k * 32 + lane;
            cpos[k] = slot < it.ce ? (a.cidx ? a.cidx[slot] : slot) : kNone;  // dense candidate lists
        }
        bool slot_live[K];
#pragma unroll
        for (int k = 0; k < K; ++k) slot_live[k] = cpos[k] != kNone && !a.dead[cpos[k]];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            // empty / dead slot: lane guards set (no borrow can reach bit 31),
            // alive guard clear -> never passes
            T[k][0] = G;
            T[k][1] = G | 0x80000000u;
            if (slot_live[k]) {
                const uint32_t c = cpos[k];
                alive |= 1u << k;
                const uint2 q = a.cqc[c];
                T[k][0] = q.x | G | CodeLayout<D>::ALIVE;
                T[k][1] = q.y | G | 0x80000000u;
                my_max = max(my_max, a.cskey[c]);
                if (warp == 0) {
                    const float4* x = reinterpret_cast<const float4*>(a.cxyz) + (size_t)c * W;
#pragma unroll
                    for (int v = 0; v < W; ++v) sm.cand[k][v][lane] = x[v];
                }
            }
        }
        const uint32_t initial = alive;
        const uint32_t bound = a.bounded ? __reduce_max_sync(FULL, my_max) : 0xFFFFFFFFu;
        __syncthreads();  // candidate coordinates staged
        bool live = __any_sync(FULL, alive != 0);

        // direct items carry their one comparator range in (lb, le)
        const uint32_t r_end = a.direct ? it.lb + 1 : it.le;
        const bool rpar = a.range_par && !a.direct;
        const uint32_t bstep = rpar ? 32u : 32u * RS3_WARPS;
        for (uint32_t r = it.lb + (rpar ? warp : 0); live && r < r_end; r += rpar ? RS3_WARPS : 1) {
            const uint2 rg = a.direct ? make_uint2(it.lb, it.le) : a.ranges[r];
            const uint32_t sb = rg.x, se = range_end(a, rg);
            uint32_t base = sb + (rpar ? 0u : warp * 32u);
            if (base >= se) continue;
            // prefetch this warp's first batch
            uint32_t idx = base + lane;
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
            for (; base < se; base += bstep) {
                // fold in kills published by the other warps
                const uint32_t dm = sm.deadmask[lane];
                if (dm & alive) {
#pragma unroll
                    for (int k = 0; k < K; ++k)
                        if ((dm >> k) & 1u) T[k][0] &= ~CodeLayout<D>::ALIVE;
                    alive &= ~dm;
                }
                const uint32_t inb = __ballot_sync(FULL, nk <= bound);  // prefix (keys sorted)
                const uint32_t lim = __popc(inb);
                __syncwarp();
                // comparators past the bound get codes that never pass
                sm.code[warp][lane] = lane < lim ? nq : make_uint2(0u, 0x80000000u);
#pragma unroll
                for (int v = 0; v < W; ++v) sm.comp[warp][lane][v] = nx[v];
                __syncwarp();
                idx = base + bstep + lane;
                if (lim == 32 && idx < se) {
                    nq = a.sqc[idx];
                    nk = a.sskey[idx];
                    const float4* x = reinterpret_cast<const float4*>(a.sxyz) + (size_t)idx * W;
#pragma unroll
                    for (int v = 0; v < W; ++v) nx[v] = x[v];
                } else {
                    nk = 0xFFFFFFFFu;
                }
                auto exact = [&](uint32_t i, const uint2 q) {
                    // exact test (core.hpp:89-96) where the codes could not rule s out
#pragma unroll
                    for (int k = 0; k < K; ++k) {
                        if (coarse_pass<G>(T[k], q)) {
                            ++nhits;
                            bool gt = false, lt = false;
#pragma unroll
                            for (int v = 0; v < W; ++v) {
                                const float4 sa = sm.comp[warp][i][v], tb = sm.cand[k][v][lane];
                                gt |= (sa.x > tb.x) | (sa.y > tb.y) | (sa.z > tb.z) | (sa.w > tb.w);
                                lt |= (sa.x < tb.x) | (sa.y < tb.y) | (sa.z < tb.z) | (sa.w < tb.w);
                            }
                            bool dom = !gt && lt;
                            if (a.x64.x && !gt) {
                                // FP64 input: confirm on the original rows
                                const uint32_t slot = it.cb + k * 32 + lane;
                                dom = dom64(a.x64, a.sid[base + i], a.cid[a.cidx ? a.cidx[slot] : slot]);
                            }
                            if (dom) {
                                alive &= ~(1u << k);
                                T[k][0] &= ~CodeLayout<D>::ALIVE;
                                atomicOr(&sm.deadmask[lane], 1u << k);
                                ntests += i + 1;
                            }
                        }
                    }
                };
                // 4 comparators x K candidates per step, one max-fold and
                // one branch. Two register buffers alternate, each loaded one
                // step ahead, so no codes are copied between steps.
                const uint4* cq = reinterpret_cast<const uint4*>(&sm.code[warp][0]);
                const uint32_t nb = (lim + 3) & ~3u;
                auto step = [&](uint32_t i, const uint4 c01, const uint4 c23) {
                    const uint2 q[4] = {make_uint2(c01.x, c01.y), make_uint2(c01.z, c01.w),
                                        make_uint2(c23.x, c23.y), make_uint2(c23.z, c23.w)};
                    uint32_t h[4 * K];
#pragma unroll
                    for (int c = 0; c < 4; ++c)
#pragma unroll
                        for (int k = 0; k < K; ++k) h[c * K + k] = coarse_hit<G>(T[k], q[c]);
                    if (max_fold<4 * K>(h) == (G | 0x80000000u)) {
#pragma unroll 1
                        for (int c = 0; c < 4; ++c) {
                            const uint2 qc = c == 0 ? q[0] : c == 1 ? q[1] : c == 2 ? q[2] : q[3];
                            if (any_coarse_pass<G, K>(T, qc)) exact(i + c, qc);
                        }
                    }
                };
                // comparators past lim carry never-pass codes, so the loop
                // runs whole pairs of steps (32 is a multiple of 8)
                const uint32_t nb8 = (nb + 7) & ~7u;
                uint4 a01 = cq[0], a23 = cq[1];
                for (uint32_t i = 0; i < nb8; i += 8) {
                    const uint4 b01 = cq[(i + 4) / 2], b23 = cq[(i + 4) / 2 + 1];
                    step(i, a01, a23);
                    if (i + 8 < nb8) {
                        a01 = cq[(i + 8) / 2];
                        a23 = cq[(i + 8) / 2 + 1];
                    }
                    step(i + 4, b01, b23);
                }
                ntests += (unsigned long long)__popc(alive) * lim;
                live = __any_sync(FULL, alive != 0);
                if (!live || lim < 32) break;  // all dominated, or past the key bound
            }
        }
        __syncthreads();
        if (warp == 0) {
            uint32_t killed = initial & (sm.deadmask[lane] | ~alive);
            while (killed) {
                const int k = __ffs(killed) - 1;
                killed &= killed - 1;
                const uint32_t slot = it.cb + k * 32 + lane;
                a.dead[a.cidx ? a.cidx[slot] : slot] = 1;
            }
        }
        __syncthreads();
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

// ------------------------------------------------------------------ BNL
// Block-nested-loops (Borzsonyi et al., ICDE 2001; the reference has no BNL,
// SPEC.md:157) for one partition per CTA with a shared-memory window of at
// most `cap` tuples. The partition is consumed in batches of BNL2_B tuples
// (one per thread). Each batch tuple t is compared with every window tuple w
// in both directions (w may dominate t: t dies; t may dominate w: w is
// evicted) and with the other batch tuples, all through the packed codes with
// exact confirmation. Survivors enter the window while it has room and spill
// to an in-place overflow list otherwise. A window tuple carries (pass,
// timestamp = overflow length when it entered); it is output once it has met
// every tuple: at the end of its pass if nothing spilled before it, else when
// the next pass has consumed that many overflow tuples.
constexpr int BNL2_B = 1024;

__device__ __forceinline__ uint4 lds128(uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
    return v;
}

template <int D>
size_t bnl2_smem(uint32_t cap) {
    constexpr int V = Dims2<D>::V;
    // window: codes (8) + key (4) + pos (4) + ts (4) + pass (1) + kill (1)
    // batch: coords (16V) + codes (8) + key (4)
    return (size_t)cap * 22 + (size_t)BNL2_B * (V * 16 + 12) + 256;
}

// dom_f4, or for FP64 input: s <= t on the float image (necessary), then
// dominates_raw on the original doubles of rows rs, rt.
template <int D>
__device__ __forceinline__ bool dom_f4x(const float4* __restrict__ s, const float4* __restrict__ t, const X64& e,
                                        uint32_t rs, uint32_t rt) {
    if (!e.x) return dom_f4<D>(s, t);
    constexpr int V = Dims2<D>::V;
    bool gt = false;
#pragma unroll
    for (int v = 0; v < V; ++v) {
        const float4 a = s[v], b = t[v];
        gt |= (a.x > b.x) | (a.y > b.y) | (a.z > b.z) | (a.w > b.w);
    }
    return !gt && dom64(e, rs, rt);
}

template <int D>
__global__ void __launch_bounds__(BNL2_B) k_bnl2(BnlArgs a, const uint2* __restrict__ qc,
                                                 const uint32_t* __restrict__ skey, uint32_t cap,
                                                 uint32_t* work_counter) {
    constexpr int V = Dims2<D>::V;
    constexpr uint32_t G = CodeLayout<D>::G;
    constexpr uint32_t GA = G | 0x80000000u;
    constexpr uint32_t ALIVE = CodeLayout<D>::ALIVE;
    constexpr int NW = BNL2_B / 32;
    extern __shared__ uint4 sm4[];
    float4* b_xyz = reinterpret_cast<float4*>(sm4);                          // batch coords [B][V]
    uint2* w_code = reinterpret_cast<uint2*>(b_xyz + BNL2_B * V);            // window codes
    uint2* b_code = w_code + cap;                                            // batch codes
    uint32_t* w_key = reinterpret_cast<uint32_t*>(b_code + BNL2_B);          // window keys
    uint32_t* b_key = w_key + cap;                                           // batch keys
    uint32_t* w_pos = b_key + BNL2_B;                                        // window -> set position
    uint32_t* w_ts = w_pos + cap;                                            // overflow length at entry
    uint8_t* w_pass = reinterpret_cast<uint8_t*>(w_ts + cap);                // pass of entry (mod 256)
    uint8_t* w_kill = w_pass + cap;                                          // 1 evicted, 2 confirmed
    __shared__ uint32_t s_wn, s_ovf_w, s_part, s_scan[NW], s_next;
    __shared__ int s_pass;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const float4* __restrict__ xyz = reinterpret_cast<const float4*>(a.xyz);
    unsigned long long ntests = 0, nhits = 0;

    // stable compaction of the window: drop entries with w_kill != 0
    // (confirmed ones are output first)
    auto compact_window = [&]() {
        const uint32_t wn0 = s_wn;
        uint32_t kept_before = 0;
        for (uint32_t c0 = 0; c0 < wn0; c0 += BNL2_B) {
            const uint32_t w = c0 + tid;
            const bool in = w < wn0;
            const uint8_t kill = in ? w_kill[w] : 0;
            const bool keep = in && kill == 0;
            uint2 q = make_uint2(0, 0);
            uint32_t pos = 0, ts = 0, key = 0;
            uint8_t ps = 0;
            if (in) pos = w_pos[w];
            if (keep) {
                q = w_code[w];
                key = w_key[w];
                ts = w_ts[w];
                ps = w_pass[w];
            }
            if (in && kill == 2) a.dead[pos] = 0;  // confirmed skyline tuple
            const unsigned bal = __ballot_sync(0xffffffffu, keep);
            if (lane == 0) s_scan[warp] = __popc(bal);
            __syncthreads();
            uint32_t off = kept_before + __popc(bal & ((1u << lane) - 1u));
            uint32_t tot = 0;
#pragma unroll
            for (int ww = 0; ww < NW; ++ww) {
                if (ww < warp) off += s_scan[ww];
                tot += s_scan[ww];
            }
            __syncthreads();
            if (keep) {
                w_code[off] = q;
                w_key[off] = key;
                w_pos[off] = pos;
                w_ts[off] = ts;
                w_pass[off] = ps;
                w_kill[off] = 0;
            }
            kept_before += tot;
            __syncthreads();
        }
        if (tid == 0) s_wn = kept_before;
        __syncthreads();
    };

    for (;;) {
        if (tid == 0) s_part = atomicAdd(work_counter, 1u);
        __syncthreads();
        const uint32_t part = s_part;
        if (part >= a.P) break;
        const uint32_t seg_b = a.seg_off[part], seg_e = a.seg_off[part + 1];
        if (seg_b == seg_e) {
            __syncthreads();
            continue;
        }
        uint32_t* ovf = a.overflow + seg_b;
        if (tid == 0) {
            s_wn = 0;
            s_pass = 0;
        }
        __syncthreads();
        uint32_t in_n = seg_e - seg_b;
        bool first = true;
        for (;;) {
            const uint32_t wn_start = s_wn;
            if (in_n == 0 && wn_start == 0) break;
            const int pass = s_pass;
            const uint8_t prev_pass = (uint8_t)(pass - 1);
            if (tid == 0) s_ovf_w = 0;
            __syncthreads();
            for (uint32_t k0 = 0;; k0 += BNL2_B) {
                // confirm window tuples of the previous pass whose timestamp is reached
                {
                    bool any = false;
                    const uint32_t wn = s_wn;
                    for (uint32_t w = tid; w < wn; w += BNL2_B) {
                        const bool c = !first && w_pass[w] == prev_pass && w_ts[w] <= k0;
                        w_kill[w] = c ? 2 : 0;
                        any |= c;
                    }
                    if (__syncthreads_or(any)) compact_window();
                }
                if (k0 >= in_n) break;
                const uint32_t bn = min((uint32_t)BNL2_B, in_n - k0);
                const bool valid = (uint32_t)tid < bn;
                uint32_t mypos = 0, tkey = 0;
                float4 t[V];
                uint2 tq = make_uint2(0, 0);
                if (valid) {
                    mypos = first ? seg_b + k0 + tid : ovf[k0 + tid];
#pragma unroll
                    for (int v = 0; v < V; ++v) {
                        t[v] = xyz[(size_t)mypos * V + v];
                        b_xyz[tid * V + v] = t[v];
                    }
                    tq = qc[mypos];
                    tkey = skey[mypos];
                    b_code[tid] = tq;
                    b_key[tid] = tkey;
                }
                __syncthreads();
                uint32_t T0 = valid ? (tq.x | G | ALIVE) : G;
                const uint32_t T1 = (valid ? tq.y : 0u) | G | 0x80000000u;
                // a window tuple can only be dominated by t if its key is >= t's
                // (dominance implies a smaller or equal coordinate sum)
                const uint32_t rkey = valid ? tkey : 0xFFFFFFFFu;
                bool alive = valid;
                const uint32_t wn = s_wn;
                bool killed_any = false;
                auto slow = [&](uint32_t w) {
                    const uint2 q = w_code[w];
                    const bool d1 = ((T0 - q.x) & (T1 - q.y) & GA) == GA;  // w may dominate t
                    const bool d2 = w_key[w] >= rkey &&                     // t may dominate w
                                    (((q.x | G | 0x80000000u) - tq.x) & ((q.y | G | 0x80000000u) - tq.y) & GA) == GA;
                    if (!(d1 | d2)) return;
                    ++nhits;
                    const float4* wx = xyz + (size_t)w_pos[w] * V;
                    float4 wv[V];
#pragma unroll
                    for (int v = 0; v < V; ++v) wv[v] = wx[v];
                    const uint32_t rw = a.x64.x ? a.id[w_pos[w]] : 0, rt = a.x64.x ? a.id[mypos] : 0;
                    if (d1 && dom_f4x<D>(wv, t, a.x64, rw, rt)) {
                        alive = false;
                        T0 &= ~ALIVE;
                    }
                    if (d2 && dom_f4x<D>(t, wv, a.x64, rt, rw)) {
                        w_kill[w] = 1;
                        killed_any = true;
                    }
                };
                uint32_t w = 0;
                // shared-window addresses as 32-bit registers (the compiler
                // otherwise re-derives the window base every step)
                uint32_t a_code = smem_u32(w_code), a_key = smem_u32(w_key);
                asm volatile("" : "+r"(a_code), "+r"(a_key));
                for (; w + 4 <= wn; w += 4) {
                    // four entries per step: forward coarse misses fold with
                    // 3-input mins, the reverse test is gated by the keys
                    const uint4 qa = lds128(a_code + w * 8);
                    const uint4 qb = lds128(a_code + w * 8 + 16);
                    const uint4 kk = lds128(a_key + w * 4);
                    const uint32_t f0 = ~((T0 - qa.x) & (T1 - qa.y)) & GA;
                    const uint32_t f1 = ~((T0 - qa.z) & (T1 - qa.w)) & GA;
                    const uint32_t f2 = ~((T0 - qb.x) & (T1 - qb.y)) & GA;
                    const uint32_t f3 = ~((T0 - qb.z) & (T1 - qb.w)) & GA;
                    const uint32_t fm = min(min(f0, f1), min(f2, f3));
                    const uint32_t km = max(max(kk.x, kk.y), max(kk.z, kk.w));
                    if (fm == 0 || km >= rkey) {
                        slow(w);
                        slow(w + 1);
                        slow(w + 2);
                        slow(w + 3);
                    }
                }
                for (; w < wn; ++w) slow(w);
                if (valid) ntests += 2ull * wn;
                // batch x batch: is t dominated by an earlier-or-equal-key batch
                // tuple? Batch keys are nondecreasing (the partition and the
                // overflow list keep key order), so the scan stops at the first
                // larger key; 4 tuples per step, coarse misses max-folded.
                auto slow_b = [&](uint32_t u) {
                    const uint2 uq = b_code[u];
                    if (u != (uint32_t)tid && b_key[u] <= tkey && ((T0 - uq.x) & (T1 - uq.y) & GA) == GA) {
                        if (dom_f4x<D>(b_xyz + u * V, t, a.x64,
                                       a.x64.x ? a.id[first ? seg_b + k0 + u : ovf[k0 + u]] : 0,
                                       a.x64.x ? a.id[mypos] : 0)) {
                            alive = false;
                            T0 &= ~ALIVE;
                        }
                    }
                };
                uint32_t u = 0;
                if (valid && alive) {
                    for (; u + 4 <= bn; u += 4) {
                        const uint4 kk = *reinterpret_cast<const uint4*>(b_key + u);
                        if (kk.x > tkey) break;
                        const uint4 qa = *reinterpret_cast<const uint4*>(b_code + u);
                        const uint4 qb = *reinterpret_cast<const uint4*>(b_code + u + 2);
                        const uint32_t f0 = ~((T0 - qa.x) & (T1 - qa.y)) & GA;
                        const uint32_t f1 = ~((T0 - qa.z) & (T1 - qa.w)) & GA;
                        const uint32_t f2 = ~((T0 - qb.x) & (T1 - qb.y)) & GA;
                        const uint32_t f3 = ~((T0 - qb.z) & (T1 - qb.w)) & GA;
                        if (min(min(f0, f1), min(f2, f3)) == 0) {
                            slow_b(u);
                            slow_b(u + 1);
                            slow_b(u + 2);
                            slow_b(u + 3);
                        }
                    }
                    for (; u < bn && b_key[u] <= tkey; ++u) slow_b(u);
                    ntests += u;
                }
                if (__syncthreads_or(killed_any)) compact_window();
                // survivors enter the window in batch order, or spill
                {
                    const unsigned bal = __ballot_sync(0xffffffffu, alive);
                    if (lane == 0) s_scan[warp] = __popc(bal);
                    __syncthreads();
                    uint32_t rank = __popc(bal & ((1u << lane) - 1u));
                    uint32_t tot = 0;
#pragma unroll
                    for (int ww = 0; ww < NW; ++ww) {
                        if (ww < warp) rank += s_scan[ww];
                        tot += s_scan[ww];
                    }
                    const uint32_t wn1 = s_wn, ow = s_ovf_w;
                    const uint32_t room = cap - wn1;
                    if (alive) {
                        if (rank < room) {
                            const uint32_t slot = wn1 + rank;
                            w_code[slot] = tq;
                            w_key[slot] = tkey;
                            w_pos[slot] = mypos;
                            w_ts[slot] = ow;  // overflow tuples written in this pass so far
                            w_pass[slot] = (uint8_t)pass;
                            w_kill[slot] = 0;
                        } else {
                            ovf[ow + (rank - room)] = mypos;  // in place: ow + spilled <= k0 + bn
                        }
                    }
                    __syncthreads();
                    if (tid == 0) {
                        const uint32_t ins = min(tot, room);
                        s_wn = wn1 + ins;
                        s_ovf_w = ow + (tot - ins);
                    }
                    __syncthreads();
                }
            }
            // end of pass: tuples that entered before any spill of this pass,
            // and every tuple of the previous pass, have met every tuple;
            // with no spill at all the whole window is final.
            {
                const uint32_t ovf_n = s_ovf_w;
                const uint32_t wn = s_wn;
                for (uint32_t w = tid; w < wn; w += BNL2_B) {
                    const bool cur = w_pass[w] == (uint8_t)pass;
                    const bool confirm = ovf_n == 0 || (cur && w_ts[w] == 0) || (!cur && w_pass[w] == prev_pass);
                    w_kill[w] = confirm ? 2 : 0;
                }
                __syncthreads();
                compact_window();
                if (tid == 0) {
                    s_pass = pass + 1;
                    s_next = ovf_n;
                }
                __syncthreads();
                in_n = s_next;
                first = false;
            }
        }
        __syncthreads();
    }
    if (a.tests) {
        ntests = warp_sum(ntests);
        if (lane == 0 && ntests) atomicAdd(a.tests, ntests);
    }
}

// ------------------------------------------------------------ prefilter
// rep_prefilter (filter.cpp:147-159) over every row: one row per thread
// (read through the sorted index, so a warp's rows have close keys). The
// representatives sit in shared memory sorted by key with their packed codes
// (quantization thresholds from a sample of the input); each row encodes
// itself from the thresholds and runs the coarse test against every
// representative with key <= the warp's bound, the exact test only where the
// codes pass. A row stops at its first dominator, a warp when all its rows
// are dominated.
// Codes are used from 32 representatives on (the count may be known on the
// device only).
// POSORDER: thread i takes sorted position i (row idx[i]; a warp's rows then
// share a partition and have neighbouring keys, so they finish together) and
// writes dead_pos[i]; after the strongest 64 representatives the CTA's rows
// still alive are regrouped into dense warps for the rest of the list.
// Otherwise thread i takes row i (coalesced stream) and writes dead_row[i].
constexpr uint32_t kAppendSmemReps = 256;

// APPEND (row order, the stream path): persistent CTAs walk bulk-copied row
// tiles with the rows' keys staged alongside (stream_row_tiles); instead of
// flags, the surviving rows are appended to app.out as
// ((key64 >> key_shift) << row_bits | row), count in *app.count — the
// survivors' (partition, key, row) sort key. Shared memory holds at most
// kAppendSmemReps representatives; a longer list is read from global memory.
template <int D, bool CODES, bool POSORDER, bool APPEND = false>
__global__ void __launch_bounds__(256) k_prefilter(const float* __restrict__ pts, uint32_t d, uint32_t n,
                                                   const uint32_t* __restrict__ idx,
                                                   const float4* __restrict__ rep_xyz,
                                                   const uint32_t* __restrict__ rep_key, const uint2* __restrict__ rep_qc,
                                                   const uint32_t* __restrict__ rep_id,
                                                   uint32_t nrep_max, const uint32_t* nrep_dev,
                                                   const float* __restrict__ thr,
                                                   uint8_t* __restrict__ dead_row, unsigned long long* tests,
                                                   X64 x64, PrefilterAppend app = {}) {
    constexpr int V = Dims2<D>::V;
    constexpr uint32_t G = CodeLayout<D>::G;
    constexpr int L = CodeLayout<D>::L, LW = CodeLayout<D>::LW, B = CodeLayout<D>::B;
    const uint32_t nrep = nrep_dev ? min(*nrep_dev, nrep_max) : nrep_max;
    // packed codes pay off from 32 representatives on (the count may only be
    // known on the device)
    const bool use_codes = CODES && nrep >= 32;
    // APPEND reserves shared memory for kAppendSmemReps representatives only
    // (the count is known on the device alone; a smaller reservation keeps
    // more CTAs resident for the row stream); more than that are read from
    // global memory (L1-cached broadcasts), guarded by their count.
    const uint32_t ncap = APPEND ? min(nrep_max, kAppendSmemReps) : nrep_max;
    const uint32_t npad = (ncap + 7) & ~7u;
    const bool greps = APPEND && nrep > ncap;
    extern __shared__ float4 s_rep_smem[];
    uint2* s_code_smem = reinterpret_cast<uint2*>(s_rep_smem + (size_t)npad * V);
    uint32_t* s_key_smem = reinterpret_cast<uint32_t*>(s_code_smem + npad);
    float* s_thr = reinterpret_cast<float*>(s_key_smem + npad);
    const float4* s_rep = greps ? rep_xyz : s_rep_smem;
    const uint32_t kmask = APPEND ? ~((1u << app.key_shift) - 1u) : 0xFFFFFFFFu;
    if (!greps) {
        for (uint32_t i = threadIdx.x; i < nrep * V; i += blockDim.x) s_rep_smem[i] = rep_xyz[i];
        for (uint32_t i = threadIdx.x; i < npad; i += blockDim.x) {
            // padding codes never pass the coarse test (bit 31 of word 1 borrows)
            if (CODES) s_code_smem[i] = i < nrep ? rep_qc[i] : make_uint2(0u, 0x80000000u);
            // APPEND compares truncated keys (the rows' keys come from key64)
            s_key_smem[i] = i < nrep ? rep_key[i] & kmask : 0xFFFFFFFFu;
        }
    }
    auto key_at = [&](uint32_t r) -> uint32_t {
        if (!greps) return s_key_smem[r];
        return r < nrep ? __ldg(rep_key + r) & kmask : 0xFFFFFFFFu;
    };
    auto code_at = [&](uint32_t r) -> uint2 {
        if (!greps) return s_code_smem[r];
        return r < nrep ? __ldg(rep_qc + r) : make_uint2(0u, 0x80000000u);
    };
    if (CODES)
        for (uint32_t i = threadIdx.x; i < D * kThr; i += blockDim.x) s_thr[i] = thr[i];
    if (APPEND && app.zero)
        for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < app.zero_words; i += gridDim.x * blockDim.x)
            app.zero[i] = 0;
    // APPEND: the row tiles stream through shared memory after the tables
    char* s_stage = reinterpret_cast<char*>(
        (reinterpret_cast<uintptr_t>(s_thr + (CODES ? D * kThr : 0)) + 15) & ~uintptr_t{15});
    __syncthreads();
    unsigned long long nt = 0;
    // APPEND: a warp's kept rows take consecutive output slots
    auto append_row = [&](const bool keep, const uint32_t row) {
        const uint32_t lane = threadIdx.x & 31;
        const uint32_t bal = __ballot_sync(0xffffffffu, keep);
        if (!bal) return;
        uint32_t base = 0;
        if (lane == 0) base = atomicAdd(app.count, (uint32_t)__popc(bal));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (keep)
            app.out[base + __popc(bal & ((1u << lane) - 1u))] =
                ((app.key64[row] >> app.key_shift) << app.row_bits) | row;
    };
    // APPEND without codes (fewer than 32 representatives), all of them in
    // shared memory: each row is tested against them in key order (the strongest
    // first) until one dominates it, a warp vote before each; no key bound
    // (a representative's key is below a row's it dominates anyway), so the
    // rows' keys are not staged
    auto few_reps = [&](const float* tile, const uint32_t r0, const uint32_t nr) {
#pragma unroll 1
        for (uint32_t r1 = 0; r1 < stream_tile_rows(d); r1 += kStreamThreads) {
            const uint32_t rr = threadIdx.x + r1;
            const bool valid = rr < nr;
            const float* x = tile + (size_t)rr * d;
            float4 t[V];
            if ((d & 3) == 0) {
#pragma unroll
                for (int v = 0; v < V; ++v)
                    t[v] = (valid && 4 * v < (int)d) ? reinterpret_cast<const float4*>(x)[v]
                                                      : make_float4(0.f, 0.f, 0.f, 0.f);
            } else {
                float xs[4 * V];
#pragma unroll
                for (int j = 0; j < 4 * V; ++j) xs[j] = (valid && (uint32_t)j < d) ? x[j] : 0.0f;
#pragma unroll
                for (int v = 0; v < V; ++v) t[v] = make_float4(xs[4 * v], xs[4 * v + 1], xs[4 * v + 2], xs[4 * v + 3]);
            }
            bool alive = valid;
#pragma unroll 1
            for (uint32_t r = 0; r < nrep && __any_sync(0xffffffffu, alive); ++r) {
                if (alive) {
                    ++nt;
                    if (dom_f4<D>(s_rep_smem + r * V, t)) alive = false;
                }
            }
            append_row(alive, r0 + rr);
        }
    };
    auto process = [&](const float* x, const uint32_t slot, const bool valid, const uint32_t row,
                       const uint64_t* key_in) {
    float4 t[V];
    uint32_t tk = 0;
    uint32_t T0 = G, T1 = G | 0x80000000u;  // never passes unless set below
    {
        float xs[4 * V];
        double sum = 0.0;
        if (APPEND && (d & 3) == 0) {
            // staged rows with d % 4 == 0: 16-byte shared loads (a quarter of
            // the bank wavefronts of scalar loads at an even row stride)
#pragma unroll
            for (int v = 0; v < V; ++v) {
                const float4 q = (valid && 4 * v < (int)d) ? reinterpret_cast<const float4*>(x)[v]
                                                            : make_float4(0.f, 0.f, 0.f, 0.f);
                xs[4 * v] = q.x; xs[4 * v + 1] = q.y; xs[4 * v + 2] = q.z; xs[4 * v + 3] = q.w;
            }
        } else {
#pragma unroll
            for (int j = 0; j < 4 * V; ++j) xs[j] = (valid && j < D && (uint32_t)j < d) ? x[j] : 0.0f;
        }
        if (APPEND) {
            // the prep pass's (truncated) key, staged with the row: no FP64
            // sum per row; with few representatives no key gating at all
            tk = !use_codes ? 0xFFFFFFFFu : (valid ? (uint32_t)*key_in : 0u);
        } else {
#pragma unroll
            for (int j = 0; j < 4 * V; ++j)
                if ((uint32_t)j < d) sum = __dadd_rn(sum, (double)xs[j]);  // same key as k_prep
            if (x64.x && valid) {
                const double* xd = x64.x + (size_t)row * d;
                sum = 0.0;
                for (uint32_t j = 0; j < d; ++j) sum = __dadd_rn(sum, xd[j]);
            }
            tk = __float_as_uint(__double2float_rn(sum));
        }
        if (use_codes && valid) {
            uint32_t w[2] = {0, 0};
#pragma unroll
            for (int j = 0; j < D; ++j) {
                w[j / L] |= quant_code<B>(s_thr + j * kThr, xs[j]) << (LW * (j % L));
            }
            T0 = w[0] | G | CodeLayout<D>::ALIVE;
            T1 = w[1] | G | 0x80000000u;
        }
#pragma unroll
        for (int v = 0; v < V; ++v) t[v] = make_float4(xs[4 * v], xs[4 * v + 1], xs[4 * v + 2], xs[4 * v + 3]);
    }
    bool alive = valid;
    const uint32_t bound = __reduce_max_sync(0xffffffffu, alive ? tk : 0u);
    bool flags_done = false;
    if (use_codes) {
        // 8 representatives per step: 8 coarse tests folded by 3-input min,
        // exact FP32 re-check only on a coarse pass; one vote per step
        auto scan = [&](uint32_t r0, uint32_t r1, uint32_t bnd, uint32_t (&Tl)[2], const float4 (&tx)[V],
                        uint32_t rowx, bool& al) {
            for (uint32_t r = r0; r < r1 && __any_sync(0xffffffffu, al); r += 8) {
                if (key_at(r) > bnd) break;  // warp-uniform: reps sorted by key
                uint2 q[8];
                if (!greps) {
                    const uint4* q4 = reinterpret_cast<const uint4*>(s_code_smem + r);
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const uint4 w = q4[k];
                        q[2 * k] = make_uint2(w.x, w.y);
                        q[2 * k + 1] = make_uint2(w.z, w.w);
                    }
                } else {
#pragma unroll
                    for (int k = 0; k < 8; ++k) q[k] = code_at(r + k);
                }
                uint32_t h[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) h[k] = coarse_hit<G>(Tl, q[k]);
                if (al) nt += min(8u, nrep - r);
                constexpr uint32_t GA = G | 0x80000000u;
                if (max_fold<8>(h) == GA) {
                    // exact checks for the representatives whose codes passed
                    uint32_t m = 0;
#pragma unroll
                    for (int k = 0; k < 8; ++k) m |= (h[k] == GA ? 1u : 0u) << k;
                    while (m && al) {
                        const int k = __ffs(m) - 1;
                        m &= m - 1;
                        if (dom_f4x<D>(s_rep + (r + k) * V, tx, x64, x64.x ? rep_id[r + k] : 0, rowx)) {
                            al = false;
                            Tl[0] &= ~CodeLayout<D>::ALIVE;
                        }
                    }
                }
            }
        };
        uint32_t Tl[2] = {T0, T1};
        const uint32_t K1 = app.regroup & ~7u;
        if constexpr (POSORDER && !APPEND) {
            if (nrep > K1) {
                // The strongest K1 representatives kill most rows; the rows
                // still alive are regrouped into dense warps for the rest, so
                // a warp no longer runs the whole list for one survivor.
                __shared__ float4 s_ct[256][V];
                __shared__ uint32_t s_cm[256][5];
                __shared__ uint32_t s_wc[8], s_nalive;
                scan(0, K1, bound, Tl, t, row, alive);
                if (valid && !alive) dead_row[slot] = 1;
                const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
                const uint32_t bal = __ballot_sync(0xffffffffu, alive);
                if (lane == 0) s_wc[wid] = __popc(bal);
                __syncthreads();
                uint32_t pos = __popc(bal & ((1u << lane) - 1u)), tot = 0;
                for (uint32_t w2 = 0; w2 < blockDim.x / 32; ++w2) {
                    pos += w2 < wid ? s_wc[w2] : 0u;
                    tot += s_wc[w2];
                }
                if (alive) {
#pragma unroll
                    for (int v = 0; v < V; ++v) s_ct[pos][v] = t[v];
                    s_cm[pos][0] = Tl[0];
                    s_cm[pos][1] = Tl[1];
                    s_cm[pos][2] = tk;
                    s_cm[pos][3] = slot;
                    s_cm[pos][4] = row;
                }
                if (threadIdx.x == 0) s_nalive = tot;
                __syncthreads();
                const uint32_t na = s_nalive;
                bool al2 = threadIdx.x < na;
                uint32_t T2[2] = {G, G | 0x80000000u}, tk2 = 0, slot2 = 0, row2 = 0;
                float4 t2[V];
#pragma unroll
                for (int v = 0; v < V; ++v) t2[v] = make_float4(0.f, 0.f, 0.f, 0.f);
                if (al2) {
#pragma unroll
                    for (int v = 0; v < V; ++v) t2[v] = s_ct[threadIdx.x][v];
                    T2[0] = s_cm[threadIdx.x][0];
                    T2[1] = s_cm[threadIdx.x][1];
                    tk2 = s_cm[threadIdx.x][2];
                    slot2 = s_cm[threadIdx.x][3];
                    row2 = s_cm[threadIdx.x][4];
                }
                if (__any_sync(0xffffffffu, al2)) {
                    const uint32_t bound2 = __reduce_max_sync(0xffffffffu, al2 ? tk2 : 0u);
                    scan(K1, nrep, bound2, T2, t2, row2, al2);
                }
                if (threadIdx.x < na && !al2) dead_row[slot2] = 1;
                flags_done = true;
            } else {
                scan(0, nrep, bound, Tl, t, row, alive);
            }
        } else {
            scan(0, nrep, bound, Tl, t, row, alive);
        }
    } else if (__any_sync(0xffffffffu, alive)) {
        uint32_t r = 0;
        for (; r < nrep; ++r) {
            const uint32_t kr = key_at(r);
            if (kr > bound) break;  // warp-uniform: reps sorted by key
            bool maybe = alive;
            if (use_codes) {
                const uint2 q = code_at(r);
                constexpr uint32_t GA = G | 0x80000000u;
                maybe = ((T0 - q.x) & (T1 - q.y) & GA) == GA;
            }
            if (maybe && kr <= tk && dom_f4x<D>(s_rep + r * V, t, x64, x64.x ? rep_id[r] : 0, row)) {
                alive = false;
                nt += r + 1;
                T0 &= ~CodeLayout<D>::ALIVE;
            }
            // few representatives: the strongest usually kill the whole warp
            if (((r & 15) == 15 || nrep <= 32) && !__any_sync(0xffffffffu, alive)) {
                ++r;
                break;
            }
        }
        if (alive) nt += r;
    }
    if (APPEND) {
        append_row(valid && alive, row);
    } else if (POSORDER) {
        if (valid && !alive && !flags_done) dead_row[slot] = 1;
    } else if (valid) {
        dead_row[row] = alive ? 0 : 1;
    }
    };
    if (APPEND) {
        stream_row_tiles(
            pts, n, d, s_stage,
            [&](const float* tile, uint32_t r0, uint32_t nr, const uint64_t* keys) {
                if (!use_codes && !greps) {
                    few_reps(tile, r0, nr);
                    return;
                }
                // warp-uniform trip count: the warp votes stay converged
#pragma unroll 1
                for (uint32_t r1 = 0; r1 < stream_tile_rows(d); r1 += kStreamThreads) {
                    const uint32_t rr = threadIdx.x + r1;
                    process(tile + (size_t)rr * d, r0 + rr, rr < nr, r0 + rr, keys + rr);
                }
            },
            use_codes || greps ? app.key64 : nullptr);  // CTA-uniform; the ring is sized for the keys
    } else {
        const uint32_t slot = blockIdx.x * blockDim.x + threadIdx.x;
        const bool valid = slot < n && (!POSORDER || !dead_row[slot]);
        const uint32_t row = (POSORDER && slot < n) ? idx[slot] : slot;
        process(pts + (size_t)row * d, slot, valid, row, nullptr);
    }
    if (tests) {
        nt = warp_sum(nt);
        if ((threadIdx.x & 31) == 0 && nt) atomicAdd(tests, nt);
    }
}

__global__ void k_gather_dead(const uint32_t* __restrict__ idx, const uint8_t* __restrict__ dead_row, uint32_t n,
                              uint8_t* __restrict__ dead_pos) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dead_pos[i] |= dead_row[idx[i]];
}

// skyline_bruteforce (core.cpp:56-73) of one small set (prune_dominated_reps,
// filter.cpp:139-145): the set in shared memory, every thread tests its
// points against all others.
template <int D>
__global__ void __launch_bounds__(1024) k_small_skyline(const float4* __restrict__ xyz, const uint32_t* __restrict__ id,
                                                        uint32_t n, uint8_t* __restrict__ dead,
                                                        unsigned long long* tests, X64 x64) {
    constexpr int V = Dims2<D>::V;
    extern __shared__ float4 s_pts[];
    for (uint32_t i = threadIdx.x; i < n * V; i += blockDim.x) s_pts[i] = xyz[i];
    __syncthreads();
    unsigned long long nt = 0;
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
        bool dom = false;
        for (uint32_t j = 0; j < n && !dom; ++j) {
            ++nt;
            if (j != i && dom_f4x<D>(s_pts + j * V, s_pts + i * V, x64, x64.x ? id[j] : 0, x64.x ? id[i] : 0))
                dom = true;
        }
        dead[i] = dom ? 1 : 0;
    }
    if (tests) {
        nt = warp_sum(nt);
        if ((threadIdx.x & 31) == 0 && nt) atomicAdd(tests, nt);
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
        default: throw Error(SKY_E_INTERNAL, std::string("packed-code kernel needs D <= 16 (") + __func__ + ")"); \
    }

template <int D, int K>
void launch_k(const Relsky2Args& a, int sm_count, cudaStream_t st) {
    const size_t smem = sizeof(Relsky3Smem<D, K>);
    ensure_smem_attr((const void*)k_relsky3<D, K>, smem);
    const int per_sm = std::max(1, occupancy_cached((const void*)k_relsky3<D, K>, RS3_THREADS, smem));
    const uint32_t grid = (uint32_t)std::min<uint64_t>(a.n_items, (uint64_t)per_sm * sm_count);
    k_relsky3<D, K><<<grid, RS3_THREADS, smem, st>>>(a);
    SKY_LAUNCH_CHECK();
}

template <int D>
void launch_bnl2_impl(const BnlArgs& a, const uint2* qc, const uint32_t* skey, uint32_t cap, uint32_t grid,
                      uint32_t* counter, cudaStream_t st) {
    cap &= ~3u;  // 4-entry loads of codes / keys
    const size_t smem = bnl2_smem<D>(cap);
    ensure_smem_attr((const void*)k_bnl2<D>, smem);
    k_bnl2<D><<<grid, BNL2_B, smem, st>>>(a, qc, skey, cap, counter);
    SKY_LAUNCH_CHECK();
}

}  // namespace

uint32_t bnl2_window_fit(int D, uint32_t want, int smem_optin) {
    uint32_t cap = want;
    SKY_DISPATCH_D16(D, {
        while (cap > 32 && bnl2_smem<DT>(cap) + 2048 > (size_t)smem_optin) cap -= 32;
    });
    return cap;
}

void launch_bnl2(int D, const BnlArgs& a, const uint2* qc, const uint32_t* skey, uint32_t cap, uint32_t grid,
                 uint32_t* counter, cudaStream_t st) {
    SKY_DISPATCH_D16(D, (launch_bnl2_impl<DT>(a, qc, skey, cap, grid, counter, st)));
}

bool launch_prefilter(int D, const float* pts, uint32_t d, const uint32_t* idx, uint32_t n, const float* rep_xyz,
                      const uint32_t* rep_key, const uint2* rep_qc, const uint32_t* rep_id, uint32_t nrep,
                      const uint32_t* nrep_dev, const float* thr, uint8_t* dead_row, uint8_t* dead_pos,
                      unsigned long long* tests, X64 x64, int smem_optin, cudaStream_t st, bool posorder) {
    if (D > 16) return false;
    const bool codes = rep_qc && thr && nrep >= 32;
    const size_t npad = (nrep + 7) & ~7u;
    const size_t smem = npad * ((D + 3) / 4) * 16 + npad * 12 + (codes ? (size_t)D * kThr * 4 : 0) + 64;
    // the sorted-position variant also holds its regrouping tables in static
    // shared memory (256 rows x (V float4 + 5 words), under 24 KB)
    const size_t stat = codes && posorder ? 24 * 1024 : 1024;
    if (smem + stat > (size_t)smem_optin) return false;
    if (!n) return true;
    SKY_DISPATCH_D16(D, {
        if (codes && posorder) {
            // many representatives, input in L2: sorted positions (a warp's
            // rows have close keys, so its key bound cuts early), flags in place
            ensure_smem_attr((const void*)k_prefilter<DT, true, true>, smem);
            PrefilterAppend rg;  // regroup point 64 (16-128 measured within noise on config 2)
            k_prefilter<DT, true, true><<<ceil_div(n, 256), 256, smem, st>>>(
                pts, d, n, idx, reinterpret_cast<const float4*>(rep_xyz), rep_key, rep_qc, rep_id, nrep, nrep_dev, thr,
                dead_pos, tests, x64, rg);
        } else if (codes) {
            // large input: rows streamed in row order (coalesced), flags
            // gathered into position order afterwards
            ensure_smem_attr((const void*)k_prefilter<DT, true, false>, smem);
            k_prefilter<DT, true, false><<<ceil_div(n, 256), 256, smem, st>>>(
                pts, d, n, idx, reinterpret_cast<const float4*>(rep_xyz), rep_key, rep_qc, rep_id, nrep, nrep_dev, thr,
                dead_row, tests, x64);
        } else {
            ensure_smem_attr((const void*)k_prefilter<DT, false, false>, smem);
            k_prefilter<DT, false, false><<<ceil_div(n, 256), 256, smem, st>>>(
                pts, d, n, idx, reinterpret_cast<const float4*>(rep_xyz), rep_key, nullptr, rep_id, nrep, nrep_dev,
                nullptr, dead_row, tests, x64);
        }
    });
    SKY_LAUNCH_CHECK();
    if (codes && posorder) return true;
    k_gather_dead<<<ceil_div(n, 256), 256, 0, st>>>(idx, dead_row, n, dead_pos);
    SKY_LAUNCH_CHECK();
    return true;
}

bool launch_prefilter_append(int D, const float* pts, uint32_t d, uint32_t n, const float* rep_xyz,
                             const uint32_t* rep_key, const uint2* rep_qc, const uint32_t* rep_id, uint32_t nrep,
                             const uint32_t* nrep_dev, const float* thr, const PrefilterAppend& app,
                             unsigned long long* tests, int smem_optin, cudaStream_t st) {
    if (D > 16 || ((uintptr_t)pts & 15)) return false;
    const bool codes = rep_qc && thr && nrep >= 32;
    const size_t npad = (std::min(nrep, kAppendSmemReps) + 7) & ~7u;
    const size_t smem = npad * ((D + 3) / 4) * 16 + npad * 12 + (codes ? (size_t)D * kThr * 4 : 0) + 64 +
                        stream_smem_bytes(d, true) + 16;
    if (smem + 1024 > (size_t)smem_optin) return false;
    if (!n) return true;
    // persistent CTAs: as many as fit, capped by the tile count
    auto go = [&](auto kern, const uint2* qc, const float* th) {
        ensure_smem_attr((const void*)kern, smem);
        const int per_sm = occupancy_cached((const void*)kern, (int)kStreamThreads, smem);
        const int sms = device_sm_count();
        const uint32_t grid = std::max<uint32_t>(1, std::min<uint32_t>(ceil_div(n, stream_tile_rows(d)),
                                                                       (uint32_t)std::max(1, per_sm) * sms));
        kern<<<grid, kStreamThreads, smem, st>>>(pts, d, n, nullptr, reinterpret_cast<const float4*>(rep_xyz), rep_key,
                                              qc, rep_id, nrep, nrep_dev, th, nullptr, tests, X64{}, app);
    };
    SKY_DISPATCH_D16(D, {
        if (codes)
            go(k_prefilter<DT, true, false, true>, rep_qc, thr);
        else
            go(k_prefilter<DT, false, false, true>, nullptr, nullptr);
    });
    SKY_LAUNCH_CHECK();
    return true;
}

bool launch_small_skyline(int D, const float* xyz, const uint32_t* id, uint32_t n, uint8_t* dead,
                          unsigned long long* tests, X64 x64, int smem_optin, cudaStream_t st) {
    if (D > 16 || n > 4096) return false;
    const size_t smem = (size_t)n * ((D + 3) / 4) * 16 + 16;
    if (smem + 1024 > (size_t)smem_optin) return false;
    if (!n) return true;
    SKY_DISPATCH_D16(D, {
        SKY_CUDA(cudaFuncSetAttribute(k_small_skyline<DT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k_small_skyline<DT><<<1, 1024, smem, st>>>(reinterpret_cast<const float4*>(xyz), id, n, dead, tests, x64);
    });
    SKY_LAUNCH_CHECK();
    return true;
}

void launch_thresholds(int D, const DevSet& s, float* thr, cudaStream_t st, const uint32_t* n_dev) {
    if (!s.n) return;
    SKY_DISPATCH_D16(D, (k_thresholds<DT><<<DT, kThrThreads, 0, st>>>(s.xyz, (DT + 3) / 4 * 4, DT, s.n, thr, n_dev)));
    SKY_LAUNCH_CHECK();
}

void launch_thresholds_rows(int D, const float* pts, uint32_t d, uint32_t n, float* thr, cudaStream_t st,
                            const uint32_t* gate, uint32_t gate_min) {
    if (!n) return;
    SKY_DISPATCH_D16(D, (k_thresholds<DT><<<DT, kThrThreads, 0, st>>>(pts, d, d, n, thr, nullptr, gate, gate_min)));
    SKY_LAUNCH_CHECK();
}

void launch_encode(int D, const DevSet& s, const float* thr, cudaStream_t st, const uint32_t* n_dev) {
    if (!s.n) return;
    SKY_DISPATCH_D16(D, (k_encode<DT><<<ceil_div(s.n, 256), 256, 0, st>>>(s, thr, n_dev)));
    SKY_LAUNCH_CHECK();
}

__global__ void __launch_bounds__(1024) k_plan_items(const uint32_t* __restrict__ dnew, uint32_t np,
                                                     const uint32_t* __restrict__ gb, const uint2* __restrict__ groups,
                                                     uint32_t max_groups, uint32_t tile, Item* __restrict__ items,
                                                     uint32_t* count) {
    // One CTA, one thread per partition (chunks of 1024). Per group level j:
    // a block scan of the tile counts of the partitions that have a j-th
    // group, then every thread writes items, each located by binary search
    // over the scanned offsets in shared memory.
    using Scan = cub::BlockScan<uint32_t, 1024>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ uint32_t s_off[1024], s_b[1024], s_e[1024], s_g[1024];
    __shared__ uint32_t s_total;
    constexpr uint32_t kGroupsSmem = 2048;
    __shared__ uint2 s_groups[kGroupsSmem];  // all groups when they fit (the usual case)
    const uint32_t ngroups = gb[np];
    const bool cached = ngroups <= kGroupsSmem;
    if (cached)
        for (uint32_t i = threadIdx.x; i < ngroups; i += 1024) s_groups[i] = groups[i];
    uint32_t base = 0;
    for (uint32_t p0 = 0; p0 < np; p0 += 1024) {
        const uint32_t p = p0 + threadIdx.x, np_here = min(1024u, np - p0);
        uint32_t tiles = 0, ng = 0;
        if (p < np) {
            s_b[threadIdx.x] = dnew[p];
            s_e[threadIdx.x] = dnew[p + 1];
            s_g[threadIdx.x] = gb[p];
            ng = gb[p + 1] - gb[p];
            tiles = (s_e[threadIdx.x] - s_b[threadIdx.x] + tile - 1) / tile;
        }
        for (uint32_t j = 0; j < max_groups; ++j) {
            uint32_t off, total;
            Scan(tmp).ExclusiveSum(j < ng ? tiles : 0u, off, total);
            s_off[threadIdx.x] = off;
            if (threadIdx.x == 0) s_total = total;
            __syncthreads();
            for (uint32_t x = threadIdx.x; x < s_total; x += 1024) {
                uint32_t lo = 0, hi = np_here;  // last q with s_off[q] <= x
                while (hi - lo > 1) {
                    const uint32_t mid = (lo + hi) >> 1;
                    if (s_off[mid] <= x) lo = mid; else hi = mid;
                }
                const uint32_t t = x - s_off[lo];
                const uint2 g = cached ? s_groups[s_g[lo] + j] : groups[s_g[lo] + j];
                const uint32_t cb = s_b[lo] + t * tile;
                items[base + x] = Item{cb, min(cb + tile, s_e[lo]), g.x, g.y};
            }
            base += s_total;
            __syncthreads();
        }
    }
    if (threadIdx.x == 0) *count = base;
}

void launch_plan_items(const uint32_t* dnew, uint32_t np, const uint32_t* gb, const uint2* groups, uint32_t max_groups,
                       uint32_t tile, Item* items, uint32_t* count, cudaStream_t st) {
    k_plan_items<<<1, 1024, 0, st>>>(dnew, np, gb, groups, max_groups, tile, items, count);
    SKY_LAUNCH_CHECK();
}

// ------------------------------------------------------ device planning
__global__ void k_partition_jobs(const uint32_t* __restrict__ coff, const uint32_t* __restrict__ soff,
                                 const uint32_t* __restrict__ n_comp, uint32_t P, uint64_t lo, uint64_t hi,
                                 Job* __restrict__ jobs) {
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= P) return;
    uint64_t rb, re;
    if (soff) {
        rb = soff[p];
        re = soff[p + 1];
    } else {
        rb = 0;
        re = *n_comp;
    }
    const uint64_t len = re - rb;
    const uint64_t l = rb + min(lo, len), h = rb + min(hi, len);
    jobs[p] = Job{coff[p], coff[p + 1], (uint32_t)l, (uint32_t)h};
}

__device__ __forceinline__ void job_shape(const Job& jb, uint32_t tile, uint32_t chunk, uint32_t max_chunks,
                                          uint32_t* ntile, uint32_t* nch, uint32_t* ch) {
    const uint32_t len = jb.hi > jb.lo ? jb.hi - jb.lo : 0;
    *ntile = (jb.ce - jb.cb + tile - 1) / tile;
    uint32_t c = chunk;
    if ((len + c - 1) / c > max_chunks) c = (len + max_chunks - 1) / max_chunks;
    *ch = c;
    *nch = len ? (len + c - 1) / c : 0;
}

__global__ void k_job_counts(const Job* __restrict__ jobs, const uint32_t* __restrict__ n_jobs, uint32_t cap,
                             uint32_t tile, uint32_t chunk, uint32_t max_chunks, uint32_t* __restrict__ counts) {
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j > cap) return;
    uint32_t c = 0;
    if (j < cap && j < *n_jobs) {
        uint32_t nt, nc, ch;
        job_shape(jobs[j], tile, chunk, max_chunks, &nt, &nc, &ch);
        c = nt * nc;
    }
    counts[j] = c;
}

// one CTA per job; chunk-major inside the job (every tile meets chunk g
// before any tile meets chunk g+1)
__global__ void k_job_items(const Job* __restrict__ jobs, const uint32_t* __restrict__ n_jobs,
                            const uint32_t* __restrict__ prefix, uint32_t tile, uint32_t chunk, uint32_t max_chunks,
                            Item* __restrict__ items) {
    const uint32_t j = blockIdx.x;
    if (j >= *n_jobs) return;
    const Job jb = jobs[j];
    uint32_t nt, nc, ch;
    job_shape(jb, tile, chunk, max_chunks, &nt, &nc, &ch);
    const uint32_t base = prefix[j], n = nt * nc;
    for (uint32_t x = threadIdx.x; x < n; x += blockDim.x) {
        const uint32_t g = x / nt, t = x - g * nt;
        const uint32_t cb = jb.cb + t * tile, lo = jb.lo + g * ch;
        items[base + x] = Item{cb, min(cb + tile, jb.ce), lo, min(lo + ch, jb.hi)};
    }
}

void launch_partition_jobs(const uint32_t* coff, const uint32_t* soff, const uint32_t* n_comp, uint32_t P,
                           uint64_t lo, uint64_t hi, Job* jobs, cudaStream_t st) {
    if (!P) return;
    k_partition_jobs<<<ceil_div(P, 256), 256, 0, st>>>(coff, soff, n_comp, P, lo, hi, jobs);
    SKY_LAUNCH_CHECK();
}
void launch_job_counts(const Job* jobs, const uint32_t* n_jobs, uint32_t cap, uint32_t tile, uint32_t chunk,
                       uint32_t max_chunks, uint32_t* counts, cudaStream_t st) {
    k_job_counts<<<ceil_div(cap + 1, 256), 256, 0, st>>>(jobs, n_jobs, cap, tile, chunk, max_chunks, counts);
    SKY_LAUNCH_CHECK();
}
void launch_job_items(const Job* jobs, const uint32_t* n_jobs, uint32_t cap, const uint32_t* prefix, uint32_t tile,
                      uint32_t chunk, uint32_t max_chunks, Item* items, cudaStream_t st) {
    if (!cap) return;
    k_job_items<<<cap, 128, 0, st>>>(jobs, n_jobs, prefix, tile, chunk, max_chunks, items);
    SKY_LAUNCH_CHECK();
}

// The three planning steps above (jobs, counts + scan, items) in one CTA
// for up to 1024 partitions: thread p builds job p and counts its items, a
// block scan places them, then the CTA writes every item (binary search of
// the item's job in the shared prefix).
__global__ void __launch_bounds__(1024) k_plan_partition_items(const uint32_t* __restrict__ coff,
                                                               const uint32_t* __restrict__ soff,
                                                               const uint32_t* __restrict__ n_comp, uint32_t P,
                                                               uint64_t lo, uint64_t hi, uint32_t tile,
                                                               uint32_t chunk, uint32_t max_chunks, uint32_t cap,
                                                               Item* __restrict__ items, uint32_t* n_items,
                                                               uint32_t grain_target) {
    using Scan = cub::BlockScan<uint32_t, 1024>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ Job s_job[1024];
    __shared__ uint32_t s_pre[1025], s_nt[1024], s_ch[1024];
    __shared__ uint32_t s_chunk;
    const uint32_t p = threadIdx.x;
    if (chunk == 0) {
        // chunk from the device counts (Runner::pick_grain's rule): halve
        // from 16384 while the launch would have fewer than grain_target items
        if (p == 0) {
            const uint64_t nc = coff[P] - coff[0];
            const uint64_t ns = n_comp ? *n_comp : (uint64_t)(soff[P] - soff[0]);
            const uint64_t pairs = nc * ns / 2;
            // small sets: down to 256 comparators per item, so a few hundred
            // rows still spread over many SMs
            uint32_t ch = 16384;
            while (ch > 256 && pairs / ((uint64_t)tile * ch) < grain_target) ch /= 2;
            s_chunk = ch;
        }
        __syncthreads();
        chunk = s_chunk;
    }
    uint32_t cnt = 0;
    if (p < P) {
        uint64_t rb, re;
        if (soff) {
            rb = soff[p];
            re = soff[p + 1];
        } else {
            rb = 0;
            re = *n_comp;
        }
        const uint64_t len = re - rb;
        const Job jb{coff[p], coff[p + 1], (uint32_t)(rb + min(lo, len)), (uint32_t)(rb + min(hi, len))};
        uint32_t nt, nc, ch;
        job_shape(jb, tile, chunk, max_chunks, &nt, &nc, &ch);
        s_job[p] = jb;
        s_nt[p] = nt;
        s_ch[p] = ch;
        cnt = nt * nc;
    }
    uint32_t pre, total;
    Scan(tmp).ExclusiveSum(cnt, pre, total);
    s_pre[p] = pre;
    if (p == 0) s_pre[1024] = total;
    __syncthreads();
    const uint32_t nout = min(total, cap);
    for (uint32_t x = threadIdx.x; x < nout; x += blockDim.x) {
        // job of item x: last j with s_pre[j] <= x (jobs with no items share a prefix)
        uint32_t a = 0, b = min(P, 1024u);
        while (b - a > 1) {
            const uint32_t m = (a + b) >> 1;
            if (s_pre[m] <= x) a = m; else b = m;
        }
        const Job jb = s_job[a];
        const uint32_t nt = s_nt[a], ch = s_ch[a], r = x - s_pre[a];
        const uint32_t g = r / nt, t = r - g * nt;
        const uint32_t cb = jb.cb + t * tile, l = jb.lo + g * ch;
        items[x] = Item{cb, min(cb + tile, jb.ce), l, min(l + ch, jb.hi)};
    }
    if (threadIdx.x == 0) *n_items = nout;
}

bool launch_plan_partition_items(const uint32_t* coff, const uint32_t* soff, const uint32_t* n_comp, uint32_t P,
                                 uint64_t lo, uint64_t hi, uint32_t tile, uint32_t chunk, uint32_t max_chunks,
                                 uint32_t cap, Item* items, uint32_t* n_items, cudaStream_t st, uint32_t grain_target) {
    if (P == 0 || P > 1024) return false;
    k_plan_partition_items<<<1, 1024, 0, st>>>(coff, soff, n_comp, P, lo, hi, tile, chunk, max_chunks, cap, items,
                                               n_items, grain_target);
    SKY_LAUNCH_CHECK();
    return true;
}

// Dense list of the live entries of dead[0, n) (base + i, ascending) and the
// segment offsets mapped onto it (off_new[p] = live entries before off[p]),
// in two launches (instead of scan init + scan + remap + compaction): per-
// block live counts, then each block takes the prefix of the blocks before
// it, scans its 8-entry-per-thread spans and writes positions and the
// offsets that fall in its range.
constexpr uint32_t kDcPer = 8, kDcThreads = 256, kDcTile = kDcPer * kDcThreads;

__global__ void __launch_bounds__(kDcThreads) k_dc_count(const uint8_t* __restrict__ dead, uint32_t n,
                                                         uint32_t* __restrict__ block_tot, const uint32_t* n_dev) {
    if (n_dev) n = min(n, *n_dev);  // entries past the device count are dead: not read
    const uint32_t i0 = blockIdx.x * kDcTile + threadIdx.x * kDcPer;
    uint32_t c = 0;
#pragma unroll
    for (uint32_t u = 0; u < kDcPer; ++u) c += (i0 + u < n && !dead[i0 + u]) ? 1u : 0u;
    c = __reduce_add_sync(0xffffffffu, c);
    __shared__ uint32_t s[kDcThreads / 32];
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0;
        for (uint32_t k = 0; k < kDcThreads / 32; ++k) t += s[k];
        block_tot[blockIdx.x] = t;
    }
}

__global__ void __launch_bounds__(kDcThreads) k_dc_emit(const uint8_t* __restrict__ dead, uint32_t n,
                                                        const uint32_t* __restrict__ block_tot,
                                                        const uint32_t* __restrict__ off, uint32_t P, uint32_t base,
                                                        uint32_t* __restrict__ dense, uint32_t* __restrict__ off_new,
                                                        uint32_t* total_out, const uint32_t* n_dev) {
    if (n_dev) n = min(n, *n_dev);
    using Scan = cub::BlockScan<uint32_t, kDcThreads>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ uint32_t s_w[kDcThreads / 32];
    // prefix of the blocks before this one (and the grand total for the last)
    uint32_t pb = 0;
    for (uint32_t k = threadIdx.x; k < blockIdx.x; k += kDcThreads) pb += block_tot[k];
    pb = __reduce_add_sync(0xffffffffu, pb);
    if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = pb;
    __syncthreads();
    uint32_t bpre = 0;
#pragma unroll
    for (uint32_t k = 0; k < kDcThreads / 32; ++k) bpre += s_w[k];
    const uint32_t i0 = blockIdx.x * kDcTile + threadIdx.x * kDcPer;
    uint32_t live = 0;
#pragma unroll
    for (uint32_t u = 0; u < kDcPer; ++u)
        if (i0 + u < n && !dead[i0 + u]) live |= 1u << u;
    uint32_t pre, agg;
    Scan(tmp).ExclusiveSum((uint32_t)__popc(live), pre, agg);
    pre += bpre;
    uint32_t o = pre;
#pragma unroll
    for (uint32_t u = 0; u < kDcPer; ++u)
        if ((live >> u) & 1u) dense[o++] = base + i0 + u;
    // offsets inside this thread's span [i0, min(i0 + kDcPer, n)); off[] is
    // sorted. Offsets at or past n (empty tail segments) get the total from
    // the last block, one per thread.
    if (i0 < n) {
        const uint32_t hi_i = min(i0 + kDcPer, n);
        uint32_t a = 0, c = P + 1;  // first p with off[p] >= i0
        while (a < c) {
            const uint32_t m = (a + c) >> 1;
            if (off[m] < i0) a = m + 1; else c = m;
        }
        for (uint32_t p = a; p <= P && off[p] < hi_i; ++p)
            off_new[p] = pre + __popc(live & ((1u << (off[p] - i0)) - 1u));
    }
    if (blockIdx.x == gridDim.x - 1) {
        const uint32_t total = bpre + agg;
        for (uint32_t p = threadIdx.x; p <= P; p += kDcThreads)
            if (off[p] >= n) off_new[p] = total;
        if (threadIdx.x == 0 && total_out) *total_out = total;
    }
}

bool launch_dense_compact(const uint8_t* dead, uint32_t n, const uint32_t* off, uint32_t P, uint32_t base,
                          uint32_t* dense, uint32_t* off_new, uint32_t* total, uint32_t* block_tot,
                          cudaStream_t st, const uint32_t* n_dev) {
    if (n == 0 || n > (64u << 20)) return false;
    const uint32_t blocks = ceil_div(n, kDcTile);
    k_dc_count<<<blocks, kDcThreads, 0, st>>>(dead, n, block_tot, n_dev);
    SKY_LAUNCH_CHECK();
    k_dc_emit<<<blocks, kDcThreads, 0, st>>>(dead, n, block_tot, off, P, base, dense, off_new, total, n_dev);
    SKY_LAUNCH_CHECK();
    return true;
}

size_t dense_compact_scratch(uint32_t n) { return (size_t)ceil_div(n, kDcTile) * sizeof(uint32_t) + 16; }

void launch_relsky2(int D, int tile, const Relsky2Args& a, int sm_count, cudaStream_t st) {
    if (!a.n_items) return;
    if (tile <= 1 * 32) {
        SKY_DISPATCH_D16(D, (launch_k<DT, 1>(a, sm_count, st)));
    } else if (tile <= 2 * 32) {
        SKY_DISPATCH_D16(D, (launch_k<DT, 2>(a, sm_count, st)));
    } else if (tile <= 4 * 32) {
        SKY_DISPATCH_D16(D, (launch_k<DT, 4>(a, sm_count, st)));
    } else if (tile <= 8 * 32) {
        SKY_DISPATCH_D16(D, (launch_k<DT, 8>(a, sm_count, st)));
    } else {
        throw Error(SKY_E_INTERNAL, "relsky item larger than one warp's candidates");
    }
}

// ----------------------------------------------------------- cell index
// (cell << 32 | skey) of every row of a set: the cell digit of each of the
// spec's dimensions is the top bits[t] bits of its packed code, dim[0] the
// least significant. Codes are monotone in the coordinate, so s <= t
// implies digit(s) <= digit(t) on every dimension.
template <int D>
__global__ void k_cell_keys(const uint2* __restrict__ qc, const uint32_t* __restrict__ skey, uint32_t n, CellSpec cs,
                            uint64_t* __restrict__ key, uint32_t* __restrict__ idx) {
    constexpr int L = CodeLayout<D>::L, LW = CodeLayout<D>::LW, B = CodeLayout<D>::B;
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint2 q = qc[i];
    uint32_t cell = 0;
    for (int t = (int)cs.k - 1; t >= 0; --t) {
        const int j = cs.dim[t];
        const uint32_t w = j / L ? q.y : q.x;
        const uint32_t code = (w >> (LW * (j % L))) & ((1u << B) - 1u);
        cell = (cell << cs.bits[t]) | (code >> (B - cs.bits[t]));
    }
    key[i] = ((uint64_t)cell << 32) | skey[i];
    idx[i] = i;
}

void launch_cell_keys(int D, const uint2* qc, const uint32_t* skey, uint32_t n, const CellSpec& cs, uint64_t* key,
                      uint32_t* idx, cudaStream_t st) {
    if (!n) return;
    SKY_DISPATCH_D16(D, (k_cell_keys<DT><<<ceil_div(n, 256), 256, 0, st>>>(qc, skey, n, cs, key, idx)));
    SKY_LAUNCH_CHECK();
}

// Rows of a dense list (dense[j], partitions doff[P+1] over j) keyed by
// (partition << (32 + K) | cell << 32 | skey), idx[j] = j.
template <int D>
__global__ void k_part_cell_keys(const uint2* __restrict__ qc, const uint32_t* __restrict__ skey,
                                 const uint32_t* __restrict__ dense, const uint32_t* __restrict__ doff, uint32_t P,
                                 uint32_t n, CellSpec cs, uint64_t* __restrict__ key, uint32_t* __restrict__ idx) {
    constexpr int L = CodeLayout<D>::L, LW = CodeLayout<D>::LW, B = CodeLayout<D>::B;
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    // partition of dense position j: the last p with doff[p] <= j
    uint32_t lo = 0, hi = P;
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (doff[mid] <= j) lo = mid; else hi = mid;
    }
    const uint32_t i = dense[j];
    const uint2 q = qc[i];
    uint32_t cell = 0, K = 0;
    for (int t = (int)cs.k - 1; t >= 0; --t) {
        const int dj = cs.dim[t];
        const uint32_t w = dj / L ? q.y : q.x;
        const uint32_t code = (w >> (LW * (dj % L))) & ((1u << B) - 1u);
        cell = (cell << cs.bits[t]) | (code >> (B - cs.bits[t]));
        K += cs.bits[t];
    }
    key[j] = ((uint64_t)lo << (32 + K)) | ((uint64_t)cell << 32) | skey[i];
    idx[j] = j;
}

void launch_part_cell_keys(int D, const uint2* qc, const uint32_t* skey, const uint32_t* dense, const uint32_t* doff,
                           uint32_t P, uint32_t n, const CellSpec& cs, uint64_t* key, uint32_t* idx, cudaStream_t st) {
    if (!n) return;
    SKY_DISPATCH_D16(D, (k_part_cell_keys<DT><<<ceil_div(n, 256), 256, 0, st>>>(qc, skey, dense, doff, P, n, cs,
                                                                                 key, idx)));
    SKY_LAUNCH_CHECK();
}

// dead[rows[i]] |= flag[i]
__global__ void k_scatter_dead(const uint8_t* __restrict__ flag, const uint32_t* __restrict__ rows, uint32_t n,
                               uint8_t* __restrict__ dead) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && flag[i]) dead[rows[i]] = 1;
}

void launch_scatter_dead(const uint8_t* flag, const uint32_t* rows, uint32_t n, uint8_t* dead, cudaStream_t st) {
    if (!n) return;
    k_scatter_dead<<<ceil_div(n, 256), 256, 0, st>>>(flag, rows, n, dead);
    SKY_LAUNCH_CHECK();
}

// ------------------------------------------------------- BNL sub-blocks
// Cut each partition [off[p], off[p+1]) into consecutive blocks of at most
// `block` rows: sub[0..*n_sub] block offsets, padded with empty blocks up to
// sub[cap] (one CTA; each thread takes a contiguous run of partitions).
__global__ void __launch_bounds__(1024) k_split_segments(const uint32_t* __restrict__ off, uint32_t P, uint32_t block,
                                                         uint32_t* __restrict__ sub, uint32_t cap) {
    __shared__ uint32_t s_tot[1024];
    const uint32_t t = threadIdx.x, per = (P + 1023) / 1024;
    const uint32_t p0 = min(P, t * per), p1 = min(P, p0 + per);
    uint32_t mine = 0;
    for (uint32_t p = p0; p < p1; ++p) mine += (off[p + 1] - off[p] + block - 1) / block;
    s_tot[t] = mine;
    __syncthreads();
    // exclusive scan of the per-thread totals (Hillis-Steele over 1024 words)
    for (uint32_t s = 1; s < 1024; s <<= 1) {
        const uint32_t v = t >= s ? s_tot[t - s] : 0u;
        __syncthreads();
        s_tot[t] += v;
        __syncthreads();
    }
    uint32_t at = s_tot[t] - mine;
    for (uint32_t p = p0; p < p1; ++p)
        for (uint32_t b = off[p]; b < off[p + 1]; b += block) sub[at++] = b;
    const uint32_t total = s_tot[1023];
    const uint32_t end = off[P];
    for (uint32_t j = total + t; j <= cap; j += 1024) sub[j] = end;
}

void launch_split_segments(const uint32_t* off, uint32_t P, uint32_t block, uint32_t* sub, uint32_t cap,
                           cudaStream_t st) {
    k_split_segments<<<1, 1024, 0, st>>>(off, P, block, sub, cap);
    SKY_LAUNCH_CHECK();
}

// ------------------------------------------------- issue-rate microbenchmark
// The packed-code test loop of k_relsky3 alone: K candidates' codes in
// registers, a warp's 32 comparator codes in shared memory read as uint4
// pairs (ld.shared.v4, as the kernel's double buffer does), 4 comparators x K
// candidates per step folded by VIMNMX3 into one branch that never fires.
// Its tests/s with every SM busy is the measured issue peak of the dominance
// core's instruction mix (the roofline denominator in bench.py).
__device__ __forceinline__ uint4 lds128v(uint32_t addr) {
    uint4 v;
    asm volatile("ld.volatile.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(addr)
                 : "memory");
    return v;
}

template <int D, int K>
__global__ void __launch_bounds__(256) k_issue_peak(uint32_t iters, uint32_t seed, unsigned long long* sink) {
    constexpr uint32_t G = CodeLayout<D>::G;
    constexpr uint32_t GA = G | 0x80000000u;
    __shared__ __align__(16) uint2 code[8][32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // never-pass comparators (word 1 borrows out of bit 31), unknown to the compiler
    code[warp][lane] = make_uint2(seed * (uint32_t)(lane + 1), 0x80000000u | (seed & 1u));
    __syncwarp();
    uint32_t T[K][2];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        T[k][0] = (seed ^ (threadIdx.x * 977u + k)) | G | CodeLayout<D>::ALIVE;
        T[k][1] = (seed * 31u + threadIdx.x + k) | G | 0x80000000u;
    }
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(&code[warp][0]);
    uint32_t hits = 0;
    for (uint32_t it = 0; it < iters; ++it) {
#pragma unroll
        for (uint32_t i = 0; i < 32; i += 4) {
            // volatile loads: ptxas may not keep one iteration's codes for the next
            const uint4 c01 = lds128v(base + i * 8), c23 = lds128v(base + i * 8 + 16);
            const uint2 q[4] = {make_uint2(c01.x, c01.y), make_uint2(c01.z, c01.w), make_uint2(c23.x, c23.y),
                                make_uint2(c23.z, c23.w)};
            uint32_t h[4 * K];
#pragma unroll
            for (int c = 0; c < 4; ++c)
#pragma unroll
                for (int k = 0; k < K; ++k) h[c * K + k] = coarse_hit<G>(T[k], q[c]);
            if (max_fold<4 * K>(h) == GA) ++hits;
        }
    }
    if (hits) atomicAdd(sink, (unsigned long long)hits);
}

template <int D, int K>
double issue_peak_impl(int sm_count, uint32_t iters, int blocks_per_sm, cudaStream_t st, unsigned long long* sink) {
    const uint32_t grid = (uint32_t)(sm_count * blocks_per_sm);
    k_issue_peak<D, K><<<grid, 256, 0, st>>>(16, 12345u, sink);  // warm-up
    SKY_LAUNCH_CHECK();
    cudaEvent_t e0, e1;
    SKY_CUDA(cudaEventCreate(&e0));
    SKY_CUDA(cudaEventCreate(&e1));
    SKY_CUDA(cudaEventRecord(e0, st));
    k_issue_peak<D, K><<<grid, 256, 0, st>>>(iters, 12345u, sink);
    SKY_LAUNCH_CHECK();
    SKY_CUDA(cudaEventRecord(e1, st));
    SKY_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    SKY_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    const double tests = (double)grid * 256.0 * iters * 32.0 * K;
    return tests / (ms / 1e3);
}

double measure_issue_peak(int D, int K, int blocks_per_sm, uint32_t iters, int sm_count, cudaStream_t st,
                          unsigned long long* sink) {
    double r = 0.0;
#define SKY_IP(KK) SKY_DISPATCH_D16(D, (r = issue_peak_impl<DT, KK>(sm_count, iters, blocks_per_sm, st, sink)))
    if (K <= 1) { SKY_IP(1); }
    else if (K <= 2) { SKY_IP(2); }
    else if (K <= 4) { SKY_IP(4); }
    else { SKY_IP(8); }
#undef SKY_IP
    return r;
}

}  // namespace sky
