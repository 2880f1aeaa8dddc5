// kernels_rand.cu — the reference's random partitioner on the GPU, bit-exact.
//
// assign_random (partition.cpp:36-54) shuffles 0..n-1 with Fisher-Yates
// driven by Rng(seed) = std::mt19937_64 (rng.hpp:15-60): for i = n..2,
// j_i = below(i) (rejection sampling, x % i), swap(v[i-1], v[j_i]); then
// partition_of[perm[k]] = k mod p. Here:
//   1. one CTA produces the mt19937_64 output stream (the twist runs as two
//      156-wide dependent phases; the standard's published parameters);
//   2. j_i = x_k % i for k = n - i, in parallel; a draw that the reference
//      would reject (x >= 2^64 - 2^64 mod i, probability ~n^2/2^65) raises a
//      flag and the caller reproduces the shuffle on the host instead;
//   3. the swap sequence is resolved without executing it: let S_p be the
//      steps with j_i = p. Position i-1 is final after step i, so
//      perm[i-1] = g(i), the value at j_i just before step i, and the value
//      at position p just before step i is f(i*) for the next-larger step i*
//      in S_p (or p itself), where f(i) = value at i-1 just before step i
//      follows the same rule on S_{i-1}. Sorting (j_i, i) gives every S_p; f
//      is resolved by pointer jumping (pointers only increase), g and the
//      partition ids in one final pass.
#include <cooperative_groups.h>
#include <cub/cub.cuh>

#include "kernels.cuh"

namespace sky {

namespace {

constexpr int MT_N = 312, MT_M = 156;
constexpr uint64_t MT_UM = 0xFFFFFFFF80000000ull, MT_LM = 0x7FFFFFFFull;

__device__ __forceinline__ uint64_t mt_tw(uint64_t a, uint64_t b) {
    const uint64_t x = (a & MT_UM) | (b & MT_LM);
    return (x >> 1) ^ ((x & 1ull) ? 0xB5026F5AA96619E9ull : 0ull);
}

__device__ __forceinline__ uint64_t mt_temper(uint64_t x) {
    x ^= (x >> 29) & 0x5555555555555555ull;
    x ^= (x << 17) & 0x71D67FFFEDA60000ull;
    x ^= (x << 37) & 0xFFF7EEE000000000ull;
    x ^= x >> 43;
    return x;
}

// Untempered mt19937_64 state sequence: x[m] = x[m-156] ^ tw(x[m-312], x[m-311]).
// Thread t < 156 of a 160+-thread CTA keeps A = x[m0-312+t] and
// B = x[m0-156+t] in registers and produces x[m0+t] = B ^ tw(A, A') and
// x[m0+156+t] = x[m0+t] ^ tw(B, B'), the primed values being thread t+1's
// (warp shuffles; shared memory across warp boundaries). Thread 155's
// B' = x[m0] is recomputed from thread 0 and 1's registers. One barrier
// per 312 outputs; the boundary slots are double-buffered by parity. Every
// thread of the CTA must call it. (A single-warp variant without barriers
// measured slower: issue bound at ~130 instructions per 312 outputs.)
__device__ void mt_generate(uint64_t A, uint64_t B, uint32_t count, uint64_t* __restrict__ out) {
    __shared__ uint64_t sA[2][8], sB[2][8], sA1[2];  // per parity: each warp's lane-0 A/B; thread 1's A
    const uint32_t t = threadIdx.x, lane = t & 31, w = t >> 5;
    uint32_t par = 0;
    for (uint32_t k0 = 0; k0 < count; k0 += MT_N, par ^= 1) {
        if (t < MT_M && lane == 0) {
            sA[par][w] = A;
            sB[par][w] = B;
        }
        if (t == 1) sA1[par] = A;
        __syncthreads();
        const uint64_t An = __shfl_down_sync(0xffffffffu, A, 1);
        const uint64_t Bn = __shfl_down_sync(0xffffffffu, B, 1);
        if (t < MT_M) {
            uint64_t A1, B1;
            if (t + 1 == MT_M) {
                // t = 155: A' = x[m0-156] = thread 0's B; B' = x[m0] recomputed
                A1 = sB[par][0];
                B1 = sB[par][0] ^ mt_tw(sA[par][0], sA1[par]);
            } else if (lane == 31) {
                A1 = sA[par][w + 1];
                B1 = sB[par][w + 1];
            } else {
                A1 = An;
                B1 = Bn;
            }
            const uint64_t v0 = B ^ mt_tw(A, A1);   // x[m0 + t]
            const uint64_t v1 = v0 ^ mt_tw(B, B1);  // x[m0 + 156 + t]
            if (k0 + t < count) out[k0 + t] = v0;
            if (k0 + MT_M + t < count) out[k0 + MT_M + t] = v1;
            A = v0;
            B = v1;
        }
    }
}

// Sequential stream: x[0..311] = seeded state (optionally to state_out);
// out[k] = x[312 + k] for k < count (untempered; the consumer tempers).
__global__ void __launch_bounds__(160) k_mt64(uint64_t seed, uint32_t count, uint64_t* __restrict__ out,
                                              uint64_t* __restrict__ state_out) {
    __shared__ uint64_t init[MT_N];
    const uint32_t t = threadIdx.x;
    if (t == 0) {
        init[0] = seed;
        for (int i = 1; i < MT_N; ++i)
            init[i] = 6364136223846793005ull * (init[i - 1] ^ (init[i - 1] >> 62)) + (uint64_t)i;
    }
    __syncthreads();
    if (state_out)
        for (uint32_t i = t; i < MT_N; i += blockDim.x) state_out[i] = init[i];
    uint64_t A = 0, B = 0;
    if (t < MT_M) {
        A = init[t];
        B = init[MT_M + t];
    }
    mt_generate(A, B, count, out);
}

// Jump-ahead stream: chunk k = blockIdx.x writes out[kJ .. min(m, (k+1)J)).
// Its start window W_kJ = sum_i g_k[i] W_i (g_k = t^(kJ) mod phi, table row
// k-1; mtjump.cpp) is a correlation of g_k's coefficient bits with the first
// 19937 + 312 stream words xs[] (seeded state + 19937 outputs), evaluated in
// shared memory over the set bits only; then the chunk runs mt_generate.
constexpr uint32_t MT_DEG = 19937, MT_XS = MT_DEG + MT_N, MT_GW = 624;

__global__ void __launch_bounds__(1024) k_mt_jump(const uint64_t* __restrict__ xs, const uint32_t* __restrict__ gtab,
                                                  uint32_t J, uint32_t m, uint64_t* __restrict__ out) {
    extern __shared__ uint64_t sm_x[];               // [MT_XS]
    uint32_t* sm_g = reinterpret_cast<uint32_t*>(sm_x + MT_XS);  // [MT_GW]
    __shared__ unsigned long long win[MT_N];
    const uint32_t k = blockIdx.x, t = threadIdx.x;
    if (k == 0) {
        for (uint32_t i = t; i < MT_N; i += blockDim.x) win[i] = xs[i];
    } else {
        for (uint32_t i = t; i < MT_XS; i += blockDim.x) sm_x[i] = xs[i];
        const uint32_t* g = gtab + (size_t)(k - 1) * MT_GW;
        for (uint32_t i = t; i < MT_GW; i += blockDim.x) sm_g[i] = g[i];
        for (uint32_t i = t; i < MT_N; i += blockDim.x) win[i] = 0;
        __syncthreads();
        // warp w takes coefficient words w, w+32, ...; lane l accumulates
        // window words l + 32r (10 independent accumulators)
        constexpr int RW = (MT_N + 31) / 32;
        const uint32_t lane = t & 31, w = t >> 5, nw = blockDim.x >> 5;
        uint64_t acc[RW];
#pragma unroll
        for (int r = 0; r < RW; ++r) acc[r] = 0;
        for (uint32_t wi = w; wi < MT_GW; wi += nw) {
            uint32_t gw = sm_g[wi];
            while (gw) {
                const uint32_t i = wi * 32 + (uint32_t)(__ffs(gw) - 1);  // i < 19937
                gw &= gw - 1;
                const uint64_t* xi = sm_x + i + lane;
#pragma unroll
                for (int r = 0; r < RW; ++r)
                    if (lane + 32 * r < MT_N) acc[r] ^= xi[32 * r];
            }
        }
#pragma unroll
        for (int r = 0; r < RW; ++r)
            if (lane + 32 * r < MT_N) atomicXor(&win[lane + 32 * r], (unsigned long long)acc[r]);
    }
    __syncthreads();
    uint64_t A = 0, B = 0;
    if (t < MT_M) {
        A = win[t];
        B = win[MT_M + t];
    }
    const uint64_t base = (uint64_t)k * J;
    const uint64_t left = base >= m ? 0ull : (uint64_t)m - base;
    const uint32_t cnt = (uint32_t)(left < J ? left : J);
    mt_generate(A, B, cnt, out + base);
}

// step i = n - k: j_i = x_k mod i; flag a rejected draw. The (j, i) pairs
// are stored in ascending-i order (slot m-1-k), so a stable sort by j alone
// leaves every S_p in ascending step order.
__global__ void k_fy_draws(const uint64_t* __restrict__ x, uint32_t n, uint32_t* __restrict__ jkey,
                           uint32_t* __restrict__ ival, uint32_t* __restrict__ jv, uint32_t* flag) {
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k + 1 >= n) return;  // n-1 steps
    const uint64_t i = (uint64_t)n - k;
    const uint64_t limit = UINT64_MAX - UINT64_MAX % i;
    const uint64_t v = mt_temper(x[k]);
    if (v >= limit) atomicOr(flag, 1u);
    const uint32_t j = (uint32_t)(v % i);
    jv[k] = j;
    const uint32_t slot = n - 2 - k;  // m - 1 - k
    jkey[slot] = j;
    ival[slot] = (uint32_t)i;
}

__global__ void k_fy_heads(const uint32_t* __restrict__ sj, uint32_t m, uint32_t* __restrict__ head) {
    const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= m) return;
    const uint32_t p = sj[q];
    if (q == 0 || sj[q - 1] != p) head[p] = q;
}

// gnext[i]: next larger step in S_{j_i}; f pointers for every step i.
__global__ void k_fy_ptrs(const uint32_t* __restrict__ sj, const uint32_t* __restrict__ si, uint32_t m,
                          const uint32_t* __restrict__ head, uint32_t n, uint32_t* __restrict__ gnext,
                          uint32_t* __restrict__ fptr, uint32_t* __restrict__ fval) {
    const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q < m) {
        const uint32_t p = sj[q], i = si[q];
        gnext[i] = (q + 1 < m && sj[q + 1] == p) ? si[q + 1] : kNone;
    }
    const uint32_t i = q + 2;  // steps 2..n
    if (i <= n) {
        const uint32_t h = head[i - 1];
        uint32_t v = kNone;
        if (h != kNone) {
            v = si[h];
            if (v == i) {
                const uint32_t h2 = h + 1;
                v = (h2 < m && sj[h2] == i - 1) ? si[h2] : kNone;
            }
        }
        if (v == kNone) {
            fval[i] = i - 1;  // position i-1 untouched before step i
            fptr[i] = kNone;
        } else {
            fval[i] = kNone;
            fptr[i] = v;
        }
    }
}

// pointer jumping until every f is resolved (cooperative: grid-wide sync)
__global__ void k_fy_jump(uint32_t n, uint32_t* __restrict__ fptr, uint32_t* __restrict__ fval, uint32_t* pending) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    const uint32_t stride = gridDim.x * blockDim.x;
    for (int round = 0; round < 64; ++round) {
        uint32_t local = 0;
        for (uint32_t i = 2 + blockIdx.x * blockDim.x + threadIdx.x; i <= n; i += stride) {
            if (fval[i] != kNone) continue;
            const uint32_t j = fptr[i];
            const uint32_t vj = ((volatile uint32_t*)fval)[j];
            if (vj != kNone) {
                fval[i] = vj;
            } else {
                fptr[i] = ((volatile uint32_t*)fptr)[j];
                ++local;
            }
        }
        local = __reduce_add_sync(0xffffffffu, local);
        if ((threadIdx.x & 31) == 0 && local) atomicAdd(pending + (round & 3), local);
        // one grid barrier per round: four rotating counters; the one reset
        // here was last read right after round-2's barrier, which every
        // thread passed before round-1's
        if (blockIdx.x == 0 && threadIdx.x == 0) pending[(round + 2) & 3] = 0;
        grid.sync();
        if (pending[round & 3] == 0) break;
    }
}

// perm[k] (k >= 1) = g(k+1); perm[0] = value at 0 after its last touch.
__global__ void k_fy_final(uint32_t n, uint64_t p, const uint32_t* __restrict__ jv, const uint32_t* __restrict__ gnext,
                           const uint32_t* __restrict__ fval, const uint32_t* __restrict__ head,
                           const uint32_t* __restrict__ si, uint32_t* __restrict__ pid) {
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    uint32_t v;
    if (k == 0) {
        const uint32_t h = head[0];
        v = h == kNone ? 0u : fval[si[h]];
    } else {
        const uint32_t i = k + 1;
        const uint32_t gn = gnext[i];
        v = gn != kNone ? fval[gn] : jv[n - i];
    }
    pid[v] = (uint32_t)(k % p);
}


// ------------------------------------------------------------ generators
// The BASELINE inputs (include/skyline_baseline_gen.h) on the device: chunk
// c of 65,536 rows is one CTA running its own mt19937_64 stream (seed ^
// 0x9E3779B97F4A7C15 * (c + 1)) block by block into a shared-memory ring
// (threads 0..155 as in mt_generate) while the rows consume it in stream
// order. Rows with a fixed number of draws (kinds 1, 3, 5) are converted by
// all threads in parallel; the anti-correlated rejection loop (kinds 2, 4)
// is one warp testing 32 consecutive attempts per step (a ballot picks the
// first accepted). Host arithmetic is restated exactly (no FMA contraction;
// float uniforms from 24 bits); the normals go through CUDA's log / cos,
// so kinds 2-4 equal the host generator wherever those round like the host
// libm (checked at the BASELINE sizes by tests/test_generate_gpu.py).
constexpr uint32_t GEN_RING = 32;         // blocks of 312 draws in the ring (78 KB)
constexpr uint32_t GEN_THREADS = 192;
constexpr uint64_t GEN_CHUNK = 65536;

__device__ __forceinline__ float gen_f32(uint64_t x) { return (float)(mt_temper(x) >> 40) * 0x1.0p-24f; }
__device__ __forceinline__ double gen_u01(uint64_t x) { return (double)(mt_temper(x) >> 11) * 0x1.0p-53; }
__device__ __forceinline__ double gen_u01_pos(uint64_t x) { return (double)((mt_temper(x) >> 11) + 1) * 0x1.0p-53; }
// Rng::normal (rng.hpp:31-37): mean + stddev * r * cos(2 pi u2), evaluated
// in the host's order without contraction
__device__ __forceinline__ double gen_normal(uint64_t x1, uint64_t x2, double mean, double stddev) {
    const double u1 = gen_u01_pos(x1), u2 = gen_u01(x2);
    const double r = sqrt(__dmul_rn(-2.0, log(u1)));
    const double c = cos(__dmul_rn(6.283185307179586476925286766559, u2));
    return __dadd_rn(mean, __dmul_rn(__dmul_rn(stddev, r), c));
}
__device__ __forceinline__ double gen_clip01(double v) { return v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v); }

__global__ void __launch_bounds__(GEN_THREADS) k_gen_baseline(int kind, uint64_t n, uint32_t d, uint64_t seed,
                                                               float* __restrict__ out, uint32_t* stuck) {
    extern __shared__ uint64_t ring[];  // [GEN_RING * MT_N]
    __shared__ uint64_t init[MT_N];
    __shared__ uint64_t sA[2][8], sB[2][8], sA1[2];
    __shared__ unsigned long long s_pos;  // next unconsumed draw (stream index)
    __shared__ unsigned long long s_q;    // anti-correlated: next attempt of the row at s_pos (0: none yet)
    __shared__ uint32_t s_row;            // next row of the chunk
    const uint32_t t = threadIdx.x, lane = t & 31, w = t >> 5;
    const uint64_t c = blockIdx.x, r0 = c * GEN_CHUNK;
    const uint32_t rows = (uint32_t)min(GEN_CHUNK, n - r0);
    if (t == 0) {
        init[0] = seed ^ (0x9E3779B97F4A7C15ull * (c + 1));
        for (int i = 1; i < MT_N; ++i)
            init[i] = 6364136223846793005ull * (init[i - 1] ^ (init[i - 1] >> 62)) + (uint64_t)i;
        s_pos = 0;
        s_q = 0;
        s_row = 0;
    }
    __syncthreads();
    uint64_t A = 0, B = 0;
    if (t < MT_M) {
        A = init[t];
        B = init[MT_M + t];
    }
    const bool fixed = kind == 1 || kind == 3 || kind == 5;
    const uint32_t per = kind == 3 ? 2 + 2 * d : d;  // draws per row (fixed kinds)
    uint64_t made = 0;                                  // draws generated so far
    uint32_t par = 0;
    while (true) {
        // produce one block if the ring has room past the unconsumed draws
        const uint64_t pos = s_pos;
        const bool room = made + MT_N <= pos - pos % MT_N + (uint64_t)(GEN_RING - 1) * MT_N;
        if (room) {
            if (t < MT_M && lane == 0) {
                sA[par][w] = A;
                sB[par][w] = B;
            }
            if (t == 1) sA1[par] = A;
        }
        __syncthreads();
        if (room) {
            const uint64_t An = __shfl_down_sync(0xffffffffu, A, 1);
            const uint64_t Bn = __shfl_down_sync(0xffffffffu, B, 1);
            if (t < MT_M) {
                uint64_t A1, B1;
                if (t + 1 == MT_M) {
                    A1 = sB[par][0];
                    B1 = sB[par][0] ^ mt_tw(sA[par][0], sA1[par]);
                } else if (lane == 31) {
                    A1 = sA[par][w + 1];
                    B1 = sB[par][w + 1];
                } else {
                    A1 = An;
                    B1 = Bn;
                }
                const uint64_t v0 = B ^ mt_tw(A, A1), v1 = v0 ^ mt_tw(B, B1);
                const uint32_t slot = (uint32_t)((made / MT_N) % GEN_RING) * MT_N;
                ring[slot + t] = v0;
                ring[slot + MT_M + t] = v1;
                A = v0;
                B = v1;
            }
            made += MT_N;
            par ^= 1;
        }
        __syncthreads();
        // consume: rows whose draws are all in the ring
        if (fixed) {
            const uint32_t row0 = s_row;
            const uint64_t ready = made / per;
            const uint32_t avail_rows = ready < rows ? (uint32_t)ready : rows;
            for (uint32_t r = row0 + t; r < avail_rows; r += GEN_THREADS) {
                const uint64_t p = (uint64_t)r * per;
                float* x = out + (r0 + r) * d;
                auto at = [&](uint64_t q) { return ring[(uint32_t)(q % (GEN_RING * MT_N))]; };
                if (kind == 1) {
                    for (uint32_t j = 0; j < d; ++j) x[j] = gen_f32(at(p + j));
                } else if (kind == 5) {
                    for (uint32_t j = 0; j < d; ++j) x[j] = (float)(mt_temper(at(p + j)) >> 60);
                } else {
                    const double v = gen_clip01(gen_normal(at(p), at(p + 1), 0.5, 0.25));
                    for (uint32_t j = 0; j < d; ++j)
                        x[j] = (float)gen_clip01(__dadd_rn(v, gen_normal(at(p + 2 + 2 * j), at(p + 3 + 2 * j), 0.0, 0.05)));
                }
            }
            __syncthreads();
            if (t == 0) {
                s_row = avail_rows;
                s_pos = (uint64_t)avail_rows * per;
            }
            __syncthreads();
            if (avail_rows >= rows) break;
        } else {
            // one warp: s (2 draws), then attempts of d uniforms until one
            // lands within the tolerance; 32 attempts per step
            if (w == 0) {
                uint64_t p = s_pos, q0 = s_q;
                uint32_t r = s_row;
                const uint64_t lim = made;
                const double tol = __dmul_rn(0.01, (double)d);
                while (r < rows) {
                    // the row's s and a full step of attempts must be in the ring
                    const uint64_t qs = q0 ? q0 : p + 2;
                    if (qs + 32ull * d > lim) break;
                    auto at = [&](uint64_t q) { return ring[(uint32_t)(q % (GEN_RING * MT_N))]; };
                    const double s = gen_clip01(gen_normal(at(p), at(p + 1), 0.5, 0.0625));
                    const double target = __dmul_rn((double)d, s);
                    uint64_t q = qs;
                    bool done = false;
                    while (!done) {
                        if (q + 32ull * d > lim) break;
                        double sum = 0.0;
                        for (uint32_t j = 0; j < d; ++j) sum = __dadd_rn(sum, (double)gen_f32(at(q + lane * d + j)));
                        const bool ok = fabs(__dsub_rn(sum, target)) <= tol;
                        const uint32_t bal = __ballot_sync(0xffffffffu, ok);
                        if (bal) {
                            const uint32_t win = __ffs(bal) - 1;
                            const uint64_t qa = q + (uint64_t)win * d;
                            float* x = out + (r0 + r) * d;
                            for (uint32_t j = lane; j < d; j += 32) x[j] = gen_f32(at(qa + j));
                            q = qa + d;
                            done = true;
                        } else {
                            q += 32ull * d;
                        }
                    }
                    if (!done) {  // more draws needed: resume this row at attempt q
                        q0 = q;
                        break;
                    }
                    p = q;
                    q0 = 0;
                    ++r;
                }
                if (lane == 0) {
                    s_pos = p;
                    s_q = q0;
                    s_row = r;
                }
            }
            __syncthreads();
            if (s_row >= rows) break;
            // a row whose attempts outrun the whole ring (probability below
            // 1e-30 per row): report it, the caller generates on the host
            if (!room && (s_q ? s_q : s_pos + 2) + 32ull * d > made) {
                if (t == 0) atomicOr(stuck, 1u);
                break;
            }
        }
    }
}

}  // namespace

size_t random_scratch_bytes(uint32_t n) {
    // x (8n) + key (8n) + key2 (8n) + jv (4n) + head (4n) + gnext/fptr/fval (12(n+1)) + pending
    return (size_t)n * 44 + 64;
}

// Partition ids of the reference's random assignment, on `st`. Returns false
// (nothing written) when a draw would have been rejected; the caller then
// reproduces the shuffle on the host. Synchronizes once to read the flag.
bool random_partition_gpu(uint32_t n, uint64_t p, uint64_t seed, uint32_t* pid, void* scratch, void* cub_tmp,
                          size_t cub_bytes, int sm_count, cudaStream_t st, uint32_t* launches,
                          const uint32_t* jump_table, uint32_t* flag_dev) {
    if (n == 0) return true;
    if (n == 1) {
        SKY_CUDA(cudaMemsetAsync(pid, 0, sizeof(uint32_t), st));
        return true;
    }
    char* s = static_cast<char*>(scratch);
    uint64_t* x = reinterpret_cast<uint64_t*>(s);
    uint64_t* key = x + n;   // jkey | ival (and the jump prefix before them)
    uint64_t* key2 = key + n;  // sj | si
    uint32_t* jkey = reinterpret_cast<uint32_t*>(key);
    uint32_t* ival = jkey + n;
    uint32_t* sj = reinterpret_cast<uint32_t*>(key2);
    uint32_t* si = sj + n;
    uint32_t* jv = reinterpret_cast<uint32_t*>(key2 + n);
    uint32_t* head = jv + n;
    uint32_t* gnext = head + n;
    uint32_t* fptr = gnext + (n + 1);
    uint32_t* fval = fptr + (n + 1);
    uint32_t* misc = fval + (n + 1);  // flag, pending[4]
    const uint32_t m = n - 1;
    SKY_CUDA(cudaMemsetAsync(misc, 0, 8 * sizeof(uint32_t), st));
    SKY_CUDA(cudaMemsetAsync(head, 0xFF, (size_t)n * sizeof(uint32_t), st));
    if (jump_table && m > (1u << 18)) {
        // many CTAs: each chunk of 2^kJumpLog2 outputs from its jumped window
        uint64_t* xs = key;  // 20249 words of scratch, consumed before k_fy_draws writes key
        k_mt64<<<1, 160, 0, st>>>(seed, MT_DEG, xs + MT_N, xs);
        const uint32_t J = 1u << kJumpLog2, chunks = (m + J - 1) / J;
        const size_t smem = (size_t)MT_XS * 8 + MT_GW * 4;
        SKY_CUDA(cudaFuncSetAttribute(k_mt_jump, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k_mt_jump<<<chunks, 1024, smem, st>>>(xs, jump_table, J, m, x);
        if (launches) *launches += 1;
    } else {
        k_mt64<<<1, 160, 0, st>>>(seed, m, x, nullptr);
    }
    k_fy_draws<<<ceil_div(m, 256), 256, 0, st>>>(x, n, jkey, ival, jv, flag_dev ? flag_dev : misc);
    int end_bit = 1;
    while (end_bit < 32 && (uint64_t{1} << end_bit) < n) ++end_bit;  // j < n
    size_t need = 0;
    SKY_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, need, jkey, sj, ival, si, (int)m, 0, end_bit, st));
    if (need > cub_bytes) throw Error(SKY_E_INTERNAL, "cub scratch too small for the random partitioner");
    SKY_CUDA(cub::DeviceRadixSort::SortPairs(cub_tmp, need, jkey, sj, ival, si, (int)m, 0, end_bit, st));
    k_fy_heads<<<ceil_div(m, 256), 256, 0, st>>>(sj, m, head);
    k_fy_ptrs<<<ceil_div(n, 256), 256, 0, st>>>(sj, si, m, head, n, gnext, fptr, fval);
    {
        int per_sm = 0;
        SKY_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_fy_jump, 256, 0));
        const int grid = std::max(1, std::min(per_sm * sm_count, (int)ceil_div(n, 256)));
        uint32_t nn = n;
        uint32_t* pending = misc + 1;
        void* args[] = {&nn, &fptr, &fval, &pending};
        SKY_CUDA(cudaLaunchCooperativeKernel((void*)k_fy_jump, grid, 256, args, 0, st));
    }
    k_fy_final<<<ceil_div(n, 256), 256, 0, st>>>(n, p, jv, gnext, fval, head, si, pid);
    SKY_LAUNCH_CHECK();
    if (launches) *launches += 7 + 4;
    if (flag_dev) return true;  // the caller checks the rejection flag at its next round trip
    uint32_t flag = 0;
    SKY_CUDA(cudaMemcpyAsync(&flag, misc, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    SKY_CUDA(cudaStreamSynchronize(st));
    return flag == 0;
}

size_t random_cub_bytes(uint32_t n) {
    if (n < 2) return 16;
    size_t need = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, need, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                    (const uint32_t*)nullptr, (uint32_t*)nullptr, (int)(n - 1), 0, 32, (cudaStream_t)0);
    return need;
}

void launch_generate_baseline(int kind, uint64_t n, uint32_t d, uint64_t seed, float* out, uint32_t* stuck,
                              cudaStream_t st) {
    if (!n) return;
    const uint64_t chunks = (n + GEN_CHUNK - 1) / GEN_CHUNK;
    const size_t smem = (size_t)GEN_RING * MT_N * sizeof(uint64_t);
    ensure_smem_attr((const void*)k_gen_baseline, smem);
    k_gen_baseline<<<(unsigned)chunks, GEN_THREADS, smem, st>>>(kind == 4 ? 2 : kind, n, d, seed, out, stuck);
    SKY_LAUNCH_CHECK();
}

}  // namespace sky
