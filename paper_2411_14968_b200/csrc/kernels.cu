// kernels.cu — sm_100a kernels of the skyline engine.
//
// HBM-bound passes (prep, scatter/gather, offsets) are written for coalesced
// row streams; the dominance core (k_relsky) and the BNL window kernel are
// compare-issue bound: comparator tiles are staged in shared memory and
// broadcast to every thread, each thread keeps RS_K candidates in registers,
// and warps leave a tile as soon as their coordinate-sum bound is passed or
// all their candidates are dominated.
#include <cub/cub.cuh>
#include <dlfcn.h>

#include <map>
#include <mutex>
#include <string>
#include <tuple>

#include "kernels.cuh"
#include "stream.cuh"

namespace sky {

// Host-side caches for launch configuration queries (the dynamic shared
// memory attribute and the occupancy of a kernel), so a run does not pay
// for them on every launch.
// Function attributes belong to the current device's context, so every cache
// is keyed by the device as well (a process may drive several GPUs).
static int current_device() {
    int dev = 0;
    SKY_CUDA(cudaGetDevice(&dev));
    return dev;
}
void ensure_smem_attr(const void* func, size_t smem) {
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, size_t> done;
    const int dev = current_device();
    // set even below 48 KB: static + dynamic shared memory past 48 KB needs it
    std::lock_guard<std::mutex> lk(mu);
    size_t& cur = done[std::make_pair(dev, func)];
    if (cur >= smem) return;
    const cudaError_t e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) {
        cudaGetLastError();  // not sticky: leave no stale error for the next launch check
        Dl_info info{};
        const char* name = dladdr(func, &info) && info.dli_sname ? info.dli_sname : "?";
        throw Error(SKY_E_INTERNAL, std::string("shared memory request of ") + std::to_string(smem) + " bytes refused for " +
                                        name + ": " + cudaGetErrorString(e));
    }
    cur = smem;
}
int occupancy_cached(const void* func, int threads, size_t smem) {
    static std::mutex mu;
    static std::map<std::tuple<int, const void*, int, size_t>, int> cache;
    const int dev = current_device();
    std::lock_guard<std::mutex> lk(mu);
    const auto key = std::make_tuple(dev, func, threads, smem);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    int per_sm = 0;
    SKY_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, func, threads, smem));
    cache[key] = per_sm;
    return per_sm;
}

int device_sm_count() {
    static std::mutex mu;
    static std::map<int, int> cache;
    const int dev = current_device();
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(dev);
    if (it != cache.end()) return it->second;
    int sms = 0;
    SKY_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    cache[dev] = sms;
    return sms;
}

int padded_dim(uint32_t d) {
    static const int widths[] = {2, 3, 4, 5, 6, 8, 10, 12, 16, 24, 32};
    for (int w : widths)
        if ((int)d <= w) return w;
    return 0;
}

#define SKY_DISPATCH_D(D, ...)                                  \
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
        case 24: { constexpr int DT = 24; __VA_ARGS__; break; } \
        case 32: { constexpr int DT = 32; __VA_ARGS__; break; } \
        default: throw Error(SKY_E_DIMENSION, "unsupported padded dimension"); \
    }

template <int D>
struct Dims {
    static constexpr int D4 = (D + 3) / 4 * 4;
    static constexpr int V = D4 / 4;  // float4 per row
};

__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ uint32_t canon_bits(float v) {
    return v == 0.0f ? 0u : __float_as_uint(v);  // -0.0 and +0.0 compare equal
}

// ------------------------------------------------------------------ prep
// One thread per row: FP64 coordinate sum (core.hpp:103-107, left to right,
// no FMA), input validation (core.cpp:21-46, partition.cpp:26-29), partition
// id for grid (partition.cpp:66-75) and angular (partition.cpp:118-148), and
// the slicing key for sliced.
// Row accessors of the prep pass: a row in memory (float or FP64 rows,
// loops not unrolled) or a float row held in registers (loops fully
// unrolled so every index is static).
struct MemRow {
    static constexpr int kUnroll = 1;
    static constexpr bool kF32 = false;  // decisions on X() (float or FP64 rows)
    const float* xf;
    const double* xd;
    __device__ __forceinline__ float f(uint32_t j) const { return xf[j]; }
    // every value as the reference sees it (float input upcasts exactly)
    __device__ __forceinline__ double X(uint32_t j) const { return xd ? xd[j] : (double)xf[j]; }
};
template <int DP>
struct RegRow {
    static constexpr int kUnroll = DP;
    static constexpr bool kF32 = true;  // float rows: validation and cells in FP32 (exact, see prep_row)
    float v[DP];
    __device__ __forceinline__ float f(uint32_t j) const { return v[j]; }
    __device__ __forceinline__ double X(uint32_t j) const { return (double)v[j]; }
};

// sign of y - x * (th + tl) for doubles x, y >= 0 in [2^-600, 2^600]:
// +1 / -1, or 0 when the difference is within the error bound (|.| <=
// 2^-98 of the operands; the threshold itself is accurate to ~2^-105)
__device__ __forceinline__ int cmp_tan(double y, double x, double th, double tl) {
    const double p = __dmul_rn(x, th);
    const double e = fma(x, th, -p);  // x*th = p + e exactly
    const double r = __dsub_rn(y, p);  // exact when p is within a factor 2 of y
    const double s = __dsub_rn(__dsub_rn(r, e), __dmul_rn(x, tl));
    const double tol = 0x1p-98 * fmax(y, p);
    return s > tol ? 1 : (s < -tol ? -1 : 0);
}

// slice of one hyperspherical angle phi = atan2(y, x) (partition.cpp:128-143)
// as the reference computes it on the host libm; *amb when the exact angle
// lies within the libm's 1-ulp latitude of a slice boundary.
__device__ __forceinline__ uint32_t angular_slice_exact(double y, double x, const double4* __restrict__ thr,
                                                        uint32_t m, double c45, bool* amb) {
    // y = sqrt(sum of squares) is +0 or positive; x >= 0 may be -0.0:
    // atan2(+0, +0) = +0 (slice 0), atan2(+0, -0) = pi (2m, clamped to m - 1)
    if (y == 0.0) return signbit(x) ? m - 1 : 0;
    double phi = -1.0;
    if (x == 0.0) {
        phi = 0x1.921fb54442d18p+0;  // atan2(y > 0, +0) = rn(pi/2)
    } else if (y == x) {
        phi = c45;  // the host libm's atan2(x, x)
    } else {
        // scale to a common exponent (the comparison is scale invariant)
        const int ex = max(ilogb(y), ilogb(x));
        const double ys = scalbn(y, -ex), xs = scalbn(x, -ex);
        if (xs < 0x1p-600) return m - 1;  // angle within 2^-600 of pi/2: above every boundary
        if (ys < 0x1p-600) return 0;      // angle within 2^-600 of 0: below every boundary
        // s = #{k : phi >= phi*_k} (the angle is above tan(phi*_k))
        uint32_t lo = 0, hi = m - 1;
        while (lo < hi) {
            const uint32_t mid = (lo + hi + 1) >> 1;
            const double4 t = thr[mid - 1];
            if (cmp_tan(ys, xs, t.z, t.w) > 0) lo = mid; else hi = mid - 1;
        }
        // the next boundary must be cleared from below: angle <= pred(phi*)
        if (lo + 1 <= m - 1) {
            const double4 t = thr[lo];
            if (cmp_tan(ys, xs, t.x, t.y) >= 0) *amb = true;
        }
        return lo;
    }
    const double v = __dmul_rn(__ddiv_rn(__dmul_rn(2.0, phi), 3.14159265358979323846), (double)m);
    const uint32_t slice = (uint32_t)v;
    return slice >= m ? m - 1 : slice;
}

// One row of the prep pass: validation, FP64 sum, partition id, sort key
// (j < DMAX covers every coordinate: DMAX >= d). Returns the sort key.
// End of a row's coordinates inside a loop over j < DMAX: a row in memory
// stops the loop; a row in registers (unrolled, DMAX = its width) skips the
// remaining iterations instead, so every index stays a compile-time
// constant and the row never goes to local memory.
#define SKY_ROW_END            \
    {                          \
        if constexpr (U == 1)  \
            break;             \
        else                   \
            continue;          \
    }

// ST >= 0: the strategy as a compile-time constant (the streamed kernels are
// instantiated per strategy, so no other strategy's code is on the row
// path); ST < 0: a.strategy at run time.
template <int DMAX, class Row, int ST = -1, bool XD = false>
__device__ __forceinline__ uint64_t prep_row(const PrepArgs& a, uint32_t i, const Row& R) {
    const int strategy = ST >= 0 ? ST : a.strategy;
    constexpr int U = Row::kUnroll;
    // XD: d == DMAX (every coordinate test below folds away at compile time)
    const int d = XD ? DMAX : (int)a.d;
    double sum = 0.0;
    uint32_t err = 0;
    uint64_t pid = 0;
    // float rows: one range test per coordinate (NaN fails it); the error
    // bits are worked out only for a row that fails (make_dataset,
    // core.cpp:32-41; cell_of, partition.cpp:26-29)
    auto f32_errors = [&](bool grid) {
        uint32_t e = 0;
#pragma unroll U
        for (int j = 0; j < DMAX; ++j) {
            if (j >= d) SKY_ROW_END;
            const float v = R.f(j);
            if (!(isfinite(v) && v >= 0.0f)) e |= kErrNonFinite;
            if (a.normalized && v > 1.0f) e |= kErrAboveOne;
            if (grid && !(v >= 0.0f && v <= 1.0f)) e |= kErrGridRange;
        }
        return e;
    };
    // the range test on raw bits: a float lies in [+0, upper] iff its bits
    // are <= upper's (negatives, -0.0 included, and NaN/inf have larger
    // bits); -0.0 fails it and is then accepted by f32_errors
    const float upper = a.normalized || strategy == SKY_GRID ? 1.0f : 3.402823466e38f;
    const uint32_t upper_bits = __float_as_uint(upper);
    if (strategy == SKY_GRID && Row::kF32) {
        // float rows: the comparisons give the same answers in FP32 as on the
        // exact upcast; cell = floor(x * m) from the product rounded toward
        // zero (floor(x*m) < m <= 2^22 is representable, so rz(x*m) lies in
        // [floor(x*m), x*m] and has the same floor)
        const uint32_t m32 = (uint32_t)a.m;
        const float mf = (float)a.m;
        uint32_t mx = 0, pid32 = 0;
#pragma unroll U
        for (int j = 0; j < DMAX; ++j) {
            if (j >= d) SKY_ROW_END;
            const float v = R.f(j);
            mx = max(mx, __float_as_uint(v));
            sum = __dadd_rn(sum, (double)v);
        }
        // pid = sum_j cell_j * m^j by Horner from the last coordinate (the
        // registers row is unrolled, so skipping j >= d keeps it exact)
#pragma unroll U
        for (int j = DMAX - 1; j >= 0; --j) {
            if (j >= d) continue;
            const uint32_t cell = min(__float2uint_rz(__fmul_rz(R.f(j), mf)), m32 - 1);
            pid32 = pid32 * m32 + cell;
        }
        if (mx > upper_bits) err = f32_errors(true);
        pid = pid32;
    } else if (strategy == SKY_GRID) {
        // m^d <= kMaxPartitions (2^22): 32-bit cell arithmetic
        uint32_t stride = 1, pid32 = 0;
        const uint32_t m32 = (uint32_t)a.m;
        const double md = (double)a.m;
#pragma unroll U
        for (int j = 0; j < DMAX; ++j) {
            if (j >= d) SKY_ROW_END;
            const double v = R.X(j);
            if (!(isfinite(v) && v >= 0.0)) err |= kErrNonFinite;
            if (a.normalized && v > 1.0) err |= kErrAboveOne;
            if (!(v >= 0.0 && v <= 1.0)) err |= kErrGridRange;
            sum = __dadd_rn(sum, v);
            uint32_t cell = __double2uint_rz(__dmul_rn(v, md));  // exact product, floor
            if (cell >= m32) cell = m32 - 1;
            pid32 += cell * stride;
            stride *= m32;
        }
        pid = pid32;
    } else if (strategy == SKY_ANGULAR) {
        uint32_t mx = 0;
#pragma unroll U
        for (int j = 0; j < DMAX; ++j) {
            if (j >= d) SKY_ROW_END;
            if (Row::kF32) {
                // float rows: the same answers as on the exact upcast
                const float v = R.f(j);
                mx = max(mx, __float_as_uint(v));
                sum = __dadd_rn(sum, (double)v);
            } else {
                const double v = R.X(j);
                if (!(isfinite(v) && v >= 0.0)) err |= kErrNonFinite;
                if (a.normalized && v > 1.0) err |= kErrAboveOne;
                sum = __dadd_rn(sum, v);
            }
        }
        if (Row::kF32 && mx > upper_bits) err = f32_errors(false);
        // hyperspherical_angles: tail sums of squares back to front; the
        // partition index sum_i slice_i * m^i (angular_index) by Horner's rule
        // over i = d-2 .. 0 (m^(d-1) <= 2^22: 32-bit arithmetic, no division)
        const double PI = 3.14159265358979323846;
        const uint32_t m32 = (uint32_t)a.m;
        // FP32 pass first: its slice value is within ~1e-6 relative of the
        // FP64 one, so a value clear of every interior boundary gives the
        // same floor; rows that come near one redo the FP64 computation.
        bool exact64 = false;
        {
            const float fm = (float)a.m, tol = 1e-4f * fmaxf(1.0f, fm / 16.0f);
            const float scale = 2.0f / 3.14159265f * fm;  // a filter value: exactness comes from the FP64 redo
            float tail32 = 0.0f;
            uint32_t pid32 = 0;
            // squares must stay normal floats for that error bound
#pragma unroll U
            for (int j = 0; j < DMAX; ++j) {
                if (j >= d) SKY_ROW_END;
                const float xj = R.f(j);
                if (xj != 0.0f && !(xj > 1e-15f && xj < 1e15f)) exact64 = true;
            }
#pragma unroll U
            for (int ii = DMAX - 1; ii >= 0; --ii) {
                if (ii > d - 1) continue;
                const float xi = R.f(ii);
                if (ii == d - 1) {
                    tail32 = xi * xi;
                    continue;
                }
                uint32_t slice;
                if (m32 <= 8 && a.tan2[0] != 0.0f) {
                    // phi_i = atan2(sqrt(tail), x_i) passes the boundary k*pi/(2m)
                    // iff tail >= x_i^2 tan^2(k*pi/(2m)) (x_i >= 0, tan^2 increasing
                    // on [0, pi/2)): no atan2 or sqrt. A row within 1e-3 (relative)
                    // of a boundary redoes FP64 below; rounding here is ~1e-6.
                    const float x2 = xi * xi;
                    slice = 0;
                    if (!(tail32 == 0.0f && !signbit(xi))) {  // atan2(+0, +0) = atan2(0, x > 0) = 0
#pragma unroll
                        for (uint32_t k = 1; k < 8; ++k) {  // static indices: no local copy of the args
                            if (k >= m32) break;
                            const float b = x2 * a.tan2[k - 1];
                            slice += tail32 >= b ? 1u : 0u;
                            if (fabsf(tail32 - b) <= 1e-3f * b) exact64 = true;
                        }
                    }
                    tail32 += x2;
                } else {
                    const float v = atan2f(sqrtf(tail32), xi) * scale;
                    tail32 += xi * xi;
                    const float r = rintf(v);
                    if (r >= 1.0f && r <= fm - 1.0f && fabsf(v - r) <= tol) exact64 = true;
                    slice = (uint32_t)fmaxf(v, 0.0f);
                    if (slice >= m32) slice = m32 - 1;
                }
                pid32 = pid32 * m32 + slice;
            }
            pid = pid32;
        }
        bool ambiguous = false;
        if (exact64) {
            uint32_t pid64 = 0;
            double tail = 0.0;
#pragma unroll U
            for (int ii = DMAX - 1; ii >= 0; --ii) {
                if (ii > d - 1) continue;
                const double xi = R.X(ii);
                if (ii == d - 1) {
                    tail = __dmul_rn(xi, xi);
                    continue;
                }
                uint32_t slice;
                if (a.ang_thr) {
                    bool amb = false;
                    slice = angular_slice_exact(__dsqrt_rn(tail), xi, a.ang_thr, m32, a.ang_c45, &amb);
                    ambiguous |= amb;
                } else {
                    // m > kAngularExactMaxM: CUDA's atan2 (within 2 ulp) and a
                    // band around each boundary resolved on the host libm
                    const double phi = atan2(sqrt(tail), xi);
                    const double v = __dmul_rn(__ddiv_rn(__dmul_rn(2.0, phi), PI), (double)a.m);
                    slice = (uint32_t)v;
                    if (slice >= m32) slice = m32 - 1;
                    const double r = rint(v);
                    if (r >= 1.0 && r <= (double)(a.m - 1) && fabs(v - r) <= 1e-9 * fmax(1.0, v)) ambiguous = true;
                }
                tail = __dadd_rn(tail, __dmul_rn(xi, xi));
                pid64 = pid64 * m32 + slice;
            }
            pid = pid64;
        }
        if (ambiguous) {
            const uint32_t k = atomicAdd(a.amb_count, 1u);
            if (k < a.amb_cap) a.amb_list[k] = i;
        }
    } else {
        float sv = 0.0f;
        uint32_t mx = 0;
#pragma unroll U
        for (int j = 0; j < DMAX; ++j) {
            if (j >= d) SKY_ROW_END;
            if (Row::kF32) {
                const float v = R.f(j);
                mx = max(mx, __float_as_uint(v));
                sum = __dadd_rn(sum, (double)v);
            } else {
                const double v = R.X(j);
                if (!(isfinite(v) && v >= 0.0)) err |= kErrNonFinite;
                if (a.normalized && v > 1.0) err |= kErrAboveOne;
                sum = __dadd_rn(sum, v);
            }
            if ((uint32_t)j == a.slice_dim) sv = R.f(j);
        }
        if (Row::kF32 && mx > upper_bits) err = f32_errors(false);
        if (strategy == SKY_RANDOM) pid = a.pid_in[i];
        if (strategy == SKY_SLICED) a.slice_key[i] = canon_bits(sv);
    }
    if (err) {
        atomicOr(a.err, err);
        pid = 0;  // the run fails at its next host check; keep every index in bounds
    }
    // monotone in sum; truncation keeps it monotone (and the partition sort
    // one radix pass shorter)
    const uint32_t skey = __float_as_uint(__double2float_rn(sum)) & ~((1u << a.key_shift) - 1u);
    const uint64_t key = (pid << 32) | skey;
    a.key64[i] = key;
    if (a.idx) a.idx[i] = i;
    return key;
}

__global__ void __launch_bounds__(256) k_prep(PrepArgs a) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < a.n)
        prep_row<32>(a, a.row_base + i,
                     MemRow{a.pts + (size_t)i * a.d, a.pts64 ? a.pts64 + (size_t)i * a.d : nullptr});
}

// Persistent prep over row tiles streamed by the bulk-copy engine; each row
// moves from the staged tile into registers with the widest shared load its
// stride allows. With a.gmin set, also the per-CTA minimum key of every
// partition (gmin[p * gridDim.x + blockIdx.x]; the stream path's representative bound).
template <int DP, int ST, bool XD>
__global__ void __launch_bounds__(kStreamThreads) k_prep_stream(PrepArgs a) {
    extern __shared__ __align__(16) char s_prep[];
    char* smem = s_prep;
    uint32_t* s_min = reinterpret_cast<uint32_t*>(smem + stream_smem_bytes(a.d));
    if (a.gmin) {
        for (uint32_t p = threadIdx.x; p < a.P; p += blockDim.x) s_min[p] = 0xFFFFFFFFu;
    }
    const uint32_t d = XD ? DP : a.d;  // XD: every row is exactly DP wide
    stream_row_tiles(a.pts, a.n, d, smem, [&](const float* tile, uint32_t r0, uint32_t nr, const uint64_t*) {
#pragma unroll 1
        for (uint32_t rr = threadIdx.x; rr < nr; rr += kStreamThreads) {
            const uint32_t i = a.row_base + r0 + rr;
            const float* x = tile + (size_t)rr * d;
            RegRow<DP> R;
            if ((d & 3) == 0) {
#pragma unroll
                for (int v = 0; v < (DP + 3) / 4; ++v) {
                    const float4 q = 4 * v < (int)d ? reinterpret_cast<const float4*>(x)[v]
                                                    : make_float4(0.f, 0.f, 0.f, 0.f);
                    if (4 * v < DP) R.v[4 * v] = q.x;
                    if (4 * v + 1 < DP) R.v[4 * v + 1] = q.y;
                    if (4 * v + 2 < DP) R.v[4 * v + 2] = q.z;
                    if (4 * v + 3 < DP) R.v[4 * v + 3] = q.w;
                }
            } else if ((d & 1) == 0) {
#pragma unroll
                for (int v = 0; v < (DP + 1) / 2; ++v) {
                    const float2 q = 2 * v < (int)d ? reinterpret_cast<const float2*>(x)[v] : make_float2(0.f, 0.f);
                    if (2 * v < DP) R.v[2 * v] = q.x;
                    if (2 * v + 1 < DP) R.v[2 * v + 1] = q.y;
                }
            } else {
#pragma unroll
                for (int j = 0; j < DP; ++j) R.v[j] = j < (int)d ? x[j] : 0.0f;
            }
            const uint64_t key = prep_row<DP, RegRow<DP>, ST, XD>(a, i, R);
            if (a.gmin) {
                // read first: after the first rows most keys are above the minimum
                const uint32_t p = (uint32_t)(key >> 32), k = (uint32_t)key;
                if (k < s_min[p]) atomicMin(s_min + p, k);
            }
        }
    });
    if (a.gmin) {
        __syncthreads();
        for (uint32_t p = threadIdx.x; p < a.P; p += blockDim.x) a.gmin[(size_t)p * gridDim.x + blockIdx.x] = s_min[p];
    }
}

// Persistent grid of the streamed prep: as many CTAs of the instantiation
// launched for (d, strategy) as fit on the SMs (the per-tile work is a
// dependent chain; resident warps hide it), at most one per tile.
// Deterministic for (n, d, P, strategy) on a device, so callers can size
// per-CTA outputs (gmin) with it.
template <int DT>
static const void* prep_stream_kernel(int strategy, bool xd) {
    if (strategy == SKY_GRID)
        return xd ? (const void*)k_prep_stream<DT, SKY_GRID, true> : (const void*)k_prep_stream<DT, SKY_GRID, false>;
    if (strategy == SKY_ANGULAR)
        return xd ? (const void*)k_prep_stream<DT, SKY_ANGULAR, true>
                  : (const void*)k_prep_stream<DT, SKY_ANGULAR, false>;
    return xd ? (const void*)k_prep_stream<DT, -1, true> : (const void*)k_prep_stream<DT, -1, false>;
}

// P: partitions whose per-CTA minima the pass keeps in shared memory (the
// stream path's a.gmin), 0 without them.
uint32_t prep_stream_grid(uint32_t n, uint32_t d, uint32_t P, int sm_count, int strategy) {
    const size_t smem = stream_smem_bytes(d) + (size_t)P * sizeof(uint32_t);
    int per_sm = 4;
    SKY_DISPATCH_D(padded_dim(d), {
        const void* k = prep_stream_kernel<DT>(strategy, padded_dim(d) == (int)d);
        ensure_smem_attr(k, smem);
        per_sm = occupancy_cached(k, (int)kStreamThreads, smem);
    });
    per_sm = std::max(1, std::min(per_sm, 8));
    return std::max<uint32_t>(1, std::min<uint32_t>(ceil_div(n, stream_tile_rows(d)), (uint32_t)per_sm * (uint32_t)sm_count));
}

void launch_prep(const PrepArgs& a, cudaStream_t st, int sm_count) {
    if (a.n == 0) return;
    if (!a.pts64 && a.d <= 32 && ((uintptr_t)a.pts & 15) == 0 && sm_count > 0) {
        // float rows, 16-byte aligned: persistent CTAs, bulk-copied row tiles
        const uint32_t pmin = a.gmin ? a.P : 0;  // minima slots only on the stream path
        const size_t smem = stream_smem_bytes(a.d) + (size_t)pmin * sizeof(uint32_t);
        const uint32_t grid = prep_stream_grid(a.n, a.d, pmin, sm_count, a.strategy);  // sets the smem attribute
        // grid and angular rows get their own instantiations (the row path
        // then holds only that strategy's code); random / sliced share one
        // and rows exactly as wide as the instantiation get one more (no
        // per-coordinate width tests)
        const bool xd = padded_dim(a.d) == (int)a.d;
#define SKY_PREP_LAUNCH(STRAT)                                              \
    SKY_DISPATCH_D(padded_dim(a.d), {                                       \
        if (xd)                                                             \
            k_prep_stream<DT, STRAT, true><<<grid, kStreamThreads, smem, st>>>(a);  \
        else                                                                \
            k_prep_stream<DT, STRAT, false><<<grid, kStreamThreads, smem, st>>>(a); \
    })
        if (a.strategy == SKY_GRID) {
            SKY_PREP_LAUNCH(SKY_GRID);
        } else if (a.strategy == SKY_ANGULAR) {
            SKY_PREP_LAUNCH(SKY_ANGULAR);
        } else {
            SKY_PREP_LAUNCH(-1);
        }
#undef SKY_PREP_LAUNCH
    } else {
        if (a.gmin) throw Error(SKY_E_INTERNAL, "partition minima need the streamed prep");
        k_prep<<<ceil_div(a.n, 256), 256, 0, st>>>(a);
    }
    SKY_LAUNCH_CHECK();
}



__global__ void k_seg_offsets(const uint64_t* __restrict__ key64, uint32_t n, uint32_t P, uint32_t* off) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t p = (uint32_t)(key64[i] >> 32);
    const int64_t prev = i ? (int64_t)(key64[i - 1] >> 32) : -1;
    for (int64_t q = prev + 1; q <= (int64_t)p; ++q) off[q] = i;
    if (i == n - 1)
        for (uint32_t q = p + 1; q <= P; ++q) off[q] = n;
}

// sorted survivor keys ((key64 >> key_shift) << row_bits | row) -> key64,
// row and the partition offsets off[P+1]
__global__ void k_unpack_survivors(const uint64_t* __restrict__ comp, uint32_t n, uint32_t row_bits,
                                   uint32_t key_shift, uint32_t P, uint64_t* __restrict__ key64,
                                   uint32_t* __restrict__ idx, uint32_t* __restrict__ off) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint64_t c = comp[i];
    const uint64_t k = (c >> row_bits) << key_shift;
    key64[i] = k;
    idx[i] = (uint32_t)(c & ((1ull << row_bits) - 1));
    const uint32_t p = (uint32_t)(k >> 32);
    const int64_t prev = i ? (int64_t)((comp[i - 1] >> row_bits) << key_shift >> 32) : -1;
    for (int64_t q = prev + 1; q <= (int64_t)p; ++q) off[q] = i;
    if (i == n - 1)
        for (uint32_t q = p + 1; q <= P; ++q) off[q] = n;
}

void launch_unpack_survivors(const uint64_t* comp, uint32_t n, uint32_t row_bits, uint32_t key_shift, uint32_t P,
                             uint64_t* key64, uint32_t* idx, uint32_t* off, cudaStream_t st) {
    if (n == 0) {
        SKY_CUDA(cudaMemsetAsync(off, 0, (P + 1) * sizeof(uint32_t), st));
        return;
    }
    k_unpack_survivors<<<ceil_div(n, 256), 256, 0, st>>>(comp, n, row_bits, key_shift, P, key64, idx, off);
    SKY_LAUNCH_CHECK();
}

void launch_seg_offsets(const uint64_t* key64, uint32_t n, uint32_t P, uint32_t* off, cudaStream_t st) {
    if (n == 0) {
        SKY_CUDA(cudaMemsetAsync(off, 0, (P + 1) * sizeof(uint32_t), st));
        return;
    }
    k_seg_offsets<<<ceil_div(n, 256), 256, 0, st>>>(key64, n, P, off);
    SKY_LAUNCH_CHECK();
}

__global__ void k_gather_rows_f64(const float* pts, const double* pts64, uint32_t d, const uint32_t* rows,
                                  uint32_t count, uint32_t row_base, double* out) {
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (uint64_t)count * d) return;
    const uint32_t k = (uint32_t)(t / d), j = (uint32_t)(t % d);
    const size_t r = (size_t)(rows[k] - row_base) * d + j;
    out[t] = pts64 ? pts64[r] : (double)pts[r];
}

void launch_gather_rows_f64(const float* pts, const double* pts64, uint32_t d, const uint32_t* rows,
                            uint32_t count, uint32_t row_base, double* out, cudaStream_t st) {
    if (!count) return;
    const uint64_t total = (uint64_t)count * d;
    k_gather_rows_f64<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(pts, pts64, d, rows, count, row_base, out);
    SKY_LAUNCH_CHECK();
}

__global__ void k_patch_pid(uint64_t* key64, const uint32_t* rows, const uint32_t* pids, uint32_t count) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const uint32_t r = rows[i];
    key64[r] = ((uint64_t)pids[i] << 32) | (key64[r] & 0xFFFFFFFFull);
}

void launch_patch_pid(uint64_t* key64, const uint32_t* rows, const uint32_t* pids, uint32_t count,
                      cudaStream_t st) {
    if (!count) return;
    k_patch_pid<<<ceil_div(count, 256), 256, 0, st>>>(key64, rows, pids, count);
    SKY_LAUNCH_CHECK();
}

// ---------------------------------------------------------------- sliced
// rank -> partition (partition.cpp:212-216)
__device__ __forceinline__ uint32_t slice_of_rank(uint64_t rank, uint64_t n, uint64_t p) {
    uint64_t index = n > 1 ? rank * p / (n - 1) : 0;
    return (uint32_t)(index >= p ? p - 1 : index);
}

// First rank belonging to slice b (b >= 1): smallest r with r*p/(n-1) >= b.
__device__ __forceinline__ uint64_t first_rank_of_slice(uint64_t b, uint64_t n, uint64_t p) {
    return (b * (n - 1) + p - 1) / p;
}

// For each slice boundary whose two sides share x[k], record the tie run
// [ra, rc) once (by the first boundary inside it).
__global__ void k_slice_runs(const uint32_t* __restrict__ key, uint32_t n, uint64_t p, uint32_t* runs,
                             uint32_t* run_count, uint32_t run_cap) {
    const uint64_t b = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x + 1;
    if (b >= p || n < 2) return;
    const uint64_t r = first_rank_of_slice(b, n, p);
    if (r == 0 || r >= n) return;
    if (key[r - 1] != key[r]) return;
    const uint32_t v = key[r];
    // run bounds by binary search
    uint64_t lo = 0, hi = r;  // first index with key == v
    while (lo < hi) {
        uint64_t mid = (lo + hi) / 2;
        if (key[mid] < v) lo = mid + 1; else hi = mid;
    }
    const uint64_t ra = lo;
    lo = r; hi = n;
    while (lo < hi) {
        uint64_t mid = (lo + hi) / 2;
        if (key[mid] <= v) lo = mid + 1; else hi = mid;
    }
    const uint64_t rc = lo;
    // owner: no earlier boundary inside [ra, rc)
    if (b > 1) {
        const uint64_t rp = first_rank_of_slice(b - 1, n, p);
        if (rp > ra) return;
    }
    const uint32_t k = atomicAdd(run_count, 1u);
    if (k < run_cap) {
        runs[2 * k] = (uint32_t)ra;
        runs[2 * k + 1] = (uint32_t)rc;
    }
}

void launch_slice_runs(const uint32_t* sorted_key, uint32_t n, uint64_t p, uint32_t* runs, uint32_t* run_count,
                       uint32_t run_cap, cudaStream_t st) {
    if (p < 2 || n < 2) return;
    k_slice_runs<<<ceil_div(p - 1, 256), 256, 0, st>>>(sorted_key, n, p, runs, run_count, run_cap);
    SKY_LAUNCH_CHECK();
}

__global__ void k_slice_assign(const uint32_t* __restrict__ rank_idx, uint32_t n, uint64_t p, uint64_t* key64) {
    const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const uint32_t row = rank_idx[r];
    key64[row] = ((uint64_t)slice_of_rank(r, n, p) << 32) | (key64[row] & 0xFFFFFFFFull);
}

void launch_slice_assign(const uint32_t* rank_idx, uint32_t n, uint64_t p, uint64_t* key64, cudaStream_t st) {
    if (!n) return;
    k_slice_assign<<<ceil_div(n, 256), 256, 0, st>>>(rank_idx, n, p, key64);
    SKY_LAUNCH_CHECK();
}

// coords_then_id_less (core.cpp:10-17) on float rows (exact: float order ==
// double order of the upcast values).
template <class T>
__device__ __forceinline__ bool lex_less(const T* pts, uint32_t d, uint32_t a, uint32_t b) {
    const T* pa = pts + (size_t)a * d;
    const T* pb = pts + (size_t)b * d;
    for (uint32_t j = 0; j < d; ++j) {
        const T x = pa[j], y = pb[j];
        if (x < y) return true;
        if (x > y) return false;
    }
    return a < b;
}

// Exact rank of each member inside its straddling tie run, then its slice.
__global__ void k_slice_fix_runs(const float* __restrict__ pts, uint32_t d, const uint32_t* __restrict__ rank_idx,
                                 uint32_t n, uint64_t p, const uint32_t* __restrict__ runs, uint64_t* key64) {
    const uint32_t ra = runs[2 * blockIdx.y], rc = runs[2 * blockIdx.y + 1];
    const uint32_t e = ra + blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= rc) return;
    const uint32_t row = rank_idx[e];
    uint32_t rank = 0;
    for (uint32_t f = ra; f < rc; ++f)
        if (f != e && lex_less(pts, d, rank_idx[f], row)) ++rank;
    key64[row] = ((uint64_t)slice_of_rank(ra + rank, n, p) << 32) | (key64[row] & 0xFFFFFFFFull);
}

void launch_slice_fix_runs(const float* pts, uint32_t d, const uint32_t* rank_idx, uint32_t n, uint64_t p,
                           const uint32_t* runs, uint32_t n_runs, uint32_t max_len, uint64_t* key64,
                           cudaStream_t st) {
    if (!n_runs) return;
    dim3 grid(ceil_div(max_len, 256), n_runs);
    k_slice_fix_runs<<<grid, 256, 0, st>>>(pts, d, rank_idx, n, p, runs, key64);
    SKY_LAUNCH_CHECK();
}

__global__ void k_gather_coord_key(const float* __restrict__ pts, uint32_t d, uint32_t j,
                                   const uint32_t* __restrict__ idx, uint32_t n, uint32_t* key) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    key[i] = canon_bits(pts[(size_t)idx[i] * d + j]);
}

void launch_gather_coord_key(const float* pts, uint32_t d, uint32_t j, const uint32_t* idx, uint32_t n,
                             uint32_t* key, cudaStream_t st) {
    if (!n) return;
    k_gather_coord_key<<<ceil_div(n, 256), 256, 0, st>>>(pts, d, j, idx, n, key);
    SKY_LAUNCH_CHECK();
}

// canonical FP64 bits: monotone for values >= 0 (-0.0 folded into +0.0)
__global__ void k_gather_coord_key64(const double* __restrict__ pts, uint32_t d, uint32_t j,
                                     const uint32_t* __restrict__ idx, uint32_t n, uint64_t* key) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double v = pts[(size_t)idx[i] * d + j];
    key[i] = v == 0.0 ? 0ull : (uint64_t)__double_as_longlong(v);
}

void launch_gather_coord_key64(const double* pts, uint32_t d, uint32_t j, const uint32_t* idx, uint32_t n,
                               uint64_t* key, cudaStream_t st) {
    if (!n) return;
    k_gather_coord_key64<<<ceil_div(n, 256), 256, 0, st>>>(pts, d, j, idx, n, key);
    SKY_LAUNCH_CHECK();
}

__global__ void k_round_rows(const double* __restrict__ in, size_t count, float* __restrict__ out) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < count) out[i] = __double2float_rn(in[i]);
}

void launch_round_rows(const double* in, size_t count, float* out, cudaStream_t st) {
    if (!count) return;
    k_round_rows<<<(unsigned)((count + 255) / 256), 256, 0, st>>>(in, count, out);
    SKY_LAUNCH_CHECK();
}

// ------------------------------------------------------- representatives
template <class T>
__device__ double row_sum(const T* pts, uint32_t d, uint32_t r) {
    const T* x = pts + (size_t)r * d;
    double s = 0.0;
    for (uint32_t j = 0; j < d; ++j) s = __dadd_rn(s, (double)x[j]);
    return s;
}

// (coord_sum, coords_then_id_less) total order of filter.cpp:74-79.
template <class T>
__device__ bool rep_less(const T* pts, uint32_t d, uint32_t a, uint32_t b) {
    const double sa = row_sum(pts, d, a), sb = row_sum(pts, d, b);
    if (sa != sb) return sa < sb;
    return lex_less(pts, d, a, b);
}

// One CTA per partition. Rows are sorted by (pid, skey, row); skey ties can
// hide (sum, lex, id) order, so the tie run that straddles position q-1 is
// resolved exactly by repeated block-wide argmin.
template <class T>
__global__ void k_rep_pick(const uint64_t* __restrict__ key64, const uint32_t* __restrict__ idx,
                           const uint32_t* __restrict__ off, const uint32_t* __restrict__ off_end,
                           const T* __restrict__ pts, uint32_t d, uint32_t q, uint32_t* cand) {
    const uint32_t p = blockIdx.x;
    const uint32_t a = off[p], b = off_end ? off_end[p] : off[p + 1];
    uint32_t* out = cand + (size_t)p * q;
    const uint32_t size = b - a;
    const uint32_t take = size < q ? size : q;
    for (uint32_t k = threadIdx.x; k < q; k += blockDim.x) out[k] = kNone;
    if (take == 0) return;
    const uint32_t v = (uint32_t)key64[a + take - 1];
    // run [ra, rb) of skey == v inside the partition
    __shared__ uint32_t s_ra, s_rb;
    if (threadIdx.x == 0) {
        uint32_t lo = a, hi = a + take - 1;
        while (lo < hi) {
            uint32_t mid = (lo + hi) / 2;
            if ((uint32_t)key64[mid] < v) lo = mid + 1; else hi = mid;
        }
        s_ra = lo;
        lo = a + take - 1; hi = b;
        while (lo < hi) {
            uint32_t mid = (lo + hi) / 2;
            if ((uint32_t)key64[mid] <= v) lo = mid + 1; else hi = mid;
        }
        s_rb = lo;
    }
    __syncthreads();
    const uint32_t ra = s_ra, rb = s_rb;
    for (uint32_t k = threadIdx.x; k < ra - a; k += blockDim.x) out[k] = idx[a + k];
    const uint32_t need = take - (ra - a);
    if (rb - ra == need) {
        for (uint32_t k = threadIdx.x; k < need; k += blockDim.x) out[ra - a + k] = idx[ra + k];
        return;
    }
    // select `need` smallest of the run under the exact order
    __shared__ uint32_t s_best[32];
    constexpr uint32_t RUN_SMEM = 1024;
    if (rb - ra <= RUN_SMEM) {
        // the run's FP64 sums once, into shared memory; then `need` rounds of
        // block argmin over (sum, lex coords, id) with lex only on equal sums
        __shared__ double s_sum[RUN_SMEM];
        __shared__ uint32_t s_rowr[RUN_SMEM];
        __shared__ uint8_t s_taken[RUN_SMEM];
        const uint32_t L = rb - ra;
        for (uint32_t e = threadIdx.x; e < L; e += blockDim.x) {
            const uint32_t row = idx[ra + e];
            s_rowr[e] = row;
            s_sum[e] = row_sum(pts, d, row);
            s_taken[e] = 0;
        }
        __syncthreads();
        auto less = [&](uint32_t x, uint32_t y) {  // run slots
            if (s_sum[x] != s_sum[y]) return s_sum[x] < s_sum[y];
            return lex_less(pts, d, s_rowr[x], s_rowr[y]);
        };
        for (uint32_t r = 0; r < need; ++r) {
            uint32_t best = kNone;
            for (uint32_t e = threadIdx.x; e < L; e += blockDim.x)
                if (!s_taken[e] && (best == kNone || less(e, best))) best = e;
            for (int o = 16; o > 0; o >>= 1) {
                const uint32_t other = __shfl_down_sync(0xffffffffu, best, o);
                if (other != kNone && (best == kNone || less(other, best))) best = other;
            }
            if ((threadIdx.x & 31) == 0) s_best[threadIdx.x >> 5] = best;
            __syncthreads();
            if (threadIdx.x == 0) {
                uint32_t bb = kNone;
                for (uint32_t w = 0; w < blockDim.x / 32; ++w) {
                    const uint32_t o = s_best[w];
                    if (o != kNone && (bb == kNone || less(o, bb))) bb = o;
                }
                s_taken[bb] = 1;
                out[ra - a + r] = s_rowr[bb];
            }
            __syncthreads();
        }
        return;
    }
    uint32_t last = kNone;
    for (uint32_t r = 0; r < need; ++r) {
        uint32_t best = kNone;
        for (uint32_t e = ra + threadIdx.x; e < rb; e += blockDim.x) {
            const uint32_t row = idx[e];
            if (last != kNone && !rep_less(pts, d, last, row)) continue;  // already taken
            if (best == kNone || rep_less(pts, d, row, best)) best = row;
        }
        // warp reduce
        for (int o = 16; o > 0; o >>= 1) {
            uint32_t other = __shfl_down_sync(0xffffffffu, best, o);
            if (other != kNone && (best == kNone || rep_less(pts, d, other, best))) best = other;
        }
        if ((threadIdx.x & 31) == 0) s_best[threadIdx.x >> 5] = best;
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t bb = kNone;
            for (uint32_t w = 0; w < blockDim.x / 32; ++w) {
                const uint32_t o = s_best[w];
                if (o != kNone && (bb == kNone || rep_less(pts, d, o, bb))) bb = o;
            }
            s_best[0] = bb;
            out[ra - a + r] = bb;
        }
        __syncthreads();
        last = s_best[0];
        __syncthreads();
    }
}

// ------------------------------------ representative candidates (stream path)
// select_representatives_sorted (filter.cpp:66-86) without sorting every row:
// the q-th smallest key of a partition is at most the q-th smallest of its
// per-chunk minima (q chunks each hold a row at or below their minimum), so
// the rows with key <= that bound contain the first q rows of the sorted
// partition and the whole tie run at position q. Only they are sorted.
//
// thr[p] = q-th smallest of gmin[., p] (0xFFFFFFFF when fewer than q chunks
// hold rows of p: then every row of p is a candidate). A warp per partition.
__global__ void k_part_thresh(const uint32_t* __restrict__ gmin, uint32_t G, uint32_t P, uint32_t q,
                              uint32_t* __restrict__ thr, uint32_t* __restrict__ bucket_count) {
    const uint32_t p = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (p >= P) return;
    if (lane == 0) bucket_count[p] = 0;  // the candidate pass counts from zero (no memset between the launches)
    uint64_t last = 0;
    for (uint32_t r = 0; r < q; ++r) {
        uint64_t best = ~0ull;
        for (uint32_t c = lane; c < G; c += 32) {
            const uint64_t v = ((uint64_t)gmin[(size_t)p * G + c] << 32) | c;
            if ((r == 0 || v > last) && v < best) best = v;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const uint64_t y = __shfl_xor_sync(0xffffffffu, best, o);
            best = y < best ? y : best;
        }
        last = best;
        if (best == ~0ull) break;
    }
    if (lane == 0) thr[p] = (uint32_t)(last >> 32);
}

// rows with key <= thr[pid] into per-partition buckets of B slots
__global__ void k_cand_bucket(const uint64_t* __restrict__ key64, uint32_t n, const uint32_t* __restrict__ thr,
                              uint32_t B, uint32_t* __restrict__ cnt, uint64_t* __restrict__ bkey,
                              uint32_t* __restrict__ brow, uint32_t* overflow) {
    // four consecutive keys per thread (two 16-byte streaming loads in flight)
    const uint32_t i0 = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
    if (i0 >= n) return;
    uint64_t k[4];
    if (i0 + 4 <= n) {
        const ulonglong2 a = __ldcs(reinterpret_cast<const ulonglong2*>(key64 + i0));
        const ulonglong2 b = __ldcs(reinterpret_cast<const ulonglong2*>(key64 + i0) + 1);
        k[0] = a.x; k[1] = a.y; k[2] = b.x; k[3] = b.y;
    } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) k[j] = i0 + j < n ? __ldcs(key64 + i0 + j) : ~0ull;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        if (k[j] == ~0ull) continue;
        const uint32_t p = (uint32_t)(k[j] >> 32);
        if ((uint32_t)k[j] > __ldg(thr + p)) continue;
        const uint32_t s = atomicAdd(cnt + p, 1u);
        if (s < B) {
            bkey[(size_t)p * B + s] = k[j];
            brow[(size_t)p * B + s] = i0 + j;
        } else {
            atomicOr(overflow, 1u);
        }
    }
}

// Ascending bitonic sort of s[0, n2) (n2 a power of two) by the block.
__device__ __forceinline__ void block_bitonic_sort(uint64_t* s, uint32_t n2) {
    for (uint32_t k = 2; k <= n2; k <<= 1) {
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            for (uint32_t i = threadIdx.x; i < n2 / 2; i += blockDim.x) {
                // i-th compare-exchange pair of this pass
                const uint32_t lo = 2 * i - (i & (j - 1)), hi = lo + j;
                const bool up = (lo & k) == 0;
                const uint64_t x = s[lo], y = s[hi];
                if ((x > y) == up) {
                    s[lo] = y;
                    s[hi] = x;
                }
            }
            __syncthreads();
        }
    }
}

// One CTA per partition: its bucket sorted by (key, row), then the first q by
// the reference order (filter.cpp:74-79): rows below the q-th key as they
// are, the tie run at position q resolved by (FP64 sum, lex coords, id) in
// `need` rounds of block argmin (k_rep_pick's rule).
__global__ void __launch_bounds__(256) k_bucket_pick(const uint64_t* __restrict__ bkey,
                                                     const uint32_t* __restrict__ brow,
                                                     const uint32_t* __restrict__ cnt, uint32_t B,
                                                     const float* __restrict__ pts, uint32_t d, uint32_t q,
                                                     uint32_t* __restrict__ cand, uint32_t run_floats) {
    // dynamic shared memory: the tie run's coordinates (run_floats floats),
    // then B slots of (key << 32 | row), FP64 sums and taken flags (B = 1,024
    // normally; the retry after a bucket overflow runs with larger buckets)
    extern __shared__ float4 s_run4[];
    uint64_t* s_c = reinterpret_cast<uint64_t*>(reinterpret_cast<float*>(s_run4) + run_floats);
    double* s_sum = reinterpret_cast<double*>(s_c + B);
    uint8_t* s_taken = reinterpret_cast<uint8_t*>(s_sum + B);
    __shared__ uint32_t s_ra, s_rb, s_best[8];
    const uint32_t p = blockIdx.x;
    const uint32_t c = min(cnt[p], B);
    uint32_t* out = cand + (size_t)p * q;
    for (uint32_t k = threadIdx.x; k < q; k += blockDim.x) out[k] = kNone;
    if (c == 0) return;
    uint32_t n2 = 1;
    while (n2 < c) n2 <<= 1;
    const size_t base = (size_t)p * B;
    for (uint32_t i = threadIdx.x; i < n2; i += blockDim.x)
        s_c[i] = i < c ? ((uint64_t)(uint32_t)bkey[base + i] << 32) | brow[base + i] : ~0ull;
    if (threadIdx.x == 0) {
        s_ra = 0;
        s_rb = c;
    }
    __syncthreads();
    block_bitonic_sort(s_c, n2);
    const uint32_t take = min(c, q);
    const uint32_t v = (uint32_t)(s_c[take - 1] >> 32);
    // tie run [ra, rb) of key v
    for (uint32_t i = threadIdx.x; i < c; i += blockDim.x) {
        const uint32_t ki = (uint32_t)(s_c[i] >> 32);
        if (ki == v && i > 0 && (uint32_t)(s_c[i - 1] >> 32) != v) s_ra = i;
        if (ki > v && (uint32_t)(s_c[i - 1] >> 32) == v) s_rb = i;
    }
    __syncthreads();
    const uint32_t ra = s_ra, rb = s_rb;
    for (uint32_t k = threadIdx.x; k < ra; k += blockDim.x) out[k] = (uint32_t)s_c[k];
    const uint32_t need = take - ra, L = rb - ra;
    if (need == L) {
        for (uint32_t k = threadIdx.x; k < need; k += blockDim.x) out[ra + k] = (uint32_t)s_c[ra + k];
        return;
    }
    // the run's rows (coordinates, FP64 sums) in shared memory: a run of
    // duplicates compares every coordinate of every pair
    float* s_run = reinterpret_cast<float*>(s_run4);  // [L][d4] when in_smem (rows padded to float4s)
    const uint32_t d4 = (d + 3) & ~3u;
    const bool in_smem = (size_t)L * d4 <= run_floats;
    if (in_smem) {
        // every coordinate of the run by its own thread (independent loads),
        // then the sums from shared memory
        // 8 loads in flight per thread (the rows are scattered: each load is a miss)
        const uint32_t total = L * d4;
        for (uint32_t k0 = threadIdx.x; k0 < total; k0 += 8 * blockDim.x) {
            float v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const uint32_t k = k0 + u * blockDim.x;
                const uint32_t e = k / d4, j = k - e * d4;
                v[u] = (k < total && j < d) ? pts[(size_t)(uint32_t)s_c[ra + e] * d + j] : 0.0f;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const uint32_t k = k0 + u * blockDim.x;
                if (k < total) s_run[k] = v[u];
            }
        }
        __syncthreads();
        for (uint32_t e = threadIdx.x; e < L; e += blockDim.x) {
            double sum = 0.0;
            for (uint32_t j = 0; j < d; ++j) sum = __dadd_rn(sum, (double)s_run[(size_t)e * d4 + j]);
            s_sum[e] = sum;
            s_taken[e] = 0;
        }
    } else {
        for (uint32_t e = threadIdx.x; e < L; e += blockDim.x) {
            s_sum[e] = row_sum(pts, d, (uint32_t)s_c[ra + e]);
            s_taken[e] = 0;
        }
    }
    __syncthreads();
    // a run of identical rows (same FP64 sum and coordinates; e.g. duplicates
    // clipped to the corner) is ordered by id alone: the bucket is sorted by
    // (key, row), so the run's first `need` are the answer
    if (in_smem) {
        __shared__ int s_diff;
        if (threadIdx.x == 0) s_diff = 0;
        __syncthreads();
        bool diff = false;
        for (uint32_t e = threadIdx.x; e < L && !diff; e += blockDim.x) {
            diff = s_sum[e] != s_sum[0];
            for (uint32_t j = 0; j < d && !diff; ++j) diff = s_run[(size_t)e * d4 + j] != s_run[j];
        }
        if (diff) s_diff = 1;
        __syncthreads();
        if (!s_diff) {
            for (uint32_t k = threadIdx.x; k < need; k += blockDim.x) out[ra + k] = (uint32_t)s_c[ra + k];
            return;
        }
    }
    auto less = [&](uint32_t x, uint32_t y) {  // run slots: (sum, lex coords, id)
        if (s_sum[x] != s_sum[y]) return s_sum[x] < s_sum[y];
        if (!in_smem) return lex_less(pts, d, (uint32_t)s_c[ra + x], (uint32_t)s_c[ra + y]);
        // padding lanes are 0 in both rows: they never decide
        const float4* a = s_run4 + (size_t)x * (d4 / 4);
        const float4* b = s_run4 + (size_t)y * (d4 / 4);
        for (uint32_t v = 0; v < d4 / 4; ++v) {
            const float4 p = a[v], q = b[v];
            if (p.x != q.x) return p.x < q.x;
            if (p.y != q.y) return p.y < q.y;
            if (p.z != q.z) return p.z < q.z;
            if (p.w != q.w) return p.w < q.w;
        }
        return (uint32_t)s_c[ra + x] < (uint32_t)s_c[ra + y];
    };
    for (uint32_t r = 0; r < need; ++r) {
        uint32_t best = kNone;
        for (uint32_t e = threadIdx.x; e < L; e += blockDim.x)
            if (!s_taken[e] && (best == kNone || less(e, best))) best = e;
        for (int o = 16; o > 0; o >>= 1) {
            const uint32_t other = __shfl_down_sync(0xffffffffu, best, o);
            if (other != kNone && (best == kNone || less(other, best))) best = other;
        }
        if ((threadIdx.x & 31) == 0) s_best[threadIdx.x >> 5] = best;
        __syncthreads();
        if (threadIdx.x < 32) {
            // the 8 warp winners by a 3-step tree in warp 0
            uint32_t bb = threadIdx.x < 8 ? s_best[threadIdx.x] : kNone;
            for (int o = 4; o > 0; o >>= 1) {
                const uint32_t other = __shfl_down_sync(0xffffffffu, bb, o);
                if (other != kNone && (bb == kNone || less(other, bb))) bb = other;
            }
            if (threadIdx.x == 0) {
                s_taken[bb] = 1;
                out[ra + r] = (uint32_t)s_c[ra + bb];
            }
        }
        __syncthreads();
    }
}

void launch_rep_candidates(const uint64_t* key64, uint32_t n, uint32_t P, uint32_t q, uint32_t G,
                           const uint32_t* gmin, uint32_t* thr, uint32_t B, uint32_t* cnt, uint64_t* bkey,
                           uint32_t* brow, const float* pts, uint32_t d, uint32_t* cand, uint32_t* overflow,
                           cudaStream_t st, cudaEvent_t pass_begin, cudaEvent_t pass_end) {
    if (B > kRepBucketBig || (B & (B - 1))) throw Error(SKY_E_INTERNAL, "candidate buckets: a power of two up to 8192 rows");
    k_part_thresh<<<ceil_div((uint64_t)P * 32, 256), 256, 0, st>>>(gmin, G, P, q, thr, cnt);
    SKY_LAUNCH_CHECK();
    // the key pass alone is timed as an HBM pass (thresholds and picks are latency-bound)
    if (pass_begin) SKY_CUDA(cudaEventRecord(pass_begin, st));
    k_cand_bucket<<<ceil_div(ceil_div(n, 4), 256), 256, 0, st>>>(key64, n, thr, B, cnt, bkey, brow, overflow);
    SKY_LAUNCH_CHECK();
    if (pass_end) SKY_CUDA(cudaEventRecord(pass_end, st));
    // <= 64 KB of run coordinates (a multiple of 4 floats: the slots after them stay 16-byte aligned)
    const uint32_t run_floats = std::min<uint32_t>(B * d, 16u * 1024) & ~3u;
    const size_t smem = run_floats * sizeof(float) + (size_t)B * (sizeof(uint64_t) + sizeof(double) + 1) + 16;
    ensure_smem_attr((const void*)k_bucket_pick, smem);
    k_bucket_pick<<<P, 256, smem, st>>>(bkey, brow, cnt, B, pts, d, q, cand, run_floats);
    SKY_LAUNCH_CHECK();
}

void launch_rep_pick(const uint64_t* key64, const uint32_t* idx, const uint32_t* off, uint32_t P,
                     const float* pts, const double* pts64, uint32_t d, uint32_t q, uint32_t* cand, cudaStream_t st,
                     const uint32_t* off_end) {
    if (!P) return;
    if (pts64)
        k_rep_pick<double><<<P, 128, 0, st>>>(key64, idx, off, off_end, pts64, d, q, cand);
    else
        k_rep_pick<float><<<P, 128, 0, st>>>(key64, idx, off, off_end, pts, d, q, cand);
    SKY_LAUNCH_CHECK();
}

// ---------------------------------------- region / random representatives
// Partition of every row (row order) from the (pid << 32 | key) sorted keys.
__global__ void k_row_pid(const uint64_t* __restrict__ key64, const uint32_t* __restrict__ idx, uint32_t n,
                          uint32_t* __restrict__ pid_row) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) pid_row[idx[i]] = (uint32_t)(key64[i] >> 32);
}

// dominance_region_volume (core.cpp:112-123): prod_j (1 - x_j) in FP64, left
// to right, each step correctly rounded as on the host. Key = ~bits(volume)
// (volumes are >= +0, so the bit pattern is monotone): an ascending stable
// sort over rows in id order gives (volume desc, id asc) (filter.cpp:103-106).
template <class T>
__global__ void k_region_keys(const T* __restrict__ pts, uint32_t d, uint32_t n, uint64_t* __restrict__ key,
                              uint32_t* __restrict__ row) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const T* x = pts + (size_t)i * d;
    double v = 1.0;
    for (uint32_t j = 0; j < d; ++j) v = __dmul_rn(v, __dsub_rn(1.0, (double)x[j]));
    key[i] = ~(uint64_t)__double_as_longlong(v);
    row[i] = i;
}

__global__ void k_iota(uint32_t n, uint32_t* __restrict__ out) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = i;
}

__global__ void k_gather_u32(const uint32_t* __restrict__ src, const uint32_t* __restrict__ idx, uint32_t n,
                             uint32_t* __restrict__ out) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = src[idx[i]];
}

// cand[p*q + k] = rows[off[p] + k] for k < min(q, |partition p|), else kNone.
__global__ void k_pick_first(const uint32_t* __restrict__ rows, const uint32_t* __restrict__ off, uint32_t P,
                             uint32_t q, uint32_t* __restrict__ cand) {
    const uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= (uint64_t)P * q) return;
    const uint32_t p = (uint32_t)(s / q), k = (uint32_t)(s % q);
    const uint32_t b = off[p], e = off[p + 1];
    cand[s] = b + k < e ? rows[b + k] : kNone;
}

// cand[s] = rows[gpos[s]] (kNone passes through).
__global__ void k_pick_gather(const uint32_t* __restrict__ rows, const uint32_t* __restrict__ gpos, uint32_t slots,
                              uint32_t* __restrict__ cand) {
    const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s < slots) cand[s] = gpos[s] == kNone ? kNone : rows[gpos[s]];
}

void launch_row_pid(const uint64_t* key64, const uint32_t* idx, uint32_t n, uint32_t* pid_row, cudaStream_t st) {
    if (!n) return;
    k_row_pid<<<ceil_div(n, 256), 256, 0, st>>>(key64, idx, n, pid_row);
    SKY_LAUNCH_CHECK();
}
void launch_region_keys(const float* pts, const double* pts64, uint32_t d, uint32_t n, uint64_t* key, uint32_t* row,
                        cudaStream_t st) {
    if (!n) return;
    if (pts64)
        k_region_keys<double><<<ceil_div(n, 256), 256, 0, st>>>(pts64, d, n, key, row);
    else
        k_region_keys<float><<<ceil_div(n, 256), 256, 0, st>>>(pts, d, n, key, row);
    SKY_LAUNCH_CHECK();
}
void launch_iota(uint32_t n, uint32_t* out, cudaStream_t st) {
    if (!n) return;
    k_iota<<<ceil_div(n, 256), 256, 0, st>>>(n, out);
    SKY_LAUNCH_CHECK();
}
void launch_gather_u32(const uint32_t* src, const uint32_t* idx, uint32_t n, uint32_t* out, cudaStream_t st) {
    if (!n) return;
    k_gather_u32<<<ceil_div(n, 256), 256, 0, st>>>(src, idx, n, out);
    SKY_LAUNCH_CHECK();
}
void launch_pick_first(const uint32_t* rows, const uint32_t* off, uint32_t P, uint32_t q, uint32_t* cand,
                       cudaStream_t st) {
    const uint64_t slots = (uint64_t)P * q;
    if (!slots) return;
    k_pick_first<<<ceil_div(slots, 256), 256, 0, st>>>(rows, off, P, q, cand);
    SKY_LAUNCH_CHECK();
}
void launch_pick_gather(const uint32_t* rows, const uint32_t* gpos, uint32_t slots, uint32_t* cand, cudaStream_t st) {
    if (!slots) return;
    k_pick_gather<<<ceil_div(slots, 256), 256, 0, st>>>(rows, gpos, slots, cand);
    SKY_LAUNCH_CHECK();
}

// select_representatives_sorted + prune_dominated_reps (filter.cpp:15-33,
// 66-86, 139-145) finished in one CTA: compact the per-partition picks, sort
// them by sum key, keep the antichain (brute force, as the reference does),
// emit them key-sorted with their count in device memory.
constexpr int REPF_ITEMS = 2, REPF_MAX = 1024 * REPF_ITEMS;

template <int D, int THREADS>
__global__ void __launch_bounds__(THREADS) k_rep_finalize(const uint32_t* __restrict__ cand, uint32_t slots,
                                                          const float* __restrict__ pts, uint32_t d, DevSet out,
                                                          uint32_t* out_count, unsigned long long* tests, X64 x64) {
    constexpr int V = Dims<D>::V;
    constexpr int MAXN = THREADS * REPF_ITEMS;
    using Scan = cub::BlockScan<uint32_t, THREADS>;
    __shared__ typename Scan::TempStorage tmp;
    extern __shared__ float4 s_xyz[];  // [MAXN][V], then rows, keys, order, dead flags
    uint32_t* s_row = reinterpret_cast<uint32_t*>(s_xyz + (size_t)MAXN * V);
    uint32_t* s_key = s_row + MAXN;
    uint32_t* s_ord = s_key + MAXN;
    uint64_t* s_sort = reinterpret_cast<uint64_t*>(s_ord + MAXN);
    uint8_t* s_dead = reinterpret_cast<uint8_t*>(s_sort + MAXN);
    __shared__ uint32_t s_n;
    const int t = threadIdx.x;
    // 1. compact the picks (slot order = partition order)
    uint32_t flags[REPF_ITEMS], rows[REPF_ITEMS];
#pragma unroll
    for (int k = 0; k < REPF_ITEMS; ++k) {
        const uint32_t sl = t * REPF_ITEMS + k;
        rows[k] = sl < slots ? cand[sl] : kNone;
        flags[k] = rows[k] != kNone;
    }
    uint32_t offs[REPF_ITEMS], total;
    Scan(tmp).ExclusiveSum(flags, offs, total);
#pragma unroll
    for (int k = 0; k < REPF_ITEMS; ++k)
        if (flags[k]) s_row[offs[k]] = rows[k];
    if (t == 0) s_n = total;
    __syncthreads();
    const uint32_t n = s_n;
    // 2. coordinates and FP64-sum keys
    // every coordinate by its own thread (independent loads), then the
    // FP64 sums from shared memory (FP64 rows: from the doubles)
    {
        float* sx = reinterpret_cast<float*>(s_xyz);
        const uint32_t total = n * 4 * V;
        for (uint32_t k0 = t; k0 < total; k0 += 4 * THREADS) {
            float v[4];  // 4 loads in flight per thread
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint32_t k = k0 + u * THREADS;
                const uint32_t i = k / (4 * V), j = k - i * (4 * V);
                v[u] = (k < total && j < d) ? pts[(size_t)s_row[i] * d + j] : 0.0f;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint32_t k = k0 + u * THREADS;
                if (k < total) sx[k] = v[u];
            }
        }
    }
    __syncthreads();
    for (uint32_t i = t; i < n; i += THREADS) {
        double sum = 0.0;
        if (x64.x) {
            sum = row_sum(x64.x, d, s_row[i]);
        } else {
            const float* sx = reinterpret_cast<const float*>(s_xyz + (size_t)i * V);
            for (uint32_t j = 0; j < d; ++j) sum = __dadd_rn(sum, (double)sx[j]);
        }
        s_key[i] = __float_as_uint(__double2float_rn(sum));
    }
    __syncthreads();
    // 3. key order (stable: ties keep slot order): bitonic sort of
    //    (key << 32 | slot)
    constexpr int NW = THREADS / 32;
    const uint32_t lane = t & 31, wid = t >> 5;
    {
        uint32_t n2 = 1;
        while (n2 < n) n2 <<= 1;
        for (uint32_t i = t; i < n2; i += THREADS) s_sort[i] = i < n ? ((uint64_t)s_key[i] << 32) | i : ~0ull;
        __syncthreads();
        block_bitonic_sort(s_sort, n2);
        for (uint32_t i = t; i < n; i += THREADS) s_ord[i] = (uint32_t)s_sort[i];
    }
    __syncthreads();
    // 4. antichain: a candidate meets the candidates in key order up to its
    //    own key (a dominator's key is <= its own); a warp per candidate,
    //    lanes split the comparators, the warp stops at the first dominator
    unsigned long long nt = 0;
    for (uint32_t pi = wid; pi < n; pi += NW) {
        const uint32_t i = s_ord[pi];
        const uint32_t ki = s_key[i];
        const float4* ti = s_xyz + (size_t)i * V;
        bool dom = false;
        for (uint32_t b = 0; b < n; b += 32) {
            const uint32_t pj = b + lane;
            bool hit = false;
            const uint32_t j = pj < n ? s_ord[pj] : 0u;
            const bool in = pj < n && s_key[j] <= ki;
            if (in && j != i) {
                ++nt;
                const float4* sj = s_xyz + (size_t)j * V;
                bool gt = false, lt = false;
#pragma unroll
                for (int v = 0; v < V; ++v) {
                    const float4 a = sj[v], c = ti[v];
                    gt |= (a.x > c.x) | (a.y > c.y) | (a.z > c.z) | (a.w > c.w);
                    lt |= (a.x < c.x) | (a.y < c.y) | (a.z < c.z) | (a.w < c.w);
                }
                hit = !gt && (x64.x ? dom64(x64, s_row[j], s_row[i]) : lt);
            }
            if (__any_sync(0xffffffffu, hit)) {
                dom = true;
                break;
            }
            if (!__all_sync(0xffffffffu, in)) break;  // keys sorted: the rest are larger
        }
        if (lane == 0) s_dead[i] = dom;
    }
    __syncthreads();
    // 5. survivors in key order
    uint32_t keep[REPF_ITEMS], kpos[REPF_ITEMS], ktot;
#pragma unroll
    for (int k = 0; k < REPF_ITEMS; ++k) {
        const uint32_t p = t * REPF_ITEMS + k;
        keep[k] = p < n && !s_dead[s_ord[p]];
    }
    Scan(tmp).ExclusiveSum(keep, kpos, ktot);
#pragma unroll
    for (int k = 0; k < REPF_ITEMS; ++k) {
        if (!keep[k]) continue;
        const uint32_t i = s_ord[t * REPF_ITEMS + k], o = kpos[k];
        float4* dst = reinterpret_cast<float4*>(out.xyz) + (size_t)o * V;
#pragma unroll
        for (int v = 0; v < V; ++v) dst[v] = s_xyz[(size_t)i * V + v];
        out.skey[o] = s_key[i];
        out.id[o] = s_row[i];
    }
    if (t == 0) *out_count = ktot;
    if (tests) {
        nt = warp_sum_u64(nt);
        if ((t & 31) == 0 && nt) atomicAdd(tests, nt);
    }
}

template <int D, int THREADS>
void rep_finalize_launch(const uint32_t* cand, uint32_t slots, const float* pts, uint32_t d, DevSet out,
                         uint32_t* out_count, unsigned long long* tests, X64 x64, size_t smem, cudaStream_t st) {
    SKY_CUDA(cudaFuncSetAttribute(k_rep_finalize<D, THREADS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_rep_finalize<D, THREADS><<<1, THREADS, smem, st>>>(cand, slots, pts, d, out, out_count, tests, x64);
}

// The same finish spread over the GPU (three launches): per-slot coordinates
// and keys; a warp per slot for its key rank and whether any other pick
// dominates it (all picks in shared memory); one CTA places the survivors by
// rank. The single-CTA kernel above runs ~130k warp instructions on one SM
// for 1280 picks.
template <int D>
__global__ void __launch_bounds__(256) k_repf_load(const uint32_t* __restrict__ cand, uint32_t slots,
                                                   const float* __restrict__ pts, uint32_t d, X64 x64,
                                                   float4* __restrict__ cx, uint32_t* __restrict__ ckey) {
    constexpr int V = Dims<D>::V;
    const uint32_t sl = blockIdx.x * blockDim.x + threadIdx.x;
    if (sl >= slots) return;
    const uint32_t r = cand[sl];
    float c[4 * V];
    double sum = 0.0;
#pragma unroll
    for (int j = 0; j < 4 * V; ++j) c[j] = (r != kNone && (uint32_t)j < d) ? pts[(size_t)r * d + j] : 0.0f;
#pragma unroll
    for (int j = 0; j < 4 * V; ++j)
        if ((uint32_t)j < d) sum = __dadd_rn(sum, (double)c[j]);
    if (x64.x && r != kNone) sum = row_sum(x64.x, d, r);
#pragma unroll
    for (int v = 0; v < V; ++v) cx[(size_t)sl * V + v] = make_float4(c[4 * v], c[4 * v + 1], c[4 * v + 2], c[4 * v + 3]);
    // sums are finite and >= 0: 0xFFFFFFFF (a NaN pattern) marks an empty slot
    ckey[sl] = r == kNone ? 0xFFFFFFFFu : __float_as_uint(__double2float_rn(sum));
}

template <int D>
__global__ void __launch_bounds__(256) k_repf_dom(const float4* __restrict__ cx, const uint32_t* __restrict__ ckey,
                                                  const uint32_t* __restrict__ cand, uint32_t slots, X64 x64,
                                                  uint32_t* __restrict__ rank, uint8_t* __restrict__ dead,
                                                  unsigned long long* tests) {
    constexpr int V = Dims<D>::V;
    extern __shared__ float4 s_x[];  // [slots][V], then keys
    uint32_t* s_k = reinterpret_cast<uint32_t*>(s_x + (size_t)slots * V);
    for (uint32_t i = threadIdx.x; i < slots * V; i += blockDim.x) s_x[i] = cx[i];
    for (uint32_t i = threadIdx.x; i < slots; i += blockDim.x) s_k[i] = ckey[i];
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t warps = gridDim.x * (blockDim.x >> 5);
    unsigned long long nt = 0;
    for (uint32_t i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < slots; i += warps) {
        const uint32_t ki = s_k[i];
        if (ki == 0xFFFFFFFFu) continue;  // empty slot (warp-uniform)
        float4 t[V];
#pragma unroll
        for (int v = 0; v < V; ++v) t[v] = s_x[(size_t)i * V + v];
        uint32_t rk = 0;
        bool hit = false;
        for (uint32_t j = lane; j < slots; j += 32) {
            const uint32_t kj = s_k[j];
            rk += (kj < ki) | ((kj == ki) & (j < i));
            if (!hit && kj <= ki && j != i) {
                ++nt;
                bool gt = false, lt = false;
#pragma unroll
                for (int v = 0; v < V; ++v) {
                    const float4 a = s_x[(size_t)j * V + v], b = t[v];
                    gt |= (a.x > b.x) | (a.y > b.y) | (a.z > b.z) | (a.w > b.w);
                    lt |= (a.x < b.x) | (a.y < b.y) | (a.z < b.z) | (a.w < b.w);
                }
                hit = !gt && (x64.x ? dom64(x64, cand[j], cand[i]) : lt);
            }
        }
        rk = __reduce_add_sync(0xffffffffu, rk);
        const bool dom = __any_sync(0xffffffffu, hit);
        if (lane == 0) {
            rank[i] = rk;
            dead[i] = dom;
        }
    }
    if (tests) {
        nt = warp_sum_u64(nt);
        if (lane == 0 && nt) atomicAdd(tests, nt);
    }
}

template <int D>
__global__ void __launch_bounds__(1024) k_repf_emit(const float4* __restrict__ cx, const uint32_t* __restrict__ ckey,
                                                    const uint32_t* __restrict__ cand, uint32_t slots,
                                                    const uint32_t* __restrict__ rank, const uint8_t* __restrict__ dead,
                                                    DevSet out, uint32_t* out_count) {
    constexpr int V = Dims<D>::V;
    using Scan = cub::BlockScan<uint32_t, 1024>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ uint32_t s_at[REPF_MAX];  // slot at each rank, kNone if dominated / unused
    for (uint32_t i = threadIdx.x; i < REPF_MAX; i += blockDim.x) s_at[i] = kNone;
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < slots; i += blockDim.x)
        if (ckey[i] != 0xFFFFFFFFu && !dead[i]) s_at[rank[i]] = i;
    __syncthreads();
    uint32_t keep[REPF_ITEMS], pos[REPF_ITEMS], total;
#pragma unroll
    for (int k = 0; k < REPF_ITEMS; ++k) keep[k] = s_at[threadIdx.x * REPF_ITEMS + k] != kNone;
    Scan(tmp).ExclusiveSum(keep, pos, total);
#pragma unroll
    for (int k = 0; k < REPF_ITEMS; ++k) {
        if (!keep[k]) continue;
        const uint32_t i = s_at[threadIdx.x * REPF_ITEMS + k], o = pos[k];
#pragma unroll
        for (int v = 0; v < V; ++v) reinterpret_cast<float4*>(out.xyz)[(size_t)o * V + v] = cx[(size_t)i * V + v];
        out.skey[o] = ckey[i];
        out.id[o] = cand[i];
    }
    if (threadIdx.x == 0) *out_count = total;
}

bool launch_rep_finalize_par(int D, const uint32_t* cand, uint32_t slots, const float* pts, uint32_t d, DevSet out,
                             uint32_t* out_count, unsigned long long* tests, X64 x64, int smem_optin, int sm_count,
                             void* scratch, cudaStream_t st) {
    if (slots > (uint32_t)REPF_MAX || slots == 0) return false;
    const int V = (D + 3) / 4;
    const size_t smem = (size_t)slots * (V * 16 + 4) + 16;
    if (smem + 1024 > (size_t)smem_optin) return false;
    char* sc = static_cast<char*>(scratch);
    float4* cx = reinterpret_cast<float4*>(sc);
    uint32_t* ckey = reinterpret_cast<uint32_t*>(sc + (size_t)REPF_MAX * V * 16);
    uint32_t* rank = ckey + REPF_MAX;
    uint8_t* dead = reinterpret_cast<uint8_t*>(rank + REPF_MAX);
    // one warp per slot, as many CTAs as fit one wave
    const uint32_t dom_grid = std::max<uint32_t>(1, std::min<uint32_t>(ceil_div(slots, 8), (uint32_t)sm_count));
    SKY_DISPATCH_D(D, {
        k_repf_load<DT><<<ceil_div(slots, 256), 256, 0, st>>>(cand, slots, pts, d, x64, cx, ckey);
        SKY_LAUNCH_CHECK();
        if (smem > 48 * 1024)
            SKY_CUDA(cudaFuncSetAttribute(k_repf_dom<DT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k_repf_dom<DT><<<dom_grid, 256, smem, st>>>(cx, ckey, cand, slots, x64, rank, dead, tests);
        SKY_LAUNCH_CHECK();
        k_repf_emit<DT><<<1, 1024, 0, st>>>(cx, ckey, cand, slots, rank, dead, out, out_count);
        SKY_LAUNCH_CHECK();
    });
    return true;
}

size_t rep_finalize_scratch_bytes(int D) { return (size_t)REPF_MAX * (((D + 3) / 4) * 16 + 9) + 64; }

bool launch_rep_finalize(int D, const uint32_t* cand, uint32_t slots, const float* pts, uint32_t d, DevSet out,
                         uint32_t* out_count, unsigned long long* tests, X64 x64, int smem_optin, cudaStream_t st) {
    if (slots > (uint32_t)REPF_MAX) return false;
    const bool small = slots <= 512u * REPF_ITEMS;
    const size_t maxn = small ? 512u * REPF_ITEMS : (size_t)REPF_MAX;
    const size_t smem = maxn * ((D + 3) / 4) * 16 + maxn * 21 + 64;
    if (smem + 16 * 1024 > (size_t)smem_optin) return false;
    SKY_DISPATCH_D(D, {
        if (small)
            rep_finalize_launch<DT, 512>(cand, slots, pts, d, out, out_count, tests, x64, smem, st);
        else
            rep_finalize_launch<DT, 1024>(cand, slots, pts, d, out, out_count, tests, x64, smem, st);
    });
    SKY_LAUNCH_CHECK();
    return true;
}

// ------------------------------------------------------------ compaction
template <int D>
__global__ void k_scatter_direct(DevSet in, const uint8_t* __restrict__ dead, const uint32_t* __restrict__ pos,
                                 DevSet out) {
    constexpr int V = Dims<D>::V;
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= in.n || dead[i]) return;
    const uint32_t o = pos[i];
    const float4* src = reinterpret_cast<const float4*>(in.xyz) + (size_t)i * V;
    float4* dst = reinterpret_cast<float4*>(out.xyz) + (size_t)o * V;
#pragma unroll
    for (int v = 0; v < V; ++v) dst[v] = src[v];
    out.skey[o] = in.skey[i];
    out.id[o] = in.id[i];
    if (in.qc && out.qc) out.qc[o] = in.qc[i];
}

void launch_scatter_direct(int D, const DevSet& in, const uint8_t* dead, const uint32_t* pos, DevSet out,
                           cudaStream_t st) {
    if (!in.n) return;
    SKY_DISPATCH_D(D, (k_scatter_direct<DT><<<ceil_div(in.n, 256), 256, 0, st>>>(in, dead, pos, out)));
    SKY_LAUNCH_CHECK();
}

template <int D>
__global__ void k_scatter_indirect(const float* __restrict__ pts, uint32_t d, const uint32_t* __restrict__ idx,
                                   const uint64_t* __restrict__ key64, uint32_t n,
                                   const uint8_t* __restrict__ dead, const uint32_t* __restrict__ pos,
                                   DevSet out) {
    constexpr int D4 = Dims<D>::D4;
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || (dead && dead[i])) return;
    const uint32_t o = pos ? pos[i] : i;
    const uint32_t row = idx[i];
    const float* x = pts + (size_t)row * d;
    float* dst = out.xyz + (size_t)o * D4;
#pragma unroll
    for (int j = 0; j < D4; ++j) dst[j] = (uint32_t)j < d ? x[j] : 0.0f;
    out.skey[o] = (uint32_t)key64[i];
    out.id[o] = row;
}

void launch_scatter_indirect(int D, const float* pts, uint32_t d, const uint32_t* idx, const uint64_t* key64,
                             uint32_t n, const uint8_t* dead, const uint32_t* pos, DevSet out, cudaStream_t st) {
    if (!n) return;
    SKY_DISPATCH_D(D, (k_scatter_indirect<DT><<<ceil_div(n, 256), 256, 0, st>>>(pts, d, idx, key64, n, dead,
                                                                               pos, out)));
    SKY_LAUNCH_CHECK();
}

// Rows of the input -> DevSet (reps, small sets). skey recomputed when
// skey_src is null.
template <int D>
__global__ void k_gather_rows(const float* __restrict__ pts, const double* __restrict__ pts64, uint32_t d,
                              const uint32_t* __restrict__ rows, uint32_t n, DevSet out) {
    constexpr int D4 = Dims<D>::D4;
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t row = rows[i];
    const float* x = pts + (size_t)row * d;
    float* dst = out.xyz + (size_t)i * D4;
#pragma unroll
    for (int j = 0; j < D4; ++j) dst[j] = (uint32_t)j < d ? x[j] : 0.0f;
    const double s = pts64 ? row_sum(pts64, d, row) : row_sum(pts, d, row);  // same key as k_prep
    out.skey[i] = __float_as_uint(__double2float_rn(s));
    out.id[i] = row;
}

void launch_gather_rows(int D, const float* pts, const double* pts64, uint32_t d, const uint32_t* rows, uint32_t n,
                        DevSet out, cudaStream_t st) {
    if (!n) return;
    SKY_DISPATCH_D(D, (k_gather_rows<DT><<<ceil_div(n, 256), 256, 0, st>>>(pts, pts64, d, rows, n, out)));
    SKY_LAUNCH_CHECK();
}

template <int D>
__global__ void k_gather_set(DevSet in, const uint32_t* __restrict__ perm, uint32_t n, DevSet out,
                             const uint32_t* n_dev) {
    constexpr int V = Dims<D>::V;
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (n_dev ? min(*n_dev, n) : n)) return;
    const uint32_t s = perm[i];
    const float4* src = reinterpret_cast<const float4*>(in.xyz) + (size_t)s * V;
    float4* dst = reinterpret_cast<float4*>(out.xyz) + (size_t)i * V;
#pragma unroll
    for (int v = 0; v < V; ++v) dst[v] = src[v];
    out.skey[i] = in.skey[s];
    out.id[i] = in.id[s];
    if (in.qc && out.qc) out.qc[i] = in.qc[s];
}

void launch_gather_set(int D, const DevSet& in, const uint32_t* perm, DevSet out, cudaStream_t st,
                       const uint32_t* n_dev) {
    if (!in.n) return;
    SKY_DISPATCH_D(D, (k_gather_set<DT><<<ceil_div(in.n, 256), 256, 0, st>>>(in, perm, in.n, out, n_dev)));
    SKY_LAUNCH_CHECK();
}

// Stable P-way merge of key-sorted runs (run p = positions off[p]..off[p+1]
// of `in`) into `out` in global key order: the same permutation as a stable
// radix sort of the concatenation. One warp per element: lanes binary-search
// the other runs (runs before p count keys <= k, runs after p keys < k, so
// equal keys keep run order), the warp sums the ranks and copies the row.
template <int D>
__global__ void __launch_bounds__(256) k_merge_runs(DevSet in, const uint32_t* __restrict__ off, uint32_t P,
                                                    uint32_t n, DevSet out, const uint32_t* n_dev) {
    constexpr int V = Dims<D>::V;
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t limit = n_dev ? min(*n_dev, n) : n;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    // persistent warps over the live count (the grid is sized for residency,
    // not for the capacity)
    for (uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < limit; i += nwarps) {
    // run of element i: the last p with off[p] <= i
    uint32_t lo = 0, hi = P;  // off[lo] <= i < off[hi]
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (__ldg(off + mid) <= i) lo = mid; else hi = mid;
    }
    const uint32_t p = lo;
    const uint32_t k = __ldg(in.skey + i);
    uint32_t rank = lane == 0 ? i - __ldg(off + p) : 0u;
    for (uint32_t q = lane; q < P; q += 32) {
        if (q == p) continue;
        uint32_t a = __ldg(off + q), b = __ldg(off + q + 1);
        const uint32_t base = a;
        if (q < p) {
            while (a < b) {  // first key > k
                const uint32_t m = (a + b) >> 1;
                if (__ldg(in.skey + m) <= k) a = m + 1; else b = m;
            }
        } else {
            while (a < b) {  // first key >= k
                const uint32_t m = (a + b) >> 1;
                if (__ldg(in.skey + m) < k) a = m + 1; else b = m;
            }
        }
        rank += a - base;
    }
    rank = __reduce_add_sync(0xffffffffu, rank);
    if (lane < (uint32_t)V)
        reinterpret_cast<float4*>(out.xyz)[(size_t)rank * V + lane] =
            reinterpret_cast<const float4*>(in.xyz)[(size_t)i * V + lane];
    if (lane == 31) {
        out.skey[rank] = k;
        out.id[rank] = in.id[i];
        if (in.qc && out.qc) out.qc[rank] = in.qc[i];
    }
    }
}

void launch_merge_runs(int D, const DevSet& in, const uint32_t* off, uint32_t P, DevSet out, cudaStream_t st,
                       const uint32_t* n_dev) {
    if (!in.n) return;
    const uint32_t grid = std::min<uint32_t>(ceil_div((uint64_t)in.n * 32, 256), (uint32_t)device_sm_count() * 8);
    SKY_DISPATCH_D(D, (k_merge_runs<DT><<<grid, 256, 0, st>>>(in, off, P, in.n, out, n_dev)));
    SKY_LAUNCH_CHECK();
}

// Ascending ids of the live candidates without a sort: a bitmap over the row
// ids (bit per input row), per-block popcounts, then each block emits its
// ids at the prefix of the blocks before it. kBmWords words per block.
constexpr uint32_t kBmWords = 2048;

__global__ void k_bm_set(const uint32_t* __restrict__ id, const uint8_t* __restrict__ dead, uint32_t n,
                         uint32_t* __restrict__ bm, const uint32_t* n_dev) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (n_dev) n = min(n, *n_dev);
    if (i >= n || dead[i]) return;
    const uint32_t v = id[i];
    atomicOr(bm + (v >> 5), 1u << (v & 31));
}

__global__ void __launch_bounds__(256) k_bm_count(const uint32_t* __restrict__ bm, uint32_t words,
                                                  uint32_t* __restrict__ block_tot) {
    const uint32_t b0 = blockIdx.x * kBmWords;
    uint32_t c = 0;
    for (uint32_t w = b0 + threadIdx.x; w < min(words, b0 + kBmWords); w += blockDim.x) c += __popc(bm[w]);
    c = __reduce_add_sync(0xffffffffu, c);
    __shared__ uint32_t s[8];
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0;
        for (int k = 0; k < 8; ++k) t += s[k];
        block_tot[blockIdx.x] = t;
    }
}

// 256 threads x 8 consecutive words per step; `total` (if set) gets the count
__global__ void __launch_bounds__(256) k_bm_emit(const uint32_t* __restrict__ bm, uint32_t words,
                                                 const uint32_t* __restrict__ block_tot, uint32_t* __restrict__ out,
                                                 uint32_t* total) {
    __shared__ uint32_t s[8];
    __shared__ uint32_t s_base;
    const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    // prefix of the blocks before this one
    uint32_t pre = 0;
    for (uint32_t b = threadIdx.x; b < blockIdx.x; b += blockDim.x) pre += block_tot[b];
    pre = __reduce_add_sync(0xffffffffu, pre);
    if (lane == 0) s[wid] = pre;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0;
        for (int k = 0; k < 8; ++k) t += s[k];
        s_base = t;
        if (total && blockIdx.x == gridDim.x - 1) *total = t + block_tot[blockIdx.x];
    }
    __syncthreads();
    // a block's ids are staged in shared memory and written out coalesced
    // when they fit (the output may be mapped host memory: full-line writes)
    constexpr uint32_t kStage = 4096;
    __shared__ uint32_t s_out[kStage];
    const bool staged = block_tot[blockIdx.x] <= kStage;
    const uint32_t gbase = s_base;
    uint32_t base = staged ? 0u : gbase;
    uint32_t* dst = staged ? s_out : out;
    const uint32_t b0 = blockIdx.x * kBmWords, b1 = min(words, b0 + kBmWords);
    for (uint32_t w0 = b0; w0 < b1; w0 += 256 * 8) {
        uint32_t v[8];
        uint32_t c = 0;
        const uint32_t wb = w0 + threadIdx.x * 8;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            v[k] = wb + k < b1 ? bm[wb + k] : 0u;
            c += __popc(v[k]);
        }
        // block exclusive scan of c
        uint32_t x = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= (uint32_t)o) x += y;
        }
        __syncthreads();
        if (lane == 31) s[wid] = x;
        __syncthreads();
        uint32_t wpre = 0, all = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            wpre += (uint32_t)k < wid ? s[k] : 0u;
            all += s[k];
        }
        uint32_t o = base + wpre + x - c;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            uint32_t m = v[k];
            while (m) {
                const uint32_t bit = __ffs(m) - 1;
                m &= m - 1;
                dst[o++] = ((wb + k) << 5) | bit;
            }
        }
        base += all;
    }
    if (staged) {
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < base; i += blockDim.x) out[gbase + i] = s_out[i];
    }
}

uint32_t bm_blocks(uint32_t n_ids) { return ceil_div(ceil_div(std::max<uint32_t>(n_ids, 1), 32), kBmWords); }

void launch_ids_bitmap(const uint32_t* id, const uint8_t* dead, uint32_t n, uint32_t n_ids, uint32_t* bm,
                       uint32_t* block_tot, uint32_t* out, uint32_t* total, cudaStream_t st, const uint32_t* n_dev) {
    const uint32_t words = ceil_div(std::max<uint32_t>(n_ids, 1), 32);
    SKY_CUDA(cudaMemsetAsync(bm, 0, (size_t)words * sizeof(uint32_t), st));
    if (n) {
        k_bm_set<<<ceil_div(n, 256), 256, 0, st>>>(id, dead, n, bm, n_dev);
        SKY_LAUNCH_CHECK();
    }
    const uint32_t blocks = bm_blocks(n_ids);
    k_bm_count<<<blocks, 256, 0, st>>>(bm, words, block_tot);
    SKY_LAUNCH_CHECK();
    k_bm_emit<<<blocks, 256, 0, st>>>(bm, words, block_tot, out, total);
    SKY_LAUNCH_CHECK();
}

__global__ void k_remap_offsets(const uint32_t* __restrict__ off_old, uint32_t P, const uint32_t* __restrict__ pos,
                                const uint8_t* __restrict__ dead, uint32_t n, uint32_t* off_new) {
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p > P) return;
    const uint32_t o = off_old[p];
    off_new[p] = o < n ? pos[o] : (n ? pos[n - 1] + (dead[n - 1] ? 0u : 1u) : 0u);
}

void launch_remap_offsets(const uint32_t* off_old, uint32_t P, const uint32_t* pos, const uint8_t* dead,
                          uint32_t n, uint32_t* off_new, cudaStream_t st) {
    k_remap_offsets<<<ceil_div(P + 1, 256), 256, 0, st>>>(off_old, P, pos, dead, n, off_new);
    SKY_LAUNCH_CHECK();
}

__global__ void k_count_total(const uint32_t* pos, const uint8_t* dead, uint32_t n, uint32_t* total) {
    *total = n ? pos[n - 1] + (dead[n - 1] ? 0u : 1u) : 0u;
}

void launch_count_total(const uint32_t* pos, const uint8_t* dead, uint32_t n, uint32_t* total, cudaStream_t st) {
    k_count_total<<<1, 1, 0, st>>>(pos, dead, n, total);
    SKY_LAUNCH_CHECK();
}

__global__ void k_compact_ids(const uint32_t* __restrict__ id, const uint8_t* __restrict__ dead,
                              const uint32_t* __restrict__ pos, uint32_t n, uint32_t* out) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || dead[i]) return;
    out[pos[i]] = id[i];
}

void launch_compact_ids(const uint32_t* id, const uint8_t* dead, const uint32_t* pos, uint32_t n, uint32_t* out,
                        cudaStream_t st) {
    if (!n) return;
    k_compact_ids<<<ceil_div(n, 256), 256, 0, st>>>(id, dead, pos, n, out);
    SKY_LAUNCH_CHECK();
}

__global__ void k_compact_pos(const uint8_t* __restrict__ dead, const uint32_t* __restrict__ pos, uint32_t n,
                              uint32_t base, uint32_t* out) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || dead[i]) return;
    out[pos[i]] = base + i;
}

void launch_compact_pos(const uint8_t* dead, const uint32_t* pos, uint32_t n, uint32_t base, uint32_t* out,
                        cudaStream_t st) {
    if (!n) return;
    k_compact_pos<<<ceil_div(n, 256), 256, 0, st>>>(dead, pos, n, base, out);
    SKY_LAUNCH_CHECK();
}

void launch_fill_u8(uint8_t* p, uint8_t v, size_t n, cudaStream_t st) {
    if (n) SKY_CUDA(cudaMemsetAsync(p, v, n, st));
}

__global__ void k_fill_tail_u8(uint8_t* __restrict__ p, uint8_t v, const uint32_t* __restrict__ count, uint32_t cap) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < cap && i >= *count) p[i] = v;
}

// dead flags of a capacity-sized set: 0 below the device count, 1 from it on
// (four flags per thread; p 4-byte aligned)
__global__ void k_fill_live_u8(uint8_t* __restrict__ p, const uint32_t* __restrict__ count, uint32_t cap) {
    const uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
    if (i >= cap) return;
    const uint32_t c = *count;
    if (i + 4 <= cap) {
        uint32_t w = 0;
#pragma unroll
        for (uint32_t k = 0; k < 4; ++k) w |= (i + k >= c ? 1u : 0u) << (8 * k);
        *reinterpret_cast<uint32_t*>(p + i) = w;
    } else {
        for (uint32_t k = i; k < cap; ++k) p[k] = k >= c ? 1 : 0;
    }
}

void launch_fill_live_u8(uint8_t* p, const uint32_t* count, uint32_t cap, cudaStream_t st) {
    if (!cap) return;
    k_fill_live_u8<<<ceil_div(ceil_div(cap, 4), 256), 256, 0, st>>>(p, count, cap);
    SKY_LAUNCH_CHECK();
}

void launch_fill_tail_u8(uint8_t* p, uint8_t v, const uint32_t* count, uint32_t cap, cudaStream_t st) {
    if (!cap) return;
    k_fill_tail_u8<<<ceil_div(cap, 256), 256, 0, st>>>(p, v, count, cap);
    SKY_LAUNCH_CHECK();
}

__global__ void k_mark_cells_dead(const uint64_t* __restrict__ key64, uint32_t n, const uint8_t* __restrict__ cell_dead,
                                  uint8_t* dead) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    dead[i] = cell_dead[(uint32_t)(key64[i] >> 32)];
}

// grid_filter (filter.cpp:37-50, engine.cpp:150-163) on the device. A
// non-empty cell a is filtered iff some non-empty cell b has b_j < a_j on
// every axis, i.e. iff a_j >= 1 everywhere and occ(a - (1,..,1)) holds, where
// occ(c) = "a non-empty cell b <= c exists" is the d-dimensional prefix OR of
// the occupancy: one running OR along each axis in turn, O(P d) instead of
// the reference's O(nonempty^2) pair loop. Cells are mixed radix m, axis 0
// the lowest digit (grid_index, partition.cpp:66-75).
__device__ __forceinline__ void grid_prefix_axis(uint8_t* e, uint32_t P, uint32_t m, uint32_t stride, uint32_t t,
                                                 uint32_t nthreads) {
    const uint32_t lines = P / m;
    for (uint32_t l = t; l < lines; l += nthreads) {
        const uint32_t base = (l / stride) * stride * m + (l % stride);
        uint8_t acc = 0;
        for (uint32_t k = 0; k < m; ++k) {
            acc |= e[base + k * stride];
            e[base + k * stride] = acc;
        }
    }
}
__device__ __forceinline__ unsigned long long grid_dead_cells(const uint32_t* off, const uint8_t* e, uint32_t P,
                                                              uint32_t m, uint32_t d, uint32_t diag, uint8_t* cell_dead,
                                                              uint32_t t, uint32_t nthreads) {
    unsigned long long rows = 0;
    for (uint32_t c = t; c < P; c += nthreads) {
        const uint32_t sz = off[c + 1] - off[c];
        bool inner = sz > 0;  // every digit >= 1
        uint32_t x = c;
        for (uint32_t j = 0; j < d && inner; ++j) {
            inner = x % m != 0;
            x /= m;
        }
        const bool dead = inner && e[c - diag];
        cell_dead[c] = dead ? 1 : 0;
        if (dead) rows += sz;
    }
    return rows;
}
// one CTA does every step (P <= kGridCtaCells): occupancy, d axis passes, dead cells
__global__ void __launch_bounds__(1024) k_grid_filter_cta(const uint32_t* __restrict__ off, uint32_t P, uint32_t m,
                                                          uint32_t d, uint32_t diag, uint8_t* e, uint8_t* cell_dead,
                                                          unsigned long long* filtered_rows) {
    for (uint32_t c = threadIdx.x; c < P; c += blockDim.x) e[c] = off[c + 1] > off[c] ? 1 : 0;
    __syncthreads();
    uint32_t stride = 1;
    for (uint32_t j = 0; j < d; ++j) {
        grid_prefix_axis(e, P, m, stride, threadIdx.x, blockDim.x);
        __syncthreads();
        stride *= m;
    }
    unsigned long long rows = grid_dead_cells(off, e, P, m, d, diag, cell_dead, threadIdx.x, blockDim.x);
    rows = warp_sum_u64(rows);
    if ((threadIdx.x & 31) == 0 && rows) atomicAdd(filtered_rows, rows);
}
__global__ void k_grid_occupancy(const uint32_t* __restrict__ off, uint32_t P, uint8_t* e) {
    const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c < P) e[c] = off[c + 1] > off[c] ? 1 : 0;
}
__global__ void k_grid_prefix_axis(uint8_t* e, uint32_t P, uint32_t m, uint32_t stride) {
    grid_prefix_axis(e, P, m, stride, blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x);
}
__global__ void k_grid_dead_cells(const uint32_t* __restrict__ off, const uint8_t* __restrict__ e, uint32_t P, uint32_t m,
                                  uint32_t d, uint32_t diag, uint8_t* cell_dead, unsigned long long* filtered_rows) {
    unsigned long long rows = grid_dead_cells(off, e, P, m, d, diag, cell_dead, blockIdx.x * blockDim.x + threadIdx.x,
                                              gridDim.x * blockDim.x);
    rows = warp_sum_u64(rows);
    if ((threadIdx.x & 31) == 0 && rows) atomicAdd(filtered_rows, rows);
}

uint32_t launch_grid_filter(const uint32_t* off, uint32_t P, uint32_t m, uint32_t d, uint8_t* occ, uint8_t* cell_dead,
                            unsigned long long* filtered_rows, cudaStream_t st) {
    SKY_CUDA(cudaMemsetAsync(filtered_rows, 0, sizeof(unsigned long long), st));
    if (!P) return 0;
    // P = m^d; the all-ones cell (1,..,1) = sum_j m^j
    uint32_t diag = 0, stride = 1;
    for (uint32_t j = 0; j < d; ++j) {
        diag += stride;
        stride *= m;
    }
    constexpr uint32_t kGridCtaCells = 1u << 15;
    if (P <= kGridCtaCells) {
        k_grid_filter_cta<<<1, 1024, 0, st>>>(off, P, m, d, diag, occ, cell_dead, filtered_rows);
        SKY_LAUNCH_CHECK();
        return 1;
    }
    k_grid_occupancy<<<ceil_div(P, 256), 256, 0, st>>>(off, P, occ);
    SKY_LAUNCH_CHECK();
    stride = 1;
    for (uint32_t j = 0; j < d; ++j) {
        k_grid_prefix_axis<<<ceil_div(P / m, 256), 256, 0, st>>>(occ, P, m, stride);
        SKY_LAUNCH_CHECK();
        stride *= m;
    }
    k_grid_dead_cells<<<ceil_div(P, 256), 256, 0, st>>>(off, occ, P, m, d, diag, cell_dead, filtered_rows);
    SKY_LAUNCH_CHECK();
    return d + 2;
}

void launch_mark_cells_dead(const uint64_t* key64, uint32_t n, const uint8_t* cell_dead, uint8_t* dead,
                            cudaStream_t st) {
    if (!n) return;
    k_mark_cells_dead<<<ceil_div(n, 256), 256, 0, st>>>(key64, n, cell_dead, dead);
    SKY_LAUNCH_CHECK();
}

// ---------------------------------------------------------- dominance core
constexpr int RS_THREADS = 128;
constexpr int RS_K = 4;
constexpr int RS_TILE = 256;

// s dominates t on D coordinates (core.hpp:89-96): s <= t everywhere and
// s < t somewhere. The <=-chain is the hot path; strictness is only checked
// on a hit.
template <int D>
__device__ __forceinline__ bool dominates_f(const float (&s)[D], const float (&t)[D]) {
    bool gt = false;
#pragma unroll
    for (int j = 0; j < D; ++j) gt |= s[j] > t[j];
    if (gt) return false;
    bool lt = false;
#pragma unroll
    for (int j = 0; j < D; ++j) lt |= s[j] < t[j];
    return lt;
}

// s <= t everywhere on the float image (necessary for FP64 dominance).
template <int D>
__device__ __forceinline__ bool le_all_f(const float (&s)[D], const float (&t)[D]) {
    bool gt = false;
#pragma unroll
    for (int j = 0; j < D; ++j) gt |= s[j] > t[j];
    return !gt;
}

template <int D, bool INDIRECT>
__global__ void __launch_bounds__(RS_THREADS) k_relsky(RelskyArgs a) {
    constexpr int V = Dims<D>::V;
    __shared__ float4 s_xyz[RS_TILE * V];
    __shared__ uint32_t s_key[RS_TILE];
    __shared__ uint32_t s_red[RS_THREADS / 32];
    __shared__ uint32_t s_end;

    const Item it = a.items[blockIdx.x];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    float t[RS_K][D];
    uint32_t tk[RS_K];
    bool alive[RS_K];
    const uint32_t pos0 = it.cb + tid * RS_K;
    uint32_t my_max = 0;
    bool any = false;
#pragma unroll
    for (int k = 0; k < RS_K; ++k) {
        const uint32_t pos = pos0 + k;
        alive[k] = pos < it.ce && !a.dead[pos];
        tk[k] = 0;
#pragma unroll
        for (int j = 0; j < D; ++j) t[k][j] = 0.0f;
        if (alive[k]) {
            if (INDIRECT) {
                const float* x = a.cxyz + (size_t)a.cidx[pos] * a.cd;
#pragma unroll
                for (int j = 0; j < D; ++j) t[k][j] = (uint32_t)j < a.cd ? x[j] : 0.0f;
                tk[k] = a.cskey[2 * (size_t)pos];  // low word of key64
            } else {
                const float4* x = reinterpret_cast<const float4*>(a.cxyz) + (size_t)pos * V;
#pragma unroll
                for (int v = 0; v < V; ++v) {
                    const float4 q = x[v];
                    if (4 * v + 0 < D) t[k][4 * v + 0] = q.x;
                    if (4 * v + 1 < D) t[k][4 * v + 1] = q.y;
                    if (4 * v + 2 < D) t[k][4 * v + 2] = q.z;
                    if (4 * v + 3 < D) t[k][4 * v + 3] = q.w;
                }
                tk[k] = a.cskey[pos];
            }
            my_max = max(my_max, tk[k]);
            any = true;
        }
    }
    bool initially[RS_K];
#pragma unroll
    for (int k = 0; k < RS_K; ++k) initially[k] = alive[k];

    uint32_t warp_max = __reduce_max_sync(0xffffffffu, my_max);
    if (lane == 0) s_red[warp] = warp_max;
    __syncthreads();
    uint32_t cta_max = 0;
#pragma unroll
    for (int w = 0; w < RS_THREADS / 32; ++w) cta_max = max(cta_max, s_red[w]);
    if (!a.bounded) warp_max = cta_max = 0xFFFFFFFFu;
    bool warp_alive = __any_sync(0xffffffffu, any);
    if (!__syncthreads_or(any)) return;

    unsigned long long ntests = 0;
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
        bool warp_range_live = warp_alive;
        for (uint32_t base = sb; base < se; base += RS_TILE) {
            const uint32_t len = min((uint32_t)RS_TILE, se - base);
            __syncthreads();
            const float4* src = reinterpret_cast<const float4*>(a.sxyz) + (size_t)base * V;
            for (uint32_t i = tid; i < len * V; i += RS_THREADS) s_xyz[i] = src[i];
            for (uint32_t i = tid; i < len; i += RS_THREADS) s_key[i] = a.sskey[base + i];
            __syncthreads();
            if (warp_range_live) {
                uint32_t i = 0;
                for (; i < len; ++i) {
                    if (s_key[i] > warp_max) break;  // warp-uniform: sorted comparators
                    float s[D];
#pragma unroll
                    for (int v = 0; v < V; ++v) {
                        const float4 q = s_xyz[i * V + v];
                        if (4 * v + 0 < D) s[4 * v + 0] = q.x;
                        if (4 * v + 1 < D) s[4 * v + 1] = q.y;
                        if (4 * v + 2 < D) s[4 * v + 2] = q.z;
                        if (4 * v + 3 < D) s[4 * v + 3] = q.w;
                    }
#pragma unroll
                    for (int k = 0; k < RS_K; ++k) {
                        const bool dom =
                            a.x64.x ? le_all_f<D>(s, t[k]) &&
                                          dom64(a.x64, a.sid[base + i],
                                                INDIRECT ? a.cidx[pos0 + k] : a.cid[pos0 + k])
                                    : dominates_f<D>(s, t[k]);
                        if (alive[k] && dom) {
                            alive[k] = false;
                            ntests += i + 1;
                        }
                    }
                    if (!__any_sync(0xffffffffu, alive[0] | alive[1] | alive[2] | alive[3])) {
                        ++i;
                        break;
                    }
                }
                int nal = 0;
#pragma unroll
                for (int k = 0; k < RS_K; ++k) nal += alive[k];
                ntests += (unsigned long long)nal * i;
                if (i < len) warp_range_live = false;
                warp_alive = __any_sync(0xffffffffu, alive[0] | alive[1] | alive[2] | alive[3]);
                if (!warp_alive) warp_range_live = false;
            }
            if (!__syncthreads_or(warp_range_live)) break;
        }
        if (!__syncthreads_or(warp_alive)) break;
    }
#pragma unroll
    for (int k = 0; k < RS_K; ++k)
        if (initially[k] && !alive[k]) a.dead[pos0 + k] = 1;
    if (a.tests) {
        ntests = warp_sum_u64(ntests);
        if (lane == 0 && ntests) atomicAdd(a.tests, ntests);
    }
}

void launch_relsky(int D, const RelskyArgs& a, cudaStream_t st) {
    if (!a.n_items) return;
    if (a.indirect) {
        SKY_DISPATCH_D(D, (k_relsky<DT, true><<<a.n_items, RS_THREADS, 0, st>>>(a)));
    } else {
        SKY_DISPATCH_D(D, (k_relsky<DT, false><<<a.n_items, RS_THREADS, 0, st>>>(a)));
    }
    SKY_LAUNCH_CHECK();
}

// ------------------------------------------------------------------- BNL
// Block-nested-loops (Börzsönyi et al., ICDE 2001) with a shared-memory
// window of at most `cap` points, restated for a CTA: the partition is
// consumed in batches of BNL_B tuples (one per thread); each batch is
// compared with the window in both directions (window tuples a batch tuple
// dominates are evicted) and with itself; survivors enter the window while it
// has room and spill to an overflow list otherwise. Window tuples carry
// (pass, timestamp = overflow length at insertion); a tuple inserted in pass
// p is confirmed once pass p+1 has consumed that many overflow tuples.
constexpr int BNL_B = 256;

template <int D>
__global__ void __launch_bounds__(BNL_B) k_bnl(BnlArgs a, uint32_t cap, uint32_t* win_pos_g, uint32_t* win_meta_g,
                                                 uint32_t* work_counter) {
    constexpr int V = Dims<D>::V;
    extern __shared__ float4 smem[];
    float4* w_xyz = smem;                                        // cap * V
    float4* b_xyz = w_xyz + (size_t)cap * V;                     // BNL_B * V
    uint8_t* w_kill = reinterpret_cast<uint8_t*>(b_xyz + BNL_B * V);  // cap
    __shared__ uint32_t s_wn, s_ovf_w, s_part, s_scan[BNL_B / 32], s_bn;
    __shared__ int s_pass;

    uint32_t* win_pos = win_pos_g + (size_t)blockIdx.x * cap;
    uint32_t* win_meta = win_meta_g + (size_t)blockIdx.x * cap;  // (pass << 24) | ts (ts < 2^24)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    unsigned long long ntests = 0;

    for (;;) {
        if (tid == 0) s_part = atomicAdd(work_counter, 1u);
        __syncthreads();
        const uint32_t part = s_part;
        if (part >= a.P) break;
        const uint32_t seg_b = a.seg_off[part], seg_e = a.seg_off[part + 1];
        if (seg_b == seg_e) { __syncthreads(); continue; }
        uint32_t* ovf = a.overflow + seg_b;  // in-place overflow list (positions)
        if (tid == 0) { s_wn = 0; s_pass = 0; }
        __syncthreads();
        uint32_t in_n = seg_e - seg_b;  // pass 0 input = the segment itself
        bool first = true;
        while (in_n > 0 || s_wn > 0) {
            const int pass = s_pass;
            if (tid == 0) s_ovf_w = 0;
            __syncthreads();
            for (uint32_t k0 = 0; k0 < in_n || k0 == 0; k0 += BNL_B) {
                // confirm window tuples of the previous pass whose timestamp
                // has been reached (they have now met every tuple)
                if (!first) {
                    const uint32_t wn = s_wn;
                    for (uint32_t w = tid; w < wn; w += BNL_B) {
                        const uint32_t meta = win_meta[w];
                        const bool prev = (meta >> 24) == ((uint32_t)(pass - 1) & 0xFFu);
                        w_kill[w] = (prev && (meta & 0xFFFFFFu) <= k0) ? 2 : 0;
                    }
                } else {
                    for (uint32_t w = tid; w < s_wn; w += BNL_B) w_kill[w] = 0;
                }
                __syncthreads();
                if (in_n == 0) break;
                // load batch
                const uint32_t bn = min((uint32_t)BNL_B, in_n - k0);
                uint32_t mypos = kNone;
                float t[D];
#pragma unroll
                for (int j = 0; j < D; ++j) t[j] = 0.0f;
                if ((uint32_t)tid < bn) {
                    mypos = first ? seg_b + k0 + tid : ovf[k0 + tid];
                    const float4* x = reinterpret_cast<const float4*>(a.xyz) + (size_t)mypos * V;
#pragma unroll
                    for (int v = 0; v < V; ++v) {
                        const float4 q = x[v];
                        b_xyz[tid * V + v] = q;
                        if (4 * v + 0 < D) t[4 * v + 0] = q.x;
                        if (4 * v + 1 < D) t[4 * v + 1] = q.y;
                        if (4 * v + 2 < D) t[4 * v + 2] = q.z;
                        if (4 * v + 3 < D) t[4 * v + 3] = q.w;
                    }
                }
                __syncthreads();
                bool alive = (uint32_t)tid < bn;
                // batch vs window (both directions)
                const uint32_t wn = s_wn;
                if (__syncthreads_or(alive)) {
                    for (uint32_t w = 0; w < wn; ++w) {
                        if (w_kill[w] == 1) continue;
                        float s[D];
#pragma unroll
                        for (int v = 0; v < V; ++v) {
                            const float4 q = w_xyz[w * V + v];
                            if (4 * v + 0 < D) s[4 * v + 0] = q.x;
                            if (4 * v + 1 < D) s[4 * v + 1] = q.y;
                            if (4 * v + 2 < D) s[4 * v + 2] = q.z;
                            if (4 * v + 3 < D) s[4 * v + 3] = q.w;
                        }
                        if (alive) {
                            bool gt = false, lt = false;
#pragma unroll
                            for (int j = 0; j < D; ++j) {
                                gt |= s[j] > t[j];
                                lt |= s[j] < t[j];
                            }
                            ntests += 2;  // both directions
                            if (a.x64.x) {
                                // float image equal or one-sided: confirm on the doubles
                                const uint32_t rw = a.id[win_pos[w]], rt = a.id[mypos];
                                if (!gt && dom64(a.x64, rw, rt)) alive = false;
                                else if (!lt && dom64(a.x64, rt, rw)) w_kill[w] = 1;
                            } else if (!gt && lt) {
                                alive = false;                          // window dominates t
                            } else if (gt && !lt) {
                                w_kill[w] = 1;                          // t dominates window tuple
                            }
                        }
                    }
                }
                // batch vs batch
                for (uint32_t b = 0; b < bn; ++b) {
                    if (!alive) break;
                    if (b == (uint32_t)tid) continue;
                    float s[D];
#pragma unroll
                    for (int v = 0; v < V; ++v) {
                        const float4 q = b_xyz[b * V + v];
                        if (4 * v + 0 < D) s[4 * v + 0] = q.x;
                        if (4 * v + 1 < D) s[4 * v + 1] = q.y;
                        if (4 * v + 2 < D) s[4 * v + 2] = q.z;
                        if (4 * v + 3 < D) s[4 * v + 3] = q.w;
                    }
                    ++ntests;
                    if (a.x64.x) {
                        if (le_all_f<D>(s, t) &&
                            dom64(a.x64, a.id[first ? seg_b + k0 + b : ovf[k0 + b]], a.id[mypos]))
                            alive = false;
                    } else if (dominates_f<D>(s, t)) {
                        alive = false;
                    }
                }
                __syncthreads();
                // remove killed (1) and confirmed (2) window tuples; compact
                {
                    const uint32_t wn0 = s_wn;
                    uint32_t kept_before = 0;
                    for (uint32_t c0 = 0; c0 < wn0; c0 += BNL_B) {
                        const uint32_t w = c0 + tid;
                        const bool in = w < wn0;
                        const uint8_t kill = in ? w_kill[w] : 0;
                        const bool keep = in && kill == 0;
                        float4 q[V];
                        uint32_t pos = 0, meta = 0;
                        if (keep) {
#pragma unroll
                            for (int v = 0; v < V; ++v) q[v] = w_xyz[w * V + v];
                            pos = win_pos[w];
                            meta = win_meta[w];
                        }
                        if (in && kill == 2) a.dead[win_pos[w]] = 0;  // confirmed skyline tuple
                        const unsigned bal = __ballot_sync(0xffffffffu, keep);
                        if (lane == 0) s_scan[warp] = __popc(bal);
                        __syncthreads();
                        uint32_t off = kept_before;
                        for (int ww = 0; ww < warp; ++ww) off += s_scan[ww];
                        off += __popc(bal & ((1u << lane) - 1u));
                        uint32_t tot = 0;
                        for (int ww = 0; ww < BNL_B / 32; ++ww) tot += s_scan[ww];
                        __syncthreads();
                        if (keep) {
#pragma unroll
                            for (int v = 0; v < V; ++v) w_xyz[off * V + v] = q[v];
                            win_pos[off] = pos;
                            win_meta[off] = meta;
                        }
                        kept_before += tot;
                        __syncthreads();
                    }
                    if (tid == 0) s_wn = kept_before;
                    __syncthreads();
                }
                // insert survivors (batch order) or spill them
                {
                    const unsigned bal = __ballot_sync(0xffffffffu, alive);
                    if (lane == 0) s_scan[warp] = __popc(bal);
                    __syncthreads();
                    uint32_t rank = __popc(bal & ((1u << lane) - 1u));
                    for (int ww = 0; ww < warp; ++ww) rank += s_scan[ww];
                    const uint32_t wn1 = s_wn, ow = s_ovf_w;
                    uint32_t room = cap - wn1;
                    if (alive) {
                        if (rank < room) {
                            const uint32_t slot = wn1 + rank;
#pragma unroll
                            for (int v = 0; v < V; ++v) w_xyz[slot * V + v] = b_xyz[tid * V + v];
                            win_pos[slot] = mypos;
                            // timestamp: overflow writes in this pass so far
                            // the pass modulo 256: a window tuple lives two passes at most
                            win_meta[slot] = ((uint32_t)pass << 24) | min(ow, 0xFFFFFFu);
                        } else {
                            ovf[ow + (rank - room)] = mypos;  // ow + ... <= k0 + tid (in place)
                        }
                    }
                    uint32_t tot = 0;
                    for (int ww = 0; ww < BNL_B / 32; ++ww) tot += s_scan[ww];
                    __syncthreads();
                    if (tid == 0) {
                        const uint32_t ins = min(tot, room);
                        s_wn = wn1 + ins;
                        s_ovf_w = ow + (tot - ins);
                    }
                    __syncthreads();
                }
            }
            // end of pass: window tuples inserted before any overflow in
            // this pass (ts == 0) are confirmed; when no overflow was written
            // every window tuple is confirmed.
            {
                const uint32_t ovf_n = s_ovf_w;
                const uint32_t wn0 = s_wn;
                for (uint32_t w = tid; w < wn0; w += BNL_B) {
                    const uint32_t meta = win_meta[w];
                    const bool cur = (meta >> 24) == ((uint32_t)pass & 0xFFu);
                    const bool confirm = ovf_n == 0 || (cur && (meta & 0xFFFFFFu) == 0) ||
                                         (!cur && (meta >> 24) == ((uint32_t)(pass - 1) & 0xFFu));
                    w_kill[w] = confirm ? 2 : 0;
                }
                __syncthreads();
                uint32_t kept_before = 0;
                for (uint32_t c0 = 0; c0 < wn0; c0 += BNL_B) {
                    const uint32_t w = c0 + tid;
                    const bool in = w < wn0;
                    const bool keep = in && w_kill[w] == 0;
                    float4 q[V];
                    uint32_t pos = 0, meta = 0;
                    if (keep) {
#pragma unroll
                        for (int v = 0; v < V; ++v) q[v] = w_xyz[w * V + v];
                        pos = win_pos[w];
                        meta = win_meta[w];
                    }
                    if (in && !keep) a.dead[win_pos[w]] = 0;
                    const unsigned bal = __ballot_sync(0xffffffffu, keep);
                    if (lane == 0) s_scan[warp] = __popc(bal);
                    __syncthreads();
                    uint32_t off = kept_before + __popc(bal & ((1u << lane) - 1u));
                    for (int ww = 0; ww < warp; ++ww) off += s_scan[ww];
                    uint32_t tot = 0;
                    for (int ww = 0; ww < BNL_B / 32; ++ww) tot += s_scan[ww];
                    __syncthreads();
                    if (keep) {
#pragma unroll
                        for (int v = 0; v < V; ++v) w_xyz[off * V + v] = q[v];
                        win_pos[off] = pos;
                        win_meta[off] = meta;
                    }
                    kept_before += tot;
                    __syncthreads();
                }
                if (tid == 0) {
                    s_wn = kept_before;
                    s_pass = pass + 1;
                    s_bn = ovf_n;
                }
                __syncthreads();
                in_n = s_bn;
                first = false;
            }
        }
        __syncthreads();
    }
    if (a.tests) {
        ntests = warp_sum_u64(ntests);
        if (lane == 0 && ntests) atomicAdd(a.tests, ntests);
    }
}

template <int D>
size_t bnl_smem_bytes(uint32_t cap) {
    constexpr int V = Dims<D>::V;
    return (size_t)cap * V * 16 + (size_t)BNL_B * V * 16 + cap + 64;
}

template <int D>
void launch_bnl_impl(const BnlArgs& a, uint32_t cap, uint32_t grid, uint32_t* win_pos, uint32_t* win_meta,
                     uint32_t* counter, cudaStream_t st) {
    const size_t smem = bnl_smem_bytes<D>(cap);
    SKY_CUDA(cudaFuncSetAttribute(k_bnl<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_bnl<D><<<grid, BNL_B, smem, st>>>(a, cap, win_pos, win_meta, counter);
    SKY_LAUNCH_CHECK();
}

uint32_t bnl_window_fit(int D, uint32_t want, int smem_optin) {
    uint32_t cap = want;
    SKY_DISPATCH_D(D, {
        while (cap > 32 && bnl_smem_bytes<DT>(cap) + 1024 > (size_t)smem_optin) cap -= 32;
    });
    return cap;
}

void launch_bnl_full(int D, const BnlArgs& a, uint32_t cap, uint32_t grid, uint32_t* win_pos, uint32_t* win_meta,
                     uint32_t* counter, cudaStream_t st) {
    SKY_DISPATCH_D(D, (launch_bnl_impl<DT>(a, cap, grid, win_pos, win_meta, counter, st)));
}

}  // namespace sky
