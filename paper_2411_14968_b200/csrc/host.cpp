// host.cpp — host-only pieces of the C ABI: the BASELINE synthetic
// generators and the multi-rank planning helpers.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <queue>
#include <random>
#include <thread>
#include <vector>

#include "../../include/skyline_b200.h"

namespace {

// Rng semantics of the reference (rng.hpp:15-51) on std::mt19937_64.
struct Rng {
    std::mt19937_64 eng;
    explicit Rng(uint64_t s) : eng(s) {}
    double uniform01() { return static_cast<double>(eng() >> 11) * 0x1.0p-53; }
    double uniform01_pos() { return static_cast<double>((eng() >> 11) + 1) * 0x1.0p-53; }
    double normal(double mean, double stddev) {  // Box-Muller
        const double u1 = uniform01_pos();
        const double u2 = uniform01();
        const double r = std::sqrt(-2.0 * std::log(u1));
        return mean + stddev * r * std::cos(6.283185307179586476925286766559 * u2);
    }
    // float32 uniform in [0,1): 24 random bits, exactly representable
    float uniform_f32() { return static_cast<float>(eng() >> 40) * 0x1.0p-24f; }
};

double clip01(double v) { return v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v); }

constexpr uint64_t kChunkRows = 65536;

void gen_chunk(int kind, uint64_t r0, uint64_t r1, uint32_t d, uint64_t seed, uint64_t chunk, float* out) {
    Rng rng(seed ^ (0x9E3779B97F4A7C15ULL * (chunk + 1)));
    for (uint64_t i = r0; i < r1; ++i) {
        float* x = out + i * d;
        switch (kind) {
            case 1:  // independent: x ~ U[0,1)^d
                for (uint32_t j = 0; j < d; ++j) x[j] = rng.uniform_f32();
                break;
            case 2:
            case 4: {  // anti-correlated: s ~ N(0.5, 0.0625) clipped; redraw x until |sum - d s| <= 0.01 d
                const double s = clip01(rng.normal(0.5, 0.0625));
                const double target = d * s, tol = 0.01 * d;
                for (;;) {
                    double sum = 0.0;
                    for (uint32_t j = 0; j < d; ++j) {
                        x[j] = rng.uniform_f32();
                        sum += (double)x[j];
                    }
                    if (std::fabs(sum - target) <= tol) break;
                }
                break;
            }
            case 3: {  // correlated: v ~ N(0.5, 0.25) clipped; x_i = clip(v + N(0, 0.05))
                const double v = clip01(rng.normal(0.5, 0.25));
                for (uint32_t j = 0; j < d; ++j) x[j] = static_cast<float>(clip01(v + rng.normal(0.0, 0.05)));
                break;
            }
            case 5:  // tie-heavy integers in [0,16)
                for (uint32_t j = 0; j < d; ++j) x[j] = static_cast<float>(rng.eng() >> 60);
                break;
        }
    }
}

}  // namespace

extern "C" {

int sky_generate(int kind, uint64_t n, uint32_t d, uint64_t seed, float* out) {
    if (kind < 1 || kind > 5 || d < 1) return SKY_E_CONFIG;
    const uint64_t chunks = (n + kChunkRows - 1) / kChunkRows;
    unsigned hw = std::thread::hardware_concurrency();
    const unsigned T = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(hw ? hw : 1, chunks));
    std::vector<std::thread> th;
    for (unsigned t = 0; t < T; ++t)
        th.emplace_back([=] {
            for (uint64_t c = t; c < chunks; c += T)
                gen_chunk(kind, c * kChunkRows, std::min(n, (c + 1) * kChunkRows), d, seed, c, out);
        });
    for (auto& x : th) x.join();
    return SKY_OK;
}

// Longest-processing-time greedy: heaviest unit first onto the least loaded
// owner (ties -> lower rank), deterministic.
int sky_plan_lpt(const uint64_t* weights, uint64_t count, int ranks, int32_t* owner) {
    if (ranks < 1) return SKY_E_CONFIG;
    std::vector<uint64_t> ix(count);
    for (uint64_t i = 0; i < count; ++i) ix[i] = i;
    std::stable_sort(ix.begin(), ix.end(), [&](uint64_t a, uint64_t b) { return weights[a] > weights[b]; });
    using E = std::pair<uint64_t, int>;
    std::priority_queue<E, std::vector<E>, std::greater<E>> load;
    for (int r = 0; r < ranks; ++r) load.push({0, r});
    for (uint64_t i : ix) {
        E e = load.top();
        load.pop();
        owner[i] = e.second;
        e.first += weights[i];
        load.push(e);
    }
    return SKY_OK;
}

// Contiguous split with balanced cost: bounds[r] = first index of rank r.
// cost_prefix has count+1 entries (cost_prefix[0] = 0).
int sky_plan_split(const uint64_t* cost_prefix, uint64_t count, int ranks, uint64_t* bounds) {
    if (ranks < 1) return SKY_E_CONFIG;
    const uint64_t total = cost_prefix[count];
    bounds[0] = 0;
    for (int r = 1; r < ranks; ++r) {
        const long double target = (long double)total * r / ranks;
        // first index whose prefix cost reaches the target
        uint64_t lo = bounds[r - 1], hi = count;
        while (lo < hi) {
            const uint64_t mid = (lo + hi) / 2;
            if ((long double)cost_prefix[mid] < target) lo = mid + 1; else hi = mid;
        }
        bounds[r] = lo;
    }
    bounds[ranks] = count;
    return SKY_OK;
}

}  // extern "C"
