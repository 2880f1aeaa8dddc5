/* skyline_baseline_gen.h — the BASELINE.json synthetic inputs, header-only.
 *
 * One definition compiled into two libraries:
 *   - libskyline_b200.so (`sky_generate`, the product's generator), and
 *   - oracle/_ref/libskyref.so (`skyref_generate_baseline`), so bench.py's
 *     `--impl reference` arm and the golden-fixture script build the exact
 *     same float32 input without loading the product library.
 *
 * Deterministic for (kind, n, d, seed) regardless of thread count: rows are
 * produced in 65,536-row chunks, chunk c by its own std::mt19937_64 seeded
 * with seed ^ (0x9E3779B97F4A7C15 * (c + 1)). Rng semantics follow the
 * reference's Rng (rng.hpp:15-51: uniform01 = (x >> 11) * 2^-53, Box-Muller
 * normal(mean, stddev)); float32 uniforms take 24 random bits so they lie in
 * [0, 1) exactly.
 *
 *   kind 1  independent: x ~ U[0,1)^d                       (configs[0])
 *   kind 2  anti-correlated: s ~ N(0.5, 0.0625) clipped to [0,1]; redraw
 *           x ~ U[0,1)^d until |sum(x) - d s| <= 0.01 d, evaluated on the
 *           stored float32 values in FP64                     (configs[1], [3])
 *   kind 3  correlated: v ~ N(0.5, 0.25) clipped; x_i = clip(v + N(0, 0.05))
 *                                                             (configs[2])
 *   kind 5  integers uniform in [0, 16) stored as float32     (configs[4])
 *   (kind 4 is an alias of kind 2.)
 */
#ifndef SKYLINE_BASELINE_GEN_H
#define SKYLINE_BASELINE_GEN_H

#ifdef __cplusplus
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <random>
#include <thread>
#include <vector>

namespace sky_baseline_gen {

struct Rng {
    std::mt19937_64 eng;
    explicit Rng(uint64_t s) : eng(s) {}
    double uniform01() { return static_cast<double>(eng() >> 11) * 0x1.0p-53; }
    double uniform01_pos() { return static_cast<double>((eng() >> 11) + 1) * 0x1.0p-53; }
    double normal(double mean, double stddev) {  // Box-Muller, rng.hpp:31-37
        const double u1 = uniform01_pos();
        const double u2 = uniform01();
        const double r = std::sqrt(-2.0 * std::log(u1));
        return mean + stddev * r * std::cos(6.283185307179586476925286766559 * u2);
    }
    float uniform_f32() { return static_cast<float>(eng() >> 40) * 0x1.0p-24f; }
};

inline double clip01(double v) { return v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v); }

constexpr uint64_t kChunkRows = 65536;

inline void gen_chunk(int kind, uint64_t r0, uint64_t r1, uint32_t d, uint64_t seed, uint64_t chunk, float* out) {
    Rng rng(seed ^ (0x9E3779B97F4A7C15ULL * (chunk + 1)));
    for (uint64_t i = r0; i < r1; ++i) {
        float* x = out + i * d;
        switch (kind) {
            case 1:
                for (uint32_t j = 0; j < d; ++j) x[j] = rng.uniform_f32();
                break;
            case 2:
            case 4: {
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
            case 3: {
                const double v = clip01(rng.normal(0.5, 0.25));
                for (uint32_t j = 0; j < d; ++j) x[j] = static_cast<float>(clip01(v + rng.normal(0.0, 0.05)));
                break;
            }
            case 5:
                for (uint32_t j = 0; j < d; ++j) x[j] = static_cast<float>(rng.eng() >> 60);
                break;
        }
    }
}

/* Returns false on a bad kind / d. out holds n*d floats, row-major. */
inline bool generate(int kind, uint64_t n, uint32_t d, uint64_t seed, float* out) {
    if (kind < 1 || kind > 5 || d < 1) return false;
    const uint64_t chunks = (n + kChunkRows - 1) / kChunkRows;
    const unsigned hw = std::thread::hardware_concurrency();
    const unsigned T = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(hw ? hw : 1, chunks));
    std::vector<std::thread> th;
    for (unsigned t = 0; t < T; ++t)
        th.emplace_back([=] {
            for (uint64_t c = t; c < chunks; c += T)
                gen_chunk(kind, c * kChunkRows, std::min(n, (c + 1) * kChunkRows), d, seed, c, out);
        });
    for (auto& x : th) x.join();
    return true;
}

}  // namespace sky_baseline_gen
#endif /* __cplusplus */
#endif /* SKYLINE_BASELINE_GEN_H */
