// host.cpp — host-only pieces of the C ABI: the BASELINE synthetic
// generators (include/skyline_baseline_gen.h) and the multi-rank planning
// helpers.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <queue>
#include <random>
#include <thread>
#include <vector>

#include "../../include/skyline_b200.h"
#include "../../include/skyline_baseline_gen.h"


extern "C" {

int sky_generate(int kind, uint64_t n, uint32_t d, uint64_t seed, float* out) {
    return sky_baseline_gen::generate(kind, n, d, seed, out) ? SKY_OK : SKY_E_CONFIG;
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
