// dom.cuh — the exact dominance test on float rows held as float4 groups.
#pragma once

#include <cuda_runtime.h>

namespace sky {

template <int D>
struct Dims2 {
    static constexpr int V = (D + 3) / 4;  // float4 per row == code words
};

// s dominates t: s <= t in every coordinate and < in one (core.hpp:89-96);
// padding coordinates are 0 in both rows
template <int D>
__device__ __forceinline__ bool dom_f4(const float4* __restrict__ s, const float4* __restrict__ t) {
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

}  // namespace sky
