// angular.cpp — slice thresholds for the exact angular partitioner
// (kernels.cuh: angular_thresholds; reference partition.cpp:118-148).
//
// The reference maps an angle phi (std::atan2 on the host libm) to
// (size_t)(2.0 * phi / 3.14159265358979323846 * m), clamped to m - 1. That
// map is monotone in phi, so slice k >= 1 starts at one double phi*_k, found
// here by bisection over the bit patterns with the reference's own double
// arithmetic. glibc's atan2 is faithful (error < 1 ulp; checked on 2e7
// near-boundary angles against quad precision), so the
// reference's slice follows from the exact angle unless that lies strictly
// between pred(phi*_k) and phi*_k; the device tests the exact angle against
// tan(pred(phi*_k)) and tan(phi*_k), computed here in quad precision and
// stored as double-doubles.
#include <cmath>
#include <cstdint>
#include <cstring>

#include <cuda_runtime.h>
#include <quadmath.h>

#include "kernels.cuh"

namespace sky {

namespace {

// partition.cpp:139-141, evaluated exactly as the reference does (no
// contraction is possible: a division then a product)
uint64_t ref_slice(double phi, uint64_t m) {
    volatile double v = 2.0 * phi;
    v = v / 3.14159265358979323846;
    v = v * static_cast<double>(m);
    const double w = v;
    return w >= 18446744073709551615.0 ? ~0ull : static_cast<uint64_t>(w);
}

double from_bits(uint64_t b) {
    double x;
    std::memcpy(&x, &b, sizeof(x));
    return x;
}

uint64_t to_bits(double x) {
    uint64_t b;
    std::memcpy(&b, &x, sizeof(b));
    return b;
}

void split(__float128 t, double* hi, double* lo) {
    *hi = static_cast<double>(t);
    *lo = static_cast<double>(t - static_cast<__float128>(*hi));
}

}  // namespace

uint64_t angular_thresholds(uint64_t m, double4* out) {
    if (m < 2 || m > kAngularExactMaxM) return 0;
    // phi ranges over [0, pi/2]; every boundary lies below rn(pi/2)
    const uint64_t top = to_bits(0x1.921fb54442d18p+0);
    uint64_t lo_bits = 0;
    for (uint64_t k = 1; k < m; ++k) {
        // smallest bit pattern b in [lo_bits, top] with ref_slice >= k
        uint64_t lo = lo_bits, hi = top;
        while (lo < hi) {
            const uint64_t mid = lo + (hi - lo) / 2;
            if (ref_slice(from_bits(mid), m) >= k) hi = mid; else lo = mid + 1;
        }
        const double phik = from_bits(lo), pred = from_bits(lo - 1);
        double4 t;
        split(tanq(static_cast<__float128>(pred)), &t.x, &t.y);
        split(tanq(static_cast<__float128>(phik)), &t.z, &t.w);
        out[k - 1] = t;
        lo_bits = lo;
    }
    return m - 1;
}

}  // namespace sky
