// mtjump.cpp — jump-ahead polynomials for std::mt19937_64, so the random
// partitioner's stream can be produced by many CTAs at once (kernels_rand.cu).
//
// The generator's 312-word state windows W_i = (x[i], ..., x[i+311]) evolve
// linearly over GF(2): W_{i+1} = A W_i. Its characteristic polynomial has the
// primitive factor phi(t) of degree 19937 (the 31 low bits of a window's
// first word never influence later words: a factor t^31 whose component
// vanishes after one step). With g(t) = t^J mod phi(t),
//     W_J = A^J W_0 = sum_i g_i W_i      (up to those 31 dead bits),
// a correlation of the coefficient bits of g with the first 19937 + 312
// words of the stream. phi is found once by Berlekamp-Massey on one output
// bit of the standard generator; g_k = t^(k J) mod phi for the chunk starts
// k J is computed once per process (seed-independent) and cached.
#include <immintrin.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <memory>
#include <mutex>
#include <random>
#include <vector>

#include "common.cuh"

namespace sky {

namespace {

constexpr int kDeg = 19937;
constexpr int kWords = (kDeg + 63) / 64;  // 312 words hold a reduced polynomial

using Poly = std::vector<uint64_t>;

inline int bit(const Poly& p, int i) { return (int)((p[i >> 6] >> (i & 63)) & 1u); }

// Berlekamp-Massey over GF(2): connection polynomial C (C[0] = 1) of the bit
// sequence s, degree L. Discrepancies are word-parallel parities of C
// against the reversed sequence.
Poly berlekamp_massey(const std::vector<uint8_t>& s, int* L_out) {
    const int N = (int)s.size();
    const int W = (N + 64) / 64 + 2;
    Poly rev(W + 2, 0);  // rev bit j = s[N-1-j]
    for (int j = 0; j < N; ++j)
        if (s[N - 1 - j]) rev[j >> 6] |= 1ull << (j & 63);
    auto rev_word = [&](int off) {  // 64 bits of rev starting at bit off
        const int w = off >> 6, b = off & 63;
        uint64_t v = rev[w] >> b;
        if (b) v |= rev[w + 1] << (64 - b);
        return v;
    };
    Poly C(W, 0), B(W, 0), T;
    C[0] = B[0] = 1;
    int L = 0, m = 1;
    for (int n = 0; n < N; ++n) {
        // d = s[n] + sum_{i=1..L} C_i s[n-i]; s[n-i] = rev bit (N-1-n+i)
        uint64_t acc = 0;
        for (int i = 1; i <= L; i += 64) {
            uint64_t cw = 0;  // C bits i .. i+63
            {
                const int w = i >> 6, b = i & 63;
                cw = C[w] >> b;
                if (b && w + 1 < W) cw |= C[w + 1] << (64 - b);
            }
            if (L - i + 1 < 64) cw &= (1ull << (L - i + 1)) - 1;
            acc ^= cw & rev_word(N - 1 - n + i);
        }
        const int d = (s[n] ^ __builtin_parityll(acc)) & 1;
        if (!d) {
            ++m;
            continue;
        }
        T = C;
        // C ^= B << m
        const int ws = m >> 6, bs = m & 63;
        for (int i = W - 1; i >= ws; --i) {
            uint64_t v = B[i - ws] << bs;
            if (bs && i - ws - 1 >= 0) v |= B[i - ws - 1] >> (64 - bs);
            C[i] ^= v;
        }
        if (2 * L <= n) {
            L = n + 1 - L;
            B = T;
            m = 1;
        } else {
            ++m;
        }
    }
    *L_out = L;
    return C;
}

// 64 x 64 -> 128 carry-less product
__attribute__((target("pclmul,sse4.1"))) inline void clmul(uint64_t a, uint64_t b, uint64_t* lo, uint64_t* hi) {
    const __m128i r = _mm_clmulepi64_si128(_mm_set_epi64x(0, (long long)a), _mm_set_epi64x(0, (long long)b), 0);
    *lo = (uint64_t)_mm_cvtsi128_si64(r);
    *hi = (uint64_t)_mm_extract_epi64(r, 1);
}

struct Field {
    Poly phi;                       // degree kDeg, monic
    std::vector<Poly> phi_shifted;  // phi << s for s in [0, 64), as words

    explicit Field(const Poly& p) : phi(p) {
        phi.resize(kWords + 2, 0);
        phi_shifted.resize(64);
        for (int s = 0; s < 64; ++s) {
            Poly q(kWords + 3, 0);
            for (int i = 0; i < (int)phi.size(); ++i) {
                q[i] ^= phi[i] << s;
                if (s && i + 1 < (int)q.size()) q[i + 1] ^= phi[i] >> (64 - s);
            }
            phi_shifted[s] = q;
        }
    }

    // p (any degree) mod phi, in place; result has kWords words
    void reduce(Poly& p) const {
        for (int i = (int)p.size() * 64 - 1; i >= kDeg; --i) {
            if (!bit(p, i)) continue;
            const int sh = i - kDeg, ws = sh >> 6, bs = sh & 63;
            const Poly& q = phi_shifted[bs];
            const int nq = std::min((int)q.size(), (int)p.size() - ws);
            for (int k = 0; k < nq; ++k) p[ws + k] ^= q[k];
        }
        p.resize(kWords);
    }

    Poly mulmod(const Poly& a, const Poly& b) const {
        Poly r(2 * kWords + 1, 0);
        for (int i = 0; i < kWords; ++i) {
            if (!a[i]) continue;
            for (int j = 0; j < kWords; ++j) {
                if (!b[j]) continue;
                uint64_t lo, hi;
                clmul(a[i], b[j], &lo, &hi);
                r[i + j] ^= lo;
                r[i + j + 1] ^= hi;
            }
        }
        reduce(r);
        return r;
    }
};

struct JumpTable {
    std::mutex mu;
    bool ready = false;
    uint32_t log2_stride = 0;
    std::unique_ptr<Field> F;
    Poly h, g;                    // h = t^J mod phi; g = t^(kJ) mod phi for the last k built
    uint32_t built = 0;
    std::vector<uint32_t> words;  // [k-1][kWords*2] u32 coefficient words of t^(kJ) mod phi
};

JumpTable g_table;

void init_table(uint32_t log2_stride) {
    // phi from one output bit of the standard generator (any seed)
    std::mt19937_64 eng(5489u);
    std::vector<uint8_t> s(2 * kDeg + 256);
    for (auto& b : s) b = (uint8_t)(eng() & 1u);
    int L = 0;
    Poly C = berlekamp_massey(s, &L);
    if (L != kDeg) throw Error(SKY_E_INTERNAL, "mt19937_64 characteristic polynomial has unexpected degree");
    // characteristic polynomial = reciprocal of the connection polynomial
    Poly phi(kWords + 1, 0);
    for (int i = 0; i <= kDeg; ++i)
        if (bit(C, i)) phi[(kDeg - i) >> 6] |= 1ull << ((kDeg - i) & 63);
    g_table.F = std::make_unique<Field>(phi);
    // h = t^(2^log2_stride) mod phi by repeated squaring of t
    Poly h(kWords, 0);
    h[0] = 2;  // t
    for (uint32_t r = 0; r < log2_stride; ++r) {
        Poly sq(2 * kWords + 1, 0);
        for (int i = 0; i < kWords; ++i) {
            uint64_t lo, hi;
            clmul(h[i], h[i], &lo, &hi);  // squaring spreads the bits
            sq[2 * i] ^= lo;
            sq[2 * i + 1] ^= hi;
        }
        g_table.F->reduce(sq);
        h = sq;
    }
    g_table.h = h;
    g_table.log2_stride = log2_stride;
    g_table.ready = true;
}

}  // namespace

// Coefficient words (u32; bit i of the polynomial = bit i%32 of word i/32)
// of t^(k * 2^log2_stride) mod phi for k = 1..chunks, row-major with 2*312
// words per k. Extended on demand, once per process (seed-independent).
const uint32_t* mt_jump_table(uint32_t log2_stride, uint32_t chunks) {
    std::lock_guard<std::mutex> lock(g_table.mu);
    if (!g_table.ready) init_table(log2_stride);
    if (g_table.log2_stride != log2_stride) throw Error(SKY_E_INTERNAL, "mt19937_64 jump stride mismatch");
    if (g_table.built < chunks) {
        g_table.words.resize((size_t)chunks * kWords * 2);
        for (uint32_t k = g_table.built + 1; k <= chunks; ++k) {
            g_table.g = k == 1 ? g_table.h : g_table.F->mulmod(g_table.g, g_table.h);
            uint32_t* dst = g_table.words.data() + (size_t)(k - 1) * kWords * 2;
            for (int i = 0; i < kWords; ++i) {
                dst[2 * i] = (uint32_t)g_table.g[i];
                dst[2 * i + 1] = (uint32_t)(g_table.g[i] >> 32);
            }
        }
        g_table.built = chunks;
    }
    return g_table.words.data();
}

int mt_jump_words() { return kWords * 2; }

}  // namespace sky
