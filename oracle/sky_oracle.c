/*
 * sky_oracle.c — TEST INFRASTRUCTURE ONLY (see sky_oracle.h).
 *
 * Plain-C restatement of the reference skyline engine, function by function,
 * each citing the reference file:line it follows (paths relative to
 * /root/reference/proj). Single-threaded: `workers` only changes scheduling
 * in the reference (engine.hpp:86-88), never results.
 */
#include "sky_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- rng.hpp */
/* std::mt19937_64 (the standard's published parameters), as pinned by
 * Rng (rng.hpp:15-51). */
typedef struct {
    uint64_t mt[312];
    int mti;
} mt64;

static void mt_seed(mt64* g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->mti = 312;
}

static uint64_t mt_next(mt64* g) {
    if (g->mti >= 312) {
        const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
        for (int i = 0; i < 312; ++i) {
            uint64_t x = (g->mt[i] & UM) | (g->mt[(i + 1) % 312] & LM);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
            g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
        }
        g->mti = 0;
    }
    uint64_t x = g->mt[g->mti++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= x >> 43;
    return x;
}

/* Rng::below (rng.hpp:40-47) */
static uint64_t rng_below(mt64* g, uint64_t n) {
    const uint64_t limit = UINT64_MAX - UINT64_MAX % n;
    uint64_t x;
    do {
        x = mt_next(g);
    } while (x >= limit);
    return x % n;
}


/* shuffle (rng.hpp:54-60) */
static void rng_shuffle(uint64_t* v, uint64_t n, mt64* g) {
    for (uint64_t i = n; i > 1; --i) {
        uint64_t j = rng_below(g, i);
        uint64_t t = v[i - 1];
        v[i - 1] = v[j];
        v[j] = t;
    }
}

void oracle_random_permutation(uint64_t n, uint64_t seed, uint64_t* perm) {
    mt64 g;
    mt_seed(&g, seed);
    for (uint64_t i = 0; i < n; ++i) perm[i] = i;
    rng_shuffle(perm, n, &g);
}

/* --------------------------------------------------------------- core.cpp */
static uint64_t g_tests; /* dominance tests executed (instrumentation) */

/* detail::dominates_raw (core.hpp:89-96) */
static int dominates_raw(const double* a, const double* b, uint32_t d) {
    int strict = 0;
    ++g_tests;
    for (uint32_t j = 0; j < d; ++j) {
        if (a[j] > b[j]) return 0;
        if (a[j] < b[j]) strict = 1;
    }
    return strict;
}

typedef struct {
    const double* x; /* row-major n x d */
    uint32_t d;
} relation;

#define ROW(R, i) ((R)->x + (size_t)(i) * (R)->d)

/* detail::coord_sum (core.hpp:103-107): left-to-right double sum */
static double coord_sum(const relation* R, uint64_t i) {
    const double* p = ROW(R, i);
    double s = 0.0;
    for (uint32_t j = 0; j < R->d; ++j) s += p[j];
    return s;
}

/* detail::coords_then_id_less (core.cpp:10-17); ids are row indices */
static int coords_then_id_cmp(const relation* R, uint64_t a, uint64_t b) {
    const double* pa = ROW(R, a);
    const double* pb = ROW(R, b);
    for (uint32_t j = 0; j < R->d; ++j) {
        if (pa[j] < pb[j]) return -1;
        if (pa[j] > pb[j]) return 1;
    }
    return a < b ? -1 : (a > b ? 1 : 0);
}

/* Stable merge sort of index arrays with a context comparator. */
typedef int (*cmp_fn)(const void* ctx, uint64_t a, uint64_t b);

static void msort_rec(uint64_t* v, uint64_t* tmp, uint64_t n, cmp_fn cmp, const void* ctx) {
    if (n < 2) return;
    if (n <= 16) {
        for (uint64_t i = 1; i < n; ++i) {
            uint64_t x = v[i];
            uint64_t j = i;
            while (j > 0 && cmp(ctx, v[j - 1], x) > 0) {
                v[j] = v[j - 1];
                --j;
            }
            v[j] = x;
        }
        return;
    }
    uint64_t h = n / 2;
    msort_rec(v, tmp, h, cmp, ctx);
    msort_rec(v + h, tmp, n - h, cmp, ctx);
    uint64_t i = 0, j = h, k = 0;
    while (i < h && j < n) tmp[k++] = (cmp(ctx, v[j], v[i]) < 0) ? v[j++] : v[i++];
    while (i < h) tmp[k++] = v[i++];
    while (j < n) tmp[k++] = v[j++];
    memcpy(v, tmp, n * sizeof(uint64_t));
}

static void msort(uint64_t* v, uint64_t n, cmp_fn cmp, const void* ctx) {
    if (n < 2) return;
    uint64_t* tmp = (uint64_t*)malloc(n * sizeof(uint64_t));
    msort_rec(v, tmp, n, cmp, ctx);
    free(tmp);
}

static int cmp_u64(const void* a, const void* b) {
    uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
    return x < y ? -1 : (x > y ? 1 : 0);
}
static int cmp_i64(const void* a, const void* b) {
    int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
    return x < y ? -1 : (x > y ? 1 : 0);
}

typedef struct {
    const relation* R;
    const double* sum;
} sum_ctx;

/* by coordinate sum only (relative_skyline's ranking, core.cpp:93-94) */
static int cmp_sum_only(const void* c, uint64_t a, uint64_t b) {
    const sum_ctx* s = (const sum_ctx*)c;
    return s->sum[a] < s->sum[b] ? -1 : (s->sum[a] > s->sum[b] ? 1 : 0);
}
/* by (sum, lex coords, id) (sequential.cpp:52-55, filter.cpp:74-79) */
static int cmp_sum_lex(const void* c, uint64_t a, uint64_t b) {
    const sum_ctx* s = (const sum_ctx*)c;
    if (s->sum[a] != s->sum[b]) return s->sum[a] < s->sum[b] ? -1 : 1;
    return coords_then_id_cmp(s->R, a, b);
}

/* skyline_bruteforce (core.cpp:56-73) over an index list; writes survivors
 * (id-sorted) into out, returns the count. */
static uint64_t bruteforce_list(const relation* R, const uint64_t* idx, uint64_t n, uint64_t* out) {
    uint64_t k = 0;
    for (uint64_t a = 0; a < n; ++a) {
        int dominated = 0;
        for (uint64_t b = 0; b < n; ++b) {
            if (a == b) continue;
            if (dominates_raw(ROW(R, idx[b]), ROW(R, idx[a]), R->d)) {
                dominated = 1;
                break;
            }
        }
        if (!dominated) out[k++] = idx[a];
    }
    qsort(out, k, sizeof(uint64_t), cmp_u64);
    return k;
}

/* relative_skyline (core.cpp:75-110): keep flags for r's rows, r's order. */
static uint64_t relative_skyline_list(const relation* R, const double* sum, const uint64_t* r,
                                      uint64_t nr, const uint64_t* c, uint64_t nc, uint64_t* out) {
    if (nr == 0) return 0;
    if (nc == 0) {
        memcpy(out, r, nr * sizeof(uint64_t));
        return nr;
    }
    uint64_t* ranked = (uint64_t*)malloc(nc * sizeof(uint64_t));
    memcpy(ranked, c, nc * sizeof(uint64_t));
    sum_ctx sc = {R, sum};
    msort(ranked, nc, cmp_sum_only, &sc);
    uint64_t k = 0;
    for (uint64_t a = 0; a < nr; ++a) {
        const uint64_t t = r[a];
        const double st = sum[t];
        int dominated = 0;
        for (uint64_t b = 0; b < nc; ++b) {
            const uint64_t s = ranked[b];
            if (sum[s] > st) break; /* core.cpp:101 */
            if (dominates_raw(ROW(R, s), ROW(R, t), R->d)) {
                dominated = 1;
                break;
            }
        }
        if (!dominated) out[k++] = t;
    }
    free(ranked);
    return k;
}

/* detail::sfs_scan (sequential.cpp:22-44): window loop, id-sorted output. */
static uint64_t sfs_scan(const relation* R, const uint64_t* ordered, uint64_t n, uint64_t* out) {
    uint64_t w = 0;
    for (uint64_t a = 0; a < n; ++a) {
        const uint64_t t = ordered[a];
        int dominated = 0;
        for (uint64_t b = 0; b < w; ++b) {
            if (dominates_raw(ROW(R, out[b]), ROW(R, t), R->d)) {
                dominated = 1;
                break;
            }
        }
        if (!dominated) out[w++] = t;
    }
    qsort(out, w, sizeof(uint64_t), cmp_u64);
    return w;
}

/* sfs (sequential.cpp:48-60) with Scoring::Sum */
static uint64_t sfs_list(const relation* R, const double* sum, const uint64_t* idx, uint64_t n,
                         uint64_t* out) {
    uint64_t* ord = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
    memcpy(ord, idx, n * sizeof(uint64_t));
    sum_ctx sc = {R, sum};
    msort(ord, n, cmp_sum_lex, &sc);
    uint64_t k = sfs_scan(R, ord, n, out);
    free(ord);
    return k;
}

/* ---------------------------------------------------------- partition.cpp */
#define K_MAX_PARTITIONS (1ULL << 22) /* partition.cpp:13 */

static uint64_t checked_pow(uint64_t base, uint64_t e) { /* partition.cpp:15-22 */
    uint64_t r = 1;
    for (uint64_t i = 0; i < e; ++i) {
        if (r > K_MAX_PARTITIONS) return K_MAX_PARTITIONS + 1;
        r *= base;
    }
    return r;
}

/* cell_of (partition.cpp:25-32); returns UINT64_MAX on NormalizationError */
static uint64_t cell_of(double v, uint64_t m) {
    if (!(v >= 0.0 && v <= 1.0)) return UINT64_MAX;
    uint64_t cell = (uint64_t)(v * (double)m);
    return cell >= m ? m - 1 : cell;
}

/* grid_index (partition.cpp:66-75) */
static uint64_t grid_index_row(const double* x, uint32_t d, uint64_t m) {
    uint64_t index = 0, stride = 1;
    for (uint32_t j = 0; j < d; ++j) {
        uint64_t c = cell_of(x[j], m);
        if (c == UINT64_MAX) return UINT64_MAX;
        index += c * stride;
        stride *= m;
    }
    return index;
}

/* hyperspherical_angles + angular_index (partition.cpp:118-148) */
static uint64_t angular_index_row(const double* x, uint32_t d, uint64_t m) {
    double tail_sq = x[d - 1] * x[d - 1];
    double angles[64];
    double* ang = d - 1 <= 64 ? angles : (double*)malloc((d - 1) * sizeof(double));
    for (uint32_t i = d - 1; i-- > 0;) {
        ang[i] = atan2(sqrt(tail_sq), x[i]);
        tail_sq += x[i] * x[i];
    }
    uint64_t index = 0, stride = 1;
    for (uint32_t i = 0; i + 1 < d; ++i) {
        uint64_t slice = (uint64_t)(2.0 * ang[i] / 3.14159265358979323846 * (double)m);
        if (slice >= m) slice = m - 1;
        index += slice * stride;
        stride *= m;
    }
    if (ang != angles) free(ang);
    return index;
}

uint64_t oracle_angular_index(const float* x, uint32_t d, uint64_t m) {
    double buf[64];
    for (uint32_t j = 0; j < d && j < 64; ++j) buf[j] = (double)x[j];
    return angular_index_row(buf, d, m);
}

uint64_t oracle_grid_index(const float* x, uint32_t d, uint64_t m) {
    double buf[64];
    for (uint32_t j = 0; j < d && j < 64; ++j) buf[j] = (double)x[j];
    return grid_index_row(buf, d, m);
}

/* snap_slices (partition.cpp:220-231) */
uint64_t oracle_snap_slices(uint64_t target_p, uint64_t k) {
    if (target_p < 1 || k < 1) return 0;
    uint64_t hi = 1;
    while (checked_pow(hi, k) < target_p && checked_pow(hi, k) <= K_MAX_PARTITIONS) ++hi;
    if (hi == 1) return 1;
    if (checked_pow(hi, k) < target_p) return hi;
    const uint64_t lo = hi - 1;
    const uint64_t above = checked_pow(hi, k) - target_p;
    const uint64_t below = target_p - checked_pow(lo, k);
    return above < below ? hi : lo;
}

typedef struct {
    int strategy;
    uint64_t count, slices;
    int presorted;
    uint64_t* partition_of;
    uint64_t* scan_order; /* NULL = natural */
} assignment;

typedef struct {
    const relation* R;
    uint64_t k;
} slice_ctx;

/* assign_sliced comparator (partition.cpp:202-209) */
static int cmp_sliced(const void* c, uint64_t a, uint64_t b) {
    const slice_ctx* s = (const slice_ctx*)c;
    const double va = ROW(s->R, a)[s->k], vb = ROW(s->R, b)[s->k];
    if (va < vb) return -1;
    if (va > vb) return 1;
    return coords_then_id_cmp(s->R, a, b);
}

/* make_assignment (partition.cpp:233-251) and the strategies it dispatches */
static int make_assignment(const relation* R, uint64_t n, const sky_config* cfg, assignment* A) {
    memset(A, 0, sizeof(*A));
    if (cfg->p < 1) return SKY_E_CONFIG;
    A->strategy = cfg->strategy;
    A->partition_of = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
    const uint32_t d = R->d;
    switch (cfg->strategy) {
        case SKY_RANDOM: { /* assign_random (partition.cpp:36-54) */
            uint64_t* perm = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
            oracle_random_permutation(n, cfg->seed, perm);
            for (uint64_t i = 0; i < n; ++i) A->partition_of[perm[i]] = i % cfg->p;
            free(perm);
            A->count = cfg->p;
            return SKY_OK;
        }
        case SKY_GRID: { /* assign_grid (partition.cpp:150-166) */
            uint64_t m = cfg->m > 0 ? cfg->m : oracle_snap_slices(cfg->p, d);
            if (m < 1) return SKY_E_CONFIG;
            if (d < 1) return SKY_E_DIMENSION;
            uint64_t count = checked_pow(m, d);
            if (count > K_MAX_PARTITIONS) return SKY_E_CONFIG;
            A->count = count;
            A->slices = m;
            for (uint64_t i = 0; i < n; ++i) {
                uint64_t g = grid_index_row(ROW(R, i), d, m);
                if (g == UINT64_MAX) return SKY_E_NORMALIZATION;
                A->partition_of[i] = g;
            }
            return SKY_OK;
        }
        case SKY_ANGULAR: { /* assign_angular (partition.cpp:168-184) */
            if (d < 2) return SKY_E_DIMENSION;
            uint64_t m = cfg->m > 0 ? cfg->m : oracle_snap_slices(cfg->p, d - 1);
            if (m < 1) return SKY_E_CONFIG;
            uint64_t count = checked_pow(m, d - 1);
            if (count > K_MAX_PARTITIONS) return SKY_E_CONFIG;
            A->count = count;
            A->slices = m;
            for (uint64_t i = 0; i < n; ++i) A->partition_of[i] = angular_index_row(ROW(R, i), d, m);
            return SKY_OK;
        }
        case SKY_SLICED: { /* assign_sliced (partition.cpp:186-218) */
            if (n > 0 && cfg->slice_dim >= d) return SKY_E_CONFIG;
            A->count = cfg->p;
            A->presorted = 1;
            A->scan_order = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
            for (uint64_t i = 0; i < n; ++i) A->scan_order[i] = i;
            slice_ctx sc = {R, cfg->slice_dim};
            msort(A->scan_order, n, cmp_sliced, &sc);
            for (uint64_t rank = 0; rank < n; ++rank) {
                uint64_t index = n > 1 ? rank * cfg->p / (n - 1) : 0;
                if (index >= cfg->p) index = cfg->p - 1;
                A->partition_of[A->scan_order[rank]] = index;
            }
            return SKY_OK;
        }
        default:
            return SKY_E_CONFIG;
    }
}

static void free_assignment(assignment* A) {
    free(A->partition_of);
    free(A->scan_order);
}

/* decode_grid_index / weak_grid_dominates / grid_dominates
 * (partition.cpp:87-116) */
static void decode_grid(uint64_t index, uint64_t m, uint32_t d, uint32_t* cells) {
    for (uint32_t j = 0; j < d; ++j) {
        cells[j] = (uint32_t)(index % m);
        index /= m;
    }
}
static int weak_grid_dominates(const uint32_t* a, const uint32_t* b, uint32_t d) {
    int equal = 1;
    for (uint32_t j = 0; j < d; ++j)
        if (a[j] != b[j]) equal = 0;
    if (equal) return 0;
    for (uint32_t j = 0; j < d; ++j)
        if (a[j] > b[j]) return 0;
    return 1;
}
static int grid_dominates(const uint32_t* a, const uint32_t* b, uint32_t d) {
    for (uint32_t j = 0; j < d; ++j)
        if (a[j] >= b[j]) return 0;
    return 1;
}

int oracle_assign(const float* pts, uint64_t n, uint32_t d, int normalized,
                  const sky_config* cfg, uint64_t* partition_of, uint64_t* count) {
    (void)normalized;
    double* x = (double*)malloc(((n && d) ? n * d : 1) * sizeof(double));
    for (uint64_t i = 0; i < n * d; ++i) x[i] = (double)pts[i];
    relation R = {x, d};
    assignment A;
    int rc = make_assignment(&R, n, cfg, &A);
    if (rc == SKY_OK) {
        memcpy(partition_of, A.partition_of, n * sizeof(uint64_t));
        *count = A.count;
    }
    free_assignment(&A);
    free(x);
    return rc;
}

/* ----------------------------------------------------- filter.cpp (reps) */
/* select_representatives_sorted (filter.cpp:66-86) + prune_dominated_reps
 * (filter.cpp:139-145). parts[i] = index list of partition i. */
static uint64_t select_reps_sorted(const relation* R, const double* sum, uint64_t** parts,
                                   const uint64_t* sizes, uint64_t P, uint64_t q, uint64_t* reps) {
    uint64_t total = 0;
    for (uint64_t i = 0; i < P; ++i) total += sizes[i] < q ? sizes[i] : q;
    uint64_t* cand = (uint64_t*)malloc((total ? total : 1) * sizeof(uint64_t));
    uint64_t k = 0;
    sum_ctx sc = {R, sum};
    for (uint64_t i = 0; i < P; ++i) {
        if (sizes[i] == 0) continue;
        uint64_t* ord = (uint64_t*)malloc(sizes[i] * sizeof(uint64_t));
        memcpy(ord, parts[i], sizes[i] * sizeof(uint64_t));
        msort(ord, sizes[i], cmp_sum_lex, &sc);
        uint64_t take = sizes[i] < q ? sizes[i] : q;
        for (uint64_t t = 0; t < take; ++t) cand[k++] = ord[t];
        free(ord);
    }
    uint64_t nr = bruteforce_list(R, cand, k, reps);
    free(cand);
    return nr;
}

/* dominance_region_volume (core.cpp:112-123): prod_j (1 - x_j), left to right */
static double region_volume(const relation* R, uint64_t i) {
    double v = 1.0;
    for (uint32_t j = 0; j < R->d; ++j) v *= 1.0 - R->x[i * R->d + j];
    return v;
}

typedef struct {
    const double* vol;
} vol_ctx;

/* (volume desc, id asc) (filter.cpp:103-106) */
static int cmp_volume(const void* c, uint64_t a, uint64_t b) {
    const vol_ctx* v = (const vol_ctx*)c;
    if (v->vol[a] != v->vol[b]) return v->vol[a] > v->vol[b] ? -1 : 1;
    return a < b ? -1 : (a > b ? 1 : 0);
}

/* select_representatives_region (filter.cpp:88-115) + prune. */
static uint64_t select_reps_region(const relation* R, uint64_t n, uint64_t** parts, const uint64_t* sizes,
                                   uint64_t P, uint64_t q, uint64_t* reps) {
    double* vol = (double*)malloc((n ? n : 1) * sizeof(double));
    for (uint64_t i = 0; i < n; ++i) vol[i] = region_volume(R, i);
    vol_ctx vc = {vol};
    uint64_t total = 0;
    for (uint64_t i = 0; i < P; ++i) total += sizes[i] < q ? sizes[i] : q;
    uint64_t* cand = (uint64_t*)malloc((total ? total : 1) * sizeof(uint64_t));
    uint64_t k = 0;
    for (uint64_t i = 0; i < P; ++i) {
        if (sizes[i] == 0) continue;
        uint64_t* ord = (uint64_t*)malloc(sizes[i] * sizeof(uint64_t));
        memcpy(ord, parts[i], sizes[i] * sizeof(uint64_t));
        msort(ord, sizes[i], cmp_volume, &vc);
        uint64_t take = sizes[i] < q ? sizes[i] : q;
        for (uint64_t t = 0; t < take; ++t) cand[k++] = ord[t];
        free(ord);
    }
    uint64_t nr = bruteforce_list(R, cand, k, reps);
    free(cand);
    free(vol);
    return nr;
}

/* select_representatives_random (filter.cpp:117-137) + prune: partial
 * Fisher-Yates over the partition's scan order with a per-partition Rng. */
static uint64_t select_reps_random(const relation* R, uint64_t** parts, const uint64_t* sizes, uint64_t P,
                                   uint64_t q, uint64_t seed, uint64_t* reps) {
    uint64_t total = 0;
    for (uint64_t i = 0; i < P; ++i) total += sizes[i] < q ? sizes[i] : q;
    uint64_t* cand = (uint64_t*)malloc((total ? total : 1) * sizeof(uint64_t));
    uint64_t k = 0;
    mt64 g;
    for (uint64_t i = 0; i < P; ++i) {
        if (sizes[i] == 0) continue;
        mt_seed(&g, seed ^ (0x9e3779b97f4a7c15ULL * (i + 1)));
        uint64_t* idx = (uint64_t*)malloc(sizes[i] * sizeof(uint64_t));
        for (uint64_t t = 0; t < sizes[i]; ++t) idx[t] = t;
        uint64_t take = sizes[i] < q ? sizes[i] : q;
        for (uint64_t t = 0; t < take; ++t) {
            uint64_t j = t + rng_below(&g, sizes[i] - t);
            uint64_t tmp = idx[t];
            idx[t] = idx[j];
            idx[j] = tmp;
        }
        for (uint64_t t = 0; t < take; ++t) cand[k++] = parts[i][idx[t]];
        free(idx);
    }
    uint64_t nr = bruteforce_list(R, cand, k, reps);
    free(cand);
    return nr;
}

/* --------------------------------------------------------------- engine.cpp */
/* validate (engine.cpp:19-32) */
static int validate(uint64_t n, uint32_t d, const sky_config* c) {
    if (c->workers < 1) return SKY_E_CONFIG;
    if (c->p < 1) return SKY_E_CONFIG;
    if (c->filter == SKY_FILTER_GRID && c->strategy != SKY_GRID) return SKY_E_CONFIG;
    if (c->filter == SKY_FILTER_REPRESENTATIVE && c->rep_q < 1) return SKY_E_CONFIG;
    if (c->strategy == SKY_ANGULAR && n > 0 && d < 2) return SKY_E_DIMENSION;
    return SKY_OK;
}

static int oracle_run_x(double* x, uint64_t n, uint32_t d, int normalized, const sky_config* cfg,
                        oracle_result* out);

int oracle_run(const float* pts, uint64_t n, uint32_t d, int normalized, const sky_config* cfg,
               oracle_result* out) {
    double* x = (double*)malloc(((n && d) ? n * d : 1) * sizeof(double));
    for (uint64_t i = 0; i < n * d; ++i) x[i] = (double)pts[i];
    return oracle_run_x(x, n, d, normalized, cfg, out);
}

int oracle_run_f64(const double* pts, uint64_t n, uint32_t d, int normalized, const sky_config* cfg,
                   oracle_result* out) {
    double* x = (double*)malloc(((n && d) ? n * d : 1) * sizeof(double));
    if (n && d) memcpy(x, pts, n * d * sizeof(double));
    return oracle_run_x(x, n, d, normalized, cfg, out);
}

/* takes ownership of x */
static int oracle_run_x(double* x, uint64_t n, uint32_t d, int normalized, const sky_config* cfg,
                        oracle_result* out) {
    memset(out, 0, sizeof(*out));
    int rc = validate(n, d, cfg);
    if (rc) {
        free(x);
        return rc;
    }
    if (cfg->filter == SKY_FILTER_REPRESENTATIVE &&
        (cfg->rep_selection < SKY_REPS_SORTED || cfg->rep_selection > SKY_REPS_RANDOM)) {
        free(x);
        return SKY_E_CONFIG;
    }
    relation R = {x, d};
    double* sum = (double*)malloc((n ? n : 1) * sizeof(double));
    for (uint64_t i = 0; i < n; ++i) sum[i] = coord_sum(&R, i);

    assignment A;
    rc = make_assignment(&R, n, cfg, &A);
    if (rc) {
        free_assignment(&A);
        free(x);
        free(sum);
        return rc;
    }
    const uint64_t P = A.count;
    out->effective_p = P;

    /* split (partition.cpp:253-273): index lists in scan order */
    uint64_t* sizes = (uint64_t*)calloc(P, sizeof(uint64_t));
    for (uint64_t i = 0; i < n; ++i) ++sizes[A.partition_of[i]];
    uint64_t** parts = (uint64_t**)malloc(P * sizeof(uint64_t*));
    uint64_t* fill = (uint64_t*)calloc(P, sizeof(uint64_t));
    for (uint64_t i = 0; i < P; ++i) parts[i] = (uint64_t*)malloc((sizes[i] ? sizes[i] : 1) * sizeof(uint64_t));
    for (uint64_t r = 0; r < n; ++r) {
        uint64_t pos = A.scan_order ? A.scan_order[r] : r;
        uint64_t pi = A.partition_of[pos];
        parts[pi][fill[pi]++] = pos;
    }
    free(fill);

    uint64_t filtered = 0;
    if (cfg->filter == SKY_FILTER_GRID) { /* engine.cpp:150-163, filter.cpp:37-64 */
        uint32_t* ca = (uint32_t*)malloc(d * sizeof(uint32_t));
        uint32_t* cb = (uint32_t*)malloc(d * sizeof(uint32_t));
        uint8_t* keep = (uint8_t*)calloc(P, 1);
        for (uint64_t i = 0; i < P; ++i) {
            if (!sizes[i]) continue;
            decode_grid(i, A.slices, d, cb);
            int dominated = 0;
            for (uint64_t j = 0; j < P && !dominated; ++j) {
                if (!sizes[j]) continue;
                decode_grid(j, A.slices, d, ca);
                if (grid_dominates(ca, cb, d)) dominated = 1;
            }
            keep[i] = !dominated;
        }
        for (uint64_t i = 0; i < P; ++i) {
            if (!keep[i] && sizes[i]) {
                filtered += sizes[i];
                sizes[i] = 0;
            }
        }
        free(ca);
        free(cb);
        free(keep);
    }

    /* representatives (engine.cpp:167-186) */
    uint64_t* reps = NULL;
    uint64_t n_reps = 0;
    int have_reps = cfg->filter == SKY_FILTER_REPRESENTATIVE;
    if (have_reps) {
        uint64_t cap = 0;
        for (uint64_t i = 0; i < P; ++i) cap += sizes[i] < cfg->rep_q ? sizes[i] : cfg->rep_q;
        reps = (uint64_t*)malloc((cap ? cap : 1) * sizeof(uint64_t));
        g_tests = 0;
        if (cfg->rep_selection == SKY_REPS_REGION) {
            /* filter.cpp:91-95: every non-empty partition must be normalized */
            if (!normalized && n > 0) {
                rc = SKY_E_NORMALIZATION;
            } else {
                n_reps = select_reps_region(&R, n, parts, sizes, P, cfg->rep_q, reps);
            }
        } else if (cfg->rep_selection == SKY_REPS_RANDOM) {
            n_reps = select_reps_random(&R, parts, sizes, P, cfg->rep_q, cfg->rep_seed, reps);
        } else {
            n_reps = select_reps_sorted(&R, sum, parts, sizes, P, cfg->rep_q, reps);
        }
        out->tests_reps = g_tests;
        if (rc) {
            for (uint64_t i = 0; i < P; ++i) free(parts[i]);
            free(parts);
            free(sizes);
            free(reps);
            free_assignment(&A);
            free(sum);
            free(x);
            return rc;
        }
    }
    out->n_reps = n_reps;

    /* compute_local_skylines (engine.cpp:41-63) */
    uint64_t** locals = (uint64_t**)malloc(P * sizeof(uint64_t*));
    uint64_t* lsz = (uint64_t*)calloc(P, sizeof(uint64_t));
    g_tests = 0;
    for (uint64_t i = 0; i < P; ++i) {
        locals[i] = (uint64_t*)malloc((sizes[i] ? sizes[i] : 1) * sizeof(uint64_t));
        if (!sizes[i]) continue;
        uint64_t* kept = parts[i];
        uint64_t nk = sizes[i];
        uint64_t* pre = NULL;
        if (have_reps && n_reps > 0) { /* rep_prefilter (filter.cpp:147-159) */
            pre = (uint64_t*)malloc(sizes[i] * sizeof(uint64_t));
            nk = relative_skyline_list(&R, sum, parts[i], sizes[i], reps, n_reps, pre);
            filtered += sizes[i] - nk;
            kept = pre;
        }
        if (A.presorted)
            lsz[i] = sfs_scan(&R, kept, nk, locals[i]); /* sfs_presorted */
        else
            lsz[i] = sfs_list(&R, sum, kept, nk, locals[i]);
        free(pre);
    }
    out->tests_local = g_tests;

    uint64_t U = 0;
    for (uint64_t i = 0; i < P; ++i) U += lsz[i];
    out->union_size = U;
    out->filtered_count = filtered;
    out->local_skyline_sizes = (uint64_t*)malloc((P ? P : 1) * sizeof(uint64_t));
    memcpy(out->local_skyline_sizes, lsz, P * sizeof(uint64_t));

    /* merge (engine.cpp:65-134) */
    g_tests = 0;
    uint64_t* fin = (uint64_t*)malloc((U ? U : 1) * sizeof(uint64_t));
    uint64_t nf = 0;
    if (cfg->merge == SKY_MERGE_SEQUENTIAL) { /* merge_sequential (engine.cpp:65-72) */
        uint64_t* pool = (uint64_t*)malloc((U ? U : 1) * sizeof(uint64_t));
        uint64_t k = 0;
        for (uint64_t i = 0; i < P; ++i)
            for (uint64_t a = 0; a < lsz[i]; ++a) pool[k++] = locals[i][a];
        nf = sfs_list(&R, sum, pool, U, fin);
        free(pool);
    } else { /* merge_noseq (engine.cpp:116-134) + potential_dominators (:74-114) */
        uint64_t* pd = (uint64_t*)malloc((U ? U : 1) * sizeof(uint64_t));
        uint32_t* ci = (uint32_t*)malloc((d ? d : 1) * sizeof(uint32_t));
        uint32_t* cj = (uint32_t*)malloc((d ? d : 1) * sizeof(uint32_t));
        for (uint64_t i = 0; i < P; ++i) {
            if (!lsz[i]) continue;
            uint64_t k = 0;
            if (A.strategy == SKY_GRID) decode_grid(i, A.slices, d, ci);
            for (uint64_t j = 0; j < P; ++j) {
                int add = 0;
                switch (A.strategy) {
                    case SKY_RANDOM:
                    case SKY_ANGULAR: add = j != i; break;
                    case SKY_GRID:
                        if (j != i && lsz[j]) {
                            decode_grid(j, A.slices, d, cj);
                            add = weak_grid_dominates(cj, ci, d);
                        }
                        break;
                    case SKY_SLICED: add = j < i; break;
                }
                if (add)
                    for (uint64_t a = 0; a < lsz[j]; ++a) pd[k++] = locals[j][a];
            }
            nf += relative_skyline_list(&R, sum, locals[i], lsz[i], pd, k, fin + nf);
        }
        free(pd);
        free(ci);
        free(cj);
    }
    out->tests_merge = g_tests;
    out->final_size = nf;
    out->n_ids = nf;
    out->ids = (int64_t*)malloc((nf ? nf : 1) * sizeof(int64_t));
    for (uint64_t i = 0; i < nf; ++i) out->ids[i] = (int64_t)fin[i];
    qsort(out->ids, nf, sizeof(int64_t), cmp_i64);

    free(fin);
    for (uint64_t i = 0; i < P; ++i) {
        free(parts[i]);
        free(locals[i]);
    }
    free(parts);
    free(locals);
    free(lsz);
    free(sizes);
    free(reps);
    free_assignment(&A);
    free(sum);
    free(x);
    return SKY_OK;
}

void oracle_result_free(oracle_result* r) {
    free(r->ids);
    free(r->local_skyline_sizes);
    memset(r, 0, sizeof(*r));
}

uint64_t oracle_bruteforce(const float* pts, uint64_t n, uint32_t d, int64_t* out) {
    double* x = (double*)malloc(((n && d) ? n * d : 1) * sizeof(double));
    for (uint64_t i = 0; i < n * d; ++i) x[i] = (double)pts[i];
    relation R = {x, d};
    uint64_t* idx = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
    uint64_t* o = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
    for (uint64_t i = 0; i < n; ++i) idx[i] = i;
    uint64_t k = bruteforce_list(&R, idx, n, o);
    for (uint64_t i = 0; i < k; ++i) out[i] = (int64_t)o[i];
    free(idx);
    free(o);
    free(x);
    return k;
}

void oracle_relative_skyline(const float* r, uint64_t nr, const float* c, uint64_t nc, uint32_t d,
                             uint8_t* keep) {
    /* One relation holding r then c so ids stay distinct. */
    uint64_t n = nr + nc;
    double* x = (double*)malloc(((n && d) ? n * d : 1) * sizeof(double));
    for (uint64_t i = 0; i < nr * d; ++i) x[i] = (double)r[i];
    for (uint64_t i = 0; i < nc * d; ++i) x[nr * d + i] = (double)c[i];
    relation R = {x, d};
    double* sum = (double*)malloc((n ? n : 1) * sizeof(double));
    for (uint64_t i = 0; i < n; ++i) sum[i] = coord_sum(&R, i);
    uint64_t* ri = (uint64_t*)malloc((nr ? nr : 1) * sizeof(uint64_t));
    uint64_t* cidx = (uint64_t*)malloc((nc ? nc : 1) * sizeof(uint64_t));
    uint64_t* o = (uint64_t*)malloc((nr ? nr : 1) * sizeof(uint64_t));
    for (uint64_t i = 0; i < nr; ++i) ri[i] = i;
    for (uint64_t i = 0; i < nc; ++i) cidx[i] = nr + i;
    uint64_t k = relative_skyline_list(&R, sum, ri, nr, cidx, nc, o);
    memset(keep, 0, nr);
    for (uint64_t i = 0; i < k; ++i) keep[o[i]] = 1;
    free(ri);
    free(cidx);
    free(o);
    free(sum);
    free(x);
}

uint64_t oracle_representatives(const float* pts, uint64_t n, uint32_t d,
                                const uint64_t* partition_of, uint64_t p, uint64_t q,
                                int64_t* out) {
    double* x = (double*)malloc(((n && d) ? n * d : 1) * sizeof(double));
    for (uint64_t i = 0; i < n * d; ++i) x[i] = (double)pts[i];
    relation R = {x, d};
    double* sum = (double*)malloc((n ? n : 1) * sizeof(double));
    for (uint64_t i = 0; i < n; ++i) sum[i] = coord_sum(&R, i);
    uint64_t* sizes = (uint64_t*)calloc(p ? p : 1, sizeof(uint64_t));
    for (uint64_t i = 0; i < n; ++i) ++sizes[partition_of[i]];
    uint64_t** parts = (uint64_t**)malloc((p ? p : 1) * sizeof(uint64_t*));
    uint64_t* fill = (uint64_t*)calloc(p ? p : 1, sizeof(uint64_t));
    for (uint64_t i = 0; i < p; ++i) parts[i] = (uint64_t*)malloc((sizes[i] ? sizes[i] : 1) * sizeof(uint64_t));
    for (uint64_t i = 0; i < n; ++i) parts[partition_of[i]][fill[partition_of[i]]++] = i;
    uint64_t* reps = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
    uint64_t k = select_reps_sorted(&R, sum, parts, sizes, p, q, reps);
    for (uint64_t i = 0; i < k; ++i) out[i] = (int64_t)reps[i];
    for (uint64_t i = 0; i < p; ++i) free(parts[i]);
    free(parts);
    free(fill);
    free(sizes);
    free(reps);
    free(sum);
    free(x);
    return k;
}
