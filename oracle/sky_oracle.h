/*
 * sky_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, single-threaded restatement of the reference engine's hot path
 * (/root/reference/proj/src/{core,sequential,partition,filter,engine}.cpp,
 * include/skyline/rng.hpp). Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it, and only as
 * the checker. The product path (paper_2411_14968_b200) never calls it.
 *
 * Parity pinned: tests/test_oracle.py checks this restatement against the
 * reference itself (oracle/_ref/libskyref.so, built from /root/reference by
 * oracle/Makefile) and against tests/golden/ fixtures generated from that
 * library by tests/golden/make_golden.py.
 */
#ifndef SKY_ORACLE_H
#define SKY_ORACLE_H

#include <stdint.h>
#include "../include/skyline_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct oracle_result {
    int64_t* ids;
    uint64_t n_ids;
    uint64_t effective_p;
    uint64_t union_size, filtered_count, final_size, n_reps;
    uint64_t* local_skyline_sizes;
    uint64_t tests_reps, tests_local, tests_merge;
} oracle_result;

/* skyline::run (engine.cpp:136-204) on float32 rows upcast to double.
 * Returns a sky_status code. */
int oracle_run(const float* pts, uint64_t n, uint32_t d, int normalized,
               const sky_config* cfg, oracle_result* out);
/* the same on FP64 rows (the reference's own coordinate type) */
int oracle_run_f64(const double* pts, uint64_t n, uint32_t d, int normalized,
                   const sky_config* cfg, oracle_result* out);
void oracle_result_free(oracle_result* r);

/* make_assignment (partition.cpp:233-251): partition_of[n], *count. */
int oracle_assign(const float* pts, uint64_t n, uint32_t d, int normalized,
                  const sky_config* cfg, uint64_t* partition_of, uint64_t* count);

/* skyline_bruteforce (core.cpp:56-73): ids ascending into out (capacity n). */
uint64_t oracle_bruteforce(const float* pts, uint64_t n, uint32_t d, int64_t* out);

/* relative_skyline (core.cpp:75-110): keep[i] for rows of r. */
void oracle_relative_skyline(const float* r, uint64_t nr, const float* c,
                             uint64_t nc, uint32_t d, uint8_t* keep);

/* snap_slices (partition.cpp:220-231). */
uint64_t oracle_snap_slices(uint64_t target_p, uint64_t k);

/* angular_index / grid_index of one point (partition.cpp:66-75,135-148). */
uint64_t oracle_angular_index(const float* x, uint32_t d, uint64_t m);
uint64_t oracle_grid_index(const float* x, uint32_t d, uint64_t m);

/* Rng (rng.hpp:15-51): mt19937_64 stream helpers for tests. */
void oracle_random_permutation(uint64_t n, uint64_t seed, uint64_t* perm);

/* select_representatives_sorted + prune (filter.cpp:66-86,139-145) with the
 * partitions given by partition_of; rep ids ascending into out. */
uint64_t oracle_representatives(const float* pts, uint64_t n, uint32_t d,
                                const uint64_t* partition_of, uint64_t p,
                                uint64_t q, int64_t* out);

#ifdef __cplusplus
}
#endif
#endif
