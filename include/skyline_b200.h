/*
 * skyline_b200.h — C ABI of the B200-native two-phase parallel skyline engine.
 *
 * This is the drop-in boundary for the reference engine's hot path
 * (arxiv 2411.14968 artifact, /root/reference/proj). Every entry point below
 * names the reference interface it replaces. Plain pointers and sizes only;
 * no C++ or torch types cross this boundary.
 *
 *   reference                                   this ABI
 *   ------------------------------------------  --------------------------------
 *   skyline::run            engine.hpp:88        sky_run
 *   skyline::EngineConfig   engine.hpp:30-38     sky_config
 *   skyline::PartitionConfig partition.hpp:21-27 sky_config.{strategy,p,m,seed,slice_dim}
 *   skyline::RunResult/PhaseMetrics engine.hpp:40-57  sky_result
 *   skyline::make_assignment partition.hpp:102   sky_assign
 *   skyline::snap_slices    partition.hpp:99     sky_snap_slices
 *   skyline::relative_skyline core.hpp:79        sky_relative_skyline
 *   skyline::sfs / skyline_bruteforce            sky_skyline
 *     (sequential.hpp:29, core.hpp:75)
 *   skyline::select_representatives_sorted +     sky_representatives
 *     prune_dominated_reps (filter.hpp:46,67)
 *   exception taxonomy core.hpp:13-34            sky_status codes
 *
 * Coordinates are float32, row-major n x d, ids are 0-based row indices
 * (core.cpp:43). The reference stores doubles; float32 -> double is exact,
 * so every comparison made here is the comparison the reference makes on the
 * upcast input.
 */
#ifndef SKYLINE_B200_H
#define SKYLINE_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define SKY_API __attribute__((visibility("default")))
#else
#define SKY_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define SKY_ABI_VERSION 3

/* Return codes mirror the reference's exception classes (core.hpp:13-34). */
typedef enum sky_status {
    SKY_OK = 0,
    SKY_E_CONFIG = 1,        /* ConfigError        core.hpp:25 */
    SKY_E_DIMENSION = 2,     /* DimensionError     core.hpp:17 */
    SKY_E_NORMALIZATION = 3, /* NormalizationError core.hpp:21 */
    SKY_E_DATA = 4,          /* DataError          core.hpp:29 */
    SKY_E_IO = 5,            /* IoError            core.hpp:32 */
    SKY_E_CUDA = 10,         /* CUDA runtime failure (no reference analogue) */
    SKY_E_NCCL = 11,         /* NCCL failure */
    SKY_E_INTERNAL = 12
} sky_status;

/* Strategy (partition.hpp:14-19). */
enum { SKY_RANDOM = 0, SKY_GRID = 1, SKY_ANGULAR = 2, SKY_SLICED = 3 };
/* FilterKind (engine.hpp:19-23). */
enum { SKY_FILTER_NONE = 0, SKY_FILTER_GRID = 1, SKY_FILTER_REPRESENTATIVE = 2 };
/* RepSelection (filter.hpp:21-25): Sorted (filter.cpp:66-86), Region
 * (filter.cpp:88-115; needs a normalized dataset), Random (filter.cpp:117-137;
 * per-partition Rng seeded from sky_config.seed). */
enum { SKY_REPS_SORTED = 0, SKY_REPS_REGION = 1, SKY_REPS_RANDOM = 2 };
/* MergeKind (engine.hpp:25-28). */
enum { SKY_MERGE_SEQUENTIAL = 0, SKY_MERGE_NOSEQ = 1 };
/* Local algorithm (new: the reference has SFS only). */
enum { SKY_LOCAL_SFS = 0, SKY_LOCAL_BNL = 1 };

typedef struct sky_config {
    /* PartitionConfig (partition.hpp:21-27) */
    int32_t strategy;
    uint64_t p;          /* target partition count */
    uint64_t m;          /* slices per dimension (grid/angular); 0 = snap from p */
    uint64_t seed;       /* random partitioning seed */
    uint64_t slice_dim;  /* sliced only */
    /* EngineConfig (engine.hpp:30-38) */
    int32_t filter;
    int32_t rep_selection;
    uint64_t rep_q;      /* default 5 (engine.hpp:34) */
    int32_t merge;
    uint64_t workers;    /* kept for validation parity (engine.cpp:20); must be >= 1 */
    /* B200 extensions */
    int32_t local_algo;       /* SKY_LOCAL_SFS | SKY_LOCAL_BNL */
    uint32_t bnl_window_cap;  /* BNL window capacity in points (0 -> 4096) */
    int32_t count_tests;      /* nonzero: kernels count dominance tests */
    /* EngineConfig::seed (engine.hpp:37): Random representative selection
     * (filter.cpp:117-137); PartitionConfig::seed above drives the random
     * partitioner. The reference CLI sets both from --seed (cli.cpp:177-184). */
    uint64_t rep_seed;
} sky_config;

/* RunResult + PhaseMetrics (engine.hpp:40-57). Owned by the library until
 * sky_result_free: `ids` comes from the library's own pool (do not free() it,
 * do not hand it to sky_free). */
typedef struct sky_result {
    int64_t* ids;               /* skyline ids, ascending (engine.cpp:132) */
    uint64_t n_ids;
    uint64_t effective_p;       /* RunResult::effective_p */
    uint64_t input_size, input_dim;
    uint64_t union_size;        /* PhaseMetrics::union_size */
    uint64_t filtered_count;    /* PhaseMetrics::filtered_count */
    uint64_t final_size;        /* PhaseMetrics::final_size */
    uint64_t* local_skyline_sizes; /* [effective_p] */
    double partition_ms, local_ms, merge_ms; /* device-timed phase durations */
    double total_ms;            /* device time of the whole run */
    uint64_t tests_reps, tests_local, tests_merge; /* executed dominance tests */
    uint64_t n_reps;            /* representatives after pruning */
    uint64_t angular_host_fixups; /* points whose angular slice sat on a boundary */
    uint64_t h2d_bytes, d2h_bytes;
    uint32_t kernel_launches;   /* kernels this library launched for the run */
    uint32_t dom_launches;      /* dominance-kernel (k_relsky/k_bnl) launches */
    double dom_kernel_ms;       /* summed CUDA-event time of those launches (option kernel_events = 1, else 0) */
    uint64_t dom_tests;         /* dominance tests they executed */
    uint64_t dom_exact_checks;  /* pairs the packed codes could not rule out */
    uint64_t exact_checks_merge;
    /* HBM streaming passes (prep, representative prefilter, candidate pass) */
    uint32_t stream_launches;
    double stream_kernel_ms;    /* summed CUDA-event time of those launches (option kernel_events = 1, else 0) */
    uint64_t stream_bytes;      /* algorithmic bytes they move (reads + writes) */
    /* multi-GPU (ABI v3) */
    uint32_t world;             /* ranks that computed the result (1: one GPU) */
    uint32_t sharded;           /* 1: rows sharded over the ranks (phase 1 per shard) */
    uint64_t exchange_bytes;    /* bytes this rank sent to its peers */
    uint64_t local_rows;        /* input rows this rank partitioned / filtered */
} sky_result;

typedef struct sky_ctx sky_ctx;

/* Context: one CUDA device, one stream, a grow-only device arena and pinned
 * staging buffers. One call in flight per context. */
SKY_API int sky_ctx_create(int device, sky_ctx** out);
SKY_API void sky_ctx_destroy(sky_ctx* ctx);
/* Multi-GPU: one rank per process. Rank 0 creates the NCCL unique id
 * (128 bytes), every rank passes it with (rank, world); sky_run on such a
 * context shards the local and merge phases over the ranks and returns the
 * full result on every rank (parallel_for fan-out of parallel.cpp:11-43
 * replaced by NCCL over NVLink). */
SKY_API int sky_nccl_unique_id(uint8_t* out, uint64_t size);
SKY_API int sky_ctx_create_dist(int device, int rank, int world, const uint8_t* unique_id, sky_ctx** out);
/* One process driving several GPUs: the reference's single run() call whose
 * phases fan out over `workers` threads (engine.hpp:30-38,88; parallel.cpp:
 * 11-43) becomes one host thread and one stream per GPU. Rank r runs on
 * devices[r]; sky_run on the group shards the input rows over the ranks
 * and returns the full result. Exchanges use NCCL (ncclCommInitAll) unless
 * SKY_GROUP_LOOPBACK is set or a device repeats: then the ranks exchange by
 * event-ordered device copies (every rank may share one GPU). */
enum { SKY_GROUP_LOOPBACK = 1 };
SKY_API int sky_ctx_create_group(const int* devices, int n, int flags, sky_ctx** out);
/* n rank contexts (rank r on devices[r]) of ONE process that exchange by
 * event-ordered device copies: each is used like a sky_ctx_create_dist
 * context from its own host thread (sky_run / sky_run_shard called
 * concurrently by the n threads). Devices may repeat. out[n]. */
SKY_API int sky_ctx_create_peers(const int* devices, int n, sky_ctx** out);
/* CUDA devices visible to this process (0 when none). */
SKY_API int sky_device_count(void);
/* (rank, world) of a context; a group context reports (0, number of GPUs). */
SKY_API int sky_ctx_world(const sky_ctx* ctx, int* rank, int* world);
/* Take the sharded multi-rank path even on a one-rank context (1 = on).
 * Results never depend on it; tests use it to run the exchange code on one
 * GPU. */
SKY_API int sky_ctx_set_sharded(sky_ctx* ctx, int on);
/* Engine options, per context (defaults are the measured best; none changes
 * a result): "stream" (-1 auto, 0 off, 1 on: the large-input path that
 * skips the full partition sort), "host_merge" (1: host-planned all-pairs
 * merge), "cap_sync" (-1 auto, 0/1: size the filtered set by the input /
 * by the exact count), "sfs_tile", "sfs_chunk", "sfs_head", "merge_tile",
 * "merge_head", "grain_items" (work granularity), "bnl_block" (rows per
 * BNL block, one CTA each; 0 = one CTA per partition), "merge_index" (1:
 * merge through a cell index of the union), "merge_cell_rows" (its target
 * rows per cell), "range_par" (ranges per work item from which each warp
 * takes whole comparator ranges; 0 = never), "profile_host",
 * "timeline" (diagnostics on stderr). SKY_E_CONFIG for an unknown name. */
SKY_API int sky_ctx_set_option(sky_ctx* ctx, const char* name, int64_t value);
SKY_API const char* sky_last_error(const sky_ctx* ctx);
/* Optional external stream (cudaStream_t passed as void*); NULL restores the
 * context's own stream. */
SKY_API int sky_ctx_set_stream(sky_ctx* ctx, void* stream);

SKY_API void sky_config_default(sky_config* cfg);

/* skyline::run (engine.hpp:88). `points` is a host pointer when
 * points_on_device == 0 (copied H2D inside the call) or a device pointer on
 * the context's device otherwise. */
SKY_API int sky_run(sky_ctx* ctx, const float* points, uint64_t n, uint32_t d,
            int normalized, int points_on_device, const sky_config* cfg,
            sky_result* out);
/* skyline::run on FP64 rows (the reference's Dataset coordinates, any
 * finite double): identical results to the reference for every input.
 * Keys, codes and coarse tests run on the rows' float32 image; every
 * dominance decision, partition id, sum and sort order that decides the
 * result is taken on the doubles (core.hpp:89-107, partition.cpp). */
SKY_API int sky_run_f64(sky_ctx* ctx, const double* points, uint64_t n, uint32_t d,
            int normalized, int points_on_device, const sky_config* cfg,
            sky_result* out);
/* skyline::run over a relation whose rows are sharded across the ranks of a
 * distributed context (one process per GPU): this rank holds `n_local`
 * consecutive rows; rank 0's rows come first, then rank 1's, ... (ids are
 * positions in that concatenation). Every rank calls it; every rank
 * receives the full result. On a one-rank context it is sky_run. */
SKY_API int sky_run_shard(sky_ctx* ctx, const float* points, uint64_t n_local, uint32_t d,
            int normalized, int points_on_device, const sky_config* cfg,
            sky_result* out);
SKY_API void sky_result_free(sky_result* r);

/* skyline::make_assignment (partition.hpp:102-103): partition_of[n] on the
 * host, effective partition count in *effective_p. */
SKY_API int sky_assign(sky_ctx* ctx, const float* points, uint64_t n, uint32_t d,
               int normalized, const sky_config* cfg, uint64_t* partition_of,
               uint64_t* effective_p);

/* skyline::snap_slices (partition.hpp:99). Host only. */
SKY_API int sky_snap_slices(uint64_t target_p, uint64_t k, uint64_t* out_m);

/* skyline::relative_skyline (core.hpp:79): keep[i] = 1 iff no row of c
 * dominates row i of r. Host arrays. */
SKY_API int sky_relative_skyline(sky_ctx* ctx, const float* r, uint64_t nr,
                         const float* c, uint64_t nc, uint32_t d,
                         uint8_t* keep, uint64_t* tests);

/* skyline::sfs / skyline_bruteforce (sequential.hpp:29, core.hpp:75): the
 * skyline ids of one relation, ascending. *out_ids is malloc'ed; free with
 * sky_free. */
SKY_API int sky_skyline(sky_ctx* ctx, const float* points, uint64_t n, uint32_t d,
                int64_t** out_ids, uint64_t* n_out, uint64_t* tests);

/* select_representatives_sorted + prune_dominated_reps (filter.cpp:66-86,
 * 139-145) over the partitions given by partition_of: rep ids ascending. */
SKY_API int sky_representatives(sky_ctx* ctx, const float* points, uint64_t n,
                        uint32_t d, const uint64_t* partition_of, uint64_t p,
                        uint64_t q, int64_t** out_ids, uint64_t* n_out);

SKY_API void sky_free(void* ptr);

/* Host-side synthetic generators for the five BASELINE configs (not part of
 * the reference API; used by bench and tests). kind: 1 uniform, 2/4
 * anticorrelated (s~N(0.5,0.0625) + rejection), 3 correlated, 5 ints [0,16).
 * Deterministic for (kind, n, d, seed) regardless of thread count. */
SKY_API int sky_generate(int kind, uint64_t n, uint32_t d, uint64_t seed, float* out);
/* The same rows generated on the context's device (dev_out: n*d floats of
 * device memory): chunk c's mt19937_64 stream in one CTA, rows consumed in
 * stream order (the rejection loop of kinds 2/4 by a warp testing 32
 * attempts per step). Integer-only kinds 1 and 5 equal sky_generate bit for
 * bit; kinds 2-4 use CUDA's log / cos in the normals and equal it wherever
 * those round like the host libm (every BASELINE config at full size, see
 * tests/test_generate_gpu.py). */
SKY_API int sky_generate_device(sky_ctx* ctx, int kind, uint64_t n, uint32_t d, uint64_t seed, float* dev_out);

/* ---- Data in and out (datagen.hpp / io.hpp of the reference) ------------ */
/* Distribution (datagen.hpp:12-16). */
enum { SKY_DIST_UNIFORM = 0, SKY_DIST_CORRELATED = 1, SKY_DIST_ANTICORRELATED = 2 };
/* skyline::generate (datagen.cpp:127-151): n rows of d doubles, normalized,
 * bit-identical to the reference for (dist, n, d, seed). out[n*d]. */
SKY_API int sky_generate_family(int dist, uint64_t n, uint32_t d, uint64_t seed, double* out);
/* skyline::normalize (datagen.cpp:153-168): column min-max to [0,1] in place. */
SKY_API int sky_normalize(double* rows, uint64_t n, uint32_t d);
/* skyline::ingest_csv (datagen.cpp:170-218): header row, selected columns in
 * the given order (all when n_columns == 0), maximize[j] != 0 negates column
 * j (Direction::Max), rows with a missing or non-numeric value dropped, then
 * column min-max normalisation. *rows is malloc'ed (free with sky_free).
 * Errors: SKY_E_IO (cannot open), SKY_E_DATA (empty / no usable rows),
 * SKY_E_CONFIG (unknown column, direction count); text in sky_host_error(). */
SKY_API int sky_ingest_csv(const char* path, const char* const* columns, uint32_t n_columns,
                   const uint8_t* maximize, uint32_t n_maximize, double** rows,
                   uint64_t* n, uint32_t* d);
/* skyline::write_csv (datagen.cpp:220-238): header d0..d{d-1}, shortest
 * round-trip doubles. */
SKY_API int sky_write_csv(const char* path, const double* rows, uint64_t n, uint32_t d);
/* Message of the last failed host-only call on this thread. */
SKY_API const char* sky_host_error(void);

/* Multi-rank planning helpers (host-only, pure functions; used by the
 * NCCL path and by the gloo tests). Longest-processing-time assignment of
 * `count` weighted units to `ranks` owners; owner[count]. */
SKY_API int sky_plan_lpt(const uint64_t* weights, uint64_t count, int ranks, int32_t* owner);
/* Balanced contiguous split of `count` candidates with per-candidate cost
 * prefix sums: bounds[ranks+1]. */
SKY_API int sky_plan_split(const uint64_t* cost_prefix, uint64_t count, int ranks, uint64_t* bounds);
/* The shard plans sky_run uses on a multi-rank context: local phase =
 * contiguous partition ranges of the filtered set (offsets off[P+1]),
 * merge phase = contiguous candidate-partition ranges of the union
 * (offsets offu[P+1]); bounds[world+1]. m = slices per dimension (grid). */
SKY_API int sky_plan_local_shards(const uint32_t* off, uint64_t P, int world, uint32_t* bounds);
SKY_API int sky_plan_merge_shards(const uint32_t* offu, uint64_t P, int world, const sky_config* cfg,
                                  uint32_t d, uint64_t m, uint32_t* bounds);

/* Measured issue peak of the dominance core: the packed-code test loop of
 * the merge/SFS kernel alone (codes in registers and shared memory, 4
 * comparators x K candidates per step, no exit) on every SM of the
 * context's device: K candidates per thread (1, 2, 4, 8), ctas_per_sm CTAs
 * of 256 threads per SM, `iters` passes over 32 comparators per thread.
 * k == 0: the best over K in {4, 8} and 2..8 CTAs per SM. *tests_per_s:
 * pair tests per second (the dominance roofline denominator); d <= 16. */
SKY_API int sky_issue_peak(sky_ctx* ctx, uint32_t d, int k, int ctas_per_sm, uint32_t iters,
                           double* tests_per_s);

SKY_API int sky_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* SKYLINE_B200_H */
