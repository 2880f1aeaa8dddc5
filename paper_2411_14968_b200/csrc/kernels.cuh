// kernels.cuh — launch wrappers for the sm_100a kernels (kernels.cu).
#pragma once

#include "common.cuh"

namespace sky {

// Internal dimensionality: d is padded with zero coordinates up to one of
// the instantiated widths (zeros never change a dominance outcome).
int padded_dim(uint32_t d);
// cached cudaFuncSetAttribute(MaxDynamicSharedMemorySize) / occupancy query
void ensure_smem_attr(const void* func, size_t smem);
int occupancy_cached(const void* func, int threads, size_t smem);  // 0 if unsupported (d > 32)
int device_sm_count();  // SMs of the current device (cached per device)

// Point set on the device in dominance-friendly layout: AoS coords with
// stride round4(D) floats (16-byte aligned rows), plus the 32-bit sort key
// (float32 image of the FP64 coordinate sum, monotone) and the input row id.
struct DevSet {
    float* xyz = nullptr;
    uint32_t* skey = nullptr;
    uint32_t* id = nullptr;
    uint2* qc = nullptr;  // packed monotone codes, two words (D <= 16), optional
    uint32_t n = 0;
};

// FP64 input (sky_run_f64): the engine keeps a float32 image of the rows for
// its layout, keys, codes and coarse tests (round-to-nearest is monotone, so
// s <= t implies rn(s) <= rn(t)), and confirms every dominance that survives
// the float test on the original doubles of the two rows.
struct X64 {
    const double* x = nullptr;  // row-major n x d input, or null (float input)
    uint32_t d = 0;
};
#ifdef __CUDACC__
// dominates_raw (core.hpp:89-96) on the original FP64 rows rs, rt.
__device__ __forceinline__ bool dom64(const X64& e, uint32_t rs, uint32_t rt) {
    const double* s = e.x + (size_t)rs * e.d;
    const double* t = e.x + (size_t)rt * e.d;
    bool lt = false;
    for (uint32_t j = 0; j < e.d; ++j) {
        const double a = s[j], b = t[j];
        if (a > b) return false;
        lt |= a < b;
    }
    return lt;
}
#endif

struct PrepArgs {
    const float* pts;
    const double* pts64;     // FP64 input (validation, sums and partition ids from the doubles)
    uint32_t n, d;
    int strategy;
    uint64_t m;
    int normalized;
    const uint32_t* pid_in;  // random: host-computed partition_of
    uint32_t slice_dim;
    uint64_t* key64;         // out: (pid << 32) | skey
    uint32_t* idx;           // out: identity
    uint32_t* slice_key;     // out (sliced): canonical bits of x[slice_dim]
    uint32_t* err;           // out: error bits
    uint32_t* amb_count;     // out (angular): rows whose slice the device cannot decide
    uint32_t* amb_list;
    uint32_t amb_cap;
    uint32_t key_shift;      // low bits of skey cleared (the partition sort skips them)
    uint32_t* gmin = nullptr;  // out (optional, streamed prep): per-CTA minimum key of each partition
    uint32_t P = 0;
    // angular, m <= 8: tan^2(k*pi/(2m)) for k = 1..m-1 (slice boundaries as
    // tangent ratios); tan2[0] == 0 means "not set" (atan2 filter instead)
    float tan2[8] = {};
    // rows [0, n) of this launch are rows row_base + [0, n) of the input
    // (pts already points at row row_base): outputs are indexed globally
    uint32_t row_base = 0;
    // angular: exact slice thresholds (angular_thresholds), one double4
    // (tan(pred(phi*_k)) hi/lo, tan(phi*_k) hi/lo) per interior boundary
    // k = 1..m-1; null -> FP64 atan2 with an ambiguity band (host libm)
    const double4* ang_thr = nullptr;
    double ang_c45 = 0.0;    // the host libm's atan2(x, x) (the y == x tie)
};
// sm_count > 0: persistent streamed prep when the rows allow it (float,
// aligned); required when a.gmin is set (grid = prep_stream_grid chunks)
void launch_prep(const PrepArgs& a, cudaStream_t st, int sm_count = 0);
uint32_t prep_stream_grid(uint32_t n, uint32_t d, uint32_t P, int sm_count, int strategy);

// Partition boundaries of a (pid << 32 | skey)-sorted key array: off[P+1].
void launch_seg_offsets(const uint64_t* key64, uint32_t n, uint32_t P, uint32_t* off, cudaStream_t st);
// sorted survivor keys of launch_prefilter_append -> key64, rows, offsets[P+1]
void launch_unpack_survivors(const uint64_t* comp, uint32_t n, uint32_t row_bits, uint32_t key_shift, uint32_t P,
                             uint64_t* key64, uint32_t* idx, uint32_t* off, cudaStream_t st);

// Exact angular slicing (partition.cpp:118-148). For an interior boundary
// k = 1..m-1 let phi*_k be the smallest double phi with
// (size_t)(2.0 * phi / pi * m) >= k (the reference's own arithmetic). The
// host libm's atan2 is faithful (error < 1 ulp), so the reference's slice is
// decided by the exact angle alone unless it lies strictly between
// pred(phi*_k) and phi*_k. Per boundary the table holds tan(pred(phi*_k)) and
// tan(phi*_k) as double-doubles (from quad precision); the device compares
// y = sqrt(tail) against x * tan(.) with an exact product. Returns the
// number of entries written (m - 1); m <= kAngularExactMaxM.
constexpr uint64_t kAngularExactMaxM = 65536;
uint64_t angular_thresholds(uint64_t m, double4* out);

// Rows (global index list) gathered as doubles for a host fix-up.
void launch_gather_rows_f64(const float* pts, const double* pts64, uint32_t d, const uint32_t* rows,
                            uint32_t count, uint32_t row_base, double* out, cudaStream_t st);

// Patch pid bits of key64 for rows listed in (rows, pids).
void launch_patch_pid(uint64_t* key64, const uint32_t* rows, const uint32_t* pids, uint32_t count,
                      cudaStream_t st);

// Sliced: pid of each row from its rank in the (x[k], lex, id) order.
//   rank_idx: rows sorted by x[k] (ties by row id); run list: tie runs that
//   straddle slice boundaries, resolved by exact lexicographic rank.
void launch_slice_runs(const uint32_t* sorted_key, uint32_t n, uint64_t p, uint32_t* runs,
                       uint32_t* run_count, uint32_t run_cap, cudaStream_t st);
void launch_slice_assign(const uint32_t* rank_idx, uint32_t n, uint64_t p, uint64_t* key64,
                         cudaStream_t st);
void launch_slice_fix_runs(const float* pts, uint32_t d, const uint32_t* rank_idx, uint32_t n, uint64_t p,
                           const uint32_t* runs, uint32_t n_runs, uint32_t max_len, uint64_t* key64,
                           cudaStream_t st);
void launch_gather_coord_key(const float* pts, uint32_t d, uint32_t j, const uint32_t* idx, uint32_t n,
                             uint32_t* key, cudaStream_t st);
void launch_gather_coord_key64(const double* pts, uint32_t d, uint32_t j, const uint32_t* idx, uint32_t n,
                               uint64_t* key, cudaStream_t st);
// float32 image (round to nearest) of FP64 rows
void launch_round_rows(const double* in, size_t count, float* out, cudaStream_t st);

// Exact top-q per partition under (FP64 sum, lex coords, id) (filter.cpp:66-86).
// region / random representatives (filter.cpp:88-137)
void launch_row_pid(const uint64_t* key64, const uint32_t* idx, uint32_t n, uint32_t* pid_row, cudaStream_t st);
void launch_region_keys(const float* pts, const double* pts64, uint32_t d, uint32_t n, uint64_t* key, uint32_t* row,
                        cudaStream_t st);
void launch_iota(uint32_t n, uint32_t* out, cudaStream_t st);
void launch_gather_u32(const uint32_t* src, const uint32_t* idx, uint32_t n, uint32_t* out, cudaStream_t st);
void launch_pick_first(const uint32_t* rows, const uint32_t* off, uint32_t P, uint32_t q, uint32_t* cand,
                       cudaStream_t st);
void launch_pick_gather(const uint32_t* rows, const uint32_t* gpos, uint32_t slots, uint32_t* cand, cudaStream_t st);
// off_end (optional): partition p spans [off[p], off_end[p]) instead of [off[p], off[p+1])
void launch_rep_pick(const uint64_t* key64, const uint32_t* idx, const uint32_t* off, uint32_t P,
                     const float* pts, const double* pts64, uint32_t d, uint32_t q, uint32_t* cand, cudaStream_t st,
                     const uint32_t* off_end = nullptr);
// stream path (representative filter over large inputs): candidate bucket slots per partition
constexpr uint32_t kRepBucket = 1024;
constexpr uint32_t kRepBucketBig = 8192;  // bucket slots of the retry after an overflow (shared memory bound)
// Stream path of the sorted representatives (select_representatives_sorted,
// filter.cpp:66-86): per-partition key bound = q-th smallest of the prep
// CTAs' minima gmin[P][G] -> rows under the bound in B-slot buckets (overflow
// flag set if one fills) -> each bucket sorted, first q picked exactly into
// cand[p * q + k] (kNone when the partition has fewer rows).
void launch_rep_candidates(const uint64_t* key64, uint32_t n, uint32_t P, uint32_t q, uint32_t G,
                           const uint32_t* gmin, uint32_t* thr, uint32_t B, uint32_t* cnt, uint64_t* bkey,
                           uint32_t* brow, const float* pts, uint32_t d, uint32_t* cand, uint32_t* overflow,
                           cudaStream_t st, cudaEvent_t pass_begin = nullptr, cudaEvent_t pass_end = nullptr);

// Representative finish on the device (<= 2048 picks): key-sorted antichain
// into `out`, count in *out_count. false: too many picks (host path).
bool launch_rep_finalize(int D, const uint32_t* cand, uint32_t slots, const float* pts, uint32_t d, DevSet out,
                         uint32_t* out_count, unsigned long long* tests, X64 x64, int smem_optin, cudaStream_t st);

// The same finish in three launches spread over the GPU (scratch:
// rep_finalize_scratch_bytes(D)). false: not applicable (use the above).
bool launch_rep_finalize_par(int D, const uint32_t* cand, uint32_t slots, const float* pts, uint32_t d, DevSet out,
                             uint32_t* out_count, unsigned long long* tests, X64 x64, int smem_optin, int sm_count,
                             void* scratch, cudaStream_t st);
size_t rep_finalize_scratch_bytes(int D);

// Compaction plumbing.
void launch_scatter_direct(int D, const DevSet& in, const uint8_t* dead, const uint32_t* pos, DevSet out,
                           cudaStream_t st);
void launch_scatter_indirect(int D, const float* pts, uint32_t d, const uint32_t* idx, const uint64_t* key64,
                             uint32_t n, const uint8_t* dead, const uint32_t* pos, DevSet out, cudaStream_t st);
void launch_gather_rows(int D, const float* pts, const double* pts64, uint32_t d, const uint32_t* rows, uint32_t n,
                        DevSet out, cudaStream_t st);
// out[i] = in[perm[i]] for i < in.n (or < *n_dev when given)
void launch_gather_set(int D, const DevSet& in, const uint32_t* perm, DevSet out, cudaStream_t st,
                       const uint32_t* n_dev = nullptr);
// stable merge of the key-sorted runs off[P+1] of `in` into `out` (key order)
// (n_dev: live count on the device, in.n the capacity)
void launch_merge_runs(int D, const DevSet& in, const uint32_t* off, uint32_t P, DevSet out, cudaStream_t st,
                       const uint32_t* n_dev = nullptr);
// ascending ids (< n_ids) of the live entries of id[n] via a bitmap; count in *total
uint32_t bm_blocks(uint32_t n_ids);
void launch_ids_bitmap(const uint32_t* id, const uint8_t* dead, uint32_t n, uint32_t n_ids, uint32_t* bm,
                       uint32_t* block_tot, uint32_t* out, uint32_t* total, cudaStream_t st,
                       const uint32_t* n_dev = nullptr);
void launch_remap_offsets(const uint32_t* off_old, uint32_t P, const uint32_t* pos, const uint8_t* dead,
                          uint32_t n, uint32_t* off_new, cudaStream_t st);
void launch_count_total(const uint32_t* pos, const uint8_t* dead, uint32_t n, uint32_t* total, cudaStream_t st);
void launch_compact_ids(const uint32_t* id, const uint8_t* dead, const uint32_t* pos, uint32_t n, uint32_t* out,
                        cudaStream_t st);
void launch_fill_u8(uint8_t* p, uint8_t v, size_t n, cudaStream_t st);
// p[i] = v for *count <= i < cap (the unused tail of a set sized by capacity)
void launch_fill_tail_u8(uint8_t* p, uint8_t v, const uint32_t* count, uint32_t cap, cudaStream_t st);
void launch_fill_live_u8(uint8_t* p, const uint32_t* count, uint32_t cap, cudaStream_t st);
// out[pos[i]] = base + i for live i (dense list of live positions)
void launch_compact_pos(const uint8_t* dead, const uint32_t* pos, uint32_t n, uint32_t base, uint32_t* out,
                        cudaStream_t st);
// grid_filter (filter.cpp:37-50) over the P = m^d cells from their row
// offsets: cell_dead[P] and the rows in filtered cells; occ[P] is scratch.
// Returns the number of launches.
uint32_t launch_grid_filter(const uint32_t* off, uint32_t P, uint32_t m, uint32_t d, uint8_t* occ, uint8_t* cell_dead,
                            unsigned long long* filtered_rows, cudaStream_t st);
void launch_mark_cells_dead(const uint64_t* key64, uint32_t n, const uint8_t* cell_dead, uint8_t* dead,
                            cudaStream_t st);

// The dominance core: for each item, candidates [cb,ce) vs every comparator
// range in ranges[lb,le). Sets dead[c] = 1 for each candidate dominated by
// some comparator with skey <= the candidate tile's key bound.
struct RelskyArgs {
    // candidates: direct (AoS DevSet) or indirect (row-major pts via idx)
    const float* cxyz;
    const uint32_t* cskey;   // direct: skey[]; indirect: key64 viewed as u32 pairs
    const uint32_t* cidx;    // indirect only
    uint32_t cd;             // indirect only: row-major stride
    bool indirect;
    const float* sxyz;
    const uint32_t* sskey;
    const Item* items;
    uint32_t n_items;
    const uint2* ranges;
    bool bounded;
    uint8_t* dead;
    unsigned long long* tests;
    X64 x64;                 // FP64 confirmation (rows: cid / cidx, sid)
    const uint32_t* cid;     // direct candidates: row id of each position
    const uint32_t* sid;     // row id of each comparator position
};
void launch_relsky(int D, const RelskyArgs& a, cudaStream_t st);

// ---- packed-code dominance core (kernels_dom.cu), D <= 16 -----------------
// Per-dimension monotone codes q(x) = #{quantile thresholds <= x}: q(s_j) >
// q(t_j) proves s_j > t_j, so a guarded lane-wise subtraction over two packed
// words rules out most non-dominating pairs; pairs that pass are confirmed
// with the exact float test.
constexpr int kCodeLevels = 128;
// thr[D][127]; n_dev: optional device row count (s.n is then an upper bound)
void launch_thresholds(int D, const DevSet& s, float* thr, cudaStream_t st, const uint32_t* n_dev = nullptr);
// fills s.qc; n_dev: optional device-side row count (s.n is then an upper bound)
void launch_encode(int D, const DevSet& s, const float* thr, cudaStream_t st, const uint32_t* n_dev = nullptr);
struct Relsky2Args {
    const uint32_t* cidx;  // optional: item candidate slots index this list of set positions
    const float* cxyz;
    const uint32_t* cskey;
    const uint2* cqc;
    const float* sxyz;
    const uint32_t* sskey;
    const uint2* sqc;
    const Item* items;
    uint32_t n_items;
    const uint2* ranges;
    bool bounded;
    uint8_t* dead;
    unsigned long long* tests;
    uint32_t* counter;   // zeroed work counter (persistent warps fetch items)
    const uint32_t* wcount;  // window lengths for dynamic ranges (y has bit 31 set)
    unsigned long long* coarse_hits;  // optional: exact checks performed
    X64 x64;                  // FP64 confirmation
    const uint32_t* cid;      // row id of each candidate position
    const uint32_t* sid;      // row id of each comparator position
    const uint32_t* n_items_dev;  // optional: item count in device memory (n_items = capacity)
    bool direct;                  // items hold their comparator range itself in (lb, le)
    // many short ranges per item (cell-indexed lists): each warp takes whole
    // ranges (w, w + 8, ...) instead of every 8th batch of each range, so no
    // range is a short burst shared by eight warps
    bool range_par = false;
};
// tile = candidates per item (<= 32 * 8, one warp); picks K from it.
void launch_relsky2(int D, int tile, const Relsky2Args& a, int sm_count, cudaStream_t st);
// tests/s of the packed-code test loop alone (k_issue_peak) on a full grid
double measure_issue_peak(int D, int K, int blocks_per_sm, uint32_t iters, int sm_count, cudaStream_t st,
                          unsigned long long* sink);
// Device-side planning. A job = candidates [cb, ce) of a candidate list x one
// comparator range [lo, hi) (sorted by key). Jobs come from device offsets;
// they expand into direct items: tiles of `tile` candidates x chunks of the
// range (at most max_chunks per job: the chunk grows for longer ranges),
// chunk-major inside a job. Item / job counts are exclusive scans of
// per-job counts (Runner::scan_u32), so every count stays on the device.
struct Job {
    uint32_t cb, ce, lo, hi;
};
// one job per partition: candidates [coff[p], coff[p+1]) vs the comparator
// sub-range [soff[p] + lo, soff[p] + hi) clipped to [soff[p], soff[p+1]) when
// soff is given ("self" lists), else [lo, hi) clipped to [0, *n_comp).
void launch_partition_jobs(const uint32_t* coff, const uint32_t* soff, const uint32_t* n_comp, uint32_t P,
                           uint64_t lo, uint64_t hi, Job* jobs, cudaStream_t st);
// counts[j] = items of job j (0 for j >= *n_jobs), j < cap
void launch_job_counts(const Job* jobs, const uint32_t* n_jobs, uint32_t cap, uint32_t tile, uint32_t chunk,
                       uint32_t max_chunks, uint32_t* counts, cudaStream_t st);
void launch_job_items(const Job* jobs, const uint32_t* n_jobs, uint32_t cap, const uint32_t* prefix, uint32_t tile,
                      uint32_t chunk, uint32_t max_chunks, Item* items, cudaStream_t st);

// jobs + counts + scan + items in one CTA (P <= 1024; false otherwise);
// *n_items = min(items, cap)
// chunk == 0: the chunk is derived on the device from the counts (>= grain_target items)
bool launch_plan_partition_items(const uint32_t* coff, const uint32_t* soff, const uint32_t* n_comp, uint32_t P,
                                 uint64_t lo, uint64_t hi, uint32_t tile, uint32_t chunk, uint32_t max_chunks,
                                 uint32_t cap, Item* items, uint32_t* n_items, cudaStream_t st,
                                 uint32_t grain_target = 0);
// dense list of live entries + remapped segment offsets (off[P+1] sorted)
// in two launches; block_tot: dense_compact_scratch(n) bytes. false: n == 0
// n_dev (optional): entries at or past *n_dev are dead and not read
bool launch_dense_compact(const uint8_t* dead, uint32_t n, const uint32_t* off, uint32_t P, uint32_t base,
                          uint32_t* dense, uint32_t* off_new, uint32_t* total, uint32_t* block_tot,
                          cudaStream_t st, const uint32_t* n_dev = nullptr);
size_t dense_compact_scratch(uint32_t n);

// Items of a relsky wave built on the device from the dense candidate
// offsets of np partitions (dnew[np+1], relative to the dense list) and each
// partition's comparator groups (groups[gb[p]..gb[p+1]) = (lb, le) into the
// wave's range array): tiles of `tile` candidates x groups, group-major.
// *count = items written (<= cap).
void launch_plan_items(const uint32_t* dnew, uint32_t np, const uint32_t* gb, const uint2* groups, uint32_t max_groups,
                       uint32_t tile, Item* items, uint32_t* count, cudaStream_t st);

// BNL local skylines: one CTA per partition segment, window capped at
// `window` points in shared memory; partition input in scan order.
struct BnlArgs {
    const float* xyz;
    const uint32_t* seg_off;  // [P+1]
    uint32_t P;
    uint32_t window;
    uint8_t* dead;            // out: 1 = dominated within its partition
    uint32_t* overflow;       // scratch: n entries
    unsigned long long* tests;
    unsigned long long* hits;  // optional: exact checks performed
    X64 x64;                   // FP64 confirmation
    const uint32_t* id;        // row id of each set position
};
// Largest window <= want whose shared-memory footprint fits smem_optin.
uint32_t bnl_window_fit(int D, uint32_t want, int smem_optin);
void launch_bnl_full(int D, const BnlArgs& a, uint32_t cap, uint32_t grid, uint32_t* win_pos, uint32_t* win_meta,
                     uint32_t* counter, cudaStream_t st);

// Cell index of a set with packed codes: k dimensions (dim[0] the least
// significant digit), dimension t split into 2^bits[t] buckets by the top
// bits of its code (halves or quartiles of the code range).
struct CellSpec {
    uint32_t k = 0;
    uint8_t dim[16] = {};
    uint8_t bits[16] = {};
    uint32_t total_bits() const {
        uint32_t b = 0;
        for (uint32_t t = 0; t < k; ++t) b += bits[t];
        return b;
    }
};
// key[i] = (cell << 32) | skey[i], idx[i] = i
void launch_cell_keys(int D, const uint2* qc, const uint32_t* skey, uint32_t n, const CellSpec& cs, uint64_t* key,
                      uint32_t* idx, cudaStream_t st);

// Rows dense[j] (partitions doff[P+1] over j): key[j] = (partition << (32 +
// K) | cell << 32 | skey), idx[j] = j
void launch_part_cell_keys(int D, const uint2* qc, const uint32_t* skey, const uint32_t* dense, const uint32_t* doff,
                           uint32_t P, uint32_t n, const CellSpec& cs, uint64_t* key, uint32_t* idx, cudaStream_t st);
// dead[rows[i]] |= flag[i]
void launch_scatter_dead(const uint8_t* flag, const uint32_t* rows, uint32_t n, uint8_t* dead, cudaStream_t st);

// The BASELINE synthetic inputs (include/skyline_baseline_gen.h) generated
// on the device, n x d float32 rows into out (kind 1..5); *stuck set if a
// rejection loop outran the stream ring (the caller then uses the host).
void launch_generate_baseline(int kind, uint64_t n, uint32_t d, uint64_t seed, float* out, uint32_t* stuck,
                              cudaStream_t st);

// Partitions off[P+1] cut into blocks of <= `block` rows: sub[cap+1] block
// offsets (empty blocks pad the tail up to cap).
void launch_split_segments(const uint32_t* off, uint32_t P, uint32_t block, uint32_t* sub, uint32_t cap,
                           cudaStream_t st);

// Packed-code BNL (D <= 16): window codes + metadata in shared memory.
uint32_t bnl2_window_fit(int D, uint32_t want, int smem_optin);
void launch_bnl2(int D, const BnlArgs& a, const uint2* qc, const uint32_t* skey, uint32_t cap, uint32_t grid,
                 uint32_t* counter, cudaStream_t st);

// Row-order prefilter that appends the survivors' sort keys
// ((key64[row] >> key_shift) << row_bits | row) to out, count in *count.
struct PrefilterAppend {
    const uint64_t* key64 = nullptr;  // row order (pid << 32 | truncated skey)
    uint64_t* out = nullptr;
    uint32_t* count = nullptr;
    uint32_t key_shift = 0, row_bits = 0;
    uint32_t regroup = 64;  // POSORDER: representatives before the CTA regroups its live rows
    // APPEND: words the pass clears on the way (the fused small tail's flags:
    // no memset between the prefilter and the tail)
    uint32_t* zero = nullptr;
    uint32_t zero_words = 0;
};
// Fused tail of a stream-path run with few prefilter survivors (small.cu).
constexpr uint32_t kSmallCap = 4096;
struct SmallTail {
    const uint64_t* surv = nullptr;  // packed survivor keys (prefilter append order)
    const uint32_t* count = nullptr; // their device count
    const float* pts = nullptr;
    uint32_t d = 0, P = 0, row_bits = 0, key_shift = 0, cap = kSmallCap;
    uint32_t* flags = nullptr;       // 3 x cap words: local dead, dead, rank; zeroed by the launcher unless
    bool flags_zeroed = false;       // the prefilter pass already cleared them (PrefilterAppend::zero)
    uint32_t* cnt = nullptr;         // P words: local skyline size per partition
    uint32_t* u_count = nullptr;     // |union| (device)
    uint32_t* total = nullptr;       // final count (device)
    uint32_t* offu = nullptr;        // P + 1 union offsets per partition (device)
    uint32_t* hid = nullptr;         // final rows ascending (mapped pinned host memory)
    unsigned long long* tests = nullptr;
    // copied into mapped pinned memory by the last kernel (also when it
    // declines): the run's counter words and the union offsets
    const uint32_t* misc = nullptr;  // kSmallMiscWords device words
    uint32_t* hmisc = nullptr;
    uint32_t* hoffu = nullptr;       // P + 1
};
constexpr uint32_t kSmallMiscWords = 32;
// all pairs of survivors (local + global dominance, ranks), then the counts,
// offsets and ascending ids (2 launches; a memset before them unless flags_zeroed)
void launch_small_tail(int D, const SmallTail& t, cudaStream_t st);

// false: not applicable (d > 16, unaligned rows, shared memory)
bool launch_prefilter_append(int D, const float* pts, uint32_t d, uint32_t n, const float* rep_xyz,
                             const uint32_t* rep_key, const uint2* rep_qc, const uint32_t* rep_id, uint32_t nrep,
                             const uint32_t* nrep_dev, const float* thr, const PrefilterAppend& app,
                             unsigned long long* tests, int smem_optin, cudaStream_t st);

// Streaming representative prefilter (false: not applicable, use k_relsky).
// Rows are tested in input order (dead_row), then folded into the sorted
// positions (dead_pos[i] |= dead_row[idx[i]]).
// nrep: host upper bound (shared-memory sizing); nrep_dev: optional device count.
bool launch_prefilter(int D, const float* pts, uint32_t d, const uint32_t* idx, uint32_t n, const float* rep_xyz,
                      const uint32_t* rep_key, const uint2* rep_qc, const uint32_t* rep_id, uint32_t nrep,
                      const uint32_t* nrep_dev, const float* thr, uint8_t* dead_row, uint8_t* dead_pos,
                      unsigned long long* tests, X64 x64, int smem_optin, cudaStream_t st, bool posorder = true);
// Quantization thresholds from a strided sample of row-major input rows.
// gate (optional): the kernel returns at once when *gate < gate_min
void launch_thresholds_rows(int D, const float* pts, uint32_t d, uint32_t n, float* thr, cudaStream_t st,
                            const uint32_t* gate = nullptr, uint32_t gate_min = 0);
// Skyline of one small set in one CTA (false: too big, use k_relsky).
bool launch_small_skyline(int D, const float* xyz, const uint32_t* id, uint32_t n, uint8_t* dead,
                          unsigned long long* tests, X64 x64, int smem_optin, cudaStream_t st);

// Random partitioner (kernels_rand.cu): bit-exact assign_random on the GPU.
size_t random_scratch_bytes(uint32_t n);
size_t random_cub_bytes(uint32_t n);
// jump_table: device copy of mt_jump_table(kJumpLog2, chunks-1) (mtjump.cpp)
// or null for the single-CTA stream.
constexpr uint32_t kJumpLog2 = 14;
inline uint32_t mt_jump_chunks(uint32_t n) { return n < 2 ? 0u : ((n - 1) + (1u << kJumpLog2) - 1) >> kJumpLog2; }
// flag_dev: when given, a rejected draw only sets *flag_dev (no sync; the
// caller checks it later and redoes the run); otherwise the function syncs,
// and returns false on a rejection (nothing written).
bool random_partition_gpu(uint32_t n, uint64_t p, uint64_t seed, uint32_t* pid, void* scratch, void* cub_tmp,
                          size_t cub_bytes, int sm_count, cudaStream_t st, uint32_t* launches,
                          const uint32_t* jump_table = nullptr, uint32_t* flag_dev = nullptr);
// host: jump polynomials t^(k 2^log2_stride) mod phi, k = 1..chunks (mtjump.cpp)
const uint32_t* mt_jump_table(uint32_t log2_stride, uint32_t chunks);
int mt_jump_words();

}  // namespace sky
