// engine_impl.cuh — internal to the engine (engine.cu, shard.cu): the context,
// device-buffer slots, work planning and the Runner that launches the
// kernels of one run on one GPU, plus the phase helpers shared by the
// single-GPU run (engine.cu run_impl) and the sharded multi-GPU run
// (shard.cu run_sharded).
#pragma once

#include <cub/cub.cuh>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <random>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "comm.hpp"
#include "kernels.cuh"

extern "C" int sky_plan_split(const uint64_t* cost_prefix, uint64_t count, int ranks, uint64_t* bounds);

// Engine options (sky_ctx_set_option): the measured defaults, changed per
// context by tests (to force a path) and by the profiling scripts.
struct sky_options {
    int32_t stream = -1;        // stream path (section 3a of DESIGN): -1 inputs > 32 MB, 0 off, 1 on
    int32_t host_merge = 0;     // 1: host-planned all-pairs merge instead of the device-planned one
    int32_t cap_sync = -1;      // filtered-set capacity: -1 exact count above 1M rows, 0 input size, 1 exact
    uint32_t sfs_tile = 0;      // candidates per SFS item (0: from the partition sizes)
    uint32_t sfs_chunk = 2048;  // comparators per SFS item
    uint32_t sfs_head = 2048;   // SFS wave 0: rows tested against the partition's first `head` rows
    int32_t sfs_auto_chunk = 1; // SFS items on sets <= 128k rows: comparator chunk from the device counts
    uint32_t merge_tile = 0;    // candidates per merge item (0: from the union size)
    uint32_t merge_head = 4096; // merge wave 0 length
    uint32_t grain_items = 4;   // work items per resident CTA
    uint32_t bnl_block = 1024;  // BNL: rows per block (one CTA each), 0 = one CTA per partition (512-1024 measured best on config 4)
    int32_t merge_index = 1;    // merge through the cell index of the union (host-planned merges)
    uint32_t merge_cell_rows = 1024;  // target rows per cell of that index
    uint32_t range_par = 4;     // ranges per item from which warps take whole ranges (0: never)
    uint32_t wave_growth = 4;   // multi-wave relative skylines: wave w+1 = growth x wave w comparators
    uint32_t wave_split_mpairs = 8192;  // split the rest into further waves above this many Mi pairs
    int32_t profile_host = 0;   // print host-side planning / wait times
    int32_t timeline = 0;       // an event after every launch, dumped per run
    int32_t small_tail = 1;     // stream path: the fused tail when <= kSmallCap rows survive the prefilter
    int32_t kernel_events = 0;  // CUDA events around the dominance launches and HBM passes (dom_kernel_ms / stream_kernel_ms of
                                // sky_result; off by default: the records between kernels cost 25-55 us per run)
};

struct sky_ctx {
    int device = 0;
    sky_options opt;
    cudaStream_t own = nullptr;
    // side stream for the input copy when it can overlap data-independent
    // work (the random partitioner), with its fork/join events
    cudaStream_t copy = nullptr;
    cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
    cudaEvent_t chunk_ev[4] = {};  // chunked input copy (prep overlaps the copy)
    cudaStream_t stream = nullptr;
    std::string err;
    sky::Arena dev;
    sky::PinnedArena pin;
    int sm_count = 148;
    int smem_optin = 0;
    cudaEvent_t ev[6] = {};
    std::vector<cudaEvent_t> dom_ev;  // (start, end) pairs, one per dominance launch of a run
    uint32_t dom_used = 0;
    std::vector<cudaEvent_t> hbm_ev;  // (start, end) pairs of the HBM streaming passes of a run
    uint32_t hbm_used = 0;
    uint32_t hbm_launches = 0;  // passes of the run (counted with or without their events)
    uint64_t hbm_bytes = 0;
    // pinned staging for async H2D copies: bump-allocated per run, never
    // reused within a run, so no launch has to wait for its copy to drain
    std::vector<std::pair<char*, size_t>> stage;
    size_t stage_cur = 0, stage_off = 0;
    uint32_t launches = 0;
    uint32_t dom_launches = 0;
    uint32_t rep_bucket = sky::kRepBucket;  // candidate bucket slots of the current run (run_impl_retry)
    uint64_t big_bucket_rows = 0;  // row count of the last run that needed the large buckets: runs of that size start with them
    double dom_ms = 0.0;
    // multi-GPU: this context is rank `rank` of `world` (one GPU each); the
    // exchanges go through `comm` (NCCL over NVLink/NVSwitch, or loopback
    // between host threads, comm.hpp). `sharded` forces the sharded run
    // even at world == 1 (tests: the exchange code on one GPU).
    int rank = 0, world = 1;
    std::unique_ptr<sky::Comm> comm;
    bool sharded = false;
    // group context (one process driving several GPUs, sky_ctx_create_group):
    // the per-rank contexts and their worker threads; sky_run fans out
    struct sky_group* group = nullptr;
    // device copy of the mt19937_64 jump polynomials (random partitioner)
    uint32_t* mt_jump = nullptr;
    uint32_t mt_jump_rows = 0;
    // SKY_PROFILE_TIMELINE: an event after every counted launch (host issue
    // time + device completion time), printed when the run drains
    std::vector<cudaEvent_t> tl_ev;
    // host round trips: spin on an event instead of a blocking stream sync
    // (the wake-up of cudaStreamSynchronize costs ~15-20 us per round trip)
    cudaEvent_t sync_ev = nullptr;
    // exact angular slice thresholds (angular_thresholds) for slices ang_m,
    // and the device copy last uploaded
    std::vector<double4> ang_host;
    uint64_t ang_m = 0, ang_dev_m = 0;
    const void* ang_dev_ptr = nullptr;
};


namespace sky {
namespace eng {

// Result id buffers (sky_result::ids). A skyline of hundreds of thousands of
// ids is megabytes: malloc hands such blocks out as fresh mappings, and
// their page faults cost more than the ids' copy (config 4: ~1 ms per run).
// Large blocks go back to a small process-wide pool in sky_result_free and
// are reused by the next run. A 16-byte header in front of the ids holds the
// capacity.
struct IdPool {
    static constexpr size_t kHeader = 16, kPooledFrom = 64 * 1024, kSlots = 4;
    std::mutex mu;
    std::vector<std::pair<char*, size_t>> free_blocks;  // (block, capacity in bytes)
    static IdPool& get() {
        static IdPool* p = new IdPool();  // never destroyed: results may outlive static teardown
        return *p;
    }
    int64_t* alloc(size_t count) {
        const size_t need = std::max<size_t>(count, 1) * sizeof(int64_t);
        if (need >= kPooledFrom) {
            std::lock_guard<std::mutex> lk(mu);
            for (size_t k = 0; k < free_blocks.size(); ++k)
                if (free_blocks[k].second >= need && free_blocks[k].second <= 4 * need) {
                    char* b = free_blocks[k].first;
                    free_blocks.erase(free_blocks.begin() + k);
                    return reinterpret_cast<int64_t*>(b + kHeader);
                }
        }
        char* b = static_cast<char*>(std::malloc(kHeader + need));
        if (!b) throw std::bad_alloc();
        *reinterpret_cast<size_t*>(b) = need;
        return reinterpret_cast<int64_t*>(b + kHeader);
    }
    void release(int64_t* ids) {
        if (!ids) return;
        char* b = reinterpret_cast<char*>(ids) - kHeader;
        const size_t cap = *reinterpret_cast<size_t*>(b);
        if (cap >= kPooledFrom) {
            std::lock_guard<std::mutex> lk(mu);
            if (free_blocks.size() < kSlots) {
                free_blocks.emplace_back(b, cap);
                return;
            }
        }
        std::free(b);
    }
};
inline int64_t* alloc_ids(size_t count) { return IdPool::get().alloc(count); }

enum Slot {
    S_PTS, S_KEY_A, S_KEY_B, S_IDX_A, S_IDX_B, S_SK_A, S_SK_B, S_PID, S_MISC, S_AMB, S_OFF_A, S_OFF_B,
    S_DEAD, S_POS, S_CUB, S_ITEMS, S_RANGES, S_REPCAND, S_REPROWS, S_RUNS,
    S_SET0, S_SET0_K, S_SET0_I, S_SET0_Q, S_SET1, S_SET1_K, S_SET1_I, S_SET1_Q,
    S_SET2, S_SET2_K, S_SET2_I, S_SET2_Q, S_SET3, S_SET3_K, S_SET3_I, S_SET3_Q,
    S_PERM_A, S_PERM_B, S_IDS_A, S_IDS_B, S_CELLDEAD, S_BNL_POS, S_BNL_META,
    S_OVF, S_SKTMP, S_THR, S_RAND, S_OFF_C, S_SIZES, S_GCOUNT, S_PTHR, S_DEADROW, S_DENSE,
    S_SCAN, S_PTS64, S_GROUPS, S_GB, S_JCNT, S_JPRE, S_JOBS, S_DNEW,
    S_ROWPID, S_AMBROWS, S_ANGT, S_RK0, S_RK1, S_RV0, S_RV1, S_RP0, S_RP1, S_GPOS, S_BM, S_BMT, S_GMIN, S_PTHR2, S_BCNT, S_BKEY, S_BROW, S_OBE, S_SURV, S_SURV2, S_REPF, S_DCBT, S_OFFG,
    // sharded multi-GPU run (shard.cu)
    S_SH_SKG, S_SH_IOTA, S_SH_RUNB, S_SH_TAB, S_SH_IDS, S_SH_TABALL, S_SH_IDSALL, S_SH_CANDG, S_SH_CNT,
    S_SH_K64R, S_SH_K64S, S_SH_PERM, S_SH_OFFM, S_SH_FULL, S_BNL_SEG,
    S_SETS, S_SETS_K, S_SETS_I, S_SETS_Q,  // rows sent to their partition owners
    S_SETR, S_SETR_K, S_SETR_I, S_SETR_Q,  // rows received from the other ranks
    S_DEAD2, S_SOFF, S_SH_OFFU, S_OFFM,
    S_SM_W, S_SM_CNT,  // the fused small tail (small.cu)
    S_GRIDOCC, S_GRIDCNT,  // grid filter: occupancy prefix OR, filtered rows
    S_COUNT
};
// pinned slots
enum PSlot { P_PID, P_MISC, P_OFF, P_ITEMS, P_RANGES, P_IDS, P_AMB, P_RUNS, P_PCOUNT, P_SH_CNT, P_SH_RUNS, P_SH_OFF };


constexpr int kTile = 512;          // candidates per relsky item (RS_THREADS * RS_K)
constexpr uint32_t kChunk = 8192;   // comparators per relsky item before bounding
constexpr uint32_t kBlock = 512;    // local block-skyline size
// candidate x comparator pairs (before bounding) below which the remaining
// comparators of a multi-wave relsky run as one last wave
constexpr uint64_t kWaveSplitPairs = 8ull << 30;
// above this many input rows the single-GPU path reads the filtered count
// back before sizing the downstream sets by it; up to it the sets keep the
// input's size as capacity and every pass is bounded by the device count
// (one round trip per run: measured 0.5% faster on config 2, 2.4% on
// config 1, even on config 5's 2M rows)
constexpr uint32_t kExactCapRows = 1u << 20;

// misc device words
enum { M_ERR = 0, M_AMB = 1, M_RUNS = 2, M_TOTAL = 3, M_BNLCTR = 4, M_WORK = 5, M_NREP = 6, M_NITEMS = 7, M_TESTS = 8 /* 4 x u64 */,
       M_HITS = 16 /* 4 x u64, per phase */,
       M_S0 = 24, M_U = 26, M_NP = 27 /* device-side set counts (single-GPU path) */,
       M_RFLAG = 28 /* random partitioner: a draw the reference would reject */,
       M_OVF = 29 /* stream path: a representative candidate bucket overflowed */ };
// the fused small tail writes P + 1 union offsets from one CTA
constexpr uint32_t kSmallMaxParts = 1u << 16;

inline uint64_t checked_pow(uint64_t base, uint64_t e) {  // partition.cpp:15-22
    uint64_t r = 1;
    for (uint64_t i = 0; i < e; ++i) {
        if (r > kMaxPartitions) return kMaxPartitions + 1;
        r *= base;
    }
    return r;
}

inline uint64_t snap_slices(uint64_t target_p, uint64_t k) {  // partition.cpp:220-231
    if (target_p < 1) throw Error(SKY_E_CONFIG, "target partition count must be >= 1");
    if (k < 1) throw Error(SKY_E_CONFIG, "snap exponent must be >= 1");
    uint64_t hi = 1;
    while (checked_pow(hi, k) < target_p && checked_pow(hi, k) <= kMaxPartitions) ++hi;
    if (hi == 1) return 1;
    if (checked_pow(hi, k) < target_p) return hi;
    const uint64_t lo = hi - 1;
    const uint64_t above = checked_pow(hi, k) - target_p;
    const uint64_t below = target_p - checked_pow(lo, k);
    return above < below ? hi : lo;
}

// Rng::below + shuffle (rng.hpp:40-60) with std::mt19937_64, the engine the
// reference pins; partition_of[perm[i]] = i mod p (partition.cpp:36-54).
inline void random_partition_of(uint64_t n, uint64_t p, uint64_t seed, uint32_t* pid) {
    std::vector<uint32_t> perm(n);
    for (uint64_t i = 0; i < n; ++i) perm[i] = (uint32_t)i;
    std::mt19937_64 eng(seed);
    for (uint64_t i = n; i > 1; --i) {
        const uint64_t limit = UINT64_MAX - UINT64_MAX % i;
        uint64_t x;
        do {
            x = eng();
        } while (x >= limit);
        std::swap(perm[i - 1], perm[x % i]);
    }
    for (uint64_t i = 0; i < n; ++i) pid[perm[i]] = (uint32_t)(i % p);
}

// hyperspherical_angles + angular_index (partition.cpp:118-148) on the host's
// libm for boundary points.
inline uint64_t angular_index_host(const double* x, uint32_t d, uint64_t m) {
    std::vector<double> ang(d - 1);
    double tail_sq = (double)x[d - 1] * (double)x[d - 1];
    for (uint32_t i = d - 1; i-- > 0;) {
        ang[i] = std::atan2(std::sqrt(tail_sq), (double)x[i]);
        tail_sq += (double)x[i] * (double)x[i];
    }
    uint64_t index = 0, stride = 1;
    for (double phi : ang) {
        uint64_t slice = (uint64_t)(2.0 * phi / 3.14159265358979323846 * (double)m);
        if (slice >= m) slice = m - 1;
        index += slice * stride;
        stride *= m;
    }
    return index;
}

// Contiguous ranges of P units over `ranks` owners with balanced weight
// (sky_plan_split); bounds[r]..bounds[r+1] belong to rank r.
template <class F>
inline std::vector<uint32_t> plan_ranges(const std::vector<uint32_t>& off, uint32_t P, int ranks, F weight) {
    (void)off;
    std::vector<uint32_t> b(ranks + 1, 0);
    b[ranks] = P;
    if (ranks == 1) return b;
    std::vector<uint64_t> prefix(P + 1, 0);
    for (uint32_t p = 0; p < P; ++p) prefix[p + 1] = prefix[p] + weight(p);
    std::vector<uint64_t> bounds(ranks + 1);
    sky_plan_split(prefix.data(), P, ranks, bounds.data());
    for (int r = 0; r <= ranks; ++r) b[r] = (uint32_t)bounds[r];
    return b;
}

// Local-phase shards: contiguous partition ranges balanced by |r_i|^2 (the
// SFS/BNL cost of a partition).
inline std::vector<uint32_t> plan_local_shards(const std::vector<uint32_t>& off, uint32_t P, int W) {
    return plan_ranges(off, P, W, [&](uint32_t p) {
        const uint64_t np = off[p + 1] - off[p];
        return np * np + np;
    });
}

inline bool weak_grid_dom(uint64_t a, uint64_t b, uint64_t m, uint32_t d);

// Potential dominators of partition i (engine.cpp:74-114) as ranges of the
// union (partition order); empty for strategies merged against all of U.
inline void pd_ranges(const std::vector<uint32_t>& offu, const std::vector<uint32_t>& nonempty, uint32_t i, int strategy,
               uint64_t m, uint32_t d, std::vector<uint2>& comps) {
    comps.clear();
    // Nearest potential dominators first: a dominated candidate usually has
    // its dominator in an adjacent slice / cell, so scanning those first lets
    // it leave early (the set, hence the result, is the reference's pd_i).
    if (strategy == SKY_SLICED) {  // pd_i = u_j, j < i (engine.cpp:106-108)
        for (auto it = nonempty.rbegin(); it != nonempty.rend(); ++it) {  // one range per slice (sorted by key)
            const uint32_t j = *it;
            if (j >= i) continue;
            comps.push_back(make_uint2(offu[j], offu[j + 1]));
        }
    } else if (strategy == SKY_GRID) {  // weakly dominating non-empty cells (engine.cpp:92-104)
        std::vector<std::pair<uint64_t, uint32_t>> cells;
        for (uint32_t j : nonempty) {
            if (j == i || !weak_grid_dom(j, i, m, d)) continue;
            uint64_t sum = 0, x = j;
            for (uint32_t k = 0; k < d; ++k) {
                sum += x % m;
                x /= m;
            }
            cells.push_back({sum, j});
        }
        std::sort(cells.begin(), cells.end(), [](const auto& a, const auto& b) {
            return a.first != b.first ? a.first > b.first : a.second > b.second;
        });
        for (const auto& c : cells) comps.push_back(make_uint2(offu[c.second], offu[c.second + 1]));
    }
}

// Merge-phase shards: contiguous candidate-partition ranges balanced by the
// number of candidate x potential-dominator pairs.
inline std::vector<uint32_t> plan_merge_shards(const std::vector<uint32_t>& offu, uint32_t P, int W, bool all_mode,
                                        int strategy, uint64_t m, uint32_t d) {
    std::vector<uint32_t> nonempty;
    for (uint32_t p = 0; p < P; ++p)
        if (offu[p + 1] > offu[p]) nonempty.push_back(p);
    std::vector<uint2> comps;
    const uint64_t U = offu[P];
    return plan_ranges(offu, P, W, [&](uint32_t i) -> uint64_t {
        const uint64_t ni = offu[i + 1] - offu[i];
        if (!ni) return 0;
        if (all_mode) return ni * U;
        pd_ranges(offu, nonempty, i, strategy, m, d, comps);
        uint64_t cmp = 0;
        for (uint2 r : comps) cmp += r.y - r.x;
        return ni * (cmp + 1);
    });
}

struct Plan {
    uint32_t tile = kTile;    // candidates per item
    uint32_t chunk = kChunk;  // comparators per item before the key bound
    std::vector<Item> items;
    std::vector<uint2> ranges;
    std::vector<uint32_t> group;  // item wave (comparator chunk index)

    // candidates [cb,ce) vs comparator ranges, split into groups of at most
    // `chunk` comparators; items of group g launch after those of group g-1
    // (so dominated candidates found by earlier chunks are skipped later).
    void add(uint32_t cb, uint32_t ce, const std::vector<uint2>& comps, uint32_t ch = 0) {
        if (!ch) ch = chunk;
        uint32_t g = 0, acc = 0;
        uint32_t lb = (uint32_t)ranges.size();
        auto flush = [&]() {
            if ((uint32_t)ranges.size() > lb) {
                items.push_back(Item{cb, ce, lb, (uint32_t)ranges.size()});
                group.push_back(g);
                ++g;
            }
            lb = (uint32_t)ranges.size();
            acc = 0;
        };
        for (uint2 r : comps) {
            uint32_t b = r.x;
            while (b < r.y) {
                const uint32_t take = std::min(r.y - b, ch - acc);
                ranges.push_back(make_uint2(b, b + take));
                b += take;
                acc += take;
                if (acc >= ch) flush();
            }
        }
        flush();
    }

    // Candidates [cb, ce) in tiles of `tile`, each tile against every group
    // of at most `chunk` comparators of `comps`; the ranges are stored once
    // and the tiles' items point at the same groups.
    void add_shared(uint32_t cb, uint32_t ce, const std::vector<uint2>& comps) {
        std::vector<uint2> groups;  // (lb, le) into `ranges`
        uint32_t acc = 0, lb = (uint32_t)ranges.size();
        for (uint2 r : comps) {
            for (uint32_t b = r.x; b < r.y;) {
                const uint32_t take = std::min(r.y - b, chunk - acc);
                ranges.push_back(make_uint2(b, b + take));
                b += take;
                acc += take;
                if (acc >= chunk) {
                    groups.push_back(make_uint2(lb, (uint32_t)ranges.size()));
                    lb = (uint32_t)ranges.size();
                    acc = 0;
                }
            }
        }
        if ((uint32_t)ranges.size() > lb) groups.push_back(make_uint2(lb, (uint32_t)ranges.size()));
        for (uint32_t b = cb; b < ce; b += tile) {
            const uint32_t e = std::min(ce, b + tile);
            for (uint32_t g = 0; g < (uint32_t)groups.size(); ++g) {
                items.push_back(Item{b, e, groups[g].x, groups[g].y});
                group.push_back(g);
            }
        }
    }

    // Launch order by wave: a stable counting pass over the group index.
    void order() {
        if (items.empty()) return;
        uint32_t G = 0;
        for (uint32_t g : group) G = std::max(G, g + 1);
        std::vector<uint32_t> start(G + 1, 0);
        for (uint32_t g : group) ++start[g + 1];
        for (uint32_t g = 0; g < G; ++g) start[g + 1] += start[g];
        std::vector<Item> it2(items.size());
        for (size_t i = 0; i < items.size(); ++i) it2[start[group[i]]++] = items[i];
        items.swap(it2);
    }
};

// For each cell of a cell index, the cells that weakly dominate it (every
// digit <=), nearest first (L1 distance over the digits, then cell id).
// Built once per digit layout and kept for the process.
inline const std::vector<std::vector<uint32_t>>& dominating_cells(const CellSpec& cs) {
    static std::mutex mu;
    static std::map<std::vector<uint8_t>, std::vector<std::vector<uint32_t>>> tables;
    const std::vector<uint8_t> layout(cs.bits, cs.bits + cs.k);
    std::lock_guard<std::mutex> lk(mu);
    std::vector<std::vector<uint32_t>>& t = tables[layout];
    if (!t.empty()) return t;
    const uint32_t k = cs.k, n = 1u << cs.total_bits();
    t.resize(n);
    std::vector<std::pair<uint32_t, uint32_t>> near;
    for (uint32_t cell = 0; cell < n; ++cell) {
        uint32_t dc[16], sh[16];
        uint32_t lim = 1;
        for (uint32_t j = 0, at = 0; j < k; ++j) {
            sh[j] = at;
            dc[j] = (cell >> at) & ((1u << cs.bits[j]) - 1u);
            at += cs.bits[j];
            lim *= dc[j] + 1;
        }
        near.clear();
        for (uint32_t r = 0; r < lim; ++r) {
            uint32_t x = r, id = 0, dist = 0;
            for (uint32_t j = 0; j < k; ++j) {
                const uint32_t dd = x % (dc[j] + 1);
                x /= dc[j] + 1;
                id |= dd << sh[j];
                dist += dc[j] - dd;
            }
            near.push_back({dist, id});
        }
        std::sort(near.begin(), near.end());
        for (const auto& p : near) t[cell].push_back(p.second);
    }
    return t;
}

class Runner {
   public:
    // Every API call ends with the stream drained (its results are read on
    // the host), so a new Runner may recycle the staging and event pools.
    Runner(sky_ctx* c) : c_(c), st_(c->stream) {
        c->dev.retire();  // the previous call drained its stream
        prof_ = c->opt.profile_host != 0;
        tl_ = c->opt.timeline != 0;
        c->stage_cur = c->stage_off = 0;
        c->dom_used = 0;
        c->hbm_used = 0;
        c->hbm_launches = 0;
        c->hbm_bytes = 0;
    }

    // Pinned bytes that stay untouched until the stream drains.
    template <class T>
    T* stage(size_t n) {
        const size_t bytes = (n ? n : 1) * sizeof(T) + 16;
        auto& v = c_->stage;
        while (true) {
            if (c_->stage_cur >= v.size()) {
                const size_t cap = std::max<size_t>(bytes, (size_t)4 << 20);
                char* p = nullptr;
                SKY_CUDA(cudaMallocHost(&p, cap));
                v.emplace_back(p, cap);
            }
            size_t off = (c_->stage_off + 15) & ~size_t{15};
            if (off + bytes <= v[c_->stage_cur].second) {
                c_->stage_off = off + bytes;
                return reinterpret_cast<T*>(v[c_->stage_cur].first + off);
            }
            ++c_->stage_cur;
            c_->stage_off = 0;
        }
    }

    // --------------------------------------------------------------- utils
    template <class T>
    T* dev(int slot, size_t n) { return c_->dev.as<T>(slot, n ? n : 1); }
    template <class T>
    T* pin(int slot, size_t n) { return c_->pin.as<T>(slot, n ? n : 1); }
    void sync(int line = __builtin_LINE()) {
        if (tl_) mark(-line);
        if (!c_->sync_ev) SKY_CUDA(cudaEventCreateWithFlags(&c_->sync_ev, cudaEventDisableTiming));
        SKY_CUDA(cudaEventRecord(c_->sync_ev, st_));
        while (true) {
            const cudaError_t e = cudaEventQuery(c_->sync_ev);
            if (e == cudaSuccess) break;
            if (e != cudaErrorNotReady) SKY_CUDA(e);
        }
        if (prof_) {
            const double t = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start_).count();
            std::fprintf(stderr, "  sync #%d at %.3f ms\n", ++n_sync_, t);
        }
    }
    bool prof_ = false;  // sky_options::profile_host (set in the constructor)
    int n_sync_ = 0;
    std::chrono::steady_clock::time_point t_start_ = std::chrono::steady_clock::now();
    void count(int k = 1, int line = __builtin_LINE()) {
        c_->launches += k;
        if (tl_) mark(line);
    }
    bool tl_ = false;  // sky_options::timeline (set in the constructor)
    std::vector<std::pair<int, double>> tl_marks_;
    void mark(int line) {
        auto& e = c_->tl_ev;
        if (e.size() <= tl_marks_.size()) {
            cudaEvent_t ev;
            SKY_CUDA(cudaEventCreate(&ev));
            e.push_back(ev);
        }
        SKY_CUDA(cudaEventRecord(e[tl_marks_.size()], st_));
        tl_marks_.emplace_back(
            line, std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start_).count());
    }
    // after the stream drained: line, host issue ms, device ms (from the first mark)
    void timeline_dump() {
        if (!tl_ || tl_marks_.empty()) return;
        float prev = 0.f;
        for (size_t k = 0; k < tl_marks_.size(); ++k) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, c_->tl_ev[0], c_->tl_ev[k]);
            std::fprintf(stderr, "TL %3zu line %5d host %8.3f dev %8.3f (+%7.3f)\n", k, tl_marks_[k].first,
                         tl_marks_[k].second, ms, ms - prev);
            prev = ms;
        }
        tl_marks_.clear();
    }

    DevSet set(int base, uint32_t n, int D) {
        DevSet s;
        const int D4 = (D + 3) / 4 * 4;
        s.xyz = dev<float>(base, (size_t)n * D4);
        s.skey = dev<uint32_t>(base + 1, n);
        s.id = dev<uint32_t>(base + 2, n);
        if (D <= 16) s.qc = dev<uint2>(base + 3, n);
        s.n = n;
        return s;
    }

    // Packed monotone codes for a set whose comparators and candidates share
    // one quantization (thresholds from a sample of `s`; `also` reuses them).
    void encode(int D, DevSet& s, DevSet* also = nullptr) {
        if (D > 16 || !s.n) return;
        float* thr = dev<float>(S_THR, (size_t)D * (kCodeLevels - 1));
        launch_thresholds(D, s, thr, st_);
        launch_encode(D, s, thr, st_);
        count(2);
        if (also && also->n) {
            launch_encode(D, *also, thr, st_);
            count();
        }
    }

    // the same with the set's row count in device memory (s.n = capacity)
    void encode_dev(int D, DevSet& s, const uint32_t* n_dev) {
        if (D > 16 || !s.n) return;
        float* thr = dev<float>(S_THR, (size_t)D * (kCodeLevels - 1));
        launch_thresholds(D, s, thr, st_, n_dev);
        launch_encode(D, s, thr, st_, n_dev);
        count(2);
    }

    template <class K, class V>
    void sort_pairs(const K* kin, K* kout, const V* vin, V* vout, uint32_t n, int bb, int eb) {
        if (!n) return;
        size_t bytes = 0;
        SKY_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, kin, kout, vin, vout, (int)n, bb, eb, st_));
        void* tmp = c_->dev.get(S_CUB, bytes);
        SKY_CUDA(cub::DeviceRadixSort::SortPairs(tmp, bytes, kin, kout, vin, vout, (int)n, bb, eb, st_));
        count(4);
    }
    template <class K>
    void sort_keys(const K* kin, K* kout, uint32_t n, int end_bit = 8 * sizeof(K)) {
        if (!n) return;
        size_t bytes = 0;
        SKY_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, bytes, kin, kout, (int)n, 0, end_bit, st_));
        void* tmp = c_->dev.get(S_CUB, bytes);
        SKY_CUDA(cub::DeviceRadixSort::SortKeys(tmp, bytes, kin, kout, (int)n, 0, end_bit, st_));
        count(4);
    }
    struct NotDead {
        __host__ __device__ uint32_t operator()(uint8_t x) const { return x ? 0u : 1u; }
    };
    // pos[i] = number of live entries before i
    void scan_live(const uint8_t* dead, uint32_t* pos, uint32_t n) {
        if (!n) return;
        cub::TransformInputIterator<uint32_t, NotDead, const uint8_t*> it(dead, NotDead());
        size_t bytes = 0;
        SKY_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, it, pos, (int)n, st_));
        void* tmp = c_->dev.get(S_CUB, bytes);
        SKY_CUDA(cub::DeviceScan::ExclusiveSum(tmp, bytes, it, pos, (int)n, st_));
        count(2);
    }

    // Keep the live rows of `in` (segments off_in[P+1]) into `out_base`;
    // new offsets land in off_out (device) and off_host. Synchronizes.
    DevSet compact(const DevSet& in, const uint8_t* dead, const uint32_t* off_in, uint32_t P, int out_base,
                   uint32_t* off_out, std::vector<uint32_t>& off_host, int D) {
        uint32_t* pos = dev<uint32_t>(S_POS, in.n);
        uint32_t* misc = dev<uint32_t>(S_MISC, 64);
        scan_live(dead, pos, in.n);
        launch_count_total(pos, dead, in.n, misc + M_TOTAL, st_);
        count();
        launch_remap_offsets(off_in, P, pos, dead, in.n, off_out, st_);
        count();
        uint32_t* h = pin<uint32_t>(P_OFF, P + 2);
        SKY_CUDA(cudaMemcpyAsync(h, off_out, (P + 1) * sizeof(uint32_t), cudaMemcpyDeviceToHost, st_));
        SKY_CUDA(cudaMemcpyAsync(h + P + 1, misc + M_TOTAL, sizeof(uint32_t), cudaMemcpyDeviceToHost, st_));
        sync();
        const uint32_t total = in.n ? h[P + 1] : 0;
        off_host.assign(h, h + P + 1);
        DevSet out = set(out_base, total, D);
        launch_scatter_direct(D, in, dead, pos, out, st_);
        count();
        return out;
    }

    // Compaction with the count kept on the device: `in` has in.n slots (a
    // capacity; slots at or past the live count must be flagged dead). The
    // result has n = in.n slots, offsets off_out and *total live rows.
    DevSet compact_dev(const DevSet& in, const uint8_t* dead, const uint32_t* off_in, uint32_t P, int out_base,
                       uint32_t* off_out, uint32_t* total, int D) {
        if (in.n) {
            // dense list of the live rows + remapped offsets + count (two
            // launches, work proportional to the live rows past the count
            // pass), then a gather bounded by the device count
            uint32_t* dense = dev<uint32_t>(S_POS, in.n);
            launch_dense_compact(dead, in.n, off_in, P, 0, dense, off_out, total,
                                 dev<uint32_t>(S_DCBT, dense_compact_scratch(in.n) / 4), st_);
            DevSet out = set(out_base, in.n, D);
            launch_gather_set(D, in, dense, out, st_, total);
            count(3);
            return out;
        }
        uint32_t* pos = dev<uint32_t>(S_POS, in.n);
        scan_live(dead, pos, in.n);
        launch_count_total(pos, dead, in.n, total, st_);
        launch_remap_offsets(off_in, P, pos, dead, in.n, off_out, st_);
        DevSet out = set(out_base, in.n, D);
        launch_scatter_direct(D, in, dead, pos, out, st_);
        count(3);
        return out;
    }

    // exclusive scan of n_plus1 words (the last output = the total)
    void scan_u32(const uint32_t* in, uint32_t* out, uint32_t n_plus1) {
        size_t bytes = 0;
        SKY_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, (int)n_plus1, st_));
        void* tmp = c_->dev.get(S_CUB, bytes);
        SKY_CUDA(cub::DeviceScan::ExclusiveSum(tmp, bytes, in, out, (int)n_plus1, st_));
        count(2);
    }

    // Direct items of device-built jobs; *n_items points at the device count.
    Item* expand_jobs(const Job* jobs, const uint32_t* n_jobs, uint32_t cap, uint32_t tile, uint32_t chunk,
                      uint32_t max_chunks, uint64_t item_cap, const uint32_t** n_items) {
        uint32_t* cnt = dev<uint32_t>(S_JCNT, cap + 1);
        uint32_t* pre = dev<uint32_t>(S_JPRE, cap + 1);
        launch_job_counts(jobs, n_jobs, cap, tile, chunk, max_chunks, cnt, st_);
        scan_u32(cnt, pre, cap + 1);
        Item* items = dev<Item>(S_ITEMS, item_cap);
        launch_job_items(jobs, n_jobs, cap, pre, tile, chunk, max_chunks, items, st_);
        count(2);
        *n_items = pre + cap;
        return items;
    }

    // One relsky launch over device-built direct items.
    void relsky_direct(int D, uint32_t tile, const RelskyArgs& base, const uint2* cq, const uint2* sq,
                       const uint32_t* dense, const Item* items, uint64_t cap, const uint32_t* n_items_dev) {
        if (x64_.x && (!base.sid || !base.cid))
            throw Error(SKY_E_INTERNAL, "FP64 confirmation needs the row ids of both sets");
        uint32_t* misc = dev<uint32_t>(S_MISC, 64);
        SKY_CUDA(cudaMemsetAsync(misc + M_WORK, 0, sizeof(uint32_t), st_));
        Relsky2Args b{};
        b.cidx = dense;
        b.cxyz = base.cxyz; b.cskey = base.cskey; b.cqc = cq;
        b.x64 = x64_; b.cid = base.cid; b.sid = base.sid;
        b.sxyz = base.sxyz; b.sskey = base.sskey; b.sqc = sq;
        b.items = items; b.n_items = (uint32_t)std::min<uint64_t>(cap, 0xFFFFFFFFu); b.n_items_dev = n_items_dev;
        b.direct = true;
        b.bounded = base.bounded; b.dead = base.dead;
        b.tests = base.tests; b.counter = misc + M_WORK;
        const int phase = base.tests ? (int)(base.tests - tests(0)) : 3;
        b.coarse_hits = reinterpret_cast<unsigned long long*>(misc + M_HITS) + phase;
        dom_begin();
        launch_relsky2(D, (int)tile, b, c_->sm_count, st_);
        dom_end();
        count();
    }

    // Local SFS with every count on the device (single GPU): the block stage
    // and both waves are planned by kernels from device offsets, so no host
    // round trip until the union's offsets are read by the caller.
    //   s0: n = capacity, *n0 live rows, partitions off0_dev[P+1].
    DevSet local_sfs_dev(int D, const DevSet& s0, const uint32_t* n0, const uint32_t* off0_dev, uint32_t P,
                         uint32_t* off_u_dev, uint32_t* n_u, bool count_tests) {
        if (D > 16) {
            // wider rows run on the exact-compare core, which the device
            // planner's packed-code launches do not cover: offsets and count
            // to the host (one round trip), then the host-planned SFS
            uint32_t* h = pin<uint32_t>(P_OFF, (size_t)P + 2);
            SKY_CUDA(cudaMemcpyAsync(h, off0_dev, ((size_t)P + 1) * sizeof(uint32_t), cudaMemcpyDeviceToHost, st_));
            SKY_CUDA(cudaMemcpyAsync(h + P + 1, n0, sizeof(uint32_t), cudaMemcpyDeviceToHost, st_));
            sync();
            const std::vector<uint32_t> off0(h, h + P + 1);
            DevSet live = s0;
            live.n = h[P + 1];
            std::vector<uint32_t> off_u;
            DevSet U = local_sfs(D, live, off0, const_cast<uint32_t*>(off0_dev), P, off_u_dev, off_u, count_tests);
            uint32_t* hn = stage<uint32_t>(1);
            *hn = U.n;
            SKY_CUDA(cudaMemcpyAsync(n_u, hn, sizeof(uint32_t), cudaMemcpyHostToDevice, st_));
            return U;
        }
        const uint32_t cap = s0.n;
        uint32_t* misc = dev<uint32_t>(S_MISC, 64);
        uint8_t* dead = dev<uint8_t>(S_DEAD, cap);
        launch_fill_live_u8(dead, n0, cap, st_);
        count();
        RelskyArgs a{};
        a.cxyz = s0.xyz; a.cskey = s0.skey; a.indirect = false;
        a.sxyz = s0.xyz; a.sskey = s0.skey; a.bounded = true; a.dead = dead;
        a.cid = s0.id; a.sid = s0.id;
        a.tests = count_tests ? tests(1) : nullptr;
        // No block stage: the first wave (every row against the strongest
        // `head` rows of its partition) already removes most dominated rows,
        // and the second runs over dense lists of the survivors.
        Job* jobs = dev<Job>(S_JOBS, P);
        const uint32_t* n_items = nullptr;
        // grain from the capacity: ~ rows per partition
        const uint64_t per = (uint64_t)cap / std::max<uint32_t>(1, P);
        // 128-candidate tiles measured ~1% faster than 256 on config 2
        uint32_t tile = per >= 512 ? 128 : 64;
        if (c_->opt.sfs_tile) tile = c_->opt.sfs_tile;
        // chunk 0: derived on the device from the live counts (a grain of
        // work items per resident CTA)
        const uint32_t chunk = c_->opt.sfs_chunk, max_chunks = 64, head = c_->opt.sfs_head;
        const uint32_t grain = (uint32_t)c_->sm_count * 2 * c_->opt.grain_items;
        // small sets (C1, C3, C5: the filtered set fits 128k rows): finer
        // chunks spread the few rows over the SMs; large sets keep sfs_chunk
        // (measured: C3 0.60 -> 0.56 ms, C2 3% slower with the finer grain)
        const bool auto_chunk = c_->opt.sfs_auto_chunk && cap <= (1u << 17);
        const uint64_t icap = ((uint64_t)cap / tile + P) * max_chunks;
        uint32_t* np_dev = misc + M_NP;
        uint32_t* hp = stage<uint32_t>(1);
        *hp = P;
        SKY_CUDA(cudaMemcpyAsync(np_dev, hp, sizeof(uint32_t), cudaMemcpyHostToDevice, st_));
        // jobs -> items: one fused planning launch for up to 1024 partitions
        auto plan = [&](const uint32_t* coff, uint64_t lo, uint64_t hi) -> Item* {
            Item* it = dev<Item>(S_ITEMS, icap);
            uint32_t* ni = misc + M_NITEMS;
            if (launch_plan_partition_items(coff, off0_dev, nullptr, P, lo, hi, tile,
                                            auto_chunk ? 0u : chunk, max_chunks,
                                            (uint32_t)std::min<uint64_t>(icap, 0xFFFFFFFFu), it, ni, st_, grain)) {
                count();
                n_items = ni;
                return it;
            }
            launch_partition_jobs(coff, off0_dev, nullptr, P, lo, hi, jobs, st_);
            count();
            return expand_jobs(jobs, np_dev, P, tile, chunk, max_chunks, icap, &n_items);
        };
        // wave 0: every row of a partition against the partition's first `head` rows
        Item* items = plan(off0_dev, 0, head);
        relsky_direct(D, tile, a, s0.qc, s0.qc, nullptr, items, icap, n_items);
        // wave 1: the live rows (dense lists) against the rest of their partition
        uint32_t* dnew = dev<uint32_t>(S_DNEW, P + 1);
        uint32_t* dense = dev<uint32_t>(S_DENSE, cap);
        if (launch_dense_compact(dead, cap, off0_dev, P, 0, dense, dnew, nullptr,
                                 dev<uint32_t>(S_DCBT, dense_compact_scratch(cap) / 4), st_, n0)) {
            count(2);
        } else {
            uint32_t* pos = dev<uint32_t>(S_POS, cap);
            scan_live(dead, pos, cap);
            launch_remap_offsets(off0_dev, P, pos, dead, cap, dnew, st_);
            launch_compact_pos(dead, pos, cap, 0, dense, st_);
            count(2);
        }
        items = plan(dnew, head, ~0ull);
        relsky_direct(D, tile, a, s0.qc, s0.qc, dense, items, icap, n_items);
        return compact_dev(s0, dead, off0_dev, P, S_SET2, off_u_dev, n_u, D);
    }

    // Sky(U) on one GPU without a host round trip (random / angular NoSeq,
    // sequential merge: u_i are antichains, so the merge is the skyline of
    // the union). U (n = capacity, live count *n_u, key-sorted partition runs
    // off_u[P+1]) is merged into key order (US, slot S_SET3), then two waves
    // as in local_sfs_dev with all of US as one partition: every row against
    // the strongest `head` rows, then the survivors against the rest. Items
    // and the comparator chunk are planned on the device from *n_u. Dead
    // flags of US (tail past *n_u set) go to *dead_out.
    DevSet merge_all_dev(int D, const DevSet& U, const uint32_t* off_u, uint32_t P, const uint32_t* n_u,
                         bool count_tests, uint8_t** dead_out) {
        const uint32_t cap = U.n;
        DevSet US = set(S_SET3, cap, D);
        launch_merge_runs(D, U, off_u, P, US, st_, n_u);
        uint8_t* dead = dev<uint8_t>(S_CELLDEAD, cap);
        launch_fill_live_u8(dead, n_u, cap, st_);
        count(2);
        *dead_out = dead;
        if (!cap) return US;
        uint32_t* misc = dev<uint32_t>(S_MISC, 64);
        uint32_t* offg = dev<uint32_t>(S_OFFG, 2);  // {0, *n_u}: the one "partition"
        SKY_CUDA(cudaMemsetAsync(offg, 0, sizeof(uint32_t), st_));
        SKY_CUDA(cudaMemcpyAsync(offg + 1, n_u, sizeof(uint32_t), cudaMemcpyDeviceToDevice, st_));
        RelskyArgs a{};
        a.cxyz = US.xyz; a.cskey = US.skey; a.cid = US.id;
        a.sxyz = US.xyz; a.sskey = US.skey; a.sid = US.id;
        a.indirect = false; a.bounded = true; a.dead = dead;
        a.tests = count_tests ? tests(2) : nullptr;
        // candidates per item from the capacity (the input size on the
        // exact-count-free path up to kExactCapRows rows, so config 2's 1M
        // input takes 256): a grain choice only
        const uint32_t tile = c_->opt.merge_tile ? c_->opt.merge_tile : (cap <= 300000 ? 128u : 256u);
        const uint32_t max_chunks = 64, head = c_->opt.merge_head;
        const uint32_t target = (uint32_t)c_->sm_count * 2 * c_->opt.grain_items;
        const uint64_t icap = ((uint64_t)cap / tile + 2) * max_chunks;
        const uint32_t icap32 = (uint32_t)std::min<uint64_t>(icap, 0xFFFFFFFFu);
        Item* items = dev<Item>(S_ITEMS, icap);
        uint32_t* ni = misc + M_NITEMS;
        launch_plan_partition_items(offg, nullptr, n_u, 1, 0, head, tile, 0, max_chunks, icap32, items, ni, st_,
                                    target);
        count();
        relsky_direct(D, tile, a, US.qc, US.qc, nullptr, items, icap, ni);
        uint32_t* dnew = dev<uint32_t>(S_DNEW, 2);
        uint32_t* dense = dev<uint32_t>(S_DENSE, cap);
        launch_dense_compact(dead, cap, offg, 1, 0, dense, dnew, nullptr,
                             dev<uint32_t>(S_DCBT, dense_compact_scratch(cap) / 4), st_, n_u);
        count(2);
        launch_plan_partition_items(dnew, nullptr, n_u, 1, head, ~0ull, tile, 0, max_chunks, icap32, items, ni, st_,
                                    target);
        count();
        relsky_direct(D, tile, a, US.qc, US.qc, dense, items, icap, ni);
        return US;
    }

    void relsky(int D, const Plan& plan, const RelskyArgs& base, const uint2* cq = nullptr,
                const uint2* sq = nullptr, const uint32_t* dense = nullptr) {
        if (plan.items.empty()) return;
        const auto t0 = std::chrono::steady_clock::now();
        struct Report {
            const Plan& p;
            std::chrono::steady_clock::time_point t0;
            sky_ctx* c;
            ~Report() {
                if (c->opt.profile_host) {
                    const double ms =
                        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
                    std::fprintf(stderr, "relsky items=%zu ranges=%zu tile=%u chunk=%u host+wait=%.3f ms dom_total=%.3f\n",
                                 p.items.size(), p.ranges.size(), p.tile, p.chunk, ms, c->dom_ms);
                }
            }
        } report{plan, t0, c_};
        Item* hi = stage<Item>(plan.items.size());
        uint2* hr = stage<uint2>(plan.ranges.size());
        std::memcpy(hi, plan.items.data(), plan.items.size() * sizeof(Item));
        std::memcpy(hr, plan.ranges.data(), plan.ranges.size() * sizeof(uint2));
        Item* di = dev<Item>(S_ITEMS, plan.items.size());
        uint2* dr = dev<uint2>(S_RANGES, plan.ranges.size());
        SKY_CUDA(cudaMemcpyAsync(di, hi, plan.items.size() * sizeof(Item), cudaMemcpyHostToDevice, st_));
        SKY_CUDA(cudaMemcpyAsync(dr, hr, plan.ranges.size() * sizeof(uint2), cudaMemcpyHostToDevice, st_));
        RelskyArgs a = base;
        a.x64 = x64_;
        if (x64_.x && (!a.sid || (!a.indirect && !a.cid)))
            throw Error(SKY_E_INTERNAL, "FP64 confirmation needs the row ids of both sets");
        a.items = di;
        a.ranges = dr;
        a.n_items = (uint32_t)plan.items.size();
        dom_begin();
        if (D <= 16 && cq && sq && !a.indirect) {
            uint32_t* misc = dev<uint32_t>(S_MISC, 64);
            SKY_CUDA(cudaMemsetAsync(misc + M_WORK, 0, sizeof(uint32_t), st_));
            Relsky2Args b{};
            b.cidx = dense;
            b.cxyz = a.cxyz; b.cskey = a.cskey; b.cqc = cq;
            b.x64 = a.x64; b.cid = a.cid; b.sid = a.sid;
            b.sxyz = a.sxyz; b.sskey = a.sskey; b.sqc = sq;
            b.items = di; b.n_items = a.n_items; b.ranges = dr; b.bounded = a.bounded; b.dead = a.dead;
            b.tests = a.tests; b.counter = misc + M_WORK;
            b.range_par = c_->opt.range_par && plan.ranges.size() >= (size_t)c_->opt.range_par * plan.items.size();
            const int phase = a.tests ? (int)(a.tests - tests(0)) : 3;
            b.coarse_hits = reinterpret_cast<unsigned long long*>(misc + M_HITS) + phase;
            launch_relsky2(D, (int)plan.tile, b, c_->sm_count, st_);
        } else {
            if (plan.tile != (uint32_t)kTile) throw Error(SKY_E_INTERNAL, "v1 relsky needs 512-candidate tiles");
            launch_relsky(D, a, st_);
        }
        dom_end();
        count();
    }

    // Multi-wave relative skyline of the candidates of partitions [qb, qe)
    // (positions offc[p]..offc[p+1] of `C`) against their comparator lists
    // (comps_of(p), most likely dominators first). Wave 0 tests every
    // candidate against the first `head` comparators of its list; wave w >= 1
    // takes the next head*3*4^(w-1) comparators. Between waves the live
    // candidates are compacted into dense per-partition lists and the next
    // wave's items are built on the device (k_plan_items), so tiles stay full
    // of live candidates without a host round trip.
    template <class CompsOf>
    void relsky_waves(int D, const std::vector<uint32_t>& offc, uint32_t qb, uint32_t qe, CompsOf comps_of,
                      const RelskyArgs& base, const uint2* cq, const uint2* sq, uint32_t tile, uint32_t chunk,
                      uint32_t head) {
        if (qb >= qe) return;
        const uint32_t np = qe - qb;
        std::vector<std::vector<uint2>> lists(np);
        uint64_t maxlen = 0;
        for (uint32_t p = qb; p < qe; ++p) {
            if (offc[p + 1] == offc[p]) continue;
            comps_of(p, lists[p - qb]);
            uint64_t len = 0;
            for (const uint2& r : lists[p - qb]) len += r.y - r.x;
            maxlen = std::max(maxlen, len);
        }
        // the sub-list [lo, hi) (in comparator counts) of a list
        auto slice = [](const std::vector<uint2>& l, uint64_t lo, uint64_t hi, std::vector<uint2>& out) {
            out.clear();
            uint64_t at = 0;
            for (const uint2& r : l) {
                const uint64_t len = r.y - r.x, b = std::max(lo, at), e = std::min(hi, at + len);
                if (b < e) out.push_back(make_uint2(r.x + (uint32_t)(b - at), r.x + (uint32_t)(e - at)));
                at += len;
                if (at >= hi) break;
            }
        };
        std::vector<uint2> sub;
        Plan A;
        A.tile = tile;
        A.chunk = chunk;
        for (uint32_t p = qb; p < qe; ++p) {
            slice(lists[p - qb], 0, head, sub);
            if (sub.empty()) continue;
            // the partition's comparator groups once, shared by all its tiles
            A.add_shared(offc[p], offc[p + 1], sub);
        }
        A.order();
        relsky(D, A, base, cq, sq);
        if (maxlen <= head) return;

        const uint32_t cb = offc[qb], cn = offc[qe] - cb;
        uint32_t* pos = dev<uint32_t>(S_POS, cn);
        uint32_t* hrel = stage<uint32_t>(np + 2);
        for (uint32_t p = qb; p <= qe; ++p) hrel[p - qb] = offc[p] - cb;
        uint32_t* drel = dev<uint32_t>(S_OFF_C, np + 1);
        uint32_t* dnew = dev<uint32_t>(S_SIZES, np + 1);
        uint32_t* dense = dev<uint32_t>(S_DENSE, cn);
        uint32_t* nitems = dev<uint32_t>(S_MISC, 64) + M_NITEMS;
        SKY_CUDA(cudaMemcpyAsync(drel, hrel, (np + 1) * sizeof(uint32_t), cudaMemcpyHostToDevice, st_));
        std::vector<uint64_t> lens(np, 0);
        for (uint32_t k = 0; k < np; ++k)
            for (const uint2& r : lists[k]) lens[k] += r.y - r.x;
        const uint64_t grow = std::max<uint32_t>(2, c_->opt.wave_growth);
        for (uint64_t lo = head, len = (grow - 1) * head; lo < maxlen; lo += len, len *= grow) {
            // split further only while the rest is worth a compaction pass
            uint64_t rest = 0;
            for (uint32_t k = 0; k < np; ++k)
                if (lens[k] > lo) rest += (uint64_t)(offc[qb + k + 1] - offc[qb + k]) * (lens[k] - lo);
            if (rest < ((uint64_t)c_->opt.wave_split_mpairs << 20)) len = maxlen - lo;
            const uint64_t hi = lo + len;
            // this wave's comparator groups per partition (host: the lists are static)
            std::vector<uint2> ranges, groups;
            std::vector<uint32_t> gb(np + 1, 0);
            uint32_t max_groups = 0;
            uint64_t cap = 0;
            for (uint32_t p = qb; p < qe; ++p) {
                slice(lists[p - qb], lo, hi, sub);
                uint32_t ng = 0, acc = 0, lb = (uint32_t)ranges.size();
                for (const uint2& r : sub) {
                    for (uint32_t b = r.x; b < r.y;) {
                        const uint32_t take = std::min(r.y - b, chunk - acc);
                        ranges.push_back(make_uint2(b, b + take));
                        b += take;
                        acc += take;
                        if (acc >= chunk) {
                            groups.push_back(make_uint2(lb, (uint32_t)ranges.size()));
                            lb = (uint32_t)ranges.size();
                            acc = 0;
                            ++ng;
                        }
                    }
                }
                if ((uint32_t)ranges.size() > lb) {
                    groups.push_back(make_uint2(lb, (uint32_t)ranges.size()));
                    ++ng;
                }
                gb[p - qb + 1] = gb[p - qb] + ng;
                max_groups = std::max(max_groups, ng);
                cap += (uint64_t)ng * ((offc[p + 1] - offc[p] + tile - 1) / tile);
            }
            if (!cap) continue;
            // dense lists of the candidates still alive
            if (launch_dense_compact(base.dead + cb, cn, drel, np, cb, dense, dnew, nullptr,
                                     dev<uint32_t>(S_DCBT, dense_compact_scratch(cn) / 4), st_)) {
                count(2);
            } else {
                scan_live(base.dead + cb, pos, cn);
                launch_remap_offsets(drel, np, pos, base.dead + cb, cn, dnew, st_);
                launch_compact_pos(base.dead + cb, pos, cn, cb, dense, st_);
                count(4);
            }
            uint2* hr = stage<uint2>(ranges.size());
            std::memcpy(hr, ranges.data(), ranges.size() * sizeof(uint2));
            uint2* hg = stage<uint2>(groups.size());
            std::memcpy(hg, groups.data(), groups.size() * sizeof(uint2));
            uint32_t* hgb = stage<uint32_t>(np + 1);
            std::memcpy(hgb, gb.data(), (np + 1) * sizeof(uint32_t));
            uint2* dr = dev<uint2>(S_RANGES, ranges.size());
            uint2* dg = dev<uint2>(S_GROUPS, groups.size());
            uint32_t* dgb = dev<uint32_t>(S_GB, np + 1);
            Item* di = dev<Item>(S_ITEMS, cap);
            SKY_CUDA(cudaMemcpyAsync(dr, hr, ranges.size() * sizeof(uint2), cudaMemcpyHostToDevice, st_));
            SKY_CUDA(cudaMemcpyAsync(dg, hg, groups.size() * sizeof(uint2), cudaMemcpyHostToDevice, st_));
            SKY_CUDA(cudaMemcpyAsync(dgb, hgb, (np + 1) * sizeof(uint32_t), cudaMemcpyHostToDevice, st_));
            launch_plan_items(dnew, np, dgb, dg, max_groups, tile, di, nitems, st_);
            count();
            relsky_dev(D, tile, base, cq, sq, dense, di, (uint32_t)cap, nitems, dr,
                       c_->opt.range_par && ranges.size() >= (size_t)c_->opt.range_par * groups.size());
        }
    }

    // One relsky launch over device-built items (count in device memory).
    void relsky_dev(int D, uint32_t tile, const RelskyArgs& base, const uint2* cq, const uint2* sq,
                    const uint32_t* dense, const Item* items, uint32_t cap, const uint32_t* n_items_dev,
                    const uint2* ranges, bool range_par = false) {
        if (x64_.x && (!base.sid || !base.cid))
            throw Error(SKY_E_INTERNAL, "FP64 confirmation needs the row ids of both sets");
        uint32_t* misc = dev<uint32_t>(S_MISC, 64);
        SKY_CUDA(cudaMemsetAsync(misc + M_WORK, 0, sizeof(uint32_t), st_));
        Relsky2Args b{};
        b.cidx = dense;
        b.cxyz = base.cxyz; b.cskey = base.cskey; b.cqc = cq;
        b.x64 = x64_; b.cid = base.cid; b.sid = base.sid;
        b.sxyz = base.sxyz; b.sskey = base.sskey; b.sqc = sq;
        b.items = items; b.n_items = cap; b.n_items_dev = n_items_dev; b.ranges = ranges;
        b.range_par = range_par;
        b.bounded = base.bounded; b.dead = base.dead;
        b.tests = base.tests; b.counter = misc + M_WORK;
        const int phase = base.tests ? (int)(base.tests - tests(0)) : 3;
        b.coarse_hits = reinterpret_cast<unsigned long long*>(misc + M_HITS) + phase;
        dom_begin();
        launch_relsky2(D, (int)tile, b, c_->sm_count, st_);
        dom_end();
        count();
    }

    // CUDA events around each dominance launch; summed once the run drained
    void dom_begin() {
        if (!c_->opt.kernel_events) return;
        auto& e = c_->dom_ev;
        while (e.size() < 2 * (size_t)(c_->dom_used + 1)) {
            cudaEvent_t ev;
            SKY_CUDA(cudaEventCreate(&ev));
            e.push_back(ev);
        }
        SKY_CUDA(cudaEventRecord(e[2 * c_->dom_used], st_));
    }
    void dom_end() {
        c_->dom_launches += c_->opt.kernel_events ? 0 : 1;
        if (!c_->opt.kernel_events) return;
        SKY_CUDA(cudaEventRecord(c_->dom_ev[2 * c_->dom_used + 1], st_));
        ++c_->dom_used;
        c_->dom_launches += 1;
    }
    // the same for the HBM streaming passes, with their algorithmic bytes
    void hbm_begin() {
        if (!c_->opt.kernel_events) return;
        auto& e = c_->hbm_ev;
        while (e.size() < 2 * (size_t)(c_->hbm_used + 1)) {
            cudaEvent_t ev;
            SKY_CUDA(cudaEventCreate(&ev));
            e.push_back(ev);
        }
        SKY_CUDA(cudaEventRecord(e[2 * c_->hbm_used], st_));
    }
    void hbm_end(uint64_t bytes) {
        ++c_->hbm_launches;
        c_->hbm_bytes += bytes;
        if (!c_->opt.kernel_events) return;
        SKY_CUDA(cudaEventRecord(c_->hbm_ev[2 * c_->hbm_used + 1], st_));
        ++c_->hbm_used;
    }
    // an event pair for a pass the launcher brackets itself (recorded there)
    void hbm_pair(uint64_t bytes, cudaEvent_t* begin, cudaEvent_t* end) {
        *begin = *end = nullptr;
        ++c_->hbm_launches;
        c_->hbm_bytes += bytes;
        if (!c_->opt.kernel_events) return;
        auto& e = c_->hbm_ev;
        while (e.size() < 2 * (size_t)(c_->hbm_used + 1)) {
            cudaEvent_t ev;
            SKY_CUDA(cudaEventCreate(&ev));
            e.push_back(ev);
        }
        *begin = e[2 * c_->hbm_used];
        *end = e[2 * c_->hbm_used + 1];
        ++c_->hbm_used;
    }
    double hbm_collect() {
        double t = 0.0;
        for (uint32_t k = 0; k < c_->hbm_used; ++k) {
            float ms = 0.f;
            SKY_CUDA(cudaEventElapsedTime(&ms, c_->hbm_ev[2 * k], c_->hbm_ev[2 * k + 1]));
            t += ms;
        }
        return t;
    }
    void dom_collect() {
        for (uint32_t k = 0; k < c_->dom_used; ++k) {
            float ms = 0.f;
            SKY_CUDA(cudaEventElapsedTime(&ms, c_->dom_ev[2 * k], c_->dom_ev[2 * k + 1]));
            c_->dom_ms += ms;
        }
        c_->dom_used = 0;
    }

    // Item granularity: candidates per item (one warp, 32*K) and comparators
    // per item before the key bound. Big items amortize comparator staging;
    // small ones keep ~16 items per resident warp slot so 148 SMs stay busy
    // and load balances. `pairs` = candidate x comparator pairs of the launch
    // (before bounding).
    void pick_grain(int D, uint64_t n_cands, uint64_t pairs, uint32_t* tile, uint32_t* chunk) const {
        if (D > 16) {
            *tile = kTile;
            *chunk = kChunk;
            return;
        }
        // ~4 items per resident CTA (8 warps share an item's comparators);
        // shrink the comparator chunk first (keeps 256-candidate tiles), the
        // candidate tile only when candidates are few
        const uint64_t target = (uint64_t)c_->sm_count * 2 * c_->opt.grain_items;
        uint32_t t = 256, ch = 16384;
        while (ch > 2048 && n_cands && pairs / ((uint64_t)t * ch) < target) ch /= 2;
        while (t > 32 && n_cands && n_cands / t < (uint64_t)c_->sm_count * 2) t /= 2;
        *tile = t;
        *chunk = ch;
    }

    // ------------------------------------------------------- exchanges
    // The rows of `mine` (rank r's block, counts[r] rows each) concatenated in
    // rank order into `all` on every rank (coordinates, keys, ids, and the
    // packed codes when `codes`; they are only comparable when every rank
    // encoded with the same thresholds).
    void allgather_set(int D, const DevSet& mine, const std::vector<uint32_t>& counts, DevSet& all, bool codes) {
        const int W = c_->world;
        const size_t D4 = (size_t)(D + 3) / 4 * 4;
        std::vector<size_t> b(W), dp(W);
        auto run = [&](const void* src, void* dst, size_t unit) {
            size_t at = 0;
            for (int q = 0; q < W; ++q) {
                b[q] = counts[q] * unit;
                dp[q] = at;
                at += b[q];
            }
            c_->comm->allgatherv(src, dst, b.data(), dp.data(), st_);
        };
        run(mine.xyz, all.xyz, D4 * sizeof(float));
        run(mine.skey, all.skey, sizeof(uint32_t));
        run(mine.id, all.id, sizeof(uint32_t));
        if (codes && all.qc) run(mine.qc, all.qc, sizeof(uint2));
    }

    // Local skylines of all ranks in partition order on every rank: sizes by
    // all-reduce, rows by a ragged all-gather (owners hold contiguous
    // partition ranges pr[W+1], so rank order is partition order).
    DevSet gather_union(int D, const DevSet& Um, const std::vector<uint32_t>& offum, const std::vector<uint32_t>& pr,
                        uint32_t P, std::vector<uint32_t>& offu, uint32_t* offu_dev, bool codes = true) {
        const int W = c_->world, rank = c_->rank;
        const uint32_t pb = pr[rank], pe = pr[rank + 1];
        uint32_t* sizes = dev<uint32_t>(S_SIZES, P);
        uint32_t* h = pin<uint32_t>(P_OFF, P + 2);
        std::memset(h, 0, P * sizeof(uint32_t));
        for (uint32_t p = pb; p < pe; ++p) h[p] = offum[p - pb + 1] - offum[p - pb];
        SKY_CUDA(cudaMemcpyAsync(sizes, h, P * sizeof(uint32_t), cudaMemcpyHostToDevice, st_));
        c_->comm->allreduce_sum_u32(sizes, P, st_);
        SKY_CUDA(cudaMemcpyAsync(h, sizes, P * sizeof(uint32_t), cudaMemcpyDeviceToHost, st_));
        sync();
        offu.assign(P + 1, 0);
        for (uint32_t p = 0; p < P; ++p) offu[p + 1] = offu[p] + h[p];
        uint32_t* ho = stage<uint32_t>(P + 1);
        std::memcpy(ho, offu.data(), (P + 1) * sizeof(uint32_t));
        SKY_CUDA(cudaMemcpyAsync(offu_dev, ho, (P + 1) * sizeof(uint32_t), cudaMemcpyHostToDevice, st_));
        DevSet Ug = set(S_SET1, offu[P], D);
        std::vector<uint32_t> counts(W);
        for (int q = 0; q < W; ++q) counts[q] = offu[pr[q + 1]] - offu[pr[q]];
        allgather_set(D, Um, counts, Ug, codes);
        return Ug;
    }

    // All ranks' survivor ids (each rank's list from its candidate range),
    // concatenated and sorted ascending into `out`; returns the count.
    uint32_t gather_ids(const uint32_t* mine, uint32_t nmine, uint32_t* out) {
        const int W = c_->world;
        uint32_t* cnt = dev<uint32_t>(S_GCOUNT, W + 1);
        uint32_t* h = pin<uint32_t>(P_RUNS, W + 1);
        h[W] = nmine;
        SKY_CUDA(cudaMemcpyAsync(cnt + W, h + W, sizeof(uint32_t), cudaMemcpyHostToDevice, st_));
        c_->comm->allgather(cnt + W, cnt, sizeof(uint32_t), st_);
        SKY_CUDA(cudaMemcpyAsync(h, cnt, W * sizeof(uint32_t), cudaMemcpyDeviceToHost, st_));
        sync();
        std::vector<size_t> bytes(W), displ(W);
        uint32_t total = 0;
        for (int q = 0; q < W; ++q) {
            bytes[q] = (size_t)h[q] * sizeof(uint32_t);
            displ[q] = (size_t)total * sizeof(uint32_t);
            total += h[q];
        }
        uint32_t* all = dev<uint32_t>(S_PERM_A, total);
        c_->comm->allgatherv(mine, all, bytes.data(), displ.data(), st_);
        sort_keys(all, out, total, 32);
        return total;
    }

    // dominance-test and exact-check counters summed over ranks
    void reduce_counters() {
        uint32_t* misc = dev<uint32_t>(S_MISC, 64);
        c_->comm->allreduce_sum_u64(reinterpret_cast<uint64_t*>(misc + M_TESTS), 3, st_);
        c_->comm->allreduce_sum_u64(reinterpret_cast<uint64_t*>(misc + M_HITS), 4, st_);
    }

    // error bits of the prep pass OR-ed over ranks (every rank raises the
    // same error), returned on the host; an all-reduce of one word per bit
    uint32_t agree_errors(uint32_t mine) {
        if (c_->world == 1) return mine;
        uint32_t* dv = dev<uint32_t>(S_GCOUNT, 8);
        uint32_t* h = pin<uint32_t>(P_RUNS, 8);
        for (int k = 0; k < 4; ++k) h[k] = (mine >> k) & 1u;
        SKY_CUDA(cudaMemcpyAsync(dv, h, 4 * sizeof(uint32_t), cudaMemcpyHostToDevice, st_));
        c_->comm->allreduce_sum_u32(dv, 4, st_);
        SKY_CUDA(cudaMemcpyAsync(h, dv, 4 * sizeof(uint32_t), cudaMemcpyDeviceToHost, st_));
        sync();
        uint32_t e = 0;
        for (int k = 0; k < 4; ++k) e |= (h[k] ? 1u : 0u) << k;
        return e;
    }

    // partition_of of assign_random (partition.cpp:36-54) on the device; the
    // host reproduces it only if a draw would have been rejected.
    // deferred: a rejected draw sets misc[M_RFLAG] instead of a host round
    // trip; the caller redoes the run eagerly (host shuffle) when it is set
    uint32_t* random_pids(uint32_t n, uint64_t P, uint64_t seed, bool deferred = false) {
        uint32_t* pid = dev<uint32_t>(S_PID, n);
        void* scratch = c_->dev.get(S_RAND, random_scratch_bytes(n));
        const size_t cb = random_cub_bytes(n);
        void* ct = c_->dev.get(S_CUB, cb);
        const uint32_t* jt = nullptr;
        const uint32_t rows = mt_jump_chunks(n) ? mt_jump_chunks(n) - 1 : 0;
        if (n - 1 > (1u << 18) && rows) {
            if (c_->mt_jump_rows < rows) {
                const uint32_t* h = mt_jump_table(kJumpLog2, rows);  // host, built once per process
                if (c_->mt_jump) SKY_CUDA(cudaFree(c_->mt_jump));
                c_->mt_jump = nullptr;
                const size_t bytes = (size_t)rows * mt_jump_words() * sizeof(uint32_t);
                SKY_CUDA(cudaMalloc(&c_->mt_jump, bytes));
                SKY_CUDA(cudaMemcpy(c_->mt_jump, h, bytes, cudaMemcpyHostToDevice));
                c_->mt_jump_rows = rows;
            }
            jt = c_->mt_jump;
        }
        uint32_t* flag = deferred ? dev<uint32_t>(S_MISC, 64) + M_RFLAG : nullptr;
        if (!random_partition_gpu(n, P, seed, pid, scratch, ct, cb, c_->sm_count, st_, &c_->launches, jt, flag)) {
            uint32_t* h = pin<uint32_t>(P_PID, n);
            random_partition_of(n, P, seed, h);
            SKY_CUDA(cudaMemcpyAsync(pid, h, (size_t)n * sizeof(uint32_t), cudaMemcpyHostToDevice, st_));
            sync();
        }
        return pid;
    }

    // exact angular slice thresholds for m (host table cached per context)
    const double4* angular_table(uint64_t m) {
        if (m > kAngularExactMaxM) return nullptr;
        if (c_->ang_m != m) {
            c_->ang_host.resize(m - 1);
            angular_thresholds(m, c_->ang_host.data());
            c_->ang_m = m;
            c_->ang_dev_m = 0;
        }
        double4* t = dev<double4>(S_ANGT, m - 1);
        if (c_->ang_dev_m != m || c_->ang_dev_ptr != t) {
            SKY_CUDA(cudaMemcpy(t, c_->ang_host.data(), (m - 1) * sizeof(double4), cudaMemcpyHostToDevice));
            c_->ang_dev_m = m;
            c_->ang_dev_ptr = t;
        }
        return t;
    }

    unsigned long long* tests(int k) {
        return reinterpret_cast<unsigned long long*>(dev<uint32_t>(S_MISC, 64) + M_TESTS) + k;
    }

    // ------------------------------------------------------ local skylines
    // SFS restated for the GPU: the partition is already in (sum key) order;
    // (1) every block of kBlock rows keeps the rows no earlier-or-equal-key
    // row of the block dominates; (2) each block survivor is tested against
    // all block survivors of its partition with key <= its own. The result is
    // exactly the partition's local skyline (sfs, sequential.cpp:48-60).
    DevSet local_sfs(int D, const DevSet& s0, const std::vector<uint32_t>& off0, uint32_t* off0_dev, uint32_t P,
                     uint32_t* off_u_dev, std::vector<uint32_t>& off_u, bool count_tests) {
        uint8_t* dead = dev<uint8_t>(S_DEAD, s0.n);
        launch_fill_u8(dead, 0, s0.n, st_);
        Plan blocks;
        blocks.tile = D <= 16 ? 256u : (uint32_t)kTile;
        for (uint32_t p = 0; p < P; ++p)
            for (uint32_t b = off0[p]; b < off0[p + 1]; b += kBlock) {
                const uint32_t e = std::min(b + kBlock, off0[p + 1]);
                for (uint32_t c = b; c < e; c += blocks.tile) blocks.add(c, std::min(e, c + blocks.tile), {make_uint2(b, e)});
            }
        RelskyArgs a{};
        a.cxyz = s0.xyz; a.cskey = s0.skey; a.indirect = false;
        a.sxyz = s0.xyz; a.sskey = s0.skey; a.bounded = true; a.dead = dead;
        a.cid = s0.id; a.sid = s0.id;
        a.tests = count_tests ? tests(1) : nullptr;
        relsky(D, blocks, a, s0.qc, s0.qc);
        std::vector<uint32_t> off1;
        uint32_t* off1_dev = dev<uint32_t>(S_OFF_B, P + 1);
        DevSet s1 = compact(s0, dead, off0_dev, P, S_SET1, off1_dev, off1, D);

        uint8_t* dead1 = dev<uint8_t>(S_DEAD, s1.n);
        launch_fill_u8(dead1, 0, s1.n, st_);
        RelskyArgs b2 = a;
        b2.cxyz = s1.xyz; b2.cskey = s1.skey; b2.sxyz = s1.xyz; b2.sskey = s1.skey; b2.dead = dead1;
        b2.cid = s1.id; b2.sid = s1.id;
        if (D <= 16 && s1.qc) {
            uint64_t pairs = 0;
            for (uint32_t p = 0; p < P; ++p) pairs += (uint64_t)(off1[p + 1] - off1[p]) * (off1[p + 1] - off1[p]) / 2;
            uint32_t tile, chunk;
            pick_grain(D, s1.n, pairs, &tile, &chunk);
            relsky_waves(D, off1, 0, P, [&](uint32_t p, std::vector<uint2>& c) {
                c.assign(1, make_uint2(off1[p], off1[p + 1]));
            }, b2, s1.qc, s1.qc, tile, chunk, 2048);
        } else {
            Plan loc;
            for (uint32_t p = 0; p < P; ++p) {
                const uint32_t b0 = off1[p], e0 = off1[p + 1];
                for (uint32_t b = b0; b < e0; b += loc.tile) loc.add(b, std::min(b + loc.tile, e0), {make_uint2(b0, e0)});
            }
            loc.order();
            relsky(D, loc, b2);
        }
        return compact(s1, dead1, off1_dev, P, S_SET2, off_u_dev, off_u, D);
    }

    // BNL local skylines (k_bnl2), window capped at cfg.bnl_window_cap.
    // With opt.bnl_block > 0 (default) each partition (rows in key order) is
    // cut into blocks of at most that many rows and one CTA runs BNL per
    // block, so the grid covers every SM however few partitions there are;
    // then every block survivor is tested against the rows of its partition
    // with key <= its own (Prop. 2 of the paper applied inside a partition:
    // the partition's skyline is the union of the block skylines minus what
    // a row of another block dominates; a dominator never has a larger key,
    // so the earlier blocks and its own hold every possible one).
    DevSet local_bnl(int D, const DevSet& s0, uint32_t* off0_dev, uint32_t P, uint32_t window, uint32_t* off_u_dev,
                     std::vector<uint32_t>& off_u, bool count_tests, uint32_t* used_window,
                     uint32_t* n_u = nullptr) {
        uint8_t* dead = dev<uint8_t>(S_DEAD, s0.n);
        launch_fill_u8(dead, 1, s0.n, st_);
        const bool packed = D <= 16 && s0.qc;
        const uint32_t want = window ? window : 4096;
        const uint32_t cap = packed ? bnl2_window_fit(D, want, c_->smem_optin) : bnl_window_fit(D, want, c_->smem_optin);
        *used_window = cap;
        uint32_t block = c_->opt.bnl_block;
        if (block > cap) block = cap;  // a block always fits the window: one pass, no overflow
        const bool blocks = packed && block >= 64 && P <= 4096;
        // a block's survivors never outgrow the block: the window shrinks to
        // it (less shared memory, two CTAs per SM)
        const uint32_t wcap = blocks ? std::min(cap, (block + 3) & ~3u) : cap;
        // BNL segments: the partitions, or their blocks (count bounded by the capacity)
        const uint32_t segs = blocks ? P + ceil_div(s0.n, block) : P;
        uint32_t* seg_off = off0_dev;
        if (blocks) {
            seg_off = dev<uint32_t>(S_BNL_SEG, (size_t)segs + 1);
            launch_split_segments(off0_dev, P, block, seg_off, segs, st_);
            count();
        }
        const uint32_t grid = std::max<uint32_t>(1, std::min<uint32_t>(segs, (uint32_t)c_->sm_count *
                                                                                 (blocks ? 2u : 1u)));
        uint32_t* wpos = dev<uint32_t>(S_BNL_POS, (size_t)grid * cap);
        uint32_t* wmeta = dev<uint32_t>(S_BNL_META, (size_t)grid * cap);
        uint32_t* ovf = dev<uint32_t>(S_OVF, s0.n);
        uint32_t* misc = dev<uint32_t>(S_MISC, 64);
        SKY_CUDA(cudaMemsetAsync(misc + M_BNLCTR, 0, sizeof(uint32_t), st_));
        BnlArgs b{};
        b.xyz = s0.xyz;
        b.seg_off = seg_off;
        b.P = segs;
        b.window = wcap;
        b.dead = dead;
        b.overflow = ovf;
        b.tests = count_tests ? tests(1) : nullptr;
        b.hits = reinterpret_cast<unsigned long long*>(misc + M_HITS) + 1;
        b.x64 = x64_;
        b.id = s0.id;
        if (s0.n) {
            dom_begin();
            if (packed)
                launch_bnl2(D, b, s0.qc, s0.skey, wcap & ~3u, grid, misc + M_BNLCTR, st_);
            else
                launch_bnl_full(D, b, cap, grid, wpos, wmeta, misc + M_BNLCTR, st_);
            dom_end();
            count();
        }
        if (blocks && s0.n && indexed_partition_sky(D, s0, dead, off0_dev, P, s0_dims_, count_tests)) {
            // reconciled through the per-partition cell index
        } else if (blocks && s0.n) {
            // block survivors (dense, per partition) against their partition
            RelskyArgs a{};
            a.cxyz = s0.xyz; a.cskey = s0.skey; a.indirect = false;
            a.sxyz = s0.xyz; a.sskey = s0.skey; a.bounded = true; a.dead = dead;
            a.cid = s0.id; a.sid = s0.id;
            a.tests = count_tests ? tests(1) : nullptr;
            const uint32_t ncap = s0.n;
            uint32_t* dnew = dev<uint32_t>(S_DNEW, P + 1);
            uint32_t* dense = dev<uint32_t>(S_DENSE, ncap);
            launch_dense_compact(dead, ncap, off0_dev, P, 0, dense, dnew, nullptr,
                                 dev<uint32_t>(S_DCBT, dense_compact_scratch(ncap) / 4), st_);
            count(2);
            const uint64_t per = (uint64_t)ncap / std::max<uint32_t>(1, P);
            const uint32_t tile = per >= 512 ? 128 : 64, chunk = c_->opt.sfs_chunk, max_chunks = 64;
            const uint64_t icap = ((uint64_t)ncap / tile + P) * max_chunks;
            Item* items = dev<Item>(S_ITEMS, icap);
            uint32_t* ni = misc + M_NITEMS;
            const uint32_t icap32 = (uint32_t)std::min<uint64_t>(icap, 0xFFFFFFFFu);
            if (!launch_plan_partition_items(dnew, off0_dev, nullptr, P, 0, ~0ull, tile, chunk, max_chunks, icap32,
                                             items, ni, st_)) {
                Job* jobs = dev<Job>(S_JOBS, P);
                uint32_t* np_dev = misc + M_NP;
                uint32_t* hp = stage<uint32_t>(1);
                *hp = P;
                SKY_CUDA(cudaMemcpyAsync(np_dev, hp, sizeof(uint32_t), cudaMemcpyHostToDevice, st_));
                launch_partition_jobs(dnew, off0_dev, nullptr, P, 0, ~0ull, jobs, st_);
                count();
                const uint32_t* n_items = nullptr;
                items = expand_jobs(jobs, np_dev, P, tile, chunk, max_chunks, icap, &n_items);
                relsky_direct(D, tile, a, s0.qc, s0.qc, dense, items, icap, n_items);
            } else {
                count();
                relsky_direct(D, tile, a, s0.qc, s0.qc, dense, items, icap, ni);
            }
        }
        // rows past the live count stay dead (the fill above), so a capacity-
        // sized set compacts with the count on the device
        if (n_u) return compact_dev(s0, dead, off0_dev, P, S_SET2, off_u_dev, n_u, D);
        return compact(s0, dead, off0_dev, P, S_SET2, off_u_dev, off_u, D);
    }

    // Relative skyline of every live row of S against its own partition
    // through a per-partition cell index (the indexed merge of §4 applied
    // inside the partitions): the live rows in (partition, cell, key) order,
    // cells = one code bit on each of K dimensions (K = log2 of the mean
    // live rows per partition / 1024, at most d), each row tested against
    // the cells of its partition that weakly dominate its own, nearest
    // first, bounded by the tile's key. Sets dead[] of the dominated rows.
    // Two host round trips (the live count, the cell offsets). false: the
    // partitions are too small for an index; nothing was done.
    bool indexed_partition_sky(int D, const DevSet& S, uint8_t* dead, const uint32_t* off_dev, uint32_t P,
                               uint32_t d, bool count_tests) {
        if (D > 16 || !S.qc || !S.n || !P || P > 4096 || !c_->opt.merge_index) return false;
        const uint32_t pb = (uint32_t)std::max(1, bits_for(P));
        uint32_t K = 0;
        for (uint64_t v = (uint64_t)S.n / P / 1024; v >= 2 && K < d && K < 10; v /= 2) ++K;
        if (K < 2 || 32 + K + pb > 64) return false;
        CellSpec cs;
        cs.k = K;
        for (uint32_t t = 0; t < K; ++t) {
            cs.dim[t] = (uint8_t)t;
            cs.bits[t] = 1;
        }
        // live rows, dense per partition, and their count
        uint32_t* dense = dev<uint32_t>(S_DENSE, S.n);
        uint32_t* dnew = dev<uint32_t>(S_DNEW, P + 1);
        launch_dense_compact(dead, S.n, off_dev, P, 0, dense, dnew, nullptr,
                             dev<uint32_t>(S_DCBT, dense_compact_scratch(S.n) / 4), st_);
        count(2);
        uint32_t* h = pin<uint32_t>(P_SH_OFF, 2);
        SKY_CUDA(cudaMemcpyAsync(h, dnew + P, sizeof(uint32_t), cudaMemcpyDeviceToHost, st_));
        sync();
        const uint32_t nl = h[0];
        if (!nl) return true;
        uint64_t* k0 = dev<uint64_t>(S_RK0, nl);
        uint64_t* k1 = dev<uint64_t>(S_RK1, nl);
        uint32_t* v0 = dev<uint32_t>(S_RV0, nl);
        uint32_t* v1 = dev<uint32_t>(S_RV1, nl);
        uint32_t* rows2 = dev<uint32_t>(S_RP0, nl);
        launch_part_cell_keys(D, S.qc, S.skey, dense, dnew, P, nl, cs, k0, v0, st_);
        count();
        sort_pairs(k0, k1, v0, v1, nl, 0, (int)(32 + K + pb));
        launch_gather_u32(dense, v1, nl, rows2, st_);
        DevSet S2 = set(S_SET1, nl, D);
        DevSet Sv = S;
        Sv.n = nl;  // the gather runs over the nl picked rows (out[i] = S[rows2[i]])
        launch_gather_set(D, Sv, rows2, S2, st_);
        const uint32_t NS = P << K;
        uint32_t* soff = dev<uint32_t>(S_SOFF, NS + 1);
        launch_seg_offsets(k1, nl, NS, soff, st_);
        count(3);
        uint32_t* hs = pin<uint32_t>(P_SH_OFF, NS + 1);
        SKY_CUDA(cudaMemcpyAsync(hs, soff, (NS + 1) * sizeof(uint32_t), cudaMemcpyDeviceToHost, st_));
        sync();
        const std::vector<uint32_t> so(hs, hs + NS + 1);
        const std::vector<std::vector<uint32_t>>& dom = dominating_cells(cs);
        const uint32_t ncell = 1u << K;
        uint64_t pairs = 0;
        std::vector<std::vector<uint2>> lists(NS);
        for (uint32_t s = 0; s < NS; ++s) {
            if (so[s + 1] == so[s]) continue;
            const uint32_t base = s & ~(ncell - 1u), cell = s & (ncell - 1u);
            uint64_t cmp = 0;
            for (uint32_t c2 : dom[cell]) {
                const uint32_t s2 = base | c2;
                if (so[s2 + 1] > so[s2]) {
                    lists[s].push_back(make_uint2(so[s2], so[s2 + 1]));
                    cmp += so[s2 + 1] - so[s2];
                }
            }
            pairs += (uint64_t)(so[s + 1] - so[s]) * cmp / 2;
        }
        uint8_t* dead2 = dev<uint8_t>(S_DEAD2, nl);
        launch_fill_u8(dead2, 0, nl, st_);
        count();
        RelskyArgs a{};
        a.cxyz = S2.xyz; a.cskey = S2.skey; a.cid = S2.id; a.indirect = false;
        a.sxyz = S2.xyz; a.sskey = S2.skey; a.sid = S2.id; a.bounded = true; a.dead = dead2;
        a.tests = count_tests ? tests(1) : nullptr;
        uint32_t tile, chunk;
        pick_grain(D, nl, pairs, &tile, &chunk);
        relsky_waves(D, so, 0, NS, [&](uint32_t s, std::vector<uint2>& out) { out = lists[s]; }, a, S2.qc, S2.qc,
                     tile, chunk, c_->opt.sfs_head);
        launch_scatter_dead(dead2, rows2, nl, dead, st_);
        count();
        return true;
    }

   public:
    sky_ctx* c_;
    X64 x64_;  // FP64 input of the current run (null for float input)
    uint32_t s0_dims_ = 0;  // coordinates per row of the current run (d)
    cudaStream_t st_;
};

inline void validate(uint64_t n, uint32_t d, const sky_config* c) {  // engine.cpp:19-32
    if (c->workers < 1) throw Error(SKY_E_CONFIG, "worker count must be >= 1");
    if (c->p < 1) throw Error(SKY_E_CONFIG, "partition count must be >= 1");
    if (c->filter == SKY_FILTER_GRID && c->strategy != SKY_GRID)
        throw Error(SKY_E_CONFIG, "grid filtering requires the grid partitioning strategy");
    if (c->filter == SKY_FILTER_REPRESENTATIVE && c->rep_q < 1)
        throw Error(SKY_E_CONFIG, "representative count q must be >= 1");
    if (c->strategy == SKY_ANGULAR && n > 0 && d < 2) throw Error(SKY_E_DIMENSION, "angular partitioning needs d >= 2");
    if (c->strategy < 0 || c->strategy > 3) throw Error(SKY_E_CONFIG, "unknown partitioning strategy");
    if (c->filter < 0 || c->filter > 2) throw Error(SKY_E_CONFIG, "unknown filter kind");
    if (c->merge < 0 || c->merge > 1) throw Error(SKY_E_CONFIG, "unknown merge kind");
    if (c->local_algo < 0 || c->local_algo > 1) throw Error(SKY_E_CONFIG, "unknown local algorithm");
    if (c->filter == SKY_FILTER_REPRESENTATIVE &&
        (c->rep_selection < SKY_REPS_SORTED || c->rep_selection > SKY_REPS_RANDOM))
        throw Error(SKY_E_CONFIG, "unknown representative selection");
}

// Effective partition count and slices (make_assignment, partition.cpp:233-251).
inline void resolve_partitions(uint64_t n, uint32_t d, const sky_config* c, uint64_t* P, uint64_t* m) {
    *m = 0;
    switch (c->strategy) {
        case SKY_RANDOM:
            *P = c->p;
            break;
        case SKY_GRID: {
            *m = c->m > 0 ? c->m : snap_slices(c->p, d);
            if (*m < 1) throw Error(SKY_E_CONFIG, "slices per dimension must be >= 1");
            if (d < 1) throw Error(SKY_E_DIMENSION, "grid partitioning needs d >= 1");
            *P = checked_pow(*m, d);
            if (*P > kMaxPartitions) throw Error(SKY_E_CONFIG, "grid partition count m^d exceeds the supported maximum");
            break;
        }
        case SKY_ANGULAR: {
            if (d < 2) throw Error(SKY_E_DIMENSION, "angular partitioning needs d >= 2");
            *m = c->m > 0 ? c->m : snap_slices(c->p, d - 1);
            if (*m < 1) throw Error(SKY_E_CONFIG, "slices per dimension must be >= 1");
            *P = checked_pow(*m, d - 1);
            if (*P > kMaxPartitions)
                throw Error(SKY_E_CONFIG, "angular partition count m^(d-1) exceeds the supported maximum");
            break;
        }
        case SKY_SLICED:
            if (n > 0 && c->slice_dim >= d) throw Error(SKY_E_CONFIG, "slice dimension out of range");
            *P = c->p;
            break;
        default:
            throw Error(SKY_E_CONFIG, "unknown partitioning strategy");
    }
    if (*P > 0xFFFFFFF0ull) throw Error(SKY_E_CONFIG, "partition count too large");
}

// weak_grid_dominates over decoded cells (partition.cpp:87-116)
inline bool weak_grid_dom(uint64_t a, uint64_t b, uint64_t m, uint32_t d) {
    bool equal = true;
    for (uint32_t j = 0; j < d; ++j) {
        const uint64_t ca = a % m, cb = b % m;
        if (ca > cb) return false;
        if (ca != cb) equal = false;
        a /= m;
        b /= m;
    }
    return !equal;
}

struct RedoEager {};  // angular boundary points seen by a deferred prep
// stream path: a candidate bucket of kRepBucket slots filled up (a tie run of
// more than 1,024 minimum keys in one partition, e.g. duplicates clipped to
// a corner): the run is redone on the stream path with kRepBucketBig slots;
// if that overflows too, on the sorted path (RedoEager)
struct RedoBigBuckets {};
[[noreturn]] inline void throw_bucket_overflow(const sky_ctx* c) {
    if (c->rep_bucket < kRepBucketBig) throw RedoBigBuckets{};
    throw RedoEager{};
}

inline void check_prep(uint32_t err, uint32_t amb, int strategy, bool eager) {
    if (err & kErrNonFinite) throw Error(SKY_E_DATA, "coordinate must be finite and >= 0");
    if (err & kErrAboveOne) throw Error(SKY_E_DATA, "normalized dataset has coordinate > 1");
    if (err & kErrGridRange) throw Error(SKY_E_NORMALIZATION, "grid index needs coordinates in [0,1]");
    if (!eager && strategy == SKY_ANGULAR && amb) throw RedoEager{};
}

// Low bits cleared from the sum key in the (pid << 32 | skey) sort key, so
// the partition sort needs 32 - shift + pb bits: 24 (3 radix passes) up to
// 32 partitions (the key keeps >= 19 bits: 10 mantissa bits), else 32 (4
// passes) up to 2^12 partitions, else none. A coarser key only adds ties;
// every bounded test scans equal keys, so results do not depend on it.
inline uint32_t key_shift_for(uint64_t P) {
    const int pb = std::max(1, bits_for(P));
    if (pb <= 5) return (uint32_t)pb + 8;
    return pb <= 12 ? (uint32_t)pb : 0u;
}

// a range of input rows whose host->device copy completes at `ready`
struct InputChunk {
    uint32_t r0, r1;
    cudaEvent_t ready;
};

struct PartitionOut {
    uint64_t* key64;   // sorted (pid << 32 | skey)
    uint32_t* idx;     // row of each sorted position
    uint32_t* off;     // device offsets [P+1]
};

// Rows whose angular slice the device left open (the exact angle within the
// host libm's 1-ulp latitude of a boundary, or m > kAngularExactMaxM): one
// gather, one copy each way, the reference's formula (partition.cpp:118-148)
// on the host libm, and the partition ids patched into key64. Returns na.
inline uint32_t angular_fixups(Runner& R, const float* pts, uint32_t d, uint64_t m, uint64_t* key64,
                               const uint32_t* amb, uint32_t na) {
    if (!na) return 0;
    cudaStream_t st = R.st_;
    double* drows = R.dev<double>(S_AMBROWS, (size_t)na * d);
    launch_gather_rows_f64(pts, R.x64_.x, d, amb, na, 0, drows, st);
    R.count();
    double* hrows = R.pin<double>(P_AMB, (size_t)na * d + na);
    SKY_CUDA(cudaMemcpyAsync(hrows, drows, (size_t)na * d * sizeof(double), cudaMemcpyDeviceToHost, st));
    R.sync();
    uint32_t* hp = reinterpret_cast<uint32_t*>(hrows + (size_t)na * d);
    for (uint32_t k = 0; k < na; ++k) hp[k] = (uint32_t)angular_index_host(hrows + (size_t)k * d, d, m);
    uint32_t* dp = R.dev<uint32_t>(S_RUNS, na);
    SKY_CUDA(cudaMemcpyAsync(dp, hp, na * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
    launch_patch_pid(key64, amb, dp, na, st);
    R.count();
    R.sync();  // the pinned pids above are reused by later phases
    return na;
}

// Phase 1a: partition ids, sum keys, validation, sort into partitions.
inline PartitionOut partition_phase(Runner& R, const float* pts, uint32_t n, uint32_t d, int normalized, int strategy,
                             uint64_t P, uint64_t m, const sky_config* cfg, const uint32_t* pid_dev,
                             uint64_t* fixups, bool eager = true, uint32_t** scan_rows = nullptr,
                             bool sort_rows = true, uint32_t* gmin = nullptr,
                             const std::vector<InputChunk>* in_chunks = nullptr) {
    cudaStream_t st = R.st_;
    uint64_t* keyA = R.dev<uint64_t>(S_KEY_A, n);
    uint64_t* keyB = R.dev<uint64_t>(S_KEY_B, n);
    uint32_t* idxA = R.dev<uint32_t>(S_IDX_A, n);
    uint32_t* idxB = R.dev<uint32_t>(S_IDX_B, n);
    uint32_t* misc = R.dev<uint32_t>(S_MISC, 64);
    const uint32_t* pid_in = strategy == SKY_RANDOM ? pid_dev : nullptr;
    if (strategy == SKY_RANDOM && !pid_in && n) throw Error(SKY_E_INTERNAL, "random strategy without partition ids");
    // angular rows the device cannot decide (see angular_thresholds): the
    // list holds every row if need be
    const uint32_t amb_cap = strategy == SKY_ANGULAR ? std::max<uint32_t>(n, 1) : 1u;
    uint32_t* amb = R.dev<uint32_t>(S_AMB, amb_cap);
    uint32_t* skA = nullptr;
    if (strategy == SKY_SLICED) skA = R.dev<uint32_t>(S_SK_A, n);
    // sort key (pid << 32 | skey): with skey's low pb bits cleared the sort
    // needs 32 key bits (4 radix passes) for P <= 2^12 partitions
    const int pb = std::max(1, bits_for(P));
    const uint32_t key_shift = key_shift_for(P);
    PrepArgs pa{pts, R.x64_.x, n, d, strategy, m, normalized, pid_in, (uint32_t)cfg->slice_dim, keyA,
                sort_rows ? idxA : nullptr, skA, misc + M_ERR, misc + M_AMB, amb, amb_cap, key_shift};
    if (gmin) {
        pa.gmin = gmin;
        pa.P = (uint32_t)P;
    }
    if (strategy == SKY_ANGULAR && m >= 2) {
        pa.ang_thr = R.angular_table(m);
        volatile double one = 1.0;
        pa.ang_c45 = std::atan2(one, one);  // the host libm's atan2(x, x) (partition.cpp:128)
    }
    if (strategy == SKY_ANGULAR && m >= 2 && m <= 8) {
        // slice boundaries k*pi/(2m) as tan^2 (k = 1..m-1) for the FP32 filter
        const double PI = 3.14159265358979323846;
        for (uint64_t k = 1; k < m; ++k) {
            const double t = std::tan((double)k * PI / (2.0 * (double)m));
            pa.tan2[k - 1] = (float)(t * t);
        }
    }
    R.hbm_begin();
    if (in_chunks && !in_chunks->empty() && !gmin && !R.x64_.x) {
        // the rows arrive in chunks on the copy stream: each chunk's prep
        // starts as soon as its copy lands (overlapping the later copies)
        for (const InputChunk& ch : *in_chunks) {
            SKY_CUDA(cudaStreamWaitEvent(st, ch.ready, 0));
            PrepArgs pc = pa;
            pc.pts = pts + (size_t)ch.r0 * d;
            pc.n = ch.r1 - ch.r0;
            pc.row_base = ch.r0;
            launch_prep(pc, st, R.c_->sm_count);
        }
    } else {
        if (in_chunks)
            for (const InputChunk& ch : *in_chunks) SKY_CUDA(cudaStreamWaitEvent(st, ch.ready, 0));
        launch_prep(pa, st, R.c_->sm_count);
    }
    // rows read once; key (8 B) written, row index (4 B) when sorting follows
    R.hbm_end((uint64_t)n * d * (R.x64_.x ? 8 : 4) + (uint64_t)n * (sort_rows ? 12 : 8) +
              (strategy == SKY_SLICED ? 4ull * n : 0ull));
    R.count();

    // errors + angular boundary points (one host round trip). Deferred mode
    // skips the round trip: the caller checks M_ERR/M_AMB at its first sync
    // (check_prep) and reruns eagerly when angular boundary points need the
    // host libm. Kernels downstream tolerate a failed prep (pids clamped).
    uint32_t* hm = R.pin<uint32_t>(P_MISC, 8);
    if (eager || strategy == SKY_SLICED) {
        SKY_CUDA(cudaMemcpyAsync(hm, misc, 4 * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
        R.sync();
        check_prep(hm[M_ERR], 0, strategy, true);
    }
    if (eager && strategy == SKY_ANGULAR && hm[M_AMB])
        *fixups = angular_fixups(R, pts, d, m, keyA, amb, std::min(hm[M_AMB], amb_cap));

    if (strategy == SKY_SLICED && n > 0) {
        // rank order by (x[k], row): radix sort of the canonical float bits
        uint32_t* skB = R.dev<uint32_t>(S_SK_B, n);
        uint32_t* rankA = R.dev<uint32_t>(S_PERM_A, n);
        uint32_t* rankB = R.dev<uint32_t>(S_PERM_B, n);
        R.sort_pairs(skA, skB, idxA, rankA, n, 0, 32);
        // tie runs straddling slice boundaries need the (lex, id) order
        const uint32_t run_cap = (uint32_t)std::min<uint64_t>(P, 1u << 20);
        uint32_t* runs = R.dev<uint32_t>(S_RUNS, 2 * (size_t)run_cap);
        SKY_CUDA(cudaMemsetAsync(misc + M_RUNS, 0, sizeof(uint32_t), st));
        launch_slice_runs(skB, n, P, runs, misc + M_RUNS, run_cap, st);
        R.count();
        SKY_CUDA(cudaMemcpyAsync(hm, misc + M_RUNS, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
        R.sync();
        const uint32_t nruns = std::min(hm[0], run_cap);
        uint64_t cost = 0;
        uint32_t max_len = 0;
        std::vector<uint32_t> hr;
        if (nruns) {
            uint32_t* h = R.pin<uint32_t>(P_RUNS, 2 * (size_t)nruns);
            SKY_CUDA(cudaMemcpyAsync(h, runs, 2 * (size_t)nruns * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
            R.sync();
            for (uint32_t k = 0; k < nruns; ++k) {
                const uint64_t L = h[2 * k + 1] - h[2 * k];
                cost += L * L;
                max_len = std::max<uint32_t>(max_len, (uint32_t)L);
            }
        }
        if (cost <= (uint64_t)1e9 && !scan_rows && !R.x64_.x) {
            launch_slice_assign(rankA, n, P, keyA, st);
            R.count();
            launch_slice_fix_runs(pts, d, rankA, n, P, runs, nruns, max_len, keyA, st);
            if (nruns) R.count();
        } else {
            // full (x[k], x[0..d-1], row) order by LSD passes over the rows
            uint32_t* cur = rankB;
            uint32_t* other = rankA;
            SKY_CUDA(cudaMemcpyAsync(cur, idxA, (size_t)n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st));
            uint64_t* k64a = R.x64_.x ? R.dev<uint64_t>(S_RK0, n) : nullptr;
            uint64_t* k64b = R.x64_.x ? R.dev<uint64_t>(S_RK1, n) : nullptr;
            for (int j = (int)d - 1; j >= -1; --j) {
                const uint32_t col = j < 0 ? (uint32_t)cfg->slice_dim : (uint32_t)j;
                if (R.x64_.x) {
                    // FP64 input: canonical double bits, 64-bit LSD passes
                    launch_gather_coord_key64(R.x64_.x, d, col, cur, n, k64a, st);
                    R.count();
                    R.sort_pairs(k64a, k64b, cur, other, n, 0, 64);
                } else {
                    launch_gather_coord_key(pts, d, col, cur, n, skA, st);
                    R.count();
                    R.sort_pairs(skA, skB, cur, other, n, 0, 32);
                }
                std::swap(cur, other);
            }
            launch_slice_assign(cur, n, P, keyA, st);
            R.count();
            if (scan_rows) {
                // exact scan order (x[k], lex coords, id): split()'s order of
                // every slice (partition.cpp:203-216, 253-273)
                *scan_rows = R.dev<uint32_t>(S_SCAN, n);
                SKY_CUDA(cudaMemcpyAsync(*scan_rows, cur, (size_t)n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st));
            }
        }
    }

    // stream path: the keys stay in row order (only the survivors of the
    // representative filter are sorted, run_impl)
    if (!sort_rows) return PartitionOut{keyA, nullptr, nullptr};
    // one radix sort by (pid, sum key); stable, so ties keep row order
    const int end_bit = 32 + pb;
    R.sort_pairs(keyA, keyB, idxA, idxB, n, (int)key_shift, std::min(64, end_bit));
    uint32_t* off = R.dev<uint32_t>(S_OFF_A, P + 1);
    launch_seg_offsets(keyB, n, (uint32_t)P, off, st);
    R.count();
    return PartitionOut{keyB, idxB, off};
}

// Representative selection finished on the host side: compact the picked
// rows, sort them by sum key and prune them to an antichain
// (select_representatives_sorted + prune_dominated_reps, filter.cpp). Used
// when the P*q candidate slots do not fit the one-CTA k_rep_finalize.
inline DevSet host_reps(Runner& R, sky_ctx* c, int D, const uint32_t* cand, uint32_t slots, const float* pts, uint32_t d,
                 bool count_tests) {
    cudaStream_t st = R.st_;
    uint32_t* hc = R.pin<uint32_t>(P_IDS, slots);
    SKY_CUDA(cudaMemcpyAsync(hc, cand, (size_t)slots * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    R.sync();
    std::vector<uint32_t> rows;
    rows.reserve(slots);
    for (size_t k = 0; k < slots; ++k)
        if (hc[k] != kNone) rows.push_back(hc[k]);
    const uint32_t nc = (uint32_t)rows.size();
    uint32_t* drows = R.dev<uint32_t>(S_REPROWS, nc);
    std::memcpy(hc, rows.data(), nc * sizeof(uint32_t));
    SKY_CUDA(cudaMemcpyAsync(drows, hc, nc * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
    DevSet cs = R.set(S_SET3, nc, D);
    launch_gather_rows(D, pts, R.x64_.x, d, drows, nc, cs, st);
    R.count();
    DevSet css = R.set(S_SET1, nc, D);
    {
        uint32_t* iota = R.dev<uint32_t>(S_PERM_A, nc);
        uint32_t* perm = R.dev<uint32_t>(S_PERM_B, nc);
        uint32_t* hio = R.pin<uint32_t>(P_RUNS, nc);
        for (uint32_t k = 0; k < nc; ++k) hio[k] = k;
        SKY_CUDA(cudaMemcpyAsync(iota, hio, nc * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
        uint32_t* sk2 = R.dev<uint32_t>(S_SKTMP, nc);
        R.sort_pairs(cs.skey, sk2, iota, perm, nc, 0, 32);
        launch_gather_set(D, cs, perm, css, st);
        R.count();
    }
    uint8_t* cdead = R.dev<uint8_t>(S_CELLDEAD, nc);
    launch_fill_u8(cdead, 0, nc, st);
    if (launch_small_skyline(D, css.xyz, css.id, nc, cdead, count_tests ? R.tests(0) : nullptr, R.x64_,
                             c->smem_optin, st)) {
        R.count();
    } else {
        Plan pp;
        for (uint32_t b = 0; b < nc; b += kTile) pp.add(b, std::min(nc, b + (uint32_t)kTile), {make_uint2(0, nc)});
        RelskyArgs ra{};
        ra.cxyz = css.xyz; ra.cskey = css.skey; ra.sxyz = css.xyz; ra.sskey = css.skey;
        ra.cid = css.id; ra.sid = css.id;
        ra.bounded = true; ra.dead = cdead; ra.tests = count_tests ? R.tests(0) : nullptr;
        R.relsky(D, pp, ra);
    }
    std::vector<uint32_t> roff;
    uint32_t* doff = R.dev<uint32_t>(S_OFF_B, 4);
    uint32_t* hz = R.pin<uint32_t>(P_MISC, 8);
    hz[4] = 0;
    hz[5] = nc;
    SKY_CUDA(cudaMemcpyAsync(doff, hz + 4, 2 * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
    return R.compact(css, cdead, doff, 1, S_SET3, doff + 2, roff, D);
}

// select_representatives_region (filter.cpp:88-115): per partition the
// first q rows by (volume desc, id asc). Two stable radix sorts: rows by
// ~volume bits, then by partition.
inline void region_candidates(Runner& R, const float* pts, uint32_t d, uint32_t n, const PartitionOut& po, uint32_t P,
                       uint32_t q, uint32_t* cand) {
    cudaStream_t st = R.st_;
    uint64_t* k0 = R.dev<uint64_t>(S_RK0, n);
    uint64_t* k1 = R.dev<uint64_t>(S_RK1, n);
    uint32_t* v0 = R.dev<uint32_t>(S_RV0, n);
    uint32_t* v1 = R.dev<uint32_t>(S_RV1, n);
    uint32_t* p0 = R.dev<uint32_t>(S_RP0, n);
    uint32_t* p1 = R.dev<uint32_t>(S_RP1, n);
    uint32_t* pid_row = R.dev<uint32_t>(S_ROWPID, n);
    launch_region_keys(pts, R.x64_.x, d, n, k0, v0, st);
    launch_row_pid(po.key64, po.idx, n, pid_row, st);
    R.count(2);
    R.sort_pairs(k0, k1, v0, v1, n, 0, 64);
    launch_gather_u32(pid_row, v1, n, p0, st);
    R.count();
    R.sort_pairs(p0, p1, v1, v0, n, 0, std::max(1, bits_for(P)));
    launch_pick_first(v0, po.off, P, q, cand, st);
    R.count();
}

// select_representatives_random (filter.cpp:117-137): the per-partition Rng
// draws (rng.hpp:40-47, std::mt19937_64) are q sequential host draws per
// partition; the picked scan positions are mapped to rows on the device.
// Scan order: row order within a partition (split, partition.cpp:262-265),
// or the exact sliced order when `scan` is given (partition.cpp:266-270).
inline void random_candidates(Runner& R, uint32_t n, const PartitionOut& po, uint32_t P, uint32_t q, const uint32_t* scan,
                       uint64_t seed, uint32_t* cand) {
    cudaStream_t st = R.st_;
    const uint32_t* rows = scan;
    if (!rows) {
        uint32_t* pid_row = R.dev<uint32_t>(S_ROWPID, n);
        uint32_t* p1 = R.dev<uint32_t>(S_RP1, n);
        uint32_t* v0 = R.dev<uint32_t>(S_RV0, n);
        uint32_t* v1 = R.dev<uint32_t>(S_RV1, n);
        launch_row_pid(po.key64, po.idx, n, pid_row, st);
        launch_iota(n, v0, st);
        R.count(2);
        R.sort_pairs(pid_row, p1, v0, v1, n, 0, std::max(1, bits_for(P)));
        rows = v1;
    }
    uint32_t* h = R.pin<uint32_t>(P_OFF, P + 2);
    SKY_CUDA(cudaMemcpyAsync(h, po.off, (P + 1) * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    R.sync();
    const uint32_t slots = P * q;
    uint32_t* gpos = R.stage<uint32_t>(slots);
    std::unordered_map<uint64_t, uint64_t> swapped;
    for (uint32_t p = 0; p < P; ++p) {
        const uint64_t size = h[p + 1] - h[p];
        const uint32_t take = (uint32_t)std::min<uint64_t>(q, size);
        for (uint32_t k = take; k < q; ++k) gpos[(size_t)p * q + k] = kNone;
        if (!size) continue;
        std::mt19937_64 eng(seed ^ (0x9e3779b97f4a7c15ULL * ((uint64_t)p + 1)));
        swapped.clear();
        auto at = [&](uint64_t i) {
            auto it = swapped.find(i);
            return it == swapped.end() ? i : it->second;
        };
        for (uint32_t k = 0; k < take; ++k) {
            // Rng::below(size - k) by rejection
            const uint64_t range = size - k;
            const uint64_t limit = UINT64_MAX - UINT64_MAX % range;
            uint64_t x;
            do {
                x = eng();
            } while (x >= limit);
            const uint64_t j = k + x % range;
            const uint64_t vk = at(k), vj = at(j);
            swapped[k] = vj;
            swapped[j] = vk;
            gpos[(size_t)p * q + k] = h[p] + (uint32_t)vj;
        }
    }
    uint32_t* dg = R.dev<uint32_t>(S_GPOS, slots);
    SKY_CUDA(cudaMemcpyAsync(dg, gpos, (size_t)slots * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
    launch_pick_gather(rows, dg, slots, cand, st);
    R.count();
}


// Cell index of the union for the merge: K = log2(|U| / cell_rows) digit
// bits (at most 12 and d), one per dimension in turn (the slice dimension
// first for sliced partitioning); no index below 16k rows. Halves on many
// dimensions prune more pairs than quartiles on few: on C4's union one bit
// on each of the 10 dimensions leaves half the comparisons of two bits on 5.
inline CellSpec cell_spec(uint32_t nU, uint32_t d, int D, const sky_config* cfg, uint32_t cell_rows) {
    CellSpec cs;
    if (D > 16 || nU < 16384 || !cell_rows || d == 0) return cs;
    uint32_t K = 0;
    for (uint64_t v = nU / cell_rows; v >= 2 && K < 12; v /= 2) ++K;
    K = std::min<uint32_t>(K, 2 * std::min<uint32_t>(d, 16));
    if (K > d) K = d;  // measured on C4: a second bit on some dimensions adds more ranges than it prunes
    if (!K) return cs;
    const uint32_t first = cfg->strategy == SKY_SLICED && cfg->slice_dim < d ? (uint32_t)cfg->slice_dim : 0;
    const uint32_t nd = std::min<uint32_t>(d, 16);
    std::vector<uint32_t> order(1, first);
    for (uint32_t j = 0; j < nd; ++j)
        if (j != first) order.push_back(j);
    cs.k = std::min(K, nd);
    for (uint32_t t = 0; t < cs.k; ++t) {
        cs.dim[t] = (uint8_t)order[t];
        cs.bits[t] = 1;
    }
    for (uint32_t t = 0, extra = K - cs.k; t < cs.k && extra; ++t, --extra) cs.bits[t] = 2;
    return cs;
}

// The final phase (merge_sequential / merge_noseq, engine.cpp:190-194) and
// the result record. U: the union of the local skylines in partition order
// (offsets offu / offu_dev), identical on every rank; with world > 1 each
// rank tests its share of the candidates and the survivors are gathered.
inline void merge_phase(Runner& R, sky_ctx* c, const sky_config* cfg, DevSet U, const std::vector<uint32_t>& offu,
                        uint32_t* offu_dev, uint32_t P, uint64_t m, uint32_t d, int D, uint32_t n, bool count_tests,
                        bool us_early, sky_result* out) {
    cudaStream_t st = c->stream;
    const int W = c->world, rank = c->rank;
    uint32_t* misc = R.dev<uint32_t>(S_MISC, 64);

    SKY_CUDA(cudaEventRecord(c->ev[2], st));
    for (uint32_t p = 0; p < P; ++p) out->local_skyline_sizes[p] = offu[p + 1] - offu[p];
    out->union_size = U.n;

    // ---------------------------------------------------------------- merge
    uint8_t* fdead = R.dev<uint8_t>(S_CELLDEAD, U.n);
    launch_fill_u8(fdead, 0, U.n, st);
    RelskyArgs ma{};
    ma.cxyz = U.xyz; ma.cskey = U.skey; ma.bounded = true; ma.dead = fdead;
    ma.cid = U.id; ma.sid = U.id;
    ma.tests = count_tests ? R.tests(2) : nullptr;
    Plan mp;
    const bool all_mode = cfg->merge == SKY_MERGE_SEQUENTIAL || cfg->strategy == SKY_RANDOM ||
                          cfg->strategy == SKY_ANGULAR;
    std::vector<uint32_t> nonempty;
    for (uint32_t p = 0; p < P; ++p)
        if (offu[p + 1] > offu[p]) nonempty.push_back(p);
    // the merge is sharded by candidate partitions, balanced by test volume
    const std::vector<uint32_t> mr = plan_merge_shards(offu, P, W, all_mode, cfg->strategy, m, d);
    const uint32_t qb = mr[rank], qe = mr[rank + 1];
    {
        uint64_t pairs = 0, cands = offu[qe] - offu[qb];
        std::vector<uint2> comps;
        for (uint32_t i = qb; i < qe; ++i) {
            const uint64_t ni = offu[i + 1] - offu[i];
            if (!ni) continue;
            if (all_mode) {
                pairs += ni * (uint64_t)U.n / 2;
            } else {
                pd_ranges(offu, nonempty, i, cfg->strategy, m, d, comps);
                for (uint2 r : comps) pairs += ni * (r.y - r.x) / 2;
            }
        }
        R.pick_grain(D, cands, pairs, &mp.tile, &mp.chunk);
    }
    const CellSpec cells = cell_spec(U.n, d, D, cfg, c->opt.merge_cell_rows);
    const bool indexed = P > 1 && D <= 16 && U.qc && cells.k > 0 && c->opt.merge_index;
    DevSet US;
    if (all_mode && P > 1 && !indexed) {
        // Sky(U) against the whole union sorted by sum key: for random and
        // angular pd_i is every other local (engine.cpp:98-103) and u_i is an
        // antichain, so testing against all of U is the same relation;
        // merge_sequential (engine.cpp:65-72) is Sky(U) by definition.
        // U's partitions are runs sorted by key: one stable P-way merge
        US = R.set(S_SET3, U.n, D);  // the same buffers as the early merge's (grow-only arena)
        if (!us_early) {
            launch_merge_runs(D, U, offu_dev, P, US, st);
            R.count();
        }
        ma.sxyz = US.xyz; ma.sskey = US.skey; ma.sid = US.id;
    } else if (P > 1) {
        ma.sxyz = U.xyz; ma.sskey = U.skey;
    }
    // Indexed Sky(U). Every merge kind yields Sky(U): the u_i are antichains
    // and pd_i (engine.cpp:74-114) holds every row of U that can dominate a
    // row of u_i (random / angular: all of U; grid: the weakly dominating
    // cells; sliced: the earlier slices, since s < t implies s <lex t), and a
    // comparison with any other row of U cannot change a test. So U is
    // ordered by (cell, key), cells = the quartiles of k code dimensions
    // (4^k cells), and a row is tested only against the cells that weakly
    // dominate its own (s <= t implies cell(s) <= cell(t) digit by digit),
    // each range bounded by the tile's key.
    DevSet UC;
    std::vector<uint32_t> coff;
    uint32_t icb = 0, ice = 0;  // this rank's cells
    if (indexed) {
        UC = R.set(S_SET3, U.n, D);
        uint64_t* k0 = R.dev<uint64_t>(S_RK0, U.n);
        uint64_t* k1 = R.dev<uint64_t>(S_RK1, U.n);
        uint32_t* v0 = R.dev<uint32_t>(S_RV0, U.n);
        uint32_t* v1 = R.dev<uint32_t>(S_RV1, U.n);
        launch_cell_keys(D, U.qc, U.skey, U.n, cells, k0, v0, st);
        R.count();
        const uint32_t ncell = 1u << cells.total_bits();
        R.sort_pairs(k0, k1, v0, v1, U.n, 0, 32 + (int)cells.total_bits());
        launch_gather_set(D, U, v1, UC, st);
        uint32_t* coff_dev = R.dev<uint32_t>(S_OFF_C, ncell + 1);
        launch_seg_offsets(k1, U.n, ncell, coff_dev, st);
        R.count(2);
        uint32_t* h = R.pin<uint32_t>(P_SH_OFF, ncell + 1);
        SKY_CUDA(cudaMemcpyAsync(h, coff_dev, (ncell + 1) * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
        R.sync();
        coff.assign(h, h + ncell + 1);
        // per cell: the non-empty weakly dominating cells, nearest first
        const std::vector<std::vector<uint32_t>>& dom = dominating_cells(cells);
        std::vector<std::vector<uint2>> lists(ncell);
        std::vector<uint64_t> cmp_rows(ncell, 0);
        for (uint32_t cell = 0; cell < ncell; ++cell) {
            if (coff[cell + 1] == coff[cell]) continue;
            lists[cell].reserve(dom[cell].size());  // one allocation per cell (the device idles while this runs)
            for (uint32_t id : dom[cell])
                if (coff[id + 1] > coff[id]) {
                    lists[cell].push_back(make_uint2(coff[id], coff[id + 1]));
                    cmp_rows[cell] += coff[id + 1] - coff[id];
                }
        }
        // each cell's list is asked for once (relsky_waves): handed over, not copied
        auto comps_of = [&](uint32_t cell, std::vector<uint2>& out) { out = std::move(lists[cell]); };
        // cells split over the ranks by test volume (candidates x comparators)
        const std::vector<uint32_t> cr = plan_ranges(coff, ncell, W, [&](uint32_t cell) -> uint64_t {
            const uint64_t nc = coff[cell + 1] - coff[cell];
            return nc ? nc * (cmp_rows[cell] / 2 + 1) : 0;
        });
        icb = cr[rank];
        ice = cr[rank + 1];
        uint64_t pairs = 0;
        for (uint32_t cell = icb; cell < ice; ++cell) pairs += (uint64_t)(coff[cell + 1] - coff[cell]) * cmp_rows[cell] / 2;
        R.pick_grain(D, coff[ice] - coff[icb], pairs, &mp.tile, &mp.chunk);
        if (c->opt.merge_tile) mp.tile = c->opt.merge_tile;
        ma.cxyz = UC.xyz; ma.cskey = UC.skey; ma.cid = UC.id;
        ma.sxyz = UC.xyz; ma.sskey = UC.skey; ma.sid = UC.id;
        R.relsky_waves(D, coff, icb, ice, comps_of, ma, UC.qc, UC.qc, mp.tile, mp.chunk, c->opt.merge_head);
    }
    // single GPU, all-pairs merge: the candidates are the union itself in
    // global key order, so a tile's key bound is as tight as it can be
    const bool global_cands = !indexed && W == 1 && all_mode && P > 1 && D <= 16 && U.qc;
    if (indexed) {
    } else if (global_cands) {
        ma.cxyz = US.xyz; ma.cskey = US.skey; ma.cid = US.id;
        const std::vector<uint32_t> offg = {0, U.n};
        R.relsky_waves(D, offg, 0, 1, [&](uint32_t, std::vector<uint2>& c) { c.assign(1, make_uint2(0, U.n)); },
                       ma, US.qc, US.qc, mp.tile, mp.chunk, c->opt.merge_head);
    } else if (P > 1) {
        const uint2* sq = all_mode ? US.qc : U.qc;
        auto comps_of = [&](uint32_t i, std::vector<uint2>& c) {
            if (all_mode)
                c.assign(1, make_uint2(0, U.n));
            else
                pd_ranges(offu, nonempty, i, cfg->strategy, m, d, c);
        };
        if (D <= 16 && U.qc) {
            // wave A: the nearest slice / cell (or the strongest keys of the
            // union), wave B: the rest over dense tiles of survivors
            std::vector<uint2> c0;
            uint32_t head = c->opt.merge_head;
            if (!all_mode)
                for (uint32_t i = qb; i < qe; ++i) {
                    comps_of(i, c0);
                    if (!c0.empty()) head = std::max(head, c0[0].y - c0[0].x);
                }
            R.relsky_waves(D, offu, qb, qe, comps_of, ma, U.qc, sq, mp.tile, mp.chunk, head);
        } else {
            std::vector<uint2> comps;
            for (uint32_t i = qb; i < qe; ++i) {
                if (offu[i + 1] == offu[i]) continue;
                comps_of(i, comps);
                if (comps.empty()) continue;
                for (uint32_t b = offu[i]; b < offu[i + 1]; b += mp.tile)
                    mp.add(b, std::min(offu[i + 1], b + mp.tile), comps, mp.chunk);
            }
            mp.order();
            R.relsky(D, mp, ma);
        }
    }

    // surviving ids of this rank's candidates, ascending (engine.cpp:128-133)
    const uint32_t cb = indexed ? coff[icb] : global_cands ? 0 : offu[qb];
    const uint32_t cn = indexed ? coff[ice] - cb : global_cands ? U.n : offu[qe] - cb;
    const uint32_t* cand_ids = indexed ? UC.id : global_cands ? US.id : U.id;
    uint32_t* hm = R.pin<uint32_t>(P_MISC, 32);
    uint32_t* idsA = R.dev<uint32_t>(S_IDS_A, std::max<uint32_t>(cn, 1));
    uint32_t* idsB = R.dev<uint32_t>(S_IDS_B, std::max<uint32_t>(cn, 1));
    uint32_t nf = 0, n_copy = 0;
    uint32_t* final_ids = idsB;
    if (W == 1) {
        // no round trip: ascending ids through a bitmap over the row ids,
        // written into a cn-slot buffer; the count travels back with them
        uint32_t* bm = R.dev<uint32_t>(S_BM, (size_t)n / 32 + 1);
        uint32_t* bt = R.dev<uint32_t>(S_BMT, bm_blocks(n));
        launch_ids_bitmap(cand_ids + cb, fdead + cb, cn, n, bm, bt, idsB, misc + M_TOTAL, st);
        R.count(cn ? 3 : 2);
        n_copy = cn;
    } else {
        uint32_t* pos = R.dev<uint32_t>(S_POS, cn);
        R.scan_live(fdead + cb, pos, cn);
        launch_count_total(pos, fdead + cb, cn, misc + M_TOTAL, st);
        R.count();
        SKY_CUDA(cudaMemcpyAsync(hm, misc + M_TOTAL, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
        R.sync();
        const uint32_t nmine = cn ? hm[0] : 0;
        launch_compact_ids(cand_ids + cb, fdead + cb, pos, cn, idsA, st);
        R.count();
        uint32_t* all = R.dev<uint32_t>(S_IDS_B, std::max<uint32_t>(U.n, 1));
        nf = R.gather_ids(idsA, nmine, all);  // all ranks' survivors, then sorted
        final_ids = all;
        n_copy = nf;
        R.reduce_counters();
    }
    SKY_CUDA(cudaEventRecord(c->ev[3], st));
    uint32_t* hid = R.pin<uint32_t>(P_IDS, n_copy);
    SKY_CUDA(cudaMemcpyAsync(hid, final_ids, (size_t)n_copy * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    SKY_CUDA(cudaMemcpyAsync(hm, misc + M_TOTAL, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    unsigned long long* ht = reinterpret_cast<unsigned long long*>(hm + 4);
    SKY_CUDA(cudaMemcpyAsync(ht, R.tests(0), 3 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    SKY_CUDA(cudaMemcpyAsync(ht + 3, misc + M_HITS, 4 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    SKY_CUDA(cudaEventRecord(c->ev[4], st));
    R.sync();
    if (W == 1) nf = cn ? hm[0] : 0;
    out->d2h_bytes += (uint64_t)n_copy * sizeof(uint32_t);
    out->ids = alloc_ids(nf);
    for (uint32_t i = 0; i < nf; ++i) out->ids[i] = hid[i];
    out->n_ids = out->final_size = nf;
    out->tests_reps = ht[0];
    out->tests_local = ht[1];
    out->tests_merge = ht[2];
    float ms = 0;
    cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]);
    out->partition_ms = ms;
    cudaEventElapsedTime(&ms, c->ev[1], c->ev[2]);
    out->local_ms = ms;
    cudaEventElapsedTime(&ms, c->ev[2], c->ev[3]);
    out->merge_ms = ms;
    cudaEventElapsedTime(&ms, c->ev[0], c->ev[4]);
    out->total_ms = ms;
    out->kernel_launches = c->launches;
    out->dom_launches = c->dom_launches;
    R.dom_collect();
    out->stream_kernel_ms = R.hbm_collect();
    out->stream_bytes = c->hbm_bytes;
    out->stream_launches = c->hbm_launches;
    R.timeline_dump();
    out->dom_kernel_ms = c->dom_ms;
    out->dom_tests = ht[0] + ht[1] + ht[2];
    out->dom_exact_checks = ht[3] + ht[4] + ht[5] + ht[6];
    out->exact_checks_merge = ht[5];
}

// ---------------------------------------------------------- sharded run
// shard.cu: phase 1 over each rank's own rows.
// first row of rank r when N rows are spread evenly over W ranks
inline uint64_t shard_row(uint64_t N, int r, int W) { return N * (uint64_t)r / (uint64_t)W; }
struct ReplicatePhase1 {};  // thrown (on every rank alike) when the input needs the replicated phase 1
bool sharded_eligible(const sky_config* cfg, uint64_t N, uint32_t d, bool f64);
// src: this rank's rows (host or device), rows_of[r]: rows of every rank
void run_sharded(sky_ctx* c, const float* src, uint32_t nl, uint32_t row0, const std::vector<uint32_t>& rows_of,
                 uint32_t d, int normalized, int on_device, const sky_config* cfg, sky_result* out);

}  // namespace eng
}  // namespace sky
