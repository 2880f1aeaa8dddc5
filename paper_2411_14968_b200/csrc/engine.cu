// engine.cu — host orchestration of the two-phase skyline on one B200 and the
// C ABI (include/skyline_b200.h).
//
// Mirrors skyline::run (reference engine.cpp:136-204) phase by phase:
//   partition   make_assignment + split      -> k_prep (+ sliced rank sort), one
//                                                radix sort by (pid, sum key)
//   local       select_representatives_sorted -> k_rep_pick, prune via k_relsky
//               rep_prefilter                 -> k_relsky over all rows (indirect)
//               sfs / sfs_presorted           -> block skylines + in-partition
//                                                relative skyline (k_relsky), or
//                                                BNL (k_bnl)
//   merge       merge_sequential / merge_noseq -> k_relsky against the union
//               + potential_dominators           (or per-strategy pd segments)
// The host side plans work items from partition offsets (one device->host
// read per phase); all dominance tests run on the GPU.
#include <cub/cub.cuh>
#include "engine_impl.cuh"

#include <condition_variable>
#include <functional>
#include <mutex>

using namespace sky;
using namespace sky::eng;

// A group context (sky_ctx_create_group): one process driving several GPUs.
// Rank r is an ordinary context on devices[r]; ranks 1.. run on persistent
// worker threads, rank 0 on the caller's thread.
struct sky_group {
    std::vector<int> devices;
    bool loopback = false;
    std::vector<sky_ctx*> ranks;
    std::vector<std::thread> workers;
    std::mutex mu;
    std::condition_variable cv, done_cv;
    uint64_t gen = 0;
    int pending = 0;
    bool stop = false;
    std::function<void(int)> job;
};

namespace {

void run_impl(sky_ctx* c, const void* points, uint64_t n64, uint32_t d, int normalized, int on_device,
              const sky_config* cfg, sky_result* out, bool eager = false, bool f64 = false) {
    std::memset(out, 0, sizeof(*out));
    validate(n64, d, cfg);
    uint64_t P64 = 0, m = 0;
    resolve_partitions(n64, d, cfg, &P64, &m);
    if (n64 >= 0xFFFFFFF0ull) throw Error(SKY_E_DATA, "at most 2^32-16 points per run");
    const uint32_t n = (uint32_t)n64;
    const uint32_t P = (uint32_t)P64;
    out->effective_p = P;
    out->input_size = n;
    out->input_dim = d;
    out->local_skyline_sizes = static_cast<uint64_t*>(std::calloc(P ? P : 1, sizeof(uint64_t)));
    c->launches = 0;
    c->dom_launches = 0;
    c->dom_ms = 0.0;
    const bool count_tests = cfg->count_tests != 0;

    if (n == 0 || d == 0) {
        // d == 0: no coordinate can be strictly better, nothing is dominated
        // (dominates_raw core.hpp:89-96); every row is its own local skyline.
        out->ids = alloc_ids(n);
        for (uint32_t i = 0; i < n; ++i) out->ids[i] = i;
        out->n_ids = out->final_size = out->union_size = n;
        if (n && cfg->strategy == SKY_RANDOM) {
            std::vector<uint32_t> pid(n);
            random_partition_of(n, P, cfg->seed, pid.data());
            for (uint32_t i = 0; i < n; ++i) out->local_skyline_sizes[pid[i]]++;
        } else if (n) {
            out->local_skyline_sizes[0] = n;
        }
        return;
    }
    const int D = padded_dim(d);
    if (!D) throw Error(SKY_E_DIMENSION, "the GPU engine supports d <= 32");

    Runner R(c);
    R.s0_dims_ = d;
    cudaStream_t st = c->stream;
    if (R.tl_) R.mark(__LINE__);

    SKY_CUDA(cudaEventRecord(c->ev[0], st));
    uint32_t* misc = R.dev<uint32_t>(S_MISC, 64);
    SKY_CUDA(cudaMemsetAsync(misc, 0, 64 * sizeof(uint32_t), st));
    const float* pts = static_cast<const float*>(points);
    if (f64) {
        // FP64 rows: keep the doubles for exact decisions, run the layout,
        // keys, codes and coarse tests on their float32 image
        const double* p64 = static_cast<const double*>(points);
        if (!on_device) {
            double* dp64 = R.dev<double>(S_PTS64, (size_t)n * d);
            SKY_CUDA(cudaMemcpyAsync(dp64, points, (size_t)n * d * sizeof(double), cudaMemcpyHostToDevice, st));
            p64 = dp64;
            out->h2d_bytes += (uint64_t)n * d * sizeof(double);
        }
        float* dp = R.dev<float>(S_PTS, (size_t)n * d);
        launch_round_rows(p64, (size_t)n * d, dp, st);
        R.count();
        pts = dp;
        R.x64_ = X64{p64, d};
    }
    // random partitioning does not read the rows: their copy runs on the
    // side stream, overlapped with the partitioner, and joins before prep
    const bool overlap_copy = !f64 && !on_device && cfg->strategy == SKY_RANDOM && c->copy;
    std::vector<InputChunk> in_chunks;
    if (!f64 && !on_device) {
        float* dp = R.dev<float>(S_PTS, (size_t)n * d);
        // copies of 4+ MB in four chunks on the side stream: the prep of a
        // chunk runs while the next one is copied (partition_phase)
        const bool chunked = !overlap_copy && c->copy && c->chunk_ev[0] && (uint64_t)n * d * 4 >= (4ull << 20);
        if (chunked) {
            SKY_CUDA(cudaEventRecord(c->fork_ev, st));
            SKY_CUDA(cudaStreamWaitEvent(c->copy, c->fork_ev, 0));
            const uint32_t per = (ceil_div(n, 4) + 255) & ~255u;
            for (uint32_t k = 0; k < 4; ++k) {
                const uint32_t r0 = std::min(n, k * per), r1 = std::min(n, r0 + per);
                if (r0 >= r1) break;
                SKY_CUDA(cudaMemcpyAsync(dp + (size_t)r0 * d, static_cast<const float*>(points) + (size_t)r0 * d,
                                         (size_t)(r1 - r0) * d * sizeof(float), cudaMemcpyHostToDevice, c->copy));
                SKY_CUDA(cudaEventRecord(c->chunk_ev[k], c->copy));
                in_chunks.push_back(InputChunk{r0, r1, c->chunk_ev[k]});
            }
        } else if (overlap_copy) {
            SKY_CUDA(cudaEventRecord(c->fork_ev, st));
            SKY_CUDA(cudaStreamWaitEvent(c->copy, c->fork_ev, 0));
            SKY_CUDA(cudaMemcpyAsync(dp, points, (size_t)n * d * sizeof(float), cudaMemcpyHostToDevice, c->copy));
            SKY_CUDA(cudaEventRecord(c->join_ev, c->copy));
        } else {
            SKY_CUDA(cudaMemcpyAsync(dp, points, (size_t)n * d * sizeof(float), cudaMemcpyHostToDevice, st));
        }
        pts = dp;
        out->h2d_bytes += (uint64_t)n * d * sizeof(float);
    }
    const bool defer_rand = !eager && c->world == 1;
    const uint32_t* pid_dev = cfg->strategy == SKY_RANDOM ? R.random_pids(n, P, cfg->seed, defer_rand) : nullptr;
    if (overlap_copy) SKY_CUDA(cudaStreamWaitEvent(st, c->join_ev, 0));
    const bool rep_random = cfg->filter == SKY_FILTER_REPRESENTATIVE && cfg->rep_selection == SKY_REPS_RANDOM;
    uint32_t* scan_rows = nullptr;  // sliced + random reps: split()'s exact scan order
    // Stream path (single GPU, sorted representatives, large input): no sort
    // of every row. Representatives come from per-partition candidate
    // buckets, the prefilter streams the rows in row order and appends the
    // survivors' (partition, key, row) sort keys, and only the survivors are
    // sorted into partitions. The same s0 as the sorted path (stable order).
    bool stream = false;
    {
        const int pb = std::max(1, bits_for(P));
        const bool want = c->opt.stream >= 0 ? c->opt.stream == 1 : (uint64_t)n * d * sizeof(float) > (32ull << 20);
        stream = want && !eager && c->world == 1 && !f64 && cfg->filter == SKY_FILTER_REPRESENTATIVE &&
                 cfg->rep_selection == SKY_REPS_SORTED && cfg->strategy != SKY_SLICED && pb <= 12 &&
                 (uint64_t)P * std::min<uint64_t>(cfg->rep_q, n) <= 2048 && cfg->rep_q <= 64 && D <= 16 &&
                 ((uintptr_t)pts & 15) == 0 && (uint64_t)P * c->rep_bucket <= (1ull << 24) &&
                 32 + bits_for(n) <= 64;
    }
    // stream path: the prep pass also leaves each CTA's minimum key per
    // partition (the representative candidate bound)
    const uint32_t prep_grid = stream ? prep_stream_grid(n, d, P, c->sm_count, cfg->strategy) : 0;
    uint32_t* gmin = stream ? R.dev<uint32_t>(S_GMIN, (size_t)prep_grid * P) : nullptr;
    PartitionOut po = partition_phase(R, pts, n, d, normalized, cfg->strategy, P, m, cfg, pid_dev,
                                      &out->angular_host_fixups, eager,
                                      rep_random && cfg->strategy == SKY_SLICED ? &scan_rows : nullptr, !stream,
                                      gmin, &in_chunks);

    uint8_t* dead = R.dev<uint8_t>(S_DEAD, n);
    uint64_t grid_filtered = 0;
    bool any_dead = false;
    if (cfg->filter == SKY_FILTER_GRID) {
        // grid_filter over non-empty cells (filter.cpp:37-50, engine.cpp:150-163):
        // the cell antichain from the partition offsets on the device (a prefix
        // OR of the occupancy along each axis); only the filtered row count
        // travels to the host
        uint8_t* cdd = R.dev<uint8_t>(S_CELLDEAD, P);
        uint8_t* occ = R.dev<uint8_t>(S_GRIDOCC, P);
        unsigned long long* gcnt = R.dev<unsigned long long>(S_GRIDCNT, 1);
        R.count(launch_grid_filter(po.off, P, (uint32_t)m, d, occ, cdd, gcnt, st));
        launch_mark_cells_dead(po.key64, n, cdd, dead, st);
        R.count();
        unsigned long long* hg = R.pin<unsigned long long>(P_PCOUNT, 1);
        SKY_CUDA(cudaMemcpyAsync(hg, gcnt, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
        R.sync();
        grid_filtered = *hg;
        any_dead = grid_filtered > 0;
    } else if (!stream) {
        launch_fill_u8(dead, 0, n, st);
    }
    SKY_CUDA(cudaEventRecord(c->ev[1], st));

    // ---------------------------------------------- representatives + filter
    uint64_t rep_filtered = 0;
    uint32_t* small_flags = nullptr;  // the small tail's flags when the stream prefilter cleared them
    if (cfg->filter == SKY_FILTER_REPRESENTATIVE) {
        const uint32_t q = (uint32_t)std::min<uint64_t>(cfg->rep_q, n);
        uint32_t* cand = R.dev<uint32_t>(S_REPCAND, (size_t)P * q);
        // filtered (grid) partitions are empty for the reps; here only the
        // representative filter is active, so every partition participates
        if ((uint64_t)P * q > 0x7FFFFFFFull) throw Error(SKY_E_CONFIG, "p * q exceeds 2^31 representative slots");
        if (cfg->rep_selection == SKY_REPS_REGION) {
            if (!normalized) throw Error(SKY_E_NORMALIZATION, "region selection requires a normalized dataset");
            region_candidates(R, pts, d, n, po, P, q, cand);
        } else if (cfg->rep_selection == SKY_REPS_RANDOM) {
            random_candidates(R, n, po, P, q, cfg->strategy == SKY_SLICED ? scan_rows : nullptr, cfg->rep_seed,
                              cand);
        } else if (stream) {
            // candidate buckets (rows under the per-partition key bound),
            // each sorted by (key, row), then the same exact pick
            uint32_t* thr = R.dev<uint32_t>(S_PTHR2, P);
            uint32_t* bcnt = R.dev<uint32_t>(S_BCNT, P);
            uint64_t* bkey = R.dev<uint64_t>(S_BKEY, (size_t)P * c->rep_bucket);
            uint32_t* brow = R.dev<uint32_t>(S_BROW, (size_t)P * c->rep_bucket);
            cudaEvent_t pb, pe;
            R.hbm_pair((uint64_t)n * 8, &pb, &pe);  // the key pass alone (thresholds and picks are latency-bound)
            launch_rep_candidates(po.key64, n, P, q, prep_grid, gmin, thr, c->rep_bucket, bcnt, bkey, brow, pts, d,
                                  cand, misc + M_OVF, st, pb, pe);
            R.count(3);
        } else {
            launch_rep_pick(po.key64, po.idx, po.off, P, pts, R.x64_.x, d, q, cand, st);
            R.count();
        }
        const uint32_t slots = P * q;
        DevSet reps = R.set(S_SET3, slots, D);  // reps.n: upper bound until the count is read back
        uint32_t* nrep_dev = misc + M_NREP;
        if (launch_rep_finalize_par(D, cand, slots, pts, d, reps, nrep_dev, count_tests ? R.tests(0) : nullptr,
                                    R.x64_, c->smem_optin, c->sm_count,
                                    R.dev<char>(S_REPF, rep_finalize_scratch_bytes(D)), st)) {
            // keys, rank + antichain (a warp per pick), placement by rank;
            // the count stays on the device
            R.count(3);
        } else if (launch_rep_finalize(D, cand, slots, pts, d, reps, nrep_dev, count_tests ? R.tests(0) : nullptr,
                                       R.x64_, c->smem_optin, st)) {
            // compact + sort + prune in one CTA; the count stays on the device
            R.count();
        } else {
            reps = host_reps(R, c, D, cand, slots, pts, d, count_tests);
            SKY_CUDA(cudaMemcpyAsync(nrep_dev, &reps.n, sizeof(uint32_t), cudaMemcpyHostToDevice, st));
            R.sync();  // &reps.n is pageable stack memory
        }

        // rep_prefilter over every row, in partition/sum order (indirect)
        float* pthr = nullptr;
        if (reps.n >= 32 && D <= 16 && reps.qc) {
            // one quantization for rows and representatives: quantiles of the input
            pthr = R.dev<float>(S_PTHR, (size_t)D * (kCodeLevels - 1));
            // codes pay off from 32 representatives on: the prefilter decides
            // on the device count, so the thresholds are skipped below it
            launch_thresholds_rows(D, pts, d, n, pthr, st, nrep_dev, 32);
            launch_encode(D, reps, pthr, st, nrep_dev);
            R.count(2);
        }
        uint8_t* dead_row = stream ? nullptr : R.dev<uint8_t>(S_DEADROW, n);
        if (stream) {
            PrefilterAppend app;
            app.key64 = po.key64;
            app.out = R.dev<uint64_t>(S_SURV, n);
            app.count = misc + M_S0;
            app.key_shift = key_shift_for(P);
            app.row_bits = (uint32_t)std::max(1, bits_for(n));
            // the fused small tail follows this pass: it clears the tail's flags on the way
            small_flags = c->world == 1 && c->opt.small_tail != 0 && (uint64_t)P <= kSmallMaxParts
                              ? R.dev<uint32_t>(S_SM_W, (size_t)3 * kSmallCap) : nullptr;
            app.zero = small_flags;
            app.zero_words = small_flags ? 3 * kSmallCap : 0;
            R.hbm_begin();
            if (!launch_prefilter_append(D, pts, d, n, reps.xyz, reps.skey, pthr ? reps.qc : nullptr, reps.id, reps.n,
                                         nrep_dev, pthr, app, count_tests ? R.tests(1) : nullptr, c->smem_optin, st))
                throw Error(SKY_E_INTERNAL, "stream prefilter not applicable");
            // rows (the rows' keys are staged too only when the device count
            // of representatives calls for codes: not counted; survivor
            // writes are few)
            R.hbm_end((uint64_t)n * 4ull * d);
            R.count();
        } else if (reps.n > 0 && (R.hbm_begin(),  // an unmatched begin is overwritten by the next
                                  launch_prefilter(D, pts, d, po.idx, n, reps.xyz, reps.skey, pthr ? reps.qc : nullptr,
                                                   reps.id, reps.n, nrep_dev, pthr, dead_row, dead,
                                                   count_tests ? R.tests(1) : nullptr, R.x64_, c->smem_optin, st,
                                                   (uint64_t)n * d * sizeof(float) <= (48ull << 20)))) {
            R.hbm_end((uint64_t)n * (4ull * d + 5));  // rows through the index, dead flags
            R.count();
            any_dead = true;
        } else if (reps.n > 0) {
            // generic relsky fallback needs the exact count on the host
            uint32_t* hn = R.pin<uint32_t>(P_MISC, 8);
            SKY_CUDA(cudaMemcpyAsync(hn, nrep_dev, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
            R.sync();
            reps.n = hn[0];
            Plan pf;
            for (uint32_t b = 0; b < n; b += kTile) pf.add(b, std::min(n, b + (uint32_t)kTile), {make_uint2(0, reps.n)});
            RelskyArgs fa{};
            fa.cxyz = pts; fa.cskey = reinterpret_cast<const uint32_t*>(po.key64); fa.cidx = po.idx; fa.cd = d;
            fa.sid = reps.id;
            // candidate keys are truncated (key_shift), the reps' are not:
            // no key bound across the two
            fa.indirect = true; fa.sxyz = reps.xyz; fa.sskey = reps.skey; fa.bounded = false; fa.dead = dead;
            fa.tests = count_tests ? R.tests(1) : nullptr;
            R.relsky(D, pf, fa);
            any_dead = true;
        }
    }

    // materialize the surviving rows in (pid, sum key) order
    const int W = c->world, rank = c->rank;
    std::vector<uint32_t> off1;
    uint32_t* off1_dev = R.dev<uint32_t>(S_OFF_B, P + 1);
    DevSet s0;
    std::vector<uint32_t> offu;
    uint32_t* offu_dev = R.dev<uint32_t>(S_OFF_A, P + 1);
    DevSet U;
    std::vector<uint32_t> pr(2, 0);
    pr[1] = P;
    // all-pairs merge on one GPU (random / angular NoSeq, sequential merge):
    // the stable merge of the union's runs into key order needs no host
    // count, so it is queued before the union's round trip and runs while
    // the host waits and plans (count and offsets stay on the device)
    const bool all_mode_merge = cfg->merge == SKY_MERGE_SEQUENTIAL || cfg->strategy == SKY_RANDOM ||
                                cfg->strategy == SKY_ANGULAR;
    bool us_early = false;
    // one GPU, all-pairs merge: the whole merge and the ids are queued before
    // the only host round trip of the step (finish_dev_merge). Its launches
    // are shaped by the union's capacity, which is the filtered set's: the
    // input size up to kExactCapRows rows, the exact filtered count above.
    // So it is taken with representative filtering only (without it the
    // capacity is every row: config 1 has a 100k capacity for a 1.4k union,
    // measured slower there) and from 8,192 capacity rows on (below that the
    // host-planned merge's round trip costs less than the capacity-sized
    // launches). The choice never changes a result.
    const bool dev_merge_cfg = W == 1 && all_mode_merge && P > 1 && D <= 16 &&
                               cfg->filter == SKY_FILTER_REPRESENTATIVE &&
                               !c->opt.host_merge;
    auto dev_merge_ok = [&](uint32_t capacity) { return dev_merge_cfg && capacity >= 8192; };
    // The only round trip of a run finished on the device: union offsets,
    // counters and test counts into pinned memory (the ids are already in
    // `hid`), then the result. `small`: the fused small tail, which may have
    // declined (too many survivors): false, with the counters left in
    // P_MISC for the general tail.
    // The small tail's last kernel writes the offsets and counter words
    // into the same pinned block itself (pin_block()).
    auto pin_block = [&]() { return R.pin<uint32_t>(P_OFF, P + 1 + kSmallMiscWords); };
    auto publish = [&](const uint32_t* hid, uint32_t ns_host, bool small) -> bool {
        static_assert(M_TESTS + 6 <= (int)kSmallMiscWords && M_HITS + 8 <= (int)kSmallMiscWords,
                      "test counters inside the copied counter words");
        uint32_t* h = pin_block();
        uint32_t* hmisc = h + P + 1;
        // test counters (3 x u64) and exact-check counters (4 x u64) are
        // counter words themselves
        const unsigned long long* hts = reinterpret_cast<const unsigned long long*>(hmisc + M_TESTS);
        const unsigned long long* hhits = reinterpret_cast<const unsigned long long*>(hmisc + M_HITS);
        if (!small) {
            SKY_CUDA(cudaMemcpyAsync(h, offu_dev, (P + 1) * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
            SKY_CUDA(cudaMemcpyAsync(hmisc, misc, kSmallMiscWords * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
        }
        SKY_CUDA(cudaEventRecord(c->ev[4], st));
        R.sync();
        if (small && hmisc[M_S0] > kSmallCap) {
            std::memcpy(R.pin<uint32_t>(P_MISC, 32), hmisc, 32 * sizeof(uint32_t));
            return false;
        }
        check_prep(hmisc[M_ERR], hmisc[M_AMB], cfg->strategy, eager);
        if (defer_rand && hmisc[M_RFLAG]) throw RedoEager{};
        if (hmisc[M_OVF]) throw_bucket_overflow(c);
        if (cfg->filter == SKY_FILTER_REPRESENTATIVE) out->n_reps = hmisc[M_NREP];
        const uint32_t ns = stream && !small ? ns_host : hmisc[M_S0];
        out->filtered_count = (uint64_t)n - ns;
        for (uint32_t p = 0; p < P; ++p) out->local_skyline_sizes[p] = h[p + 1] - h[p];
        out->union_size = hmisc[M_U];
        const uint32_t nf = hmisc[M_TOTAL];
        out->d2h_bytes += (uint64_t)nf * sizeof(uint32_t);
        out->ids = alloc_ids(nf);
        for (uint32_t i = 0; i < nf; ++i) out->ids[i] = hid[i];
        out->n_ids = out->final_size = nf;
        out->tests_reps = hts[0];
        out->tests_local = hts[1];
        out->tests_merge = hts[2];
        float ms = 0;
        cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]);
        out->partition_ms = ms;
        // the fused small tail ends the local phase at the end of the run (no
        // merge phase, no events of its own)
        cudaEventElapsedTime(&ms, c->ev[1], c->ev[small ? 4 : 2]);
        out->local_ms = ms;
        ms = 0;
        if (!small) cudaEventElapsedTime(&ms, c->ev[2], c->ev[3]);
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
        out->dom_tests = hts[0] + hts[1] + hts[2];
        out->dom_exact_checks = hhits[0] + hhits[1] + hhits[2] + hhits[3];
        out->exact_checks_merge = hhits[2];
        return true;
    };
    auto finish_dev_merge = [&](const DevSet& Ucap, uint32_t ns_host) {
        SKY_CUDA(cudaEventRecord(c->ev[2], st));
        uint8_t* fdead = nullptr;
        DevSet US = R.merge_all_dev(D, Ucap, offu_dev, P, misc + M_U, count_tests, &fdead);
        SKY_CUDA(cudaEventRecord(c->ev[3], st));
        // ascending ids written by the emit kernel straight into pinned host
        // memory (mapped under UVA): no copy of a capacity-sized buffer
        const uint32_t cap = Ucap.n;
        uint32_t* hid = R.pin<uint32_t>(P_IDS, std::max<uint32_t>(cap, 1));
        uint32_t* bm = R.dev<uint32_t>(S_BM, (size_t)n / 32 + 1);
        uint32_t* bt = R.dev<uint32_t>(S_BMT, bm_blocks(n));
        launch_ids_bitmap(US.id, fdead, cap, n, bm, bt, hid, misc + M_TOTAL, st, misc + M_U);
        R.count(cap ? 3 : 2);
        publish(hid, ns_host, false);
    };
    // stream path, few survivors: sort, local skylines, union, merge and ids
    // in five capacity-sized launches and one round trip (small.cu); false
    // when the survivors exceed the capacity (nothing was changed)
    auto finish_small = [&]() -> bool {
        SmallTail t;
        t.surv = R.dev<uint64_t>(S_SURV, n);
        t.count = misc + M_S0;
        t.pts = pts;
        t.d = d;
        t.P = P;
        t.row_bits = (uint32_t)std::max(1, bits_for(n));
        t.key_shift = key_shift_for(P);
        t.cap = kSmallCap;
        t.flags = R.dev<uint32_t>(S_SM_W, (size_t)3 * kSmallCap);
        t.flags_zeroed = small_flags == t.flags;
        t.cnt = R.dev<uint32_t>(S_SM_CNT, P);
        t.u_count = misc + M_U;
        t.total = misc + M_TOTAL;
        t.offu = offu_dev;
        t.hid = R.pin<uint32_t>(P_IDS, kSmallCap);
        t.tests = count_tests ? R.tests(1) : nullptr;
        t.misc = misc;
        t.hoffu = pin_block();
        t.hmisc = t.hoffu + P + 1;
        launch_small_tail(D, t, st);
        R.count(2);
        // one pass gives the local skylines and the merge: the merge phase
        // is empty and the local phase ends with the run (publish)
        return publish(t.hid, 0, true);
    };
    auto early_merge = [&](const DevSet& Ucap) {
        if (!(all_mode_merge && P > 1)) return;
        DevSet USc = R.set(S_SET3, Ucap.n, D);  // capacity; the live count is misc[M_U]
        launch_merge_runs(D, Ucap, offu_dev, P, USc, st, misc + M_U);
        R.count();
        us_early = true;
    };
    if (W == 1 && stream) {
        // few survivors: the fused tail (its round trip also brings the
        // counters when it declines)
        const bool small_tried = c->opt.small_tail != 0 && (uint64_t)P <= kSmallMaxParts;
        if (small_tried && finish_small()) return;
        // survivors of the stream prefilter: count (round trip), sort by
        // (partition, key, row), unpack into partition order
        uint32_t* hc = R.pin<uint32_t>(P_MISC, 32);
        if (!small_tried) {
            SKY_CUDA(cudaMemcpyAsync(hc, misc, 32 * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
            R.sync();
        }
        check_prep(hc[M_ERR], hc[M_AMB], cfg->strategy, eager);
        if (hc[M_OVF]) throw_bucket_overflow(c);  // a candidate bucket filled up: larger buckets, then the sorted path
        const uint32_t ns = hc[M_S0];
        const uint32_t rb = (uint32_t)std::max(1, bits_for(n));
        uint64_t* surv = R.dev<uint64_t>(S_SURV, n);
        uint64_t* surv2 = R.dev<uint64_t>(S_SURV2, std::max<uint32_t>(ns, 1));
        R.sort_keys(surv, surv2, ns, 32 + std::max(1, bits_for(P)) - (int)key_shift_for(P) + (int)rb);
        uint64_t* k64 = R.dev<uint64_t>(S_KEY_B, std::max<uint32_t>(ns, 1));
        uint32_t* rows = R.dev<uint32_t>(S_IDX_B, std::max<uint32_t>(ns, 1));
        launch_unpack_survivors(surv2, ns, rb, key_shift_for(P), P, k64, rows, off1_dev, st);
        R.count();
        s0 = R.set(S_SET0, ns, D);
        launch_scatter_indirect(D, pts, d, rows, k64, ns, nullptr, nullptr, s0, st);
        R.count();
        R.encode_dev(D, s0, misc + M_S0);
        if (cfg->local_algo == SKY_LOCAL_BNL) {
            uint32_t used = 0;
            std::vector<uint32_t> unused;
            U = R.local_bnl(D, s0, off1_dev, P, cfg->bnl_window_cap, offu_dev, unused, count_tests, &used,
                            misc + M_U);
        } else {
            U = R.local_sfs_dev(D, s0, misc + M_S0, off1_dev, P, offu_dev, misc + M_U, count_tests);
        }
        if (dev_merge_ok(U.n)) {
            finish_dev_merge(U, ns);
            return;
        }
        early_merge(U);
        uint32_t* h = R.pin<uint32_t>(P_OFF, P + 1 + 32);
        SKY_CUDA(cudaMemcpyAsync(h, offu_dev, (P + 1) * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
        SKY_CUDA(cudaMemcpyAsync(h + P + 1, misc, 32 * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
        R.sync();
        const uint32_t* hmisc = h + P + 1;
        check_prep(hmisc[M_ERR], hmisc[M_AMB], cfg->strategy, eager);
        if (defer_rand && hmisc[M_RFLAG]) throw RedoEager{};
        out->n_reps = hmisc[M_NREP];
        rep_filtered = (uint64_t)n - ns;
        offu.assign(h, h + P + 1);
        U.n = hmisc[M_U];
    } else if (W == 1) {
        // Single GPU: every count stays on the device until the union of the
        // local skylines is known (one host round trip for this phase).
        uint32_t* pos = R.dev<uint32_t>(S_POS, n);
        R.scan_live(dead, pos, n);
        launch_count_total(pos, dead, n, misc + M_S0, st);
        launch_remap_offsets(po.off, P, pos, dead, n, off1_dev, st);
        R.count(2);
        // capacity of the filtered set: n, or for large inputs the exact
        // count (one early round trip), so later passes are not sized by n
        uint32_t cap0 = n;
        if (c->opt.cap_sync > 0 || (c->opt.cap_sync < 0 && n > kExactCapRows)) {
            uint32_t* hc = R.pin<uint32_t>(P_MISC, 8);
            SKY_CUDA(cudaMemcpyAsync(hc, misc + M_S0, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
            R.sync();
            cap0 = hc[0];
        }
        s0 = R.set(S_SET0, cap0, D);
        launch_scatter_indirect(D, pts, d, po.idx, po.key64, n, dead, pos, s0, st);
        R.count();
        R.encode_dev(D, s0, misc + M_S0);
        if (cfg->local_algo == SKY_LOCAL_BNL) {
            uint32_t used = 0;
            std::vector<uint32_t> unused;
            U = R.local_bnl(D, s0, off1_dev, P, cfg->bnl_window_cap, offu_dev, unused, count_tests, &used,
                            misc + M_U);
        } else {
            U = R.local_sfs_dev(D, s0, misc + M_S0, off1_dev, P, offu_dev, misc + M_U, count_tests);
        }
        if (dev_merge_ok(U.n) && grid_filtered == 0) {
            finish_dev_merge(U, 0);
            return;
        }
        early_merge(U);
        uint32_t* h = R.pin<uint32_t>(P_OFF, P + 1 + 32);
        SKY_CUDA(cudaMemcpyAsync(h, offu_dev, (P + 1) * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
        SKY_CUDA(cudaMemcpyAsync(h + P + 1, misc, 32 * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
        R.sync();
        const uint32_t* hmisc = h + P + 1;
        check_prep(hmisc[M_ERR], hmisc[M_AMB], cfg->strategy, eager);
        if (defer_rand && hmisc[M_RFLAG]) throw RedoEager{};  // redo with the host shuffle
        if (cfg->filter == SKY_FILTER_REPRESENTATIVE) out->n_reps = hmisc[M_NREP];
        rep_filtered = (uint64_t)n - hmisc[M_S0] - grid_filtered;
        offu.assign(h, h + P + 1);
        U.n = hmisc[M_U];
    } else {
        uint32_t* pos = R.dev<uint32_t>(S_POS, n);
        R.scan_live(dead, pos, n);
        launch_count_total(pos, dead, n, misc + M_TOTAL, st);
        launch_remap_offsets(po.off, P, pos, dead, n, off1_dev, st);
        R.count(2);
        uint32_t* h = R.pin<uint32_t>(P_OFF, P + 8);
        SKY_CUDA(cudaMemcpyAsync(h, off1_dev, (P + 1) * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
        SKY_CUDA(cudaMemcpyAsync(h + P + 1, misc, 8 * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
        R.sync();
        const uint32_t* hmisc = h + P + 1;
        check_prep(hmisc[M_ERR], hmisc[M_AMB], cfg->strategy, eager);
        if (cfg->filter == SKY_FILTER_REPRESENTATIVE) out->n_reps = hmisc[M_NREP];
        off1.assign(h, h + P + 1);
        const uint32_t total = hmisc[M_TOTAL];
        s0 = R.set(S_SET0, total, D);
        launch_scatter_indirect(D, pts, d, po.idx, po.key64, n, any_dead ? dead : nullptr, any_dead ? pos : nullptr,
                                s0, st);
        R.count();
        rep_filtered = (uint64_t)n - total - grid_filtered;
        R.encode(D, s0);

        // ----------------------------------------------------- local skylines
        // Multi-GPU: every rank holds the same s0 (phase 1a above is
        // replicated); the local phase is sharded by contiguous, cost-balanced
        // partition ranges, and the local skylines are all-gathered over NCCL.
        pr = plan_local_shards(off1, P, W);
        const uint32_t pb = pr[rank], pe = pr[rank + 1];
        // view of this rank's partitions
        const uint32_t base = off1[pb], cnt = off1[pe] - base;
        const int D4 = (D + 3) / 4 * 4;
        DevSet mine = s0;
        mine.xyz = s0.xyz + (size_t)base * D4;
        mine.skey = s0.skey + base;
        mine.id = s0.id + base;
        mine.qc = s0.qc ? s0.qc + base : nullptr;
        mine.n = cnt;
        const uint32_t Pm = pe - pb;
        std::vector<uint32_t> offm(Pm + 1);
        for (uint32_t k = 0; k <= Pm; ++k) offm[k] = off1[pb + k] - base;
        uint32_t* offm_dev = R.dev<uint32_t>(S_OFFM, Pm + 1);  // not S_OFF_C: the local waves use it
        {
            uint32_t* hs = R.stage<uint32_t>(Pm + 1);
            std::memcpy(hs, offm.data(), (Pm + 1) * sizeof(uint32_t));
            SKY_CUDA(cudaMemcpyAsync(offm_dev, hs, (Pm + 1) * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
        }
        std::vector<uint32_t> offum;
        DevSet Um;
        if (cfg->local_algo == SKY_LOCAL_BNL) {
            uint32_t used = 0;
            Um = R.local_bnl(D, mine, offm_dev, Pm, cfg->bnl_window_cap, offu_dev, offum, count_tests, &used);
        } else {
            Um = R.local_sfs(D, mine, offm, offm_dev, Pm, offu_dev, offum, count_tests);
        }
        U = R.gather_union(D, Um, offum, pr, P, offu, offu_dev);
    }
    out->filtered_count = grid_filtered + rep_filtered;
    merge_phase(R, c, cfg, U, offu, offu_dev, P, m, d, D, n, count_tests, us_early, out);
}

template <class F>
int guarded(sky_ctx* c, F&& f) {
    try {
        if (c) SKY_CUDA(cudaSetDevice(c->device));
        cudaGetLastError();  // a failed call of an earlier run must not fail this one's launch checks
        f();
        if (c) c->err.clear();
        return SKY_OK;
    } catch (const Error& e) {
        if (c) c->err = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        if (c) c->err = "host out of memory";
        return SKY_E_INTERNAL;
    } catch (const std::exception& e) {
        if (c) c->err = e.what();
        return SKY_E_INTERNAL;
    }
}


// run_impl with its eager retry (angular boundary rows, rejected random draws)
void run_impl_retry(sky_ctx* c, const void* points, uint64_t n, uint32_t d, int normalized, int on_device,
                    const sky_config* cfg, sky_result* out, bool f64) {
    struct BucketReset {  // whatever happens, the next run starts with the normal buckets
        sky_ctx* c;
        ~BucketReset() { c->rep_bucket = sky::kRepBucket; }
    } reset{c};
    try {
        // a relation whose last run overflowed the normal buckets (queried
        // again, same size) starts with the large ones
        if (n && c->big_bucket_rows == n) c->rep_bucket = kRepBucketBig;
        try {
            run_impl(c, points, n, d, normalized, on_device, cfg, out, false, f64);
        } catch (const RedoBigBuckets&) {
            sky_result_free(out);
            c->rep_bucket = kRepBucketBig;
            c->big_bucket_rows = n;
            run_impl(c, points, n, d, normalized, on_device, cfg, out, false, f64);
        }
    } catch (const RedoEager&) {
        sky_result_free(out);
        if (c->rep_bucket == kRepBucketBig) c->big_bucket_rows = 0;  // the large buckets did not help either
        run_impl(c, points, n, d, normalized, on_device, cfg, out, true, f64);
    }
}

// every rank's value of one word, on the host
std::vector<uint32_t> allgather_host_u32(sky_ctx* c, uint32_t mine) {
    const int W = c->world;
    uint32_t* dv = static_cast<uint32_t*>(c->dev.get(S_GCOUNT, (W + 1) * sizeof(uint32_t) + 16));
    uint32_t* h = static_cast<uint32_t*>(c->pin.get(P_RUNS, (W + 1) * sizeof(uint32_t) + 16));
    h[W] = mine;
    SKY_CUDA(cudaMemcpyAsync(dv + W, h + W, sizeof(uint32_t), cudaMemcpyHostToDevice, c->stream));
    c->comm->allgather(dv + W, dv, sizeof(uint32_t), c->stream);
    SKY_CUDA(cudaMemcpyAsync(h, dv, W * sizeof(uint32_t), cudaMemcpyDeviceToHost, c->stream));
    SKY_CUDA(cudaStreamSynchronize(c->stream));
    return std::vector<uint32_t>(h, h + W);
}

int device_of(const void* p, int dflt) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return dflt;
    }
    return at.type == cudaMemoryTypeDevice ? at.device : dflt;
}

// One rank of a multi-rank context (world > 1, or the sharded path forced at
// world 1). `points`: the whole relation, the same on every rank (shard ==
// false; rank r then works on rows [N*r/W, N*(r+1)/W)), or this rank's own
// rows (shard == true; ranks hold consecutive row ranges in rank order).
void run_rank(sky_ctx* c, const void* points, uint64_t n_arg, uint32_t d, int normalized, int on_device,
              const sky_config* cfg, sky_result* out, bool f64, bool shard) {
    const int W = c->world, r = c->rank;
    std::memset(out, 0, sizeof(*out));
    if (n_arg >= 0xFFFFFFF0ull) throw Error(SKY_E_DATA, "at most 2^32-16 points per run");
    std::vector<uint32_t> rows_of(W);
    uint64_t N = 0;
    if (shard) {
        rows_of = allgather_host_u32(c, (uint32_t)n_arg);
        for (uint32_t v : rows_of) N += v;
    } else {
        N = n_arg;
        for (int q = 0; q < W; ++q) rows_of[q] = (uint32_t)(shard_row(N, q + 1, W) - shard_row(N, q, W));
    }
    if (N >= 0xFFFFFFF0ull) throw Error(SKY_E_DATA, "at most 2^32-16 points per run");
    uint32_t row0 = 0;
    for (int q = 0; q < r; ++q) row0 += rows_of[q];
    const size_t esz = f64 ? sizeof(double) : sizeof(float);
    validate(N, d, cfg);
    if (sharded_eligible(cfg, N, d, f64)) {
        const char* base = static_cast<const char*>(points) + (shard ? 0 : (size_t)row0 * d * esz);
        try {
            run_sharded(c, reinterpret_cast<const float*>(base), rows_of[r], row0, rows_of, d, normalized, on_device,
                        cfg, out);
            return;
        } catch (const ReplicatePhase1&) {
            sky_result_free(out);
            std::memset(out, 0, sizeof(*out));
        }
    }
    // replicated phase 1: every rank partitions and filters the whole relation
    const void* full = points;
    int full_dev = on_device;
    const size_t bytes = (size_t)N * d * esz;
    if (shard || (on_device && device_of(points, c->device) != c->device)) {
        char* dst = static_cast<char*>(c->dev.get(S_SH_FULL, bytes + 16));
        if (shard) {
            // this rank's rows on its device, then every rank's rows on every rank
            const size_t mine = (size_t)rows_of[r] * d * esz;
            char* own = static_cast<char*>(c->dev.get(S_SH_SKG, mine + 16));
            if (mine) SKY_CUDA(cudaMemcpyAsync(own, points, mine, cudaMemcpyDefault, c->stream));
            std::vector<size_t> b(W), dp(W);
            size_t at = 0;
            for (int q = 0; q < W; ++q) {
                b[q] = (size_t)rows_of[q] * d * esz;
                dp[q] = at;
                at += b[q];
            }
            c->comm->allgatherv(own, dst, b.data(), dp.data(), c->stream);
        } else if (bytes) {
            SKY_CUDA(cudaMemcpyAsync(dst, points, bytes, cudaMemcpyDefault, c->stream));
        }
        SKY_CUDA(cudaStreamSynchronize(c->stream));
        full = dst;
        full_dev = 1;
    }
    run_impl_retry(c, full, N, d, normalized, full_dev, cfg, out, f64);
    out->world = (uint32_t)W;
    out->local_rows = N;
}

}  // namespace

// ===================================================================== C ABI
extern "C" {

int sky_abi_version(void) { return SKY_ABI_VERSION; }

void sky_config_default(sky_config* cfg) {
    std::memset(cfg, 0, sizeof(*cfg));
    cfg->strategy = SKY_RANDOM;
    cfg->p = 1;
    cfg->rep_q = 5;  // engine.hpp:34
    cfg->merge = SKY_MERGE_SEQUENTIAL;
    cfg->workers = 1;
    cfg->local_algo = SKY_LOCAL_SFS;
    cfg->bnl_window_cap = 4096;
    cfg->count_tests = 1;
    cfg->rep_seed = 0;
}

int sky_ctx_create(int device, sky_ctx** out) {
    *out = nullptr;
    sky_ctx* c = new sky_ctx();
    c->device = device;
    int rc = guarded(c, [&] {
        SKY_CUDA(cudaSetDevice(device));
        SKY_CUDA(cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking));
        SKY_CUDA(cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking));
        SKY_CUDA(cudaEventCreateWithFlags(&c->fork_ev, cudaEventDisableTiming));
        SKY_CUDA(cudaEventCreateWithFlags(&c->join_ev, cudaEventDisableTiming));
        for (auto& e : c->chunk_ev) SKY_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        c->stream = c->own;
        SKY_CUDA(cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device));
        SKY_CUDA(cudaDeviceGetAttribute(&c->smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
        for (auto& e : c->ev) SKY_CUDA(cudaEventCreate(&e));
    });
    if (rc != SKY_OK) {
        static thread_local std::string last;
        last = c->err;
        delete c;
        return rc;
    }
    *out = c;
    return SKY_OK;
}

int sky_nccl_unique_id(uint8_t* out, uint64_t size) {
    return guarded(nullptr, [&] {
        if (size < nccl_unique_id_bytes()) throw Error(SKY_E_CONFIG, "unique id buffer too small");
        nccl_unique_id(out);
    });
}

int sky_ctx_create_dist(int device, int rank, int world, const uint8_t* unique_id, sky_ctx** out) {
    *out = nullptr;
    if (world < 1 || rank < 0 || rank >= world) return SKY_E_CONFIG;
    sky_ctx* c = nullptr;
    int rc = sky_ctx_create(device, &c);
    if (rc != SKY_OK) return rc;
    rc = guarded(c, [&] {
        c->rank = rank;
        c->world = world;
        c->comm = make_nccl_comm(device, rank, world, unique_id);
    });
    if (rc != SKY_OK) {
        sky_ctx_destroy(c);
        return rc;
    }
    *out = c;
    return SKY_OK;
}

namespace {

void group_worker(sky_group* g, int r) {
    uint64_t seen = 0;
    while (true) {
        std::function<void(int)> job;
        {
            std::unique_lock<std::mutex> lk(g->mu);
            g->cv.wait(lk, [&] { return g->stop || g->gen != seen; });
            if (g->stop) return;
            seen = g->gen;
            job = g->job;
        }
        job(r);
        std::lock_guard<std::mutex> lk(g->mu);
        if (--g->pending == 0) g->done_cv.notify_all();
    }
}

// run job(r) on every rank concurrently (rank 0 on this thread)
void group_dispatch(sky_group* g, const std::function<void(int)>& job) {
    const int W = (int)g->ranks.size();
    {
        std::lock_guard<std::mutex> lk(g->mu);
        g->job = job;
        g->pending = W - 1;
        ++g->gen;
    }
    g->cv.notify_all();
    job(0);
    std::unique_lock<std::mutex> lk(g->mu);
    g->done_cv.wait(lk, [&] { return g->pending == 0; });
}

void make_group_comms(sky_group* g) {
    const int W = (int)g->ranks.size();
    for (sky_ctx* r : g->ranks) r->comm.reset();
    if (g->loopback) {
        auto lg = std::make_shared<LoopbackGroup>(W);
        for (int r = 0; r < W; ++r) {
            SKY_CUDA(cudaSetDevice(g->devices[r]));
            g->ranks[r]->comm = std::make_unique<LoopbackComm>(lg, r, g->devices[r]);
        }
    } else {
        auto cs = make_nccl_comms(g->devices);
        for (int r = 0; r < W; ++r) g->ranks[r]->comm = std::move(cs[r]);
    }
    for (int r = 0; r < W; ++r) {
        g->ranks[r]->rank = r;
        g->ranks[r]->world = W;
    }
}

void destroy_rank_ctx(sky_ctx* c) {
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    c->comm.reset();
    for (auto& e : c->ev)
        if (e) cudaEventDestroy(e);
    for (auto& e : c->dom_ev)
        if (e) cudaEventDestroy(e);
    for (auto& e : c->tl_ev)
        if (e) cudaEventDestroy(e);
    for (auto& e : c->hbm_ev)
        if (e) cudaEventDestroy(e);
    if (c->sync_ev) cudaEventDestroy(c->sync_ev);
    for (auto& b : c->stage) cudaFreeHost(b.first);
    if (c->mt_jump) cudaFree(c->mt_jump);
    c->dev.release();
    if (c->own) cudaStreamDestroy(c->own);
    if (c->copy) cudaStreamDestroy(c->copy);
    if (c->fork_ev) cudaEventDestroy(c->fork_ev);
    if (c->join_ev) cudaEventDestroy(c->join_ev);
    for (auto& e : c->chunk_ev)
        if (e) cudaEventDestroy(e);
    delete c;
}

// sky_run / sky_run_f64 on a group: every rank works on its row slice of the
// host (or device) rows; rank 0's result is returned (all ranks hold it)
int group_run(sky_ctx* gc, const void* points, uint64_t n, uint32_t d, int normalized, int on_device,
              const sky_config* cfg, sky_result* out, bool f64) {
    sky_group* g = gc->group;
    const int W = (int)g->ranks.size();
    std::vector<sky_result> res(W);
    std::vector<int> rcs(W, SKY_OK);
    group_dispatch(g, [&](int r) {
        sky_ctx* c = g->ranks[r];
        rcs[r] = guarded(c, [&] {
            try {
                run_rank(c, points, n, d, normalized, on_device, cfg, &res[r], f64, false);
            } catch (...) {
                sky_result_free(&res[r]);
                for (sky_ctx* q : g->ranks)
                    if (q->comm) q->comm->abort();  // unblock the ranks waiting in an exchange
                throw;
            }
        });
    });
    int first = -1;
    for (int r = 0; r < W; ++r)
        if (rcs[r] != SKY_OK && (first < 0 || g->ranks[first]->err.find("aborted by another rank") != std::string::npos))
            first = r;
    if (first >= 0) {
        gc->err = g->ranks[first]->err;
        for (int r = 0; r < W; ++r) sky_result_free(&res[r]);
        std::memset(out, 0, sizeof(*out));
        try {
            make_group_comms(g);  // aborted exchanges cannot be reused
        } catch (const Error& e) {
            gc->err += std::string("; rebuilding the exchanges failed: ") + e.what();
        }
        return rcs[first];
    }
    *out = res[0];
    for (int r = 1; r < W; ++r) {
        const sky_result& x = res[r];
        if (x.n_ids != out->n_ids || x.union_size != out->union_size) {
            for (int k = 0; k < W; ++k) sky_result_free(&res[k]);
            std::memset(out, 0, sizeof(*out));
            gc->err = "ranks returned different results";
            return SKY_E_INTERNAL;
        }
        out->partition_ms = std::max(out->partition_ms, x.partition_ms);
        out->local_ms = std::max(out->local_ms, x.local_ms);
        out->merge_ms = std::max(out->merge_ms, x.merge_ms);
        out->total_ms = std::max(out->total_ms, x.total_ms);
        out->dom_kernel_ms = std::max(out->dom_kernel_ms, x.dom_kernel_ms);
        out->stream_kernel_ms = std::max(out->stream_kernel_ms, x.stream_kernel_ms);
        out->kernel_launches += x.kernel_launches;
        out->dom_launches += x.dom_launches;
        out->stream_launches += x.stream_launches;
        out->stream_bytes += x.stream_bytes;
        out->h2d_bytes += x.h2d_bytes;
        out->exchange_bytes += x.exchange_bytes;
        out->local_rows += x.local_rows;
        out->angular_host_fixups += x.angular_host_fixups;
        sky_result free_me = x;
        sky_result_free(&free_me);
    }
    gc->err.clear();
    return SKY_OK;
}

}  // namespace

int sky_ctx_create_group(const int* devices, int n, int flags, sky_ctx** out) {
    *out = nullptr;
    if (n < 1 || !devices) return SKY_E_CONFIG;
    sky_group* g = new sky_group();
    g->devices.assign(devices, devices + n);
    g->loopback = (flags & SKY_GROUP_LOOPBACK) != 0;
    for (int a = 0; a < n; ++a)
        for (int b = a + 1; b < n; ++b)
            if (devices[a] == devices[b]) g->loopback = true;  // NCCL needs distinct devices
    sky_ctx* gc = new sky_ctx();
    gc->device = devices[0];
    gc->group = g;
    gc->world = n;
    int rc = SKY_OK;
    for (int r = 0; r < n && rc == SKY_OK; ++r) {
        sky_ctx* c = nullptr;
        rc = sky_ctx_create(devices[r], &c);
        if (rc == SKY_OK) g->ranks.push_back(c);
    }
    if (rc == SKY_OK) rc = guarded(gc, [&] { make_group_comms(g); });
    if (rc != SKY_OK) {
        for (sky_ctx* c : g->ranks) destroy_rank_ctx(c);
        delete g;
        delete gc;
        return rc;
    }
    for (int r = 1; r < n; ++r) g->workers.emplace_back(group_worker, g, r);
    *out = gc;
    return SKY_OK;
}

int sky_ctx_create_peers(const int* devices, int n, sky_ctx** out) {
    if (n < 1 || !devices || !out) return SKY_E_CONFIG;
    for (int r = 0; r < n; ++r) out[r] = nullptr;
    auto lg = std::make_shared<LoopbackGroup>(n);
    int rc = SKY_OK;
    for (int r = 0; r < n && rc == SKY_OK; ++r) {
        rc = sky_ctx_create(devices[r], &out[r]);
        if (rc == SKY_OK)
            rc = guarded(out[r], [&] {
                out[r]->rank = r;
                out[r]->world = n;
                out[r]->comm = std::make_unique<LoopbackComm>(lg, r, devices[r]);
            });
    }
    if (rc != SKY_OK)
        for (int r = 0; r < n; ++r) {
            sky_ctx_destroy(out[r]);
            out[r] = nullptr;
        }
    return rc;
}

int sky_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

int sky_ctx_world(const sky_ctx* c, int* rank, int* world) {
    if (!c) return SKY_E_CONFIG;
    if (rank) *rank = c->group ? 0 : c->rank;
    if (world) *world = c->world;
    return SKY_OK;
}

int sky_ctx_set_sharded(sky_ctx* c, int on) {
    if (!c) return SKY_E_CONFIG;
    return guarded(c, [&] {
        if (c->group) {
            for (sky_ctx* r : c->group->ranks) r->sharded = on != 0;
            return;
        }
        c->sharded = on != 0;
        if (c->sharded && !c->comm) {
            // a one-rank exchange group, so the sharded path has its collectives
            auto lg = std::make_shared<LoopbackGroup>(1);
            c->comm = std::make_unique<LoopbackComm>(lg, 0, c->device);
        }
    });
}

int sky_ctx_set_option(sky_ctx* c, const char* name, int64_t v) {
    if (!c || !name) return SKY_E_CONFIG;
    if (c->group) {
        for (sky_ctx* r : c->group->ranks) {
            const int rc = sky_ctx_set_option(r, name, v);
            if (rc != SKY_OK) return rc;
        }
        return SKY_OK;
    }
    sky_options& o = c->opt;
    const std::string k(name);
    const int32_t s = (int32_t)std::max<int64_t>(-1, std::min<int64_t>(v, 1));
    const uint32_t u = (uint32_t)std::max<int64_t>(0, std::min<int64_t>(v, 1 << 30));
    if (k == "stream") o.stream = s;
    else if (k == "host_merge") o.host_merge = s > 0;
    else if (k == "cap_sync") o.cap_sync = s;
    else if (k == "sfs_tile") o.sfs_tile = u;
    else if (k == "sfs_chunk" && u) o.sfs_chunk = u;
    else if (k == "sfs_head" && u) o.sfs_head = u;
    else if (k == "merge_tile") o.merge_tile = u;
    else if (k == "merge_head" && u) o.merge_head = u;
    else if (k == "grain_items" && u) o.grain_items = u;
    else if (k == "bnl_block") o.bnl_block = u;
    else if (k == "merge_index") o.merge_index = s > 0;
    else if (k == "merge_cell_rows" && u) o.merge_cell_rows = u;
    else if (k == "range_par") o.range_par = u;
    else if (k == "sfs_auto_chunk") o.sfs_auto_chunk = s > 0;
    else if (k == "wave_growth" && u >= 2) o.wave_growth = u;
    else if (k == "wave_split_mpairs") o.wave_split_mpairs = u;
    else if (k == "profile_host") o.profile_host = s > 0;
    else if (k == "timeline") o.timeline = s > 0;
    else if (k == "small_tail") o.small_tail = s > 0;
    else if (k == "kernel_events") o.kernel_events = s > 0;
    else {
        c->err = "unknown option or value: " + k;
        return SKY_E_CONFIG;
    }
    return SKY_OK;
}

void sky_ctx_destroy(sky_ctx* c) {
    if (!c) return;
    if (sky_group* g = c->group) {
        {
            std::lock_guard<std::mutex> lk(g->mu);
            g->stop = true;
        }
        g->cv.notify_all();
        for (auto& t : g->workers) t.join();
        for (sky_ctx* r : g->ranks) destroy_rank_ctx(r);
        delete g;
        delete c;
        return;
    }
    destroy_rank_ctx(c);
}

const char* sky_last_error(const sky_ctx* c) { return c ? c->err.c_str() : "no context"; }

int sky_ctx_set_stream(sky_ctx* c, void* stream) {
    c->stream = stream ? static_cast<cudaStream_t>(stream) : c->own;
    return SKY_OK;
}

// the per-call helpers below run on one GPU: a group's rank 0
static sky_ctx* single_gpu(sky_ctx* c) { return c && c->group ? c->group->ranks[0] : c; }

static int run_guarded(sky_ctx* c, const void* points, uint64_t n, uint32_t d, int normalized, int on_device,
                       const sky_config* cfg, sky_result* out, bool f64) {
    if (c && c->group) return group_run(c, points, n, d, normalized, on_device, cfg, out, f64);
    return guarded(c, [&] {
        try {
            if (c->world > 1 || c->sharded)
                run_rank(c, points, n, d, normalized, on_device, cfg, out, f64, false);
            else
                run_impl_retry(c, points, n, d, normalized, on_device, cfg, out, f64);
        } catch (...) {
            sky_result_free(out);
            throw;
        }
    });
}

int sky_run(sky_ctx* c, const float* points, uint64_t n, uint32_t d, int normalized, int on_device,
            const sky_config* cfg, sky_result* out) {
    return run_guarded(c, points, n, d, normalized, on_device, cfg, out, false);
}

int sky_run_f64(sky_ctx* c, const double* points, uint64_t n, uint32_t d, int normalized, int on_device,
                const sky_config* cfg, sky_result* out) {
    return run_guarded(c, points, n, d, normalized, on_device, cfg, out, true);
}

int sky_run_shard(sky_ctx* c, const float* points, uint64_t n_local, uint32_t d, int normalized, int on_device,
                  const sky_config* cfg, sky_result* out) {
    if (c && c->group) {
        c->err = "sky_run_shard takes a distributed (one rank per process) context; use sky_run on a group";
        return SKY_E_CONFIG;
    }
    if (c && c->world == 1 && !c->sharded) return run_guarded(c, points, n_local, d, normalized, on_device, cfg, out, false);
    return guarded(c, [&] {
        try {
            run_rank(c, points, n_local, d, normalized, on_device, cfg, out, false, true);
        } catch (...) {
            sky_result_free(out);
            throw;
        }
    });
}

void sky_result_free(sky_result* r) {
    if (!r) return;
    IdPool::get().release(r->ids);
    std::free(r->local_skyline_sizes);
    r->ids = nullptr;
    r->local_skyline_sizes = nullptr;
}

int sky_snap_slices(uint64_t target_p, uint64_t k, uint64_t* out_m) {
    return guarded(nullptr, [&] { *out_m = snap_slices(target_p, k); });
}

int sky_assign(sky_ctx* c, const float* points, uint64_t n64, uint32_t d, int normalized, const sky_config* cfg,
               uint64_t* partition_of, uint64_t* effective_p) {
    c = single_gpu(c);
    return guarded(c, [&] {
        if (cfg->p < 1) throw Error(SKY_E_CONFIG, "partition count must be >= 1");
        uint64_t P64, m;
        resolve_partitions(n64, d, cfg, &P64, &m);
        *effective_p = P64;
        if (n64 == 0) return;
        if (d == 0) throw Error(SKY_E_DIMENSION, "assignment needs d >= 1");
        const uint32_t n = (uint32_t)n64;
        Runner R(c);
        float* dp = R.dev<float>(S_PTS, (size_t)n * d);
        SKY_CUDA(cudaMemcpyAsync(dp, points, (size_t)n * d * sizeof(float), cudaMemcpyHostToDevice, c->stream));
        const uint32_t* pid_dev = cfg->strategy == SKY_RANDOM ? R.random_pids(n, P64, cfg->seed) : nullptr;
        uint64_t fix = 0;
        PartitionOut po = partition_phase(R, dp, n, d, normalized, cfg->strategy, P64, m, cfg, pid_dev, &fix);
        std::vector<uint64_t> key(n);
        std::vector<uint32_t> idx(n);
        SKY_CUDA(cudaMemcpyAsync(key.data(), po.key64, n * sizeof(uint64_t), cudaMemcpyDeviceToHost, c->stream));
        SKY_CUDA(cudaMemcpyAsync(idx.data(), po.idx, n * sizeof(uint32_t), cudaMemcpyDeviceToHost, c->stream));
        R.sync();
        for (uint32_t i = 0; i < n; ++i) partition_of[idx[i]] = key[i] >> 32;
    });
}

int sky_relative_skyline(sky_ctx* c, const float* r, uint64_t nr64, const float* cp, uint64_t nc64, uint32_t d,
                         uint8_t* keep, uint64_t* tests_out) {
    c = single_gpu(c);
    return guarded(c, [&] {
        const uint32_t nr = (uint32_t)nr64, nc = (uint32_t)nc64;
        if (tests_out) *tests_out = 0;
        std::memset(keep, 1, nr);
        if (nr == 0 || nc == 0 || d == 0) return;  // relative_skyline (core.cpp:81-84)
        const int D = padded_dim(d);
        if (!D) throw Error(SKY_E_DIMENSION, "the GPU engine supports d <= 32");
        Runner R(c);
        cudaStream_t st = c->stream;
        // rows of r then c in one upload
        float* dp = R.dev<float>(S_PTS, (size_t)(nr + nc) * d);
        SKY_CUDA(cudaMemcpyAsync(dp, r, (size_t)nr * d * sizeof(float), cudaMemcpyHostToDevice, st));
        SKY_CUDA(cudaMemcpyAsync(dp + (size_t)nr * d, cp, (size_t)nc * d * sizeof(float), cudaMemcpyHostToDevice, st));
        uint32_t* misc = R.dev<uint32_t>(S_MISC, 64);
        SKY_CUDA(cudaMemsetAsync(misc, 0, 64 * sizeof(uint32_t), st));
        uint64_t* key = R.dev<uint64_t>(S_KEY_A, nr + nc);
        uint32_t* idx = R.dev<uint32_t>(S_IDX_A, nr + nc);
        PrepArgs pa{dp, nullptr, nr + nc, d, SKY_SLICED + 100, 0, 0, nullptr, 0, key, idx, nullptr, misc + M_ERR,
                    misc + M_AMB, nullptr, 0, 0};
        launch_prep(pa, st);
        // comparators sorted by sum key
        uint64_t* keyB = R.dev<uint64_t>(S_KEY_B, nc);
        uint32_t* idxB = R.dev<uint32_t>(S_IDX_B, nc);
        R.sort_pairs(key + nr, keyB, idx + nr, idxB, nc, 0, 32);
        DevSet S = R.set(S_SET1, nc, D);
        launch_scatter_indirect(D, dp, d, idxB, keyB, nc, nullptr, nullptr, S, st);
        DevSet T = R.set(S_SET0, nr, D);
        launch_scatter_indirect(D, dp, d, idx, key, nr, nullptr, nullptr, T, st);
        uint8_t* dead = R.dev<uint8_t>(S_DEAD, nr);
        launch_fill_u8(dead, 0, nr, st);
        R.encode(D, S, &T);
        Plan pl;
        pl.tile = D <= 16 ? 128u : (uint32_t)kTile;
        for (uint32_t b = 0; b < nr; b += pl.tile) pl.add(b, std::min(nr, b + pl.tile), {make_uint2(0, nc)});
        pl.order();
        RelskyArgs a{};
        a.cxyz = T.xyz; a.cskey = T.skey; a.sxyz = S.xyz; a.sskey = S.skey; a.dead = dead;
        a.cid = T.id; a.sid = S.id;
        a.tests = R.tests(0);
        // candidates are in input order, so the key bound is per warp (still
        // sound on any order: a dominator never has a larger key)
        a.bounded = true;
        R.relsky(D, pl, a, T.qc, S.qc);
        std::vector<uint8_t> h(nr);
        unsigned long long t[5] = {0, 0, 0, 0, 0};
        SKY_CUDA(cudaMemcpyAsync(h.data(), dead, nr, cudaMemcpyDeviceToHost, st));
        SKY_CUDA(cudaMemcpyAsync(t, R.tests(0), sizeof(t[0]), cudaMemcpyDeviceToHost, st));
        SKY_CUDA(cudaMemcpyAsync(t + 1, R.dev<uint32_t>(S_MISC, 64) + M_HITS, 4 * sizeof(t[0]),
                                 cudaMemcpyDeviceToHost, st));
        R.sync();
        for (uint32_t i = 0; i < nr; ++i) keep[i] = h[i] ? 0 : 1;
        if (tests_out) *tests_out = t[0];
    });
}

int sky_skyline(sky_ctx* c, const float* points, uint64_t n, uint32_t d, int64_t** out_ids, uint64_t* n_out,
                uint64_t* tests_out) {
    c = single_gpu(c);
    return guarded(c, [&] {
        // one partition: Sky(r) is the local skyline of the only partition
        sky_config cfg;
        sky_config_default(&cfg);
        cfg.strategy = SKY_SLICED;
        cfg.p = 1;
        sky_result r;
        run_impl(c, points, n, d, 0, 0, &cfg, &r);
        // a plain malloc block for sky_free (the result's own ids are pooled)
        *out_ids = static_cast<int64_t*>(std::malloc((r.n_ids ? r.n_ids : 1) * sizeof(int64_t)));
        if (*out_ids) std::memcpy(*out_ids, r.ids, r.n_ids * sizeof(int64_t));
        *n_out = r.n_ids;
        if (tests_out) *tests_out = r.tests_local + r.tests_merge;
        sky_result_free(&r);
        if (!*out_ids) throw std::bad_alloc();
    });
}

int sky_representatives(sky_ctx* c, const float* points, uint64_t n64, uint32_t d, const uint64_t* partition_of,
                        uint64_t p, uint64_t q, int64_t** out_ids, uint64_t* n_out) {
    c = single_gpu(c);
    return guarded(c, [&] {
        *out_ids = nullptr;
        *n_out = 0;
        if (q < 1) throw Error(SKY_E_CONFIG, "representative count q must be >= 1");
        const uint32_t n = (uint32_t)n64;
        if (n == 0) {
            *out_ids = static_cast<int64_t*>(std::malloc(sizeof(int64_t)));
            return;
        }
        const int D = padded_dim(d);
        if (!D) throw Error(SKY_E_DIMENSION, "the GPU engine supports 1 <= d <= 32");
        // run the partition + reps steps through the engine with a host-given
        // assignment (random strategy with an explicit partition_of)
        Runner R(c);
        cudaStream_t st = c->stream;
        float* dp = R.dev<float>(S_PTS, (size_t)n * d);
        SKY_CUDA(cudaMemcpyAsync(dp, points, (size_t)n * d * sizeof(float), cudaMemcpyHostToDevice, st));
        uint32_t* hp = R.pin<uint32_t>(P_PID, n);
        for (uint32_t i = 0; i < n; ++i) hp[i] = (uint32_t)partition_of[i];
        uint32_t* misc = R.dev<uint32_t>(S_MISC, 64);
        SKY_CUDA(cudaMemsetAsync(misc, 0, 64 * sizeof(uint32_t), st));
        sky_config cfg;
        sky_config_default(&cfg);
        cfg.p = p;
        uint32_t* pd = R.dev<uint32_t>(S_PID, n);
        SKY_CUDA(cudaMemcpyAsync(pd, hp, (size_t)n * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
        uint64_t fix = 0;
        PartitionOut po = partition_phase(R, dp, n, d, 0, SKY_RANDOM, p, 0, &cfg, pd, &fix);
        const uint32_t qq = (uint32_t)std::min<uint64_t>(q, n);
        uint32_t* cand = R.dev<uint32_t>(S_REPCAND, (size_t)p * qq);
        launch_rep_pick(po.key64, po.idx, po.off, (uint32_t)p, dp, nullptr, d, qq, cand, st);
        std::vector<uint32_t> hc((size_t)p * qq);
        SKY_CUDA(cudaMemcpyAsync(hc.data(), cand, hc.size() * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
        R.sync();
        std::vector<float> rows;
        std::vector<int64_t> ids;
        for (uint32_t v : hc)
            if (v != kNone) {
                ids.push_back(v);
                rows.insert(rows.end(), points + (size_t)v * d, points + (size_t)(v + 1) * d);
            }
        // prune: the skyline of the candidates (prune_dominated_reps)
        std::vector<int64_t> sk;
        uint64_t ns = 0;
        if (!ids.empty()) {
            sky_config c2;
            sky_config_default(&c2);
            c2.strategy = SKY_SLICED;
            c2.p = 1;
            sky_result r;
            run_impl(c, rows.data(), ids.size(), d, 0, 0, &c2, &r);
            sk.assign(r.ids, r.ids + r.n_ids);
            ns = r.n_ids;
            sky_result_free(&r);
        }
        std::vector<int64_t> outv;
        for (uint64_t k = 0; k < ns; ++k) outv.push_back(ids[sk[k]]);
        std::sort(outv.begin(), outv.end());
        *out_ids = static_cast<int64_t*>(std::malloc((outv.size() ? outv.size() : 1) * sizeof(int64_t)));
        std::memcpy(*out_ids, outv.data(), outv.size() * sizeof(int64_t));
        *n_out = outv.size();
    });
}

void sky_free(void* p) { std::free(p); }

int sky_generate_device(sky_ctx* c, int kind, uint64_t n, uint32_t d, uint64_t seed, float* dev_out) {
    c = single_gpu(c);
    return guarded(c, [&] {
        if (kind < 1 || kind > 5 || d < 1) throw Error(SKY_E_CONFIG, "generator kind 1..5 and d >= 1");
        if (!n) return;
        uint32_t* stuck = static_cast<uint32_t*>(c->dev.get(S_GCOUNT, 64));
        SKY_CUDA(cudaMemsetAsync(stuck, 0, sizeof(uint32_t), c->stream));
        launch_generate_baseline(kind, n, d, seed, dev_out, stuck, c->stream);
        uint32_t h = 0;
        SKY_CUDA(cudaMemcpyAsync(&h, stuck, sizeof(uint32_t), cudaMemcpyDeviceToHost, c->stream));
        SKY_CUDA(cudaStreamSynchronize(c->stream));
        if (h) {
            // a rejection loop outran the device ring: the host generator
            std::vector<float> rows(n * d);
            if (sky_generate(kind, n, d, seed, rows.data()) != SKY_OK) throw Error(SKY_E_CONFIG, "generator failed");
            SKY_CUDA(cudaMemcpy(dev_out, rows.data(), rows.size() * sizeof(float), cudaMemcpyHostToDevice));
        }
    });
}

int sky_issue_peak(sky_ctx* c, uint32_t d, int k, int ctas_per_sm, uint32_t iters, double* tests_per_s) {
    c = single_gpu(c);
    return guarded(c, [&] {
        const int D = padded_dim(d);
        if (!D || D > 16) throw Error(SKY_E_DIMENSION, "the packed-code core covers d <= 16");
        unsigned long long* sink = static_cast<unsigned long long*>(c->dev.get(S_MISC, 64 * sizeof(uint32_t)));
        if (k > 0) {
            if (ctas_per_sm < 1 || ctas_per_sm > 8 || iters < 1) throw Error(SKY_E_CONFIG, "bad microbenchmark shape");
            *tests_per_s = measure_issue_peak(D, k, ctas_per_sm, iters, c->sm_count, c->stream, sink);
            return;
        }
        double best = 0.0;
        for (int K : {4, 8})
            for (int bps : {2, 4, 8}) {
                const uint32_t iters = (uint32_t)(40000 / (K / 4) / (bps / 2));
                best = std::max(best, measure_issue_peak(D, K, bps, iters, c->sm_count, c->stream, sink));
            }
        *tests_per_s = best;
    });
}

int sky_plan_local_shards(const uint32_t* off, uint64_t P, int world, uint32_t* bounds) {
    return guarded(nullptr, [&] {
        if (world < 1) throw Error(SKY_E_CONFIG, "world must be >= 1");
        std::vector<uint32_t> o(off, off + P + 1);
        const auto b = plan_local_shards(o, (uint32_t)P, world);
        std::memcpy(bounds, b.data(), (world + 1) * sizeof(uint32_t));
    });
}

int sky_plan_merge_shards(const uint32_t* offu, uint64_t P, int world, const sky_config* cfg, uint32_t d,
                          uint64_t m, uint32_t* bounds) {
    return guarded(nullptr, [&] {
        if (world < 1) throw Error(SKY_E_CONFIG, "world must be >= 1");
        std::vector<uint32_t> o(offu, offu + P + 1);
        const bool all_mode = cfg->merge == SKY_MERGE_SEQUENTIAL || cfg->strategy == SKY_RANDOM ||
                              cfg->strategy == SKY_ANGULAR;
        const auto b = plan_merge_shards(o, (uint32_t)P, world, all_mode, cfg->strategy, m, d);
        std::memcpy(bounds, b.data(), (world + 1) * sizeof(uint32_t));
    });
}

}  // extern "C"
