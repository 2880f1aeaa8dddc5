// shard.cu — the multi-GPU run with phase 1 sharded by input rows (SURVEY
// §8(e)); one rank per GPU, exchanges through sky::Comm (NCCL or loopback).
//
// The reference runs every phase over the whole dataset in one process
// (skyline::run, engine.cpp:136-204) and fans the per-partition work out
// over threads (parallel_for, parallel.cpp:11-43). Here rank r holds rows
// [row0, row0 + nl) of the N-row relation and:
//
//  1a partition   k_prep over its own rows (partition ids, FP64 sum keys,
//                 validation); error bits agreed over the ranks. Random: the
//                 global Fisher-Yates permutation (partition.cpp:36-54) on
//                 every rank, its own slice used. Sliced (partition.cpp:
//                 186-218): the slice-key column is all-gathered and sorted
//                 on every rank; tie runs that straddle a slice boundary are
//                 ordered on a table of their rows' coordinates assembled
//                 from the owners by an all-reduce.
//  1b reps        the first q rows of each partition by (sum, lex, id) among
//                 its own rows (filter.cpp:66-86), all-gathered (P*q slots per
//                 rank), the global first q per partition picked from the
//                 W*q candidates (the global first q are among them), pruned
//                 to an antichain on every rank (prune_dominated_reps,
//                 filter.cpp:139-145): identical representatives everywhere.
//     prefilter   its own rows against the representatives (rep_prefilter,
//                 filter.cpp:147-159); survivors sorted by (partition, key,
//                 row).
//     routing     per-partition survivor counts all-gathered; partitions
//                 owned by contiguous ranges balanced by |r_i|^2; one
//                 all-to-all moves every survivor to its owner, which
//                 re-sorts by (partition, key, id) (sender order = id order
//                 on ties: ranks hold ascending row ranges).
//     local       SFS / BNL over the owned partitions (compute_local_
//                 skylines, engine.cpp:41-63).
//  2  merge       local skylines all-gathered in partition order (the union
//                 U, identical everywhere), candidates split over the ranks
//                 by test volume, survivors all-gathered (merge_phase).
//
// Configurations this path does not cover (FP64 rows, grid filtering,
// region/random representatives, d > 16, P > 4096, sliced inputs whose tie
// runs are too long) take the replicated phase 1 of run_impl.
#include "engine_impl.cuh"

namespace sky {
namespace eng {

namespace {

// ------------------------------------------------------------------ kernels
// sliced: partition id of the rank's own rows from the global rank order
// (k_slice_assign restricted to rows [row0, row0 + nl), key64 indexed locally)
__global__ void k_slice_assign_range(const uint32_t* __restrict__ rank_idx, uint32_t n, uint64_t p,
                                     uint64_t* key64, uint32_t row0, uint32_t nl) {
    const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const uint32_t row = rank_idx[r];
    if (row - row0 >= nl) return;  // unsigned: also rows below row0
    uint64_t index = n > 1 ? (uint64_t)r * p / (n - 1) : 0;
    if (index >= p) index = p - 1;
    key64[row - row0] = (index << 32) | (key64[row - row0] & 0xFFFFFFFFull);
}

// rows of the straddling tie runs, concatenated run by run (run j starts at
// table row runb[j]); only this rank's rows are written, the rest stay zero
__global__ void k_run_rows(const uint32_t* __restrict__ rank_idx, const uint32_t* __restrict__ runs,
                           const uint32_t* __restrict__ runb, const float* __restrict__ pts, uint32_t d,
                           uint32_t row0, uint32_t nl, float* __restrict__ table) {
    const uint32_t j = blockIdx.y;
    const uint32_t ra = runs[2 * j], rc = runs[2 * j + 1];
    const uint32_t e = ra + blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= rc) return;
    const uint32_t row = rank_idx[e];
    if (row - row0 >= nl) return;
    const float* x = pts + (size_t)(row - row0) * d;
    float* t = table + (size_t)(runb[j] + (e - ra)) * d;
    for (uint32_t k = 0; k < d; ++k) t[k] = x[k];
}

// exact rank inside each straddling run by (lex coords, id) on the table
// (k_slice_fix_runs, partition.cpp:202-216), written for the own rows
__global__ void k_slice_fix_runs_tab(const float* __restrict__ table, uint32_t d,
                                     const uint32_t* __restrict__ rank_idx, uint32_t n, uint64_t p,
                                     const uint32_t* __restrict__ runs, const uint32_t* __restrict__ runb,
                                     uint64_t* key64, uint32_t row0, uint32_t nl) {
    const uint32_t j = blockIdx.y;
    const uint32_t ra = runs[2 * j], rc = runs[2 * j + 1];
    const uint32_t e = ra + blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= rc) return;
    const uint32_t row = rank_idx[e];
    if (row - row0 >= nl) return;
    const float* me = table + (size_t)(runb[j] + (e - ra)) * d;
    uint32_t rank = 0;
    for (uint32_t f = ra; f < rc; ++f) {
        if (f == e) continue;
        const float* o = table + (size_t)(runb[j] + (f - ra)) * d;
        int c = 0;
        for (uint32_t k = 0; k < d && !c; ++k) c = o[k] < me[k] ? -1 : (o[k] > me[k] ? 1 : 0);
        if (c < 0 || (c == 0 && rank_idx[f] < row)) ++rank;
    }
    uint64_t index = n > 1 ? (uint64_t)(ra + rank) * p / (n - 1) : 0;
    if (index >= p) index = p - 1;
    key64[row - row0] = (index << 32) | (key64[row - row0] & 0xFFFFFFFFull);
}

// the rank's representative picks as table rows: coordinates (zeros for an
// empty slot) and global row ids (kNone for an empty slot)
__global__ void k_cand_rows(const uint32_t* __restrict__ cand, uint32_t slots, const float* __restrict__ pts,
                            uint32_t d, uint32_t row0, float* __restrict__ tab, uint32_t* __restrict__ ids) {
    const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= slots) return;
    const uint32_t r = cand[s];
    ids[s] = r == kNone ? kNone : row0 + r;
    for (uint32_t k = 0; k < d; ++k) tab[(size_t)s * d + k] = r == kNone ? 0.0f : pts[(size_t)r * d + k];
}

// Global first q of partition p among the ranks' picks (slots r*P*q + p*q + k):
// rank of each candidate under (FP64 coordinate sum, lex coords, id)
// (filter.cpp:74-79); out[p*q + rank] = slot for rank < q.
__global__ void __launch_bounds__(256) k_rep_merge(const float* __restrict__ tab, const uint32_t* __restrict__ ids,
                                                   uint32_t W, uint32_t P, uint32_t q, uint32_t d,
                                                   uint32_t* __restrict__ out) {
    extern __shared__ __align__(8) unsigned char s_rm[];
    const uint32_t p = blockIdx.x;
    const uint32_t C = W * q;
    double* s_sum = reinterpret_cast<double*>(s_rm);
    uint32_t* s_slot = reinterpret_cast<uint32_t*>(s_sum + C);
    for (uint32_t k = threadIdx.x; k < q; k += blockDim.x) out[(size_t)p * q + k] = kNone;
    for (uint32_t c = threadIdx.x; c < C; c += blockDim.x) {
        const uint32_t r = c / q, k = c % q;
        const uint32_t slot = (r * P + p) * q + k;
        s_slot[c] = slot;
        double s = 0.0;
        if (ids[slot] != kNone)
            for (uint32_t j = 0; j < d; ++j) s = __dadd_rn(s, (double)tab[(size_t)slot * d + j]);
        s_sum[c] = s;
    }
    __syncthreads();
    for (uint32_t c = threadIdx.x; c < C; c += blockDim.x) {
        const uint32_t sc = s_slot[c];
        const uint32_t idc = ids[sc];
        if (idc == kNone) continue;
        const double mc = s_sum[c];
        uint32_t rank = 0;
        for (uint32_t o = 0; o < C && rank < q; ++o) {
            const uint32_t so = s_slot[o];
            const uint32_t ido = ids[so];
            if (o == c || ido == kNone) continue;
            const double mo = s_sum[o];
            bool less = mo < mc;
            if (mo == mc) {
                int cmp = 0;
                for (uint32_t j = 0; j < d && !cmp; ++j) {
                    const float a = tab[(size_t)so * d + j], b = tab[(size_t)sc * d + j];
                    cmp = a < b ? -1 : (a > b ? 1 : 0);
                }
                less = cmp < 0 || (cmp == 0 && ido < idc);
            }
            rank += less ? 1u : 0u;
        }
        if (rank < q) out[(size_t)p * q + rank] = sc;
    }
}

__global__ void k_seg_counts(const uint32_t* __restrict__ off, uint32_t P, uint32_t* __restrict__ cnt) {
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p < P) cnt[p] = off[p + 1] - off[p];
}

__global__ void k_add_u32(uint32_t* __restrict__ v, uint32_t n, uint32_t add) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) v[i] += add;
}

// received rows: partition ids relative to the owner's first partition, and
// the 32-bit sum key of each row
__global__ void k_rebase_keys(uint64_t* __restrict__ k64, uint32_t n, uint32_t pb, uint32_t* __restrict__ skey) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint64_t k = k64[i] - ((uint64_t)pb << 32);
    k64[i] = k;
    skey[i] = (uint32_t)k;
}

}  // namespace

// The configuration is covered by the sharded phase 1 (else run_impl's
// replicated phase 1 runs on every rank).
bool sharded_eligible(const sky_config* cfg, uint64_t N, uint32_t d, bool f64) {
    if (f64 || N == 0 || d == 0) return false;
    const int D = padded_dim(d);
    if (!D || D > 16) return false;
    uint64_t P = 0, m = 0;
    resolve_partitions(N, d, cfg, &P, &m);
    if (bits_for(P) > 12) return false;
    if (cfg->filter == SKY_FILTER_NONE) return true;
    if (cfg->filter != SKY_FILTER_REPRESENTATIVE || cfg->rep_selection != SKY_REPS_SORTED) return false;
    const uint64_t q = std::min<uint64_t>(cfg->rep_q, N);
    return q <= 64 && P * q <= 2048;
}

void run_sharded(sky_ctx* c, const float* src, uint32_t nl, uint32_t row0, const std::vector<uint32_t>& rows_of,
                 uint32_t d, int normalized, int on_device, const sky_config* cfg, sky_result* out) {
    const int W = c->world, rank = c->rank;
    Comm& comm = *c->comm;
    uint64_t N64 = 0;
    for (uint32_t v : rows_of) N64 += v;
    std::memset(out, 0, sizeof(*out));
    validate(N64, d, cfg);
    uint64_t P64 = 0, m = 0;
    resolve_partitions(N64, d, cfg, &P64, &m);
    const uint32_t N = (uint32_t)N64, P = (uint32_t)P64;
    out->effective_p = P;
    out->input_size = N;
    out->input_dim = d;
    out->world = (uint32_t)W;
    out->sharded = 1;
    out->local_rows = nl;
    out->local_skyline_sizes = static_cast<uint64_t*>(std::calloc(P ? P : 1, sizeof(uint64_t)));
    c->launches = 0;
    c->dom_launches = 0;
    c->dom_ms = 0.0;
    const bool count_tests = cfg->count_tests != 0;
    const int D = padded_dim(d);
    const int strategy = cfg->strategy;
    const bool reps_on = cfg->filter == SKY_FILTER_REPRESENTATIVE;

    Runner R(c);
    R.s0_dims_ = d;
    cudaStream_t st = c->stream;
    SKY_CUDA(cudaEventRecord(c->ev[0], st));
    uint32_t* misc = R.dev<uint32_t>(S_MISC, 64);
    SKY_CUDA(cudaMemsetAsync(misc, 0, 64 * sizeof(uint32_t), st));
    uint64_t sent = 0;  // bytes this rank sends to its peers

    // ----------------------------------------------------------- own rows
    const float* pts = src;
    {
        int dev_of_src = c->device;
        if (on_device) {
            cudaPointerAttributes at{};
            SKY_CUDA(cudaPointerGetAttributes(&at, src));
            dev_of_src = at.device;
        }
        // the streamed kernels need 16-byte aligned rows on this device
        if (!on_device || dev_of_src != c->device || ((uintptr_t)src & 15)) {
            float* dp = R.dev<float>(S_PTS, (size_t)nl * d);
            if (nl) SKY_CUDA(cudaMemcpyAsync(dp, src, (size_t)nl * d * sizeof(float), cudaMemcpyDefault, st));
            if (!on_device) out->h2d_bytes += (uint64_t)nl * d * sizeof(float);
            pts = dp;
        }
    }

    // -------------------------------------------- 1a: partition own rows
    const uint32_t* pid_in = nullptr;
    if (strategy == SKY_RANDOM) pid_in = R.random_pids(N, P, cfg->seed, false) + row0;
    const uint32_t key_shift = key_shift_for(P);
    const int pb = std::max(1, bits_for(P));
    const uint32_t q = reps_on ? (uint32_t)std::min<uint64_t>(cfg->rep_q, N) : 0;
    // representative candidates from per-CTA partition minima (no sort of
    // the own rows) when the rows are many
    bool stream_reps = reps_on && strategy != SKY_SLICED && (uint64_t)nl * d * sizeof(float) > (32ull << 20) &&
                       (uint64_t)P * kRepBucket <= (1ull << 31);
    const uint32_t prep_grid = stream_reps ? prep_stream_grid(nl, d, P, c->sm_count, strategy) : 0;
    uint64_t* keyA = R.dev<uint64_t>(S_KEY_A, nl);
    uint32_t* skA = strategy == SKY_SLICED ? R.dev<uint32_t>(S_SK_A, nl) : nullptr;
    const uint32_t amb_cap = strategy == SKY_ANGULAR ? std::max<uint32_t>(nl, 1) : 1u;
    uint32_t* amb = R.dev<uint32_t>(S_AMB, amb_cap);
    uint32_t* gmin = stream_reps ? R.dev<uint32_t>(S_GMIN, (size_t)prep_grid * P) : nullptr;
    PrepArgs pa{pts, nullptr, nl, d, strategy, m, normalized, pid_in, (uint32_t)cfg->slice_dim, keyA, nullptr, skA,
                misc + M_ERR, misc + M_AMB, amb, amb_cap, key_shift};
    if (gmin) {
        pa.gmin = gmin;
        pa.P = P;
    }
    if (strategy == SKY_ANGULAR && m >= 2) {
        pa.ang_thr = R.angular_table(m);
        volatile double one = 1.0;
        pa.ang_c45 = std::atan2(one, one);  // the host libm's atan2(x, x) (partition.cpp:128)
        if (m <= 8) {
            const double PI = 3.14159265358979323846;
            for (uint64_t k = 1; k < m; ++k) {
                const double t = std::tan((double)k * PI / (2.0 * (double)m));
                pa.tan2[k - 1] = (float)(t * t);
            }
        }
    }
    R.hbm_begin();
    launch_prep(pa, st, c->sm_count);
    R.hbm_end((uint64_t)nl * d * 4 + (uint64_t)nl * 8 + (skA ? 4ull * nl : 0ull));
    R.count();
    // errors (agreed: every rank raises the same) and angular boundary rows
    uint32_t* hm = R.pin<uint32_t>(P_MISC, 8);
    SKY_CUDA(cudaMemcpyAsync(hm, misc, 4 * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    R.sync();
    const uint32_t n_amb = std::min(hm[M_AMB], amb_cap);
    check_prep(R.agree_errors(hm[M_ERR]), 0, strategy, true);
    if (strategy == SKY_ANGULAR && n_amb) {
        out->angular_host_fixups = angular_fixups(R, pts, d, m, keyA, amb, n_amb);
        stream_reps = false;  // the partition minima predate the fixed ids
    }

    if (strategy == SKY_SLICED && N > 0) {
        // the slice-key column of every rank, in global row order
        uint32_t* skG = R.dev<uint32_t>(S_SH_SKG, N);
        uint32_t* skB = R.dev<uint32_t>(S_SK_B, N);
        uint32_t* iota = R.dev<uint32_t>(S_SH_IOTA, N);
        uint32_t* rankA = R.dev<uint32_t>(S_PERM_A, N);
        {
            std::vector<size_t> b(W), dp(W);
            size_t at = 0;
            for (int k = 0; k < W; ++k) {
                b[k] = (size_t)rows_of[k] * 4;
                dp[k] = at;
                at += b[k];
            }
            comm.allgatherv(skA, skG, b.data(), dp.data(), st);
            sent += (uint64_t)nl * 4 * (W - 1);
        }
        launch_iota(N, iota, st);
        R.count();
        R.sort_pairs(skG, skB, iota, rankA, N, 0, 32);
        const uint32_t run_cap = (uint32_t)std::min<uint64_t>(P, 1u << 20);
        uint32_t* runs = R.dev<uint32_t>(S_RUNS, 2 * (size_t)run_cap);
        SKY_CUDA(cudaMemsetAsync(misc + M_RUNS, 0, sizeof(uint32_t), st));
        launch_slice_runs(skB, N, P, runs, misc + M_RUNS, run_cap, st);
        R.count();
        SKY_CUDA(cudaMemcpyAsync(hm, misc + M_RUNS, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
        R.sync();
        const uint32_t nruns = std::min(hm[0], run_cap);
        std::vector<uint32_t> runb(nruns + 1, 0);
        uint64_t cost = 0;
        uint32_t max_len = 0;
        if (nruns) {
            uint32_t* h = R.pin<uint32_t>(P_SH_RUNS, 2 * (size_t)nruns);
            SKY_CUDA(cudaMemcpyAsync(h, runs, 2 * (size_t)nruns * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
            R.sync();
            // the kernel lists the runs in atomic order: sort them, so every
            // rank lays out the run table (assembled by an all-reduce) alike
            std::vector<uint2> rl(nruns);
            for (uint32_t k = 0; k < nruns; ++k) rl[k] = make_uint2(h[2 * k], h[2 * k + 1]);
            std::sort(rl.begin(), rl.end(), [](const uint2& a, const uint2& b) { return a.x < b.x; });
            uint32_t* hs = R.stage<uint32_t>(2 * (size_t)nruns);
            for (uint32_t k = 0; k < nruns; ++k) {
                hs[2 * k] = rl[k].x;
                hs[2 * k + 1] = rl[k].y;
                const uint32_t L = rl[k].y - rl[k].x;
                runb[k + 1] = runb[k] + L;
                cost += (uint64_t)L * L;
                max_len = std::max(max_len, L);
            }
            SKY_CUDA(cudaMemcpyAsync(runs, hs, 2 * (size_t)nruns * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
        }
        // every rank sees the same runs: the same decision everywhere
        if (cost > (uint64_t)1e9) throw ReplicatePhase1{};
        {
            uint32_t grid = ceil_div(N, 256);
            k_slice_assign_range<<<grid, 256, 0, st>>>(rankA, N, P, keyA, row0, nl);
            SKY_LAUNCH_CHECK();
            R.count();
        }
        if (nruns) {
            const uint32_t L = runb[nruns];
            uint32_t* hb = R.stage<uint32_t>(nruns + 1);
            std::memcpy(hb, runb.data(), (nruns + 1) * sizeof(uint32_t));
            uint32_t* db = R.dev<uint32_t>(S_SH_RUNB, nruns + 1);
            SKY_CUDA(cudaMemcpyAsync(db, hb, (nruns + 1) * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
            float* tab = R.dev<float>(S_SH_TAB, (size_t)L * d);
            SKY_CUDA(cudaMemsetAsync(tab, 0, (size_t)L * d * sizeof(float), st));
            const dim3 grid(ceil_div(max_len, 256), nruns);
            k_run_rows<<<grid, 256, 0, st>>>(rankA, runs, db, pts, d, row0, nl, tab);
            SKY_LAUNCH_CHECK();
            comm.allreduce_sum_f32(tab, (size_t)L * d, st);
            sent += (uint64_t)L * d * 4;
            k_slice_fix_runs_tab<<<grid, 256, 0, st>>>(tab, d, rankA, N, P, runs, db, keyA, row0, nl);
            SKY_LAUNCH_CHECK();
            R.count(2);
        }
    }
    SKY_CUDA(cudaEventRecord(c->ev[1], st));

    // the own rows in (partition, key, row) order (sorted path)
    uint64_t* keyB = nullptr;
    uint32_t* idxB = nullptr;
    uint32_t* offL = nullptr;
    auto sort_own = [&]() {
        if (keyB) return;
        keyB = R.dev<uint64_t>(S_KEY_B, nl);
        idxB = R.dev<uint32_t>(S_IDX_B, nl);
        uint32_t* iota = R.dev<uint32_t>(S_IDX_A, nl);
        launch_iota(nl, iota, st);
        R.count();
        R.sort_pairs(keyA, keyB, iota, idxB, nl, (int)key_shift, std::min(64, 32 + pb));
        offL = R.dev<uint32_t>(S_OFF_A, P + 1);
        launch_seg_offsets(keyB, nl, P, offL, st);
        R.count();
    };

    // -------------------------------- 1b: representatives + prefilter
    uint64_t* k64 = nullptr;  // survivors: (pid << 32 | key), partition order
    uint32_t* rows = nullptr;
    uint32_t* off1 = R.dev<uint32_t>(S_OFF_B, P + 1);
    uint32_t ns = 0;
    if (reps_on) {
        const uint32_t slots = P * q;
        uint32_t* cand = R.dev<uint32_t>(S_REPCAND, slots);
        bool have = false;
        if (stream_reps) {
            uint32_t* thr = R.dev<uint32_t>(S_PTHR2, P);
            uint32_t* bcnt = R.dev<uint32_t>(S_BCNT, P);
            uint64_t* bkey = R.dev<uint64_t>(S_BKEY, (size_t)P * kRepBucket);
            uint32_t* brow = R.dev<uint32_t>(S_BROW, (size_t)P * kRepBucket);
            cudaEvent_t pb, pe;
            R.hbm_pair((uint64_t)nl * 8, &pb, &pe);
            launch_rep_candidates(keyA, nl, P, q, prep_grid, gmin, thr, kRepBucket, bcnt, bkey, brow, pts, d, cand,
                                  misc + M_OVF, st, pb, pe);
            R.count(3);
            SKY_CUDA(cudaMemcpyAsync(hm, misc + M_OVF, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
            R.sync();
            have = hm[0] == 0;  // a bucket that filled up: pick from the sorted rows
        }
        if (!have) {
            sort_own();
            launch_rep_pick(keyB, idxB, offL, P, pts, nullptr, d, q, cand, st);
            R.count();
        }
        // the picks of every rank, then the global first q of each partition
        float* tab = R.dev<float>(S_SH_TAB, (size_t)slots * d);
        uint32_t* ids = R.dev<uint32_t>(S_SH_IDS, slots);
        k_cand_rows<<<ceil_div(slots, 256), 256, 0, st>>>(cand, slots, pts, d, row0, tab, ids);
        SKY_LAUNCH_CHECK();
        R.count();
        float* taball = R.dev<float>(S_SH_TABALL, (size_t)W * slots * d);
        uint32_t* idsall = R.dev<uint32_t>(S_SH_IDSALL, (size_t)W * slots);
        comm.allgather(tab, taball, (size_t)slots * d * sizeof(float), st);
        comm.allgather(ids, idsall, (size_t)slots * sizeof(uint32_t), st);
        sent += (uint64_t)slots * (d * 4 + 4) * (W - 1);
        uint32_t* candg = R.dev<uint32_t>(S_SH_CANDG, slots);
        const size_t smem = (size_t)W * q * (sizeof(double) + sizeof(uint32_t));
        ensure_smem_attr((const void*)k_rep_merge, smem);
        k_rep_merge<<<P, 256, smem, st>>>(taball, idsall, (uint32_t)W, P, q, d, candg);
        SKY_LAUNCH_CHECK();
        R.count();
        DevSet reps = R.set(S_SET3, slots, D);
        uint32_t* nrep_dev = misc + M_NREP;
        // every rank prunes the same picks: count the tests once
        unsigned long long* rt = count_tests && rank == 0 ? R.tests(0) : nullptr;
        if (launch_rep_finalize_par(D, candg, slots, taball, d, reps, nrep_dev, rt, X64{}, c->smem_optin,
                                    c->sm_count, R.dev<char>(S_REPF, rep_finalize_scratch_bytes(D)), st)) {
            R.count(3);
        } else if (launch_rep_finalize(D, candg, slots, taball, d, reps, nrep_dev, rt, X64{}, c->smem_optin, st)) {
            R.count();
        } else {
            throw Error(SKY_E_INTERNAL, "representative finish not applicable");
        }
        float* pthr = nullptr;
        if (reps.qc) {
            pthr = R.dev<float>(S_PTHR, (size_t)D * (kCodeLevels - 1));
            launch_thresholds_rows(D, pts, d, nl, pthr, st, nrep_dev, 32);
            launch_encode(D, reps, pthr, st, nrep_dev);
            R.count(2);
        }
        PrefilterAppend app;
        app.key64 = keyA;
        app.out = R.dev<uint64_t>(S_SURV, nl);
        app.count = misc + M_S0;
        app.key_shift = key_shift;
        app.row_bits = (uint32_t)std::max(1, bits_for(nl));
        R.hbm_begin();
        if (!launch_prefilter_append(D, pts, d, nl, reps.xyz, reps.skey, pthr ? reps.qc : nullptr, reps.id, reps.n,
                                     nrep_dev, pthr, app, count_tests ? R.tests(1) : nullptr, c->smem_optin, st))
            throw Error(SKY_E_INTERNAL, "stream prefilter not applicable");
        R.hbm_end((uint64_t)nl * (4ull * d + 8));
        R.count();
        uint32_t* hc = R.pin<uint32_t>(P_MISC, 32);
        SKY_CUDA(cudaMemcpyAsync(hc, misc, 32 * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
        R.sync();
        ns = hc[M_S0];
        out->n_reps = hc[M_NREP];
        uint64_t* surv2 = R.dev<uint64_t>(S_SURV2, std::max<uint32_t>(ns, 1));
        R.sort_keys(app.out, surv2, ns, 32 + pb - (int)key_shift + (int)app.row_bits);
        k64 = R.dev<uint64_t>(S_KEY_B, std::max<uint32_t>(ns, 1));
        rows = R.dev<uint32_t>(S_IDX_B, std::max<uint32_t>(ns, 1));
        launch_unpack_survivors(surv2, ns, app.row_bits, key_shift, P, k64, rows, off1, st);
        R.count();
    } else {
        sort_own();
        k64 = keyB;
        rows = idxB;
        ns = nl;
        SKY_CUDA(cudaMemcpyAsync(off1, offL, (P + 1) * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st));
    }

    // ----------------------------------------------------------- routing
    // per-partition survivor counts of every rank
    uint32_t* cnt = R.dev<uint32_t>(S_SH_CNT, (size_t)(W + 1) * P);
    k_seg_counts<<<ceil_div(P, 256), 256, 0, st>>>(off1, P, cnt + (size_t)W * P);
    SKY_LAUNCH_CHECK();
    R.count();
    comm.allgather(cnt + (size_t)W * P, cnt, (size_t)P * sizeof(uint32_t), st);
    sent += (uint64_t)P * 4 * (W - 1);
    uint32_t* hcnt = R.pin<uint32_t>(P_SH_CNT, (size_t)W * P);
    SKY_CUDA(cudaMemcpyAsync(hcnt, cnt, (size_t)W * P * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    R.sync();
    std::vector<uint32_t> offS(P + 1, 0);
    for (uint32_t p = 0; p < P; ++p) {
        uint64_t s = 0;
        for (int k = 0; k < W; ++k) s += hcnt[(size_t)k * P + p];
        offS[p + 1] = offS[p] + (uint32_t)s;
    }
    out->filtered_count = (uint64_t)N - offS[P];
    // owners: contiguous partition ranges balanced by |r_i|^2
    const std::vector<uint32_t> pr = plan_local_shards(offS, P, W);
    const uint32_t pbeg = pr[rank], pend = pr[rank + 1], Pm = pend - pbeg;
    std::vector<uint32_t> offMine(P + 1, 0);  // this rank's survivors per partition (prefix)
    for (uint32_t p = 0; p < P; ++p) offMine[p + 1] = offMine[p] + hcnt[(size_t)rank * P + p];
    std::vector<size_t> sb(W), sd(W), rb(W), rd(W);
    uint32_t n_recv = 0;
    for (int k = 0; k < W; ++k) {
        sd[k] = offMine[pr[k]];
        sb[k] = offMine[pr[k + 1]] - offMine[pr[k]];
        uint32_t r = 0;
        for (uint32_t p = pbeg; p < pend; ++p) r += hcnt[(size_t)k * P + p];
        rd[k] = n_recv;
        rb[k] = r;
        n_recv += r;
    }
    // the survivors as sendable rows (coordinates padded to D4, global ids)
    DevSet snd = R.set(S_SETS, std::max<uint32_t>(ns, 1), D);
    snd.n = ns;
    launch_scatter_indirect(D, pts, d, rows, k64, ns, nullptr, nullptr, snd, st);
    if (ns) {
        k_add_u32<<<ceil_div(ns, 256), 256, 0, st>>>(snd.id, ns, row0);
        SKY_LAUNCH_CHECK();
    }
    R.count(2);
    DevSet rcv = R.set(S_SETR, std::max<uint32_t>(n_recv, 1), D);
    rcv.n = n_recv;
    uint64_t* k64r = R.dev<uint64_t>(S_SH_K64R, std::max<uint32_t>(n_recv, 1));
    const size_t D4 = (size_t)(D + 3) / 4 * 4;
    auto a2a = [&](const void* s, void* r, size_t unit) {
        std::vector<size_t> b1(W), d1(W), b2(W), d2(W);
        for (int k = 0; k < W; ++k) {
            b1[k] = sb[k] * unit;
            d1[k] = sd[k] * unit;
            b2[k] = rb[k] * unit;
            d2[k] = rd[k] * unit;
            if (k != rank) sent += b1[k];
        }
        comm.alltoallv(s, b1.data(), d1.data(), r, b2.data(), d2.data(), st);
    };
    a2a(snd.xyz, rcv.xyz, D4 * sizeof(float));
    a2a(k64, k64r, sizeof(uint64_t));
    a2a(snd.id, rcv.id, sizeof(uint32_t));
    // owned partitions in (partition, key, id) order
    DevSet s0 = R.set(S_SET0, std::max<uint32_t>(n_recv, 1), D);
    s0.n = n_recv;
    uint32_t* offm = R.dev<uint32_t>(S_SH_OFFM, Pm + 1);
    if (n_recv) {
        k_rebase_keys<<<ceil_div(n_recv, 256), 256, 0, st>>>(k64r, n_recv, pbeg, rcv.skey);
        SKY_LAUNCH_CHECK();
        uint64_t* k64s = R.dev<uint64_t>(S_SH_K64S, n_recv);
        uint32_t* iota = R.dev<uint32_t>(S_SH_IOTA, n_recv);
        uint32_t* perm = R.dev<uint32_t>(S_SH_PERM, n_recv);
        launch_iota(n_recv, iota, st);
        R.count(2);
        R.sort_pairs(k64r, k64s, iota, perm, n_recv, (int)key_shift, std::min(64, 32 + std::max(1, bits_for(Pm))));
        DevSet rcv_nq = rcv;
        rcv_nq.qc = nullptr;
        launch_gather_set(D, rcv_nq, perm, s0, st);
        launch_seg_offsets(k64s, n_recv, Pm, offm, st);
        R.count(2);
    } else {
        SKY_CUDA(cudaMemsetAsync(offm, 0, (Pm + 1) * sizeof(uint32_t), st));
    }

    // ------------------------------------------ local skylines (owned)
    uint32_t* hn = R.stage<uint32_t>(1);
    *hn = n_recv;
    SKY_CUDA(cudaMemcpyAsync(misc + M_S0, hn, sizeof(uint32_t), cudaMemcpyHostToDevice, st));
    uint32_t* offum_dev = R.dev<uint32_t>(S_SH_OFFU, Pm + 1);  // not S_OFF_C: the local phase's waves use it
    DevSet Um;
    std::vector<uint32_t> offum(Pm + 1, 0);
    if (n_recv && Pm) {
        R.encode_dev(D, s0, misc + M_S0);
        if (cfg->local_algo == SKY_LOCAL_BNL) {
            uint32_t used = 0;
            std::vector<uint32_t> unused;
            Um = R.local_bnl(D, s0, offm, Pm, cfg->bnl_window_cap, offum_dev, unused, count_tests, &used, misc + M_U);
        } else {
            Um = R.local_sfs_dev(D, s0, misc + M_S0, offm, Pm, offum_dev, misc + M_U, count_tests);
        }
        uint32_t* h = R.pin<uint32_t>(P_SH_OFF, Pm + 1);
        SKY_CUDA(cudaMemcpyAsync(h, offum_dev, (Pm + 1) * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
        R.sync();
        offum.assign(h, h + Pm + 1);
    } else {
        Um = R.set(S_SET2, 1, D);
        Um.n = 0;
    }

    // -------------------------------------------- union on every rank
    std::vector<uint32_t> offu;
    uint32_t* offu_dev = R.dev<uint32_t>(S_OFF_A, P + 1);
    // codes are re-derived from the union itself (the ranks' local
    // quantizations differ), so every rank encodes the same U identically
    DevSet U = R.gather_union(D, Um, offum, pr, P, offu, offu_dev, false);
    sent += (uint64_t)offum[Pm] * (D4 * 4 + 8) * (W - 1);
    R.encode(D, U);
    out->exchange_bytes = sent;
    merge_phase(R, c, cfg, U, offu, offu_dev, P, m, d, D, N, count_tests, false, out);
    out->world = (uint32_t)W;
    out->sharded = 1;
    out->local_rows = nl;
    out->exchange_bytes = sent;
}

}  // namespace eng
}  // namespace sky
