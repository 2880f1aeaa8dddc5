// ref_shim.cpp — TEST INFRASTRUCTURE ONLY.
//
// extern "C" entry points over the UNMODIFIED reference engine
// (/root/reference/proj/src/*.cpp, compiled in place by oracle/Makefile into
// oracle/_ref/libskyref.so). Used by tests to pin oracle/sky_oracle.c, by
// tests/golden/make_golden.py to produce fixtures, and by bench.py's
// `--impl reference` arm to time the reference's own CPU path.
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "skyline/core.hpp"
#include "skyline/datagen.hpp"
#include "skyline/engine.hpp"
#include "skyline/filter.hpp"
#include "skyline/partition.hpp"
#include "skyline/sequential.hpp"
#include "../include/skyline_b200.h"
#include "../include/skyline_baseline_gen.h"

using namespace skyline;

namespace {

template <class T>
Dataset to_dataset(const T* pts, uint64_t n, uint32_t d, int normalized) {
    Dataset r;
    r.d = d;
    r.normalized = normalized != 0;
    r.points.resize(n);
    for (uint64_t i = 0; i < n; ++i) {
        r.points[i].coords.assign(pts + i * d, pts + (i + 1) * d);  // float -> double, exact
        r.points[i].id = static_cast<PointId>(i);
    }
    return r;
}

EngineConfig to_engine(const sky_config* c) {
    EngineConfig e;
    e.partition.strategy = static_cast<Strategy>(c->strategy);
    e.partition.p = c->p;
    e.partition.m = c->m;
    e.partition.seed = c->seed;
    e.partition.slice_dim = c->slice_dim;
    e.filter = static_cast<FilterKind>(c->filter);
    e.rep_selection = static_cast<RepSelection>(c->rep_selection);
    e.rep_q = c->rep_q;
    e.merge = static_cast<MergeKind>(c->merge);
    e.workers = c->workers;
    e.seed = c->rep_seed;
    return e;
}

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return SKY_OK;
    } catch (const ConfigError&) {
        return SKY_E_CONFIG;
    } catch (const DimensionError&) {
        return SKY_E_DIMENSION;
    } catch (const NormalizationError&) {
        return SKY_E_NORMALIZATION;
    } catch (const DataError&) {
        return SKY_E_DATA;
    } catch (const IoError&) {
        return SKY_E_IO;
    } catch (...) {
        return SKY_E_INTERNAL;
    }
}

}  // namespace

extern "C" {

struct skyref_result {
    int64_t* ids;
    uint64_t n_ids;
    uint64_t effective_p;
    uint64_t union_size, filtered_count, final_size, n_reps;
    uint64_t* local_skyline_sizes;
    double partition_ms, local_ms, merge_ms, run_ms;
};

int skyref_hardware_concurrency(void) {
    unsigned n = std::thread::hardware_concurrency();
    return n ? static_cast<int>(n) : 1;
}

// skyline::run on float32 rows upcast to double. run_ms is the steady_clock
// time of run() alone (engine.cpp:144-194 phase timers summed by the caller).
extern "C++" {
template <class T>
int run_any(const T* pts, uint64_t n, uint32_t d, int normalized, const sky_config* cfg, skyref_result* out) {
    std::memset(out, 0, sizeof(*out));
    return guarded([&] {
        const Dataset r = to_dataset(pts, n, d, normalized);
        const EngineConfig e = to_engine(cfg);
        auto t0 = std::chrono::steady_clock::now();
        RunResult res = run(r, e);
        auto t1 = std::chrono::steady_clock::now();
        out->run_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
        out->n_ids = res.skyline.size();
        out->ids = static_cast<int64_t*>(std::malloc((out->n_ids ? out->n_ids : 1) * sizeof(int64_t)));
        for (uint64_t i = 0; i < out->n_ids; ++i) out->ids[i] = res.skyline.points[i].id;
        out->effective_p = res.effective_p;
        out->union_size = res.metrics.union_size;
        out->filtered_count = res.metrics.filtered_count;
        out->final_size = res.metrics.final_size;
        const auto& ls = res.metrics.local_skyline_sizes;
        out->local_skyline_sizes =
            static_cast<uint64_t*>(std::malloc((ls.size() ? ls.size() : 1) * sizeof(uint64_t)));
        for (size_t i = 0; i < ls.size(); ++i) out->local_skyline_sizes[i] = ls[i];
        out->partition_ms = res.metrics.partition_ms;
        out->local_ms = res.metrics.local_ms;
        out->merge_ms = res.metrics.merge_ms;
    });
}
}  // extern "C++"

int skyref_run(const float* pts, uint64_t n, uint32_t d, int normalized, const sky_config* cfg,
               skyref_result* out) {
    return run_any(pts, n, d, normalized, cfg, out);
}

// skyline::run on FP64 rows (the reference's own coordinate type).
int skyref_run_f64(const double* pts, uint64_t n, uint32_t d, int normalized, const sky_config* cfg,
                   skyref_result* out) {
    return run_any(pts, n, d, normalized, cfg, out);
}

// skyline::generate (datagen.cpp:127-151): dist 0 uniform, 1 correlated,
// 2 anticorrelated; rows into out[n*d].
// BASELINE.json's synthetic inputs (include/skyline_baseline_gen.h): the
// same bytes the product's sky_generate writes, so the reference arm and the
// golden script never load the product library to build their input.
int skyref_generate_baseline(int kind, uint64_t n, uint32_t d, uint64_t seed, float* out) {
    return sky_baseline_gen::generate(kind, n, d, seed, out) ? SKY_OK : SKY_E_CONFIG;
}

int skyref_generate(int dist, uint64_t n, uint64_t d, uint64_t seed, double* out) {
    return guarded([&] {
        GenSpec g;
        g.distribution = static_cast<Distribution>(dist);
        g.n = n;
        g.d = d;
        g.seed = seed;
        const Dataset r = generate(g);
        for (uint64_t i = 0; i < n; ++i)
            for (uint64_t j = 0; j < d; ++j) out[i * d + j] = r.points[i].coords[j];
    });
}

// skyline::ingest_csv (datagen.cpp:170-218); *rows malloc'ed.
int skyref_ingest_csv(const char* path, const char* const* cols, uint32_t ncols, const uint8_t* maxflags,
                      uint32_t nmax, double** rows, uint64_t* n, uint32_t* d) {
    *rows = nullptr;
    *n = 0;
    *d = 0;
    return guarded([&] {
        std::vector<std::string> columns(cols, cols + ncols);
        std::vector<Direction> dirs;
        for (uint32_t j = 0; j < nmax; ++j) dirs.push_back(maxflags[j] ? Direction::Max : Direction::Min);
        const Dataset r = ingest_csv(path, columns, dirs);
        *n = r.size();
        *d = static_cast<uint32_t>(r.d);
        *rows = static_cast<double*>(std::malloc((r.size() * r.d ? r.size() * r.d : 1) * sizeof(double)));
        for (uint64_t i = 0; i < r.size(); ++i)
            for (uint64_t j = 0; j < r.d; ++j) (*rows)[i * r.d + j] = r.points[i].coords[j];
    });
}

// skyline::write_csv (datagen.cpp:220-238).
int skyref_write_csv(const char* path, const double* rows, uint64_t n, uint32_t d) {
    return guarded([&] {
        Dataset r;
        r.d = d;
        r.points.resize(n);
        for (uint64_t i = 0; i < n; ++i) {
            r.points[i].coords.assign(rows + i * d, rows + (i + 1) * d);
            r.points[i].id = static_cast<PointId>(i);
        }
        write_csv(r, path);
    });
}

void skyref_free(void* p) { std::free(p); }

void skyref_result_free(skyref_result* r) {
    std::free(r->ids);
    std::free(r->local_skyline_sizes);
    std::memset(r, 0, sizeof(*r));
}

int skyref_assign(const float* pts, uint64_t n, uint32_t d, int normalized, const sky_config* cfg,
                  uint64_t* partition_of, uint64_t* count) {
    return guarded([&] {
        const Dataset r = to_dataset(pts, n, d, normalized);
        PartitionAssignment a = make_assignment(r, to_engine(cfg).partition);
        for (uint64_t i = 0; i < n; ++i) partition_of[i] = a.partition_of[i];
        *count = a.partition_count;
    });
}

uint64_t skyref_bruteforce(const float* pts, uint64_t n, uint32_t d, int64_t* out) {
    const Dataset r = to_dataset(pts, n, d, 0);
    SkylineSet s = skyline_bruteforce(r);
    for (size_t i = 0; i < s.size(); ++i) out[i] = s.points[i].id;
    return s.size();
}

uint64_t skyref_sfs(const float* pts, uint64_t n, uint32_t d, int64_t* out) {
    const Dataset r = to_dataset(pts, n, d, 0);
    SkylineSet s = sfs(r);
    for (size_t i = 0; i < s.size(); ++i) out[i] = s.points[i].id;
    return s.size();
}

void skyref_relative_skyline(const float* rp, uint64_t nr, const float* cp, uint64_t nc, uint32_t d,
                             uint8_t* keep) {
    const Dataset r = to_dataset(rp, nr, d, 0);
    Dataset c = to_dataset(cp, nc, d, 0);
    for (auto& pt : c.points) pt.id += static_cast<PointId>(nr);
    Dataset k = relative_skyline(r, c);
    std::memset(keep, 0, nr);
    for (const Point& t : k.points) keep[t.id] = 1;
}

uint64_t skyref_snap_slices(uint64_t target_p, uint64_t k) {
    uint64_t m = 0;
    guarded([&] { m = snap_slices(target_p, k); });
    return m;
}

uint64_t skyref_angular_index(const float* x, uint32_t d, uint64_t m) {
    Point t;
    t.coords.assign(x, x + d);
    return angular_index(t, m);
}

uint64_t skyref_grid_index(const float* x, uint32_t d, uint64_t m) {
    Point t;
    t.coords.assign(x, x + d);
    uint64_t g = UINT64_MAX;
    guarded([&] { g = grid_index(t, m); });
    return g;
}

uint64_t skyref_representatives(const float* pts, uint64_t n, uint32_t d, const uint64_t* partition_of,
                                uint64_t p, uint64_t q, int64_t* out) {
    const Dataset r = to_dataset(pts, n, d, 0);
    std::vector<Dataset> parts(p);
    for (auto& part : parts) part.d = d;
    for (uint64_t i = 0; i < n; ++i) parts[partition_of[i]].points.push_back(r.points[i]);
    Representatives reps = select_representatives_sorted(parts, q, 1);
    std::vector<int64_t> ids;
    for (const Point& t : reps.points) ids.push_back(t.id);
    std::sort(ids.begin(), ids.end());
    for (size_t i = 0; i < ids.size(); ++i) out[i] = ids[i];
    return ids.size();
}

}  // extern "C"
