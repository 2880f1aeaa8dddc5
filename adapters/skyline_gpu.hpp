// skyline_gpu.hpp — drop-in adapter: the reference engine API (skyline::run,
// /root/reference/proj/include/skyline/engine.hpp:88) served by the B200
// engine through the C ABI in include/skyline_b200.h.
//
// A maintainer of the reference adds this header next to engine.hpp and calls
// skyline::gpu::run(dataset, config) where skyline::run was called; the
// returned RunResult carries the same skyline (id-sorted Points) and the same
// PhaseMetrics fields (engine.hpp:40-57). Errors come back as the reference's
// exception classes (core.hpp:13-34).
//
// Any finite double coordinates: rows that are all float32 values go through
// sky_run, others through sky_run_f64 (FP64 decisions, identical results).
// d <= 32 and one sky_ctx per thread.
//
// Several GPUs from one reference thread: Context::devices({0, 1, ...}) (or
// Context::first(n)) makes a group context; run(ctx, dataset, config) then
// shards the rows over the GPUs (one host thread and stream per GPU inside
// the library, NCCL between them) and returns the same RunResult. The
// reference's EngineConfig::workers fans out threads (engine.hpp:30-38);
// Context::for_workers(config.workers) maps it onto min(workers, visible
// GPUs) devices.
#pragma once

#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "skyline/core.hpp"
#include "skyline/engine.hpp"
#include "skyline/sequential.hpp"
#include "skyline_b200.h"

namespace skyline::gpu {

inline void throw_status(int rc, const char* msg) {
    const std::string m = msg ? msg : "";
    switch (rc) {
        case SKY_OK: return;
        case SKY_E_CONFIG: throw ConfigError(m);
        case SKY_E_DIMENSION: throw DimensionError(m);
        case SKY_E_NORMALIZATION: throw NormalizationError(m);
        case SKY_E_DATA: throw DataError(m);
        case SKY_E_IO: throw IoError(m);
        default: throw SkylineError("skyline_b200: " + m);
    }
}

struct Context {
    sky_ctx* ctx = nullptr;
    explicit Context(int device = 0) { throw_status(sky_ctx_create(device, &ctx), "sky_ctx_create failed"); }
    // one process, several GPUs (rank r on devices[r]); flags: SKY_GROUP_LOOPBACK
    static std::unique_ptr<Context> devices(const std::vector<int>& devs, int flags = 0) {
        std::unique_ptr<Context> c(new Context(nullptr));
        throw_status(sky_ctx_create_group(devs.data(), static_cast<int>(devs.size()), flags, &c->ctx),
                     "sky_ctx_create_group failed");
        return c;
    }
    // devices 0..n-1
    static std::unique_ptr<Context> first(int n) {
        std::vector<int> devs(n > 0 ? n : 1);
        for (size_t i = 0; i < devs.size(); ++i) devs[i] = static_cast<int>(i);
        return devs.size() == 1 ? std::unique_ptr<Context>(new Context(0)) : devices(devs);
    }
    // EngineConfig::workers -> min(workers, visible GPUs) devices
    static std::unique_ptr<Context> for_workers(size_t workers) {
        int visible = sky_device_count();
        if (visible < 1) visible = 1;
        const size_t n = workers < 1 ? 1 : (workers < static_cast<size_t>(visible) ? workers : visible);
        return first(static_cast<int>(n));
    }
    int world() const {
        int r = 0, w = 1;
        sky_ctx_world(ctx, &r, &w);
        return w;
    }
    ~Context() { sky_ctx_destroy(ctx); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;

   private:
    explicit Context(std::nullptr_t) {}
};

inline sky_config to_sky(const EngineConfig& e) {
    sky_config c;
    sky_config_default(&c);
    c.strategy = static_cast<int32_t>(e.partition.strategy);
    c.p = e.partition.p;
    c.m = e.partition.m;
    c.seed = e.partition.seed;
    c.slice_dim = e.partition.slice_dim;
    c.filter = static_cast<int32_t>(e.filter);
    c.rep_selection = static_cast<int32_t>(e.rep_selection);
    c.rep_q = e.rep_q;
    c.merge = static_cast<int32_t>(e.merge);
    c.rep_seed = e.seed;
    c.workers = e.workers;
    return c;
}

// skyline::run on the GPU (engine.hpp:88). Ids of the input points are
// preserved (core.cpp:43 assigns them in row order; Dataset ids are used as
// given here).
inline RunResult run(Context& g, const Dataset& r, const EngineConfig& config) {
    const size_t n = r.size(), d = r.d;
    std::vector<float> rows(n * d);
    std::vector<double> rows64;
    bool exact32 = true;
    for (size_t i = 0; i < n; ++i) {
        const Point& t = r.points[i];
        if (t.dim() != d) throw DimensionError("ragged dataset");
        for (size_t j = 0; j < d; ++j) {
            const float f = static_cast<float>(t.coords[j]);
            if (static_cast<double>(f) != t.coords[j] && !std::isnan(t.coords[j])) exact32 = false;
            rows[i * d + j] = f;
        }
    }
    if (!exact32) {
        rows64.resize(n * d);
        for (size_t i = 0; i < n; ++i)
            for (size_t j = 0; j < d; ++j) rows64[i * d + j] = r.points[i].coords[j];
    }
    const sky_config c = to_sky(config);
    sky_result res;
    const int rc = exact32 ? sky_run(g.ctx, rows.data(), n, static_cast<uint32_t>(d), r.normalized ? 1 : 0, 0, &c,
                                     &res)
                           : sky_run_f64(g.ctx, rows64.data(), n, static_cast<uint32_t>(d), r.normalized ? 1 : 0,
                                         0, &c, &res);
    throw_status(rc, sky_last_error(g.ctx));
    RunResult out;
    out.config = config;
    out.effective_p = res.effective_p;
    out.input_size = n;
    out.input_dim = d;
    out.skyline.points.reserve(res.n_ids);
    for (uint64_t k = 0; k < res.n_ids; ++k) out.skyline.points.push_back(r.points[res.ids[k]]);
    PhaseMetrics& m = out.metrics;
    m.partition_ms = res.partition_ms;
    m.local_ms = res.local_ms;
    m.merge_ms = res.merge_ms;
    m.local_skyline_sizes.assign(res.local_skyline_sizes, res.local_skyline_sizes + res.effective_p);
    m.union_size = res.union_size;
    m.filtered_count = res.filtered_count;
    m.final_size = res.final_size;
    sky_result_free(&res);
    return out;
}

// skyline::sfs (sequential.hpp:29) on the GPU: the skyline of one relation,
// id-sorted. The scoring function only orders the reference's scan, so every
// monotone score gives the same set; VolumeComplement is monotone on [0,1]
// coordinates only (sequential.hpp:14-16) and is accepted there.
inline SkylineSet sfs(Context& g, const Dataset& r, Scoring f = Scoring::Sum) {
    if (f == Scoring::VolumeComplement)
        for (const Point& t : r.points)
            for (double v : t.coords)
                if (!(v >= 0.0 && v <= 1.0))
                    throw NormalizationError("VolumeComplement scoring needs coordinates in [0,1]");
    Dataset copy = r;
    copy.normalized = false;  // any finite non-negative data (sky_skyline semantics)
    EngineConfig one;         // one sliced partition, no filter: Sky(r) itself
    one.partition.strategy = Strategy::Sliced;
    one.partition.p = 1;
    RunResult res = run(g, copy, one);
    return std::move(res.skyline);
}

}  // namespace skyline::gpu
