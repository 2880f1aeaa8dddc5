// adapter_check: the drop-in adapter (adapters/skyline_gpu.hpp) against the
// reference itself, through the reference's own types. Test infrastructure:
// it links the reference engine (oracle/_ref/libskyref.so) only as the
// checker. For each configuration it builds a Dataset with the reference's
// generator, runs skyline::run (reference, CPU) and skyline::gpu::run (B200),
// and compares the skylines (ids and coordinates) and every PhaseMetrics
// count. Exit status = number of mismatching configurations.
#include <cstdio>
#include <string>
#include <vector>

#include "skyline/datagen.hpp"
#include "skyline/engine.hpp"
#include "skyline/sequential.hpp"
#include "skyline_gpu.hpp"

using namespace skyline;

static bool same(const RunResult& a, const RunResult& b, std::string& why) {
    if (a.skyline.size() != b.skyline.size()) return why = "skyline size", false;
    for (size_t i = 0; i < a.skyline.size(); ++i) {
        if (a.skyline.points[i].id != b.skyline.points[i].id) return why = "skyline ids", false;
        if (a.skyline.points[i].coords != b.skyline.points[i].coords) return why = "skyline coords", false;
    }
    if (a.effective_p != b.effective_p) return why = "effective_p", false;
    if (a.metrics.local_skyline_sizes != b.metrics.local_skyline_sizes) return why = "local sizes", false;
    if (a.metrics.union_size != b.metrics.union_size) return why = "union_size", false;
    if (a.metrics.filtered_count != b.metrics.filtered_count) return why = "filtered_count", false;
    if (a.metrics.final_size != b.metrics.final_size) return why = "final_size", false;
    return true;
}

int main() {
    gpu::Context g1(0);
    // the same calls through a two-rank group context (rows sharded over
    // the ranks; both ranks on device 0, exchanging through device copies)
    auto g2 = gpu::Context::devices({0, 0}, SKY_GROUP_LOOPBACK);
    int bad = 0, runs = 0;
  for (gpu::Context* gp : {&g1, g2.get()}) {
    gpu::Context& g = *gp;
    const Distribution dists[] = {Distribution::Uniform, Distribution::Correlated, Distribution::Anticorrelated};
    for (Distribution dist : dists) {
        for (size_t d : {2, 4, 6}) {
            const Dataset data = generate(GenSpec{dist, 20000, d, 31 + d});
            for (Strategy s : {Strategy::Random, Strategy::Grid, Strategy::Angular, Strategy::Sliced}) {
                for (int f = 0; f < 3; ++f) {
                    for (MergeKind m : {MergeKind::Sequential, MergeKind::NoSeq}) {
                        EngineConfig c;
                        c.partition.strategy = s;
                        c.partition.p = 16;
                        c.partition.seed = 5;
                        c.seed = 9;
                        c.merge = m;
                        c.workers = 4;
                        c.rep_q = 4;
                        if (f == 1) c.filter = FilterKind::Representative, c.rep_selection = RepSelection::Sorted;
                        if (f == 2) c.filter = FilterKind::Representative, c.rep_selection = RepSelection::Region;
                        const RunResult want = run(data, c);
                        const RunResult got = gpu::run(g, data, c);
                        std::string why;
                        ++runs;
                        if (!same(want, got, why)) {
                            ++bad;
                            std::printf("MISMATCH (%s): gpus %d dist %d d=%zu strategy %d filter %d merge %d\n",
                                        why.c_str(), g.world(), (int)dist, d, (int)s, f, (int)m);
                        }
                    }
                }
            }
            // sfs under both scoring functions (normalized data)
            for (Scoring sc : {Scoring::Sum, Scoring::VolumeComplement}) {
                const SkylineSet want = sfs(data, sc);
                const SkylineSet got = gpu::sfs(g, data, sc);
                ++runs;
                bool ok = want.size() == got.size();
                for (size_t i = 0; ok && i < want.size(); ++i) ok = want.points[i].id == got.points[i].id;
                if (!ok) {
                    ++bad;
                    std::printf("MISMATCH sfs scoring %d dist %d d=%zu\n", (int)sc, (int)dist, d);
                }
            }
        }
    }
  }
    std::printf("adapter_check: %d runs, %d mismatches\n", runs, bad);
    return bad;
}
