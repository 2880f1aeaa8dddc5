// skyline-cli (GPU): the reference's command-line driver (cli.cpp:241-447)
// served by libskyline_b200.so. Same subcommands (generate / run / bench),
// options, defaults, output formats (run_result_to_json, io.cpp:84-105; the
// CSV bench rows, cli.cpp:95-122) and exit codes (0 ok, 1 usage error, 2
// runtime error). GPU-only extras: --device, --local-algo, --bnl-window.
//
// Datasets are the reference's own: generate() and ingest_csv() restated in
// the library (sky_generate_family / sky_ingest_csv, bit-identical) and run
// through sky_run_f64, so every number in the output matches the reference.
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <map>
#include <optional>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "skyline_b200.h"

namespace {

struct UsageError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct RuntimeError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// ------------------------------------------------------------ names (io.cpp)
const char* strategy_name(int s) {
    switch (s) {
        case SKY_RANDOM: return "random";
        case SKY_GRID: return "grid";
        case SKY_ANGULAR: return "angular";
        case SKY_SLICED: return "sliced";
    }
    return "unknown";
}
const char* merge_name(int m) { return m == SKY_MERGE_SEQUENTIAL ? "sequential" : "noseq"; }
const char* dist_name(int d) {
    switch (d) {
        case SKY_DIST_UNIFORM: return "uniform";
        case SKY_DIST_CORRELATED: return "correlated";
        case SKY_DIST_ANTICORRELATED: return "anticorrelated";
    }
    return "unknown";
}
const char* filter_name(int f, int sel) {
    if (f == SKY_FILTER_NONE) return "none";
    if (f == SKY_FILTER_GRID) return "grid";
    if (f == SKY_FILTER_REPRESENTATIVE)
        return sel == SKY_REPS_REGION ? "rep-region" : sel == SKY_REPS_RANDOM ? "rep-random" : "rep-sorted";
    return "unknown";
}
// parse errors are ConfigErrors in the reference (io.cpp:44-83); callers map
// them to usage errors where cli.cpp does
struct ConfigErr : std::runtime_error {
    using std::runtime_error::runtime_error;
};
int parse_strategy(const std::string& s) {
    if (s == "random") return SKY_RANDOM;
    if (s == "grid") return SKY_GRID;
    if (s == "angular") return SKY_ANGULAR;
    if (s == "sliced") return SKY_SLICED;
    throw ConfigErr("unknown strategy '" + s + "'");
}
int parse_merge(const std::string& s) {
    if (s == "sequential") return SKY_MERGE_SEQUENTIAL;
    if (s == "noseq") return SKY_MERGE_NOSEQ;
    throw ConfigErr("unknown merge mode '" + s + "'");
}
int parse_dist(const std::string& s) {
    if (s == "uniform" || s == "uni") return SKY_DIST_UNIFORM;
    if (s == "correlated" || s == "corr") return SKY_DIST_CORRELATED;
    if (s == "anticorrelated" || s == "ant") return SKY_DIST_ANTICORRELATED;
    throw ConfigErr("unknown distribution '" + s + "'");
}
void parse_filter(const std::string& s, int32_t& f, int32_t& sel) {
    if (s == "none") f = SKY_FILTER_NONE;
    else if (s == "grid") f = SKY_FILTER_GRID;
    else if (s == "rep-sorted") f = SKY_FILTER_REPRESENTATIVE, sel = SKY_REPS_SORTED;
    else if (s == "rep-region") f = SKY_FILTER_REPRESENTATIVE, sel = SKY_REPS_REGION;
    else if (s == "rep-random") f = SKY_FILTER_REPRESENTATIVE, sel = SKY_REPS_RANDOM;
    else throw ConfigErr("unknown filter '" + s + "'");
}

// --------------------------------------------------------------- JSON text
// Doubles as nlohmann::json::dump prints them: shortest round-trip digits,
// fixed notation for decimal exponents in (-4, 15], else d.ddde+XX.
std::string json_double(double v) {
    if (!std::isfinite(v)) return "null";
    if (v == 0.0) return std::signbit(v) ? "-0.0" : "0.0";
    char buf[64];
    auto [p, ec] = std::to_chars(buf, buf + sizeof(buf), v, std::chars_format::scientific);
    (void)ec;
    std::string s(buf, p);
    std::string sign;
    if (s[0] == '-') sign = "-", s.erase(0, 1);
    const size_t epos = s.find('e');
    std::string digits = s.substr(0, epos);
    digits.erase(std::remove(digits.begin(), digits.end(), '.'), digits.end());
    const int e10 = std::stoi(s.substr(epos + 1));
    const int k = (int)digits.size(), n = e10 + 1;  // value = 0.digits * 10^n
    std::string out;
    if (k <= n && n <= 15) {
        out = digits + std::string(n - k, '0') + ".0";
    } else if (0 < n && n <= 15) {
        out = digits.substr(0, n) + "." + digits.substr(n);
    } else if (-4 < n && n <= 0) {
        out = "0." + std::string(-n, '0') + digits;
    } else {
        out = digits.substr(0, 1);
        if (k > 1) out += "." + digits.substr(1);
        const int ex = n - 1;
        char eb[16];
        std::snprintf(eb, sizeof eb, "e%c%02d", ex < 0 ? '-' : '+', ex < 0 ? -ex : ex);
        out += eb;
    }
    return sign + out;
}

std::string json_string(const std::string& s) {
    std::string o = "\"";
    for (char c : s) {
        if (c == '"' || c == '\\') o += '\\', o += c;
        else if ((unsigned char)c < 0x20) {
            char b[8];
            std::snprintf(b, sizeof b, "\\u%04x", c);
            o += b;
        } else o += c;
    }
    return o + "\"";
}

// ----------------------------------------------------------------- dataset
struct Data {
    std::vector<double> rows;
    uint64_t n = 0;
    uint32_t d = 0;
    std::string label;
};

void check(int rc, const char* what) {
    if (rc != SKY_OK) throw RuntimeError(std::string(what) + ": " + sky_host_error());
}

struct Gen {
    int dist;
    uint64_t n, d, seed;
};

Gen parse_gen(const std::string& text, uint64_t seed) {
    std::vector<std::string> parts;
    std::stringstream ss(text);
    std::string part;
    while (std::getline(ss, part, ',')) parts.push_back(part);
    if (parts.size() != 3) throw UsageError("--gen expects 'distribution,N,d', got '" + text + "'");
    Gen g{};
    try {
        g.dist = parse_dist(parts[0]);
    } catch (const ConfigErr& e) {
        throw UsageError(e.what());
    }
    try {
        size_t pos = 0;
        g.n = std::stoull(parts[1], &pos);
        g.d = std::stoull(parts[2], &pos);
    } catch (const std::exception&) {
        throw UsageError("--gen expects numeric N and d, got '" + text + "'");
    }
    if (g.d < 1) throw UsageError("--gen needs d >= 1");
    g.seed = seed;
    return g;
}

Data generate(const Gen& g) {
    Data r;
    r.n = g.n;
    r.d = (uint32_t)g.d;
    r.rows.resize(g.n * g.d);
    check(sky_generate_family(g.dist, g.n, (uint32_t)g.d, g.seed, r.rows.data()), "generate");
    r.label = dist_name(g.dist);
    return r;
}

// ------------------------------------------------------------ option parse
struct Args {
    std::map<std::string, std::vector<std::string>> opt;  // --name -> values (vectors split on ',')
    std::map<std::string, int> count;
    bool has(const std::string& k) const { return count.count(k) && count.at(k) > 0; }
    std::string str(const std::string& k, const std::string& def) const {
        auto it = opt.find(k);
        return it == opt.end() || it->second.empty() ? def : it->second.back();
    }
    uint64_t u64(const std::string& k, uint64_t def) const {
        if (!has(k)) return def;
        const std::string v = str(k, "");
        uint64_t x = 0;
        auto [p, ec] = std::from_chars(v.data(), v.data() + v.size(), x);
        if (ec != std::errc{} || p != v.data() + v.size())
            throw UsageError(k + ": Value " + v + " could not be converted");
        return x;
    }
    std::vector<std::string> list(const std::string& k, std::vector<std::string> def) const {
        auto it = opt.find(k);
        if (it == opt.end()) return def;
        std::vector<std::string> out;
        for (const auto& v : it->second) {
            std::stringstream ss(v);
            std::string part;
            while (std::getline(ss, part, ',')) out.push_back(part);
        }
        return out;
    }
};

Args parse_args(int argc, char** argv, int first, const std::vector<std::string>& opts,
                const std::vector<std::string>& flags) {
    Args a;
    for (int i = first; i < argc; ++i) {
        std::string t = argv[i];
        std::string val;
        bool inline_val = false;
        const size_t eq = t.find('=');
        if (t.rfind("--", 0) == 0 && eq != std::string::npos) {
            val = t.substr(eq + 1);
            t = t.substr(0, eq);
            inline_val = true;
        }
        if (std::find(flags.begin(), flags.end(), t) != flags.end()) {
            a.count[t]++;
            continue;
        }
        if (std::find(opts.begin(), opts.end(), t) == opts.end())
            throw UsageError("The following argument was not expected: " + std::string(argv[i]));
        if (!inline_val) {
            if (i + 1 >= argc) throw UsageError(t + " requires an argument");
            val = argv[++i];
        }
        a.opt[t].push_back(val);
        a.count[t]++;
    }
    return a;
}

uint64_t list_u64(const std::string& k, const std::string& v) {
    uint64_t x = 0;
    auto [p, ec] = std::from_chars(v.data(), v.data() + v.size(), x);
    if (ec != std::errc{} || p != v.data() + v.size()) throw UsageError(k + ": Value " + v + " could not be converted");
    return x;
}

// ------------------------------------------------------------- engine call
struct Result {
    sky_result r{};
    bool ok = false;
    ~Result() {
        if (ok) sky_result_free(&r);
    }
};

struct Gpu {
    sky_ctx* ctx = nullptr;
    // one GPU (`device`), or `gpus` > 1 devices device..device+gpus-1 driven
    // from this process (a group context: rows sharded over the GPUs)
    Gpu(int device, int gpus) {
        if (gpus <= 1) {
            if (sky_ctx_create(device, &ctx) != SKY_OK) throw RuntimeError("cannot create a GPU context");
            return;
        }
        std::vector<int> devs;
        for (int k = 0; k < gpus; ++k) devs.push_back(device + k);
        if (sky_ctx_create_group(devs.data(), gpus, 0, &ctx) != SKY_OK)
            throw RuntimeError("cannot create a " + std::to_string(gpus) + "-GPU context");
    }
    ~Gpu() { sky_ctx_destroy(ctx); }
    // status codes mirror the reference's exception classes (core.hpp:13-34)
    void run(const Data& data, const sky_config& cfg, Result& out) {
        const int rc = sky_run_f64(ctx, data.rows.data(), data.n, data.d, 1, 0, &cfg, &out.r);
        if (rc != SKY_OK) throw RuntimeError(sky_last_error(ctx));
        out.ok = true;
    }
};

const char* kCsvHeader =
    "distribution,n,d,seed,repetition,strategy,filter,merge,target_p,"
    "effective_p,workers,rep_q,partition_ms,local_ms,merge_ms,filtered,"
    "union_size,skyline_size,status,message";

std::string sanitize(std::string s) {
    for (char& c : s)
        if (c == ',' || c == '\n' || c == '\r') c = ';';
    return s;
}

std::string csv_row(const std::string& dist, uint64_t n, uint64_t d, uint64_t seed, uint64_t rep,
                    const sky_config& c, const sky_result* r, const std::string& status, const std::string& msg) {
    std::ostringstream row;  // default ostream formatting, as the reference prints
    row << dist << ',' << n << ',' << d << ',' << seed << ',' << rep << ',' << strategy_name(c.strategy) << ','
        << filter_name(c.filter, c.rep_selection) << ',' << merge_name(c.merge) << ',' << c.p << ',';
    if (r) row << r->effective_p;
    row << ',' << c.workers << ',' << c.rep_q << ',';
    if (r)
        row << r->partition_ms << ',' << r->local_ms << ',' << r->merge_ms << ',' << r->filtered_count << ','
            << r->union_size << ',' << r->final_size;
    else
        row << ",,,,,";
    row << ',' << status << ',' << sanitize(msg);
    return row.str();
}

void write_text(const std::string& path, const std::string& text) {
    if (path.empty()) {
        std::cout << text << '\n';
        return;
    }
    std::ofstream out(path);
    if (!out) throw RuntimeError("cannot write " + path);
    out << text << '\n';
    if (!out) throw RuntimeError("write failed for " + path);
}

sky_config base_config() {
    sky_config c;
    sky_config_default(&c);
    return c;
}

void apply_gpu_extras(const Args& a, sky_config& c) {
    const std::string la = a.str("--local-algo", "sfs");
    if (la == "sfs") c.local_algo = SKY_LOCAL_SFS;
    else if (la == "bnl") c.local_algo = SKY_LOCAL_BNL;
    else throw UsageError("unknown local algorithm '" + la + "'");
    c.bnl_window_cap = (uint32_t)a.u64("--bnl-window", 4096);
}

void apply_preset(const std::string& name, sky_config& c) {
    struct P {
        int s, f, sel, m;
    };
    static const std::map<std::string, P> presets = {
        {"random", {SKY_RANDOM, SKY_FILTER_NONE, SKY_REPS_SORTED, SKY_MERGE_SEQUENTIAL}},
        {"grid", {SKY_GRID, SKY_FILTER_NONE, SKY_REPS_SORTED, SKY_MERGE_SEQUENTIAL}},
        {"angular", {SKY_ANGULAR, SKY_FILTER_NONE, SKY_REPS_SORTED, SKY_MERGE_SEQUENTIAL}},
        {"sliced", {SKY_SLICED, SKY_FILTER_NONE, SKY_REPS_SORTED, SKY_MERGE_SEQUENTIAL}},
        {"sliced+", {SKY_SLICED, SKY_FILTER_REPRESENTATIVE, SKY_REPS_SORTED, SKY_MERGE_SEQUENTIAL}},
        {"angular+", {SKY_ANGULAR, SKY_FILTER_REPRESENTATIVE, SKY_REPS_SORTED, SKY_MERGE_SEQUENTIAL}},
        {"noseq", {SKY_SLICED, SKY_FILTER_NONE, SKY_REPS_SORTED, SKY_MERGE_NOSEQ}},
    };
    auto it = presets.find(name);
    if (it == presets.end()) throw UsageError("unknown preset '" + name + "'");
    c.strategy = it->second.s;
    c.filter = it->second.f;
    if (it->second.f == SKY_FILTER_REPRESENTATIVE) c.rep_selection = it->second.sel;
    c.merge = it->second.m;
}

// ---------------------------------------------------------------- commands
int do_generate(int argc, char** argv) {
    Args a = parse_args(argc, argv, 2, {"--gen", "--seed", "--out"}, {});
    if (!a.has("--gen") || !a.has("--out")) throw UsageError("--gen and --out are required");
    const Gen g = parse_gen(a.str("--gen", ""), a.u64("--seed", 0));
    const Data data = generate(g);
    const std::string out = a.str("--out", "");
    check(sky_write_csv(out.c_str(), data.rows.data(), data.n, data.d), "write_csv");
    std::cout << "N=" << g.n << " d=" << g.d << " seed=" << g.seed << " distribution=" << dist_name(g.dist)
              << " -> " << out << '\n';
    return 0;
}

int do_run(int argc, char** argv) {
    Args a = parse_args(argc, argv, 2,
                        {"--input", "--gen", "--seed", "--columns", "--max-columns", "--preset", "--strategy",
                         "--filter", "--merge", "--partitions", "--slices", "--slice-dim", "--reps-q", "--workers",
                         "--out", "--format", "--device", "--gpus", "--local-algo", "--bnl-window"},
                        {"--oracle", "--no-timings"});
    const uint64_t seed = a.u64("--seed", 0);
    // load_input (cli.cpp:157-196)
    if (a.has("--input") == a.has("--gen")) throw UsageError("exactly one of --input and --gen is required");
    const std::vector<std::string> columns = a.list("--columns", {});
    const std::vector<std::string> maxcols = a.list("--max-columns", {});
    Data data;
    if (a.has("--gen")) {
        if (!columns.empty() || !maxcols.empty()) throw UsageError("--columns/--max-columns apply to --input only");
        data = generate(parse_gen(a.str("--gen", ""), seed));
    } else {
        std::vector<uint8_t> maximize;
        if (!maxcols.empty()) {
            if (columns.empty()) throw UsageError("--max-columns requires --columns");
            maximize.assign(columns.size(), 0);
            for (const auto& m : maxcols) {
                auto it = std::find(columns.begin(), columns.end(), m);
                if (it == columns.end()) throw UsageError("--max-columns entry '" + m + "' is not in --columns");
                maximize[it - columns.begin()] = 1;
            }
        }
        std::vector<const char*> cp;
        for (const auto& c : columns) cp.push_back(c.c_str());
        double* rows = nullptr;
        uint64_t n = 0;
        uint32_t d = 0;
        const std::string path = a.str("--input", "");
        check(sky_ingest_csv(path.c_str(), cp.data(), (uint32_t)cp.size(), maximize.data(),
                             (uint32_t)maximize.size(), &rows, &n, &d),
              "ingest");
        data.rows.assign(rows, rows + n * d);
        sky_free(rows);
        data.n = n;
        data.d = d;
        data.label = "file";
    }
    // build_config (cli.cpp:198-224)
    sky_config c = base_config();
    c.p = a.u64("--partitions", 8);
    c.m = a.u64("--slices", 0);
    c.seed = seed;
    c.rep_seed = seed;
    c.slice_dim = a.u64("--slice-dim", 0);
    c.rep_q = a.u64("--reps-q", 5);
    c.workers = a.u64("--workers", 1);
    c.strategy = SKY_RANDOM;
    c.filter = SKY_FILTER_NONE;
    c.merge = SKY_MERGE_SEQUENTIAL;
    const std::string preset = a.str("--preset", "");
    if (!preset.empty()) apply_preset(preset, c);
    try {
        if (preset.empty() || a.has("--strategy")) c.strategy = parse_strategy(a.str("--strategy", "random"));
        if (preset.empty() || a.has("--filter")) parse_filter(a.str("--filter", "none"), c.filter, c.rep_selection);
        if (preset.empty() || a.has("--merge")) c.merge = parse_merge(a.str("--merge", "sequential"));
    } catch (const ConfigErr& e) {
        throw UsageError(e.what());
    }
    apply_gpu_extras(a, c);

    Gpu gpu((int)a.u64("--device", 0), (int)a.u64("--gpus", 1));
    Result res;
    gpu.run(data, c, res);
    std::optional<bool> oracle_match;
    if (a.has("--oracle")) {
        // the skyline of the whole relation in one partition (no partitioning,
        // no filter, no merge) against the configured run
        sky_config o = base_config();
        o.strategy = SKY_SLICED;
        o.p = 1;
        Result ref;
        gpu.run(data, o, ref);
        oracle_match = ref.r.n_ids == res.r.n_ids &&
                       std::equal(ref.r.ids, ref.r.ids + ref.r.n_ids, res.r.ids);
    }
    const std::string format = a.str("--format", "json");
    const bool timings = !a.has("--no-timings");
    const sky_result& r = res.r;
    if (format == "json") {
        std::string s = "{";
        s += "\"strategy\":" + json_string(strategy_name(c.strategy));
        s += ",\"filter\":" + json_string(filter_name(c.filter, c.rep_selection));
        s += ",\"merge\":" + json_string(merge_name(c.merge));
        s += ",\"workers\":" + std::to_string(c.workers);
        s += ",\"effective_p\":" + std::to_string(r.effective_p);
        s += ",\"partition_ms\":" + json_double(timings ? r.partition_ms : 0.0);
        s += ",\"local_ms\":" + json_double(timings ? r.local_ms : 0.0);
        s += ",\"merge_ms\":" + json_double(timings ? r.merge_ms : 0.0);
        s += ",\"filtered\":" + std::to_string(r.filtered_count);
        s += ",\"union_size\":" + std::to_string(r.union_size);
        s += ",\"skyline_size\":" + std::to_string(r.final_size);
        if (oracle_match) s += std::string(",\"oracle_match\":") + (*oracle_match ? "true" : "false");
        s += ",\"skyline\":[";
        for (uint64_t k = 0; k < r.n_ids; ++k) {
            s += k ? ",[" : "[";
            const double* x = data.rows.data() + (size_t)r.ids[k] * data.d;
            for (uint32_t j = 0; j < data.d; ++j) s += (j ? "," : "") + json_double(x[j]);
            s += "]";
        }
        s += "]}";
        write_text(a.str("--out", ""), s);
    } else if (format == "csv") {
        write_text(a.str("--out", ""), std::string(kCsvHeader) + '\n' +
                                           csv_row(data.label, data.n, data.d, seed, 0, c, &r, "ok", ""));
    } else {
        throw UsageError("unknown format '" + format + "'");
    }
    if (!a.str("--out", "").empty()) {
        std::cout << "skyline_size=" << r.final_size << " union_size=" << r.union_size
                  << " filtered=" << r.filtered_count << " effective_p=" << r.effective_p;
        if (oracle_match) std::cout << " oracle_match=" << (*oracle_match ? "true" : "false");
        std::cout << " -> " << a.str("--out", "") << '\n';
    }
    return 0;
}

int do_bench(int argc, char** argv) {
    Args a = parse_args(argc, argv, 2,
                        {"--dist", "--n", "--d", "--strategy", "--filter", "--merge", "--partitions", "--workers",
                         "--repetitions", "--reps-q", "--seed", "--out", "--device", "--gpus", "--local-algo", "--bnl-window"},
                        {});
    const auto dists = a.list("--dist", {"anticorrelated"});
    const auto ns = a.list("--n", {"100000"});
    const auto ds = a.list("--d", {"4"});
    const auto strategies = a.list("--strategy", {"sliced"});
    const auto filters = a.list("--filter", {"none"});
    const auto merges = a.list("--merge", {"sequential"});
    const auto parts = a.list("--partitions", {"8"});
    const auto workers = a.list("--workers", {"1"});
    const uint64_t reps = a.u64("--repetitions", 1), q = a.u64("--reps-q", 5), seed = a.u64("--seed", 0);
    sky_config extras = base_config();
    apply_gpu_extras(a, extras);
    Gpu gpu((int)a.u64("--device", 0), (int)a.u64("--gpus", 1));
    std::ostringstream table;
    table << kCsvHeader << '\n';
    Data data;
    std::string cached;
    for (const auto& dn : dists) {
        int dist;
        try {
            dist = parse_dist(dn);
        } catch (const ConfigErr& e) {
            throw RuntimeError(e.what());
        }
        for (const auto& nt : ns) {
            const uint64_t n = list_u64("--n", nt);
            for (const auto& dt : ds) {
                const uint64_t d = list_u64("--d", dt);
                for (uint64_t rep = 0; rep < reps; ++rep) {
                    // one dataset per (distribution, n, d, repetition): strategies
                    // compete on identical data (cli.cpp:304-313)
                    const uint64_t ds_seed = seed + rep;
                    const std::string key = dn + '/' + nt + '/' + dt + '/' + std::to_string(ds_seed);
                    if (key != cached) {
                        data = generate(Gen{dist, n, d, ds_seed});
                        data.label = dn;
                        cached = key;
                    }
                    for (const auto& st : strategies)
                        for (const auto& fl : filters)
                            for (const auto& mg : merges)
                                for (const auto& pt : parts)
                                    for (const auto& wk : workers) {
                                        sky_config c = extras;
                                        c.p = list_u64("--partitions", pt);
                                        c.seed = ds_seed;
                                        c.rep_seed = ds_seed;
                                        c.rep_q = q;
                                        c.workers = list_u64("--workers", wk);
                                        std::string status = "ok", msg;
                                        Result res;
                                        const sky_result* rp = nullptr;
                                        try {
                                            c.strategy = parse_strategy(st);
                                            parse_filter(fl, c.filter, c.rep_selection);
                                            c.merge = parse_merge(mg);
                                            gpu.run(data, c, res);
                                            rp = &res.r;
                                        } catch (const std::exception& e) {
                                            status = "error";
                                            msg = e.what();
                                        }
                                        table << csv_row(dn, n, d, ds_seed, rep, c, rp, status, msg) << '\n';
                                    }
                }
            }
        }
    }
    std::string text = table.str();
    if (!text.empty() && text.back() == '\n') text.pop_back();
    write_text(a.str("--out", ""), text);
    return 0;
}

void usage(std::ostream& os) {
    os << "Parallel skyline computation on B200: partitioning strategies, filtering optimizations, and a fully "
          "parallel merge.\n"
          "Usage: skyline-cli [generate|run|bench] [OPTIONS]\n"
          "  generate --gen dist,N,d [--seed S] --out PATH\n"
          "  run (--input CSV [--columns a,b] [--max-columns a] | --gen dist,N,d) [--seed S] [--preset P]\n"
          "      [--strategy random|grid|angular|sliced] [--filter none|grid|rep-sorted|rep-region|rep-random]\n"
          "      [--merge sequential|noseq] [--partitions P] [--slices M] [--slice-dim K] [--reps-q Q]\n"
          "      [--workers W] [--oracle] [--no-timings] [--out PATH] [--format json|csv]\n"
          "  bench [--dist a,b] [--n N,..] [--d D,..] [--strategy ..] [--filter ..] [--merge ..]\n"
          "        [--partitions ..] [--workers ..] [--repetitions R] [--reps-q Q] [--seed S] [--out PATH]\n"
          "  GPU options (run, bench): --device I, --gpus N (devices I..I+N-1), --local-algo sfs|bnl,\n"
          "    --bnl-window W\n";
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        std::cerr << "A subcommand is required\n";
        usage(std::cerr);
        return 1;
    }
    const std::string cmd = argv[1];
    if (cmd == "-h" || cmd == "--help") {
        usage(std::cout);
        return 0;
    }
    try {
        if (cmd == "generate") return do_generate(argc, argv);
        if (cmd == "run") return do_run(argc, argv);
        if (cmd == "bench") return do_bench(argc, argv);
        throw UsageError("The following argument was not expected: " + cmd);
    } catch (const UsageError& e) {
        std::cerr << "error: " << e.what() << '\n';
        return 1;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << '\n';
        return 2;
    }
}
