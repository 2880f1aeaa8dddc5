// dataio.cpp — the steps either side of the hot path:
// the reference's dataset generators, CSV ingest with min-max
// normalisation, and CSV output, behind the C ABI. Host code: the generators
// are one sequential mt19937_64 stream whose rejection loops depend on glibc
// log/cos results (datagen.cpp:16-57), so bit-identical datasets come from
// running that stream on the host; ingest is parse-bound.
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <limits>
#include <random>
#include <string>
#include <string_view>
#include <vector>

#include "../../include/skyline_b200.h"

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

// Rng (rng.hpp:15-51) on std::mt19937_64
struct Stream {
    std::mt19937_64 eng;
    explicit Stream(uint64_t s) : eng(s) {}
    double u01() { return static_cast<double>(eng() >> 11) * 0x1.0p-53; }
    double u01_pos() { return static_cast<double>((eng() >> 11) + 1) * 0x1.0p-53; }
    double normal(double mean, double stddev) {
        const double u1 = u01_pos();
        const double u2 = u01();
        const double r = std::sqrt(-2.0 * std::log(u1));
        return mean + stddev * r * std::cos(6.283185307179586476925286766559 * u2);
    }
};

// One point of each family (datagen.cpp:16-57).
void draw(int dist, Stream& g, uint32_t d, double* x) {
    if (dist == SKY_DIST_UNIFORM) {
        for (uint32_t j = 0; j < d; ++j) x[j] = g.u01();
    } else if (dist == SKY_DIST_CORRELATED) {
        const double base = g.u01();
        for (uint32_t j = 0; j < d; ++j) {
            double v;
            do {
                v = base + g.normal(0.0, 0.05);
            } while (v < 0.0 || v > 1.0);
            x[j] = v;
        }
    } else {  // anticorrelated: a level near 0.5, a uniform direction rescaled onto it
        double level;
        do {
            level = g.normal(0.5, 0.05);
        } while (level < 0.0 || level > 1.0);
        for (;;) {
            double sum = 0.0;
            for (uint32_t j = 0; j < d; ++j) {
                x[j] = g.u01();
                sum += x[j];
            }
            if (sum == 0.0) continue;
            const double scale = level * static_cast<double>(d) / sum;
            bool ok = true;
            for (uint32_t j = 0; j < d && ok; ++j) {
                x[j] *= scale;
                ok = x[j] <= 1.0;
            }
            if (ok) return;
        }
    }
}

// Column-wise min-max to [0,1]; constant columns -> 0; values above 1 after
// rounding are clamped (datagen.cpp:60-78).
void minmax_columns(double* rows, uint64_t n, uint32_t d) {
    if (!n) return;
    std::vector<double> lo(d, std::numeric_limits<double>::infinity());
    std::vector<double> hi(d, -std::numeric_limits<double>::infinity());
    for (uint64_t i = 0; i < n; ++i)
        for (uint32_t j = 0; j < d; ++j) {
            lo[j] = std::min(lo[j], rows[i * d + j]);
            hi[j] = std::max(hi[j], rows[i * d + j]);
        }
    for (uint64_t i = 0; i < n; ++i)
        for (uint32_t j = 0; j < d; ++j) {
            const double range = hi[j] - lo[j];
            double& v = rows[i * d + j];
            v = range > 0.0 ? (v - lo[j]) / range : 0.0;
            if (v > 1.0) v = 1.0;
        }
}

std::string_view trim_view(std::string_view s) {
    while (!s.empty() && (s.front() == ' ' || s.front() == '\t')) s.remove_prefix(1);
    while (!s.empty() && (s.back() == ' ' || s.back() == '\t' || s.back() == '\r')) s.remove_suffix(1);
    return s;
}

// A finite number spanning the whole (trimmed) field (datagen.cpp:80-93).
bool parse_number(std::string_view f, double& out) {
    f = trim_view(f);
    if (f.empty()) return false;
    const char* end = f.data() + f.size();
    auto [ptr, ec] = std::from_chars(f.data(), end, out);
    return ec == std::errc{} && ptr == end && std::isfinite(out);
}

void split_commas(std::string_view line, std::vector<std::string_view>& out) {
    out.clear();
    size_t start = 0;
    for (;;) {
        const size_t c = line.find(',', start);
        if (c == std::string_view::npos) {
            out.push_back(line.substr(start));
            return;
        }
        out.push_back(line.substr(start, c - start));
        start = c + 1;
    }
}

}  // namespace

extern "C" {

const char* sky_host_error(void) { return g_err.c_str(); }

int sky_generate_family(int dist, uint64_t n, uint32_t d, uint64_t seed, double* out) {
    if (d < 1) return fail(SKY_E_CONFIG, "dimensionality must be >= 1");
    if (dist < SKY_DIST_UNIFORM || dist > SKY_DIST_ANTICORRELATED) return fail(SKY_E_CONFIG, "unknown distribution");
    Stream g(seed);
    for (uint64_t i = 0; i < n; ++i) draw(dist, g, d, out + i * d);
    return SKY_OK;
}

int sky_normalize(double* rows, uint64_t n, uint32_t d) {
    minmax_columns(rows, n, d);
    return SKY_OK;
}

int sky_ingest_csv(const char* path, const char* const* columns, uint32_t n_columns, const uint8_t* maximize,
                   uint32_t n_maximize, double** rows_out, uint64_t* n_out, uint32_t* d_out) {
    *rows_out = nullptr;
    *n_out = 0;
    *d_out = 0;
    if (n_maximize && n_columns && n_maximize != n_columns)
        return fail(SKY_E_CONFIG, "directions must be empty or match the selected columns");
    std::ifstream in(path);
    if (!in) return fail(SKY_E_IO, std::string("cannot open ") + path);
    std::string line;
    if (!std::getline(in, line)) return fail(SKY_E_DATA, std::string("empty file: ") + path);
    std::vector<std::string_view> fields;
    split_commas(line, fields);
    std::vector<std::string> header;
    for (auto f : fields) header.emplace_back(trim_view(f));
    std::vector<size_t> sel;
    if (!n_columns) {
        for (size_t j = 0; j < header.size(); ++j) sel.push_back(j);
    } else {
        for (uint32_t k = 0; k < n_columns; ++k) {
            auto it = std::find(header.begin(), header.end(), std::string(columns[k]));
            if (it == header.end())
                return fail(SKY_E_CONFIG, std::string("unknown column '") + columns[k] + "' in " + path);
            sel.push_back(static_cast<size_t>(it - header.begin()));
        }
    }
    if (n_maximize && n_maximize != sel.size())
        return fail(SKY_E_CONFIG, "directions must be empty or match the selected columns");
    const uint32_t d = static_cast<uint32_t>(sel.size());
    std::vector<double> rows;
    std::vector<double> row(d);
    while (std::getline(in, line)) {
        if (trim_view(line).empty()) continue;
        split_commas(line, fields);
        bool ok = true;
        for (uint32_t j = 0; j < d && ok; ++j) ok = sel[j] < fields.size() && parse_number(fields[sel[j]], row[j]);
        if (!ok) continue;  // a missing or non-numeric value drops the row
        for (uint32_t j = 0; j < d; ++j)
            if (j < n_maximize && maximize[j]) row[j] = -row[j];
        rows.insert(rows.end(), row.begin(), row.end());
    }
    const uint64_t n = d ? rows.size() / d : 0;
    if (n == 0) return fail(SKY_E_DATA, std::string("no usable rows in ") + path);
    minmax_columns(rows.data(), n, d);
    double* out = static_cast<double*>(std::malloc(rows.size() * sizeof(double)));
    if (!out) return fail(SKY_E_INTERNAL, "out of host memory");
    std::memcpy(out, rows.data(), rows.size() * sizeof(double));
    *rows_out = out;
    *n_out = n;
    *d_out = d;
    return SKY_OK;
}

int sky_write_csv(const char* path, const double* rows, uint64_t n, uint32_t d) {
    std::ofstream out(path);
    if (!out) return fail(SKY_E_IO, std::string("cannot write ") + path);
    for (uint32_t j = 0; j < d; ++j) out << (j ? "," : "") << 'd' << j;
    out << '\n';
    char buf[64];
    for (uint64_t i = 0; i < n; ++i) {
        for (uint32_t j = 0; j < d; ++j) {
            if (j) out << ',';
            auto [ptr, ec] = std::to_chars(buf, buf + sizeof(buf), rows[i * d + j]);  // shortest round trip
            (void)ec;
            out.write(buf, ptr - buf);
        }
        out << '\n';
    }
    if (!out) return fail(SKY_E_IO, std::string("write failed for ") + path);
    return SKY_OK;
}

}  // extern "C"
