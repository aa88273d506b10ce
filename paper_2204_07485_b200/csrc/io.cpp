// io.cpp — dataset ingestion ahead of the hot path: the reference's loaders
// (io::load io.hpp:31-37 / io.cpp:224-243 with load_delimited :82-124,
// load_tsplib :126-174, select_columns :176-195) re-implemented natively, then
// the device upload (bm_dataset_create) and, when asked, the device
// min-max normalisation (bm_dataset_min_max_normalize, io.cpp:245-264).
//
// Same results and errors as the reference: every cell is trimmed and parsed
// with strtod and must be consumed whole (parse_cell io.cpp:30-43); blank lines
// are not rows (csv: empty, whitespace: all-space); a trailing '\r' is
// dropped; the first data row fixes the field count (ragged rows are an
// error); ParseError messages carry the same 1-based line / column.  The
// delimited formats are parsed in parallel over line ranges (host threads);
// the first error in file order is the one reported.
// Citations are relative to /root/reference/proj/src.
#include <algorithm>
#include <cctype>
#include <cerrno>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <optional>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "bigmeans_b200.h"

namespace bm {
extern thread_local std::string g_last_error;
}

namespace {

thread_local uint64_t t_parse_line = 0, t_parse_column = 0;

struct ParseError : std::runtime_error {  // ParseError common.hpp:28-42
    uint64_t line, column;
    ParseError(const std::string& what, uint64_t l, uint64_t c)
        : std::runtime_error(what + " (line " + std::to_string(l) + ", column " + std::to_string(c) + ")"),
          line(l),
          column(c) {}
};
struct ConfigErr : std::runtime_error {
    explicit ConfigErr(const std::string& w) : std::runtime_error(w) {}
};
struct StateErr : std::runtime_error {
    explicit StateErr(const std::string& w) : std::runtime_error(w) {}
};

template <class F>
bm_status guarded_io(F&& f) {
    try {
        f();
        return BM_OK;
    } catch (const ParseError& e) {
        bm::g_last_error = e.what();
        t_parse_line = e.line;
        t_parse_column = e.column;
        return BM_PARSE_ERROR;
    } catch (const ConfigErr& e) {
        bm::g_last_error = e.what();
        return BM_CONFIG_ERROR;
    } catch (const StateErr& e) {
        bm::g_last_error = e.what();
        return BM_STATE_ERROR;
    } catch (const std::exception& e) {
        bm::g_last_error = e.what();
        return BM_INTERNAL_ERROR;
    }
}

inline bool is_space(char c) { return std::isspace(static_cast<unsigned char>(c)) != 0; }

// The whole file (a missing file is the reference's StateError, io.cpp:84-86).
std::string read_file(const char* path) {
    std::FILE* f = std::fopen(path, "rb");
    if (!f) throw StateErr(std::string("cannot open dataset file '") + path + "'");
    std::string buf;
    char tmp[1 << 16];
    size_t got;
    while ((got = std::fread(tmp, 1, sizeof(tmp), f)) > 0) buf.append(tmp, got);
    std::fclose(f);
    return buf;
}

// parse_cell (io.cpp:30-43): trimmed, non-empty, strtod consumes all of it.
double parse_cell(const char* b, const char* e, uint64_t line, uint64_t column, std::string& scratch) {
    while (b < e && is_space(*b)) ++b;
    while (e > b && is_space(e[-1])) --e;
    if (b == e) throw ParseError("missing value", line, column);
    scratch.assign(b, e);
    char* end = nullptr;
    const double v = std::strtod(scratch.c_str(), &end);
    if (end != scratch.c_str() + scratch.size())
        throw ParseError("malformed numeric cell '" + scratch + "'", line, column);
    return v;
}

struct Line {
    const char* b;
    const char* e;  // without '\n' (and without a trailing '\r')
};

// getline semantics: a final line without '\n' counts if non-empty.
std::vector<Line> split_lines(const std::string& text) {
    std::vector<Line> lines;
    const char* p = text.data();
    const char* end = p + text.size();
    while (p < end) {
        const char* nl = static_cast<const char*>(std::memchr(p, '\n', end - p));
        const char* le = nl ? nl : end;
        const char* e = le;
        if (e > p && e[-1] == '\r') --e;  // io.cpp:96-98
        lines.push_back({p, e});
        p = nl ? nl + 1 : end;
    }
    return lines;
}

struct RowResult {
    bool data = false;       // a data row (not blank / header)
    uint32_t fields = 0;
    uint64_t err_col = 0;    // a cell error in this row (column), 0 = none
    std::string err_what;
};

// load_delimited (io.cpp:82-124), parsed in parallel over line ranges.
void parse_delimited(const std::string& text, bool csv, bool has_header, int threads, std::vector<double>& values,
                     uint64_t& m, uint64_t& n) {
    const std::vector<Line> lines = split_lines(text);
    const uint64_t L = lines.size();
    std::vector<RowResult> rows(L);
    std::vector<std::vector<double>> part_vals;
    const int T = std::max(1, std::min<int>(threads, static_cast<int>((L + 4095) / 4096)));
    part_vals.resize(T);
    auto work = [&](int t) {
        const uint64_t l0 = L * t / T, l1 = L * (t + 1) / T;
        std::string scratch;
        std::vector<double>& out = part_vals[t];
        for (uint64_t i = l0; i < l1; ++i) {
            RowResult& r = rows[i];
            if (has_header && i == 0) continue;  // io.cpp:99-102
            const char* b = lines[i].b;
            const char* e = lines[i].e;
            if (csv ? b == e : std::all_of(b, e, is_space)) continue;  // io.cpp:103-105
            r.data = true;
            uint32_t f = 0;
            try {
                if (csv) {  // split_csv (io.cpp:45-57)
                    const char* s = b;
                    for (;;) {
                        const char* c = static_cast<const char*>(std::memchr(s, ',', e - s));
                        const char* fe = c ? c : e;
                        out.push_back(parse_cell(s, fe, i + 1, f + 1, scratch));
                        ++f;
                        if (!c) break;
                        s = c + 1;
                    }
                } else {  // split_whitespace (io.cpp:59-67)
                    const char* s = b;
                    while (true) {
                        while (s < e && is_space(*s)) ++s;
                        if (s == e) break;
                        const char* fe = s;
                        while (fe < e && !is_space(*fe)) ++fe;
                        out.push_back(parse_cell(s, fe, i + 1, f + 1, scratch));
                        ++f;
                        s = fe;
                    }
                }
            } catch (const ParseError& pe) {
                r.err_col = pe.column;
                r.err_what = pe.what();
                // drop this row's partial values (the run stops at the first error anyway)
                out.resize(out.size() - f);
                r.fields = f;
                continue;
            }
            r.fields = f;
        }
    };
    if (T == 1) {
        work(0);
    } else {
        std::vector<std::thread> th;
        for (int t = 0; t < T; ++t) th.emplace_back(work, t);
        for (auto& x : th) x.join();
    }
    // file order: the first data row fixes the field count (io.cpp:113-121)
    uint64_t expected = 0, first_data_line = 0;
    bool have_first = false;
    for (uint64_t i = 0; i < L; ++i) {
        const RowResult& r = rows[i];
        if (!r.data) continue;
        if (r.err_col)  // the row's first cell error (its message without the location suffix)
            throw ParseError(r.err_what.substr(0, r.err_what.rfind(" (line ")), i + 1, r.err_col);
        if (!have_first) {
            have_first = true;
            expected = r.fields;
            first_data_line = i + 1;
        } else if (r.fields != expected) {
            throw ParseError("ragged row: expected " + std::to_string(expected) + " fields, got " +
                                 std::to_string(r.fields),
                             i + 1, r.fields + 1);
        }
    }
    if (!have_first)  // from_rows (io.cpp:69-80): "no data rows"
        throw ParseError("no data rows", first_data_line == 0 ? L + 1 : first_data_line, 1);
    m = 0;
    for (uint64_t i = 0; i < L; ++i) m += rows[i].data ? 1 : 0;
    n = expected;
    values.clear();
    values.reserve(m * n);
    for (int t = 0; t < T; ++t) values.insert(values.end(), part_vals[t].begin(), part_vals[t].end());
}

// load_tsplib (io.cpp:126-174).
void parse_tsplib(const std::string& text, std::vector<double>& values, uint64_t& m, uint64_t& n) {
    const std::vector<Line> lines = split_lines(text);
    std::string scratch;
    std::optional<uint64_t> dimension;
    bool in_coords = false;
    uint64_t line_no = 0;
    values.clear();
    m = 0;
    for (const Line& ln : lines) {
        ++line_no;
        const char* b = ln.b;
        const char* e = ln.e;
        while (b < e && is_space(*b)) ++b;
        while (e > b && is_space(e[-1])) --e;
        const std::string t(b, e);
        if (!in_coords) {
            if (t == "NODE_COORD_SECTION") {
                in_coords = true;
                continue;
            }
            const size_t colon = t.find(':');
            if (colon != std::string::npos) {
                std::string key = t.substr(0, colon);
                const size_t kb = key.find_first_not_of(" \t\n\v\f\r");
                const size_t ke = key.find_last_not_of(" \t\n\v\f\r");
                key = kb == std::string::npos ? std::string() : key.substr(kb, ke - kb + 1);
                if (key == "DIMENSION") {
                    const std::string rest = t.substr(colon + 1);
                    dimension = static_cast<uint64_t>(parse_cell(rest.data(), rest.data() + rest.size(), line_no, 2,
                                                                 scratch));
                }
            }
            continue;
        }
        if (t.empty()) continue;
        if (t == "EOF") break;
        // split_whitespace
        std::vector<std::pair<const char*, const char*>> f;
        const char* s = t.data();
        const char* te = s + t.size();
        while (true) {
            while (s < te && is_space(*s)) ++s;
            if (s == te) break;
            const char* fe = s;
            while (fe < te && !is_space(*fe)) ++fe;
            f.push_back({s, fe});
            s = fe;
        }
        if (f.size() != 3)
            throw ParseError("node line must be 'index x y'", line_no, f.size() < 3 ? f.size() + 1 : 4);
        parse_cell(f[0].first, f[0].second, line_no, 1, scratch);  // index column: validated, then dropped
        values.push_back(parse_cell(f[1].first, f[1].second, line_no, 2, scratch));
        values.push_back(parse_cell(f[2].first, f[2].second, line_no, 3, scratch));
        ++m;
    }
    if (!in_coords) throw ParseError("NODE_COORD_SECTION not found", line_no, 1);
    if (dimension.has_value() && m != *dimension)
        throw ParseError("DIMENSION says " + std::to_string(*dimension) + " nodes but " + std::to_string(m) +
                             " were read",
                         line_no, 1);
    if (m == 0) throw ParseError("no data rows", line_no, 1);  // from_rows
    n = 2;
}

void parse_any(const char* path, int32_t format, int32_t has_header, const uint64_t* columns, uint64_t ncolumns,
               int32_t threads, std::vector<double>& values, uint64_t& m, uint64_t& n) {
    if (format < 0 || format > 2) throw ConfigErr("unknown dataset format");
    const std::string text = read_file(path);
    const int T = threads > 0 ? threads : std::max(1u, std::thread::hardware_concurrency());
    if (format == BM_FORMAT_TSPLIB) parse_tsplib(text, values, m, n);
    else parse_delimited(text, format == BM_FORMAT_CSV, has_header != 0, T, values, m, n);
    // Dataset ctor (core.cpp:19-32): every value finite (before any column selection)
    for (double v : values)
        if (!std::isfinite(v)) throw ConfigErr("dataset contains a non-finite value");
    if (columns) {  // select_columns (io.cpp:176-195)
        if (ncolumns == 0) throw ConfigErr("column selection must not be empty");
        for (uint64_t c = 0; c < ncolumns; ++c)
            if (columns[c] >= n)
                throw ConfigErr("selected column " + std::to_string(columns[c]) + " does not exist (n=" +
                                std::to_string(n) + ")");
        std::vector<double> sel;
        sel.reserve(m * ncolumns);
        for (uint64_t i = 0; i < m; ++i)
            for (uint64_t c = 0; c < ncolumns; ++c) sel.push_back(values[i * n + columns[c]]);
        values.swap(sel);
        n = ncolumns;
    }
}

}  // namespace

extern "C" {

bm_status bm_parse_file(const char* path, int32_t format, int32_t has_header, const uint64_t* columns,
                        uint64_t ncolumns, int32_t threads, double** values, uint64_t* m, uint64_t* n) {
    return guarded_io([&] {
        std::vector<double> v;
        uint64_t mm = 0, nn = 0;
        parse_any(path, format, has_header, columns, ncolumns, threads, v, mm, nn);
        double* out = static_cast<double*>(std::malloc(std::max<size_t>(v.size(), 1) * sizeof(double)));
        if (!out) throw std::runtime_error("out of host memory");
        std::memcpy(out, v.data(), v.size() * sizeof(double));
        *values = out;
        *m = mm;
        *n = nn;
    });
}

void bm_free_values(double* values) { std::free(values); }

bm_status bm_dataset_load(const char* path, int32_t format, int32_t has_header, int32_t normalize,
                          const uint64_t* columns, uint64_t ncolumns, int32_t threads, int device,
                          bm_dataset** out) {
    std::vector<double> v;
    uint64_t m = 0, n = 0;
    bm_status st = guarded_io([&] { parse_any(path, format, has_header, columns, ncolumns, threads, v, m, n); });
    if (st != BM_OK) return st;
    bm_dataset* d = nullptr;
    st = bm_dataset_create(v.data(), m, n, BM_F64, device, &d);
    if (st != BM_OK || !normalize) {
        if (st == BM_OK) *out = d;
        return st;
    }
    bm_dataset* nd = nullptr;  // min_max_normalize (io.cpp:245-264) on the device
    st = bm_dataset_min_max_normalize(d, &nd);
    bm_dataset_destroy(d);
    if (st == BM_OK) *out = nd;
    return st;
}

bm_status bm_last_parse_location(uint64_t* line, uint64_t* column) {
    if (line) *line = t_parse_line;
    if (column) *column = t_parse_column;
    return BM_OK;
}

}  // extern "C"
