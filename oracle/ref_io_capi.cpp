// ref_io_capi.cpp — TEST INFRASTRUCTURE: a C entry over the UNMODIFIED
// reference loader io::load (/root/reference/proj/src/io.cpp:224-243), compiled
// into oracle/_ref with the reference sources, so tests can check the B200
// ingestion (paper_2204_07485_b200/csrc/io.cpp) against it: values, column
// selection, min-max normalisation and every error (kind, message, line, column).
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "bigmeans/io.hpp"

using namespace bigmeans;

namespace {
thread_local std::string g_io_err;
}

extern "C" {

const char* ref_io_last_error() { return g_io_err.c_str(); }

// 0 ok, 1 ConfigError, 2 StateError, 5 ParseError (eline / ecol set), 4 other
int ref_io_load(const char* path, int format, int has_header, int normalize, const uint64_t* cols, uint64_t ncols,
                int has_cols, double** values, uint64_t* m, uint64_t* n, uint64_t* eline, uint64_t* ecol) {
    try {
        io::DatasetSpec spec;
        spec.path = path;
        spec.format = format == 0 ? io::Format::csv : format == 1 ? io::Format::whitespace : io::Format::tsplib;
        spec.has_header = has_header != 0;
        spec.normalize = normalize != 0;
        if (has_cols) spec.columns = std::vector<std::size_t>(cols, cols + ncols);
        const Dataset d = io::load(spec);
        *m = d.m();
        *n = d.n();
        *values = static_cast<double*>(std::malloc(std::max<size_t>(d.values().size(), 1) * sizeof(double)));
        std::memcpy(*values, d.values().data(), d.values().size() * sizeof(double));
        return 0;
    } catch (const ParseError& e) {
        g_io_err = e.what();
        *eline = e.line();
        *ecol = e.column();
        return 5;
    } catch (const ConfigError& e) {
        g_io_err = e.what();
        return 1;
    } catch (const StateError& e) {
        g_io_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_io_err = e.what();
        return 4;
    }
}

void ref_io_free(double* v) { std::free(v); }

}  // extern "C"
