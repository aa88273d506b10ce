// dropin_common.hpp — shared pieces of the drop-in translation units that
// replace the reference's src/big_means.cpp and src/local_search.cpp
// (/root/reference/proj/src): status -> exception mapping (common.hpp:21-49)
// and the per-Dataset device cache.
#pragma once

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <list>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "bigmeans/core.hpp"
#include "bigmeans_b200.h"

namespace bigmeans {
namespace dropin {

inline void rethrow(bm_status st) {
    if (st == BM_OK) return;
    const std::string msg = bm_last_error();
    if (st == BM_CONFIG_ERROR) throw ConfigError(msg);
    if (st == BM_STATE_ERROR) throw StateError(msg);
    throw std::runtime_error(msg);
}

inline int device_of_thread() {
    const char* e = std::getenv("BIGMEANS_DEVICE");
    return e ? std::atoi(e) : 0;
}

// Device copies of (host, immutable; core.hpp:13-15) Datasets, cached so that
// repeated calls on one Dataset (choose_chunk_size_hint's probes, bench runs
// over n_exec seeds, the acceptance corpora) upload it once.  A cache hit needs
// the same values buffer, shape, device and content: the 64-bit content
// fingerprint (an order-free sum of mixed (index, bits) pairs, computed with
// OpenMP) guards against a new Dataset reusing a freed buffer's address.
// The cache holds at most kCacheEntries handles (least recently used evicted).
struct Handle {
    bm_dataset* h = nullptr;
    ~Handle() {
        if (h) bm_dataset_destroy(h);
    }
};

struct CacheKey {
    const double* data;
    std::size_t m, n;
    int device;
    std::uint64_t fingerprint;
    bool operator==(const CacheKey& o) const {
        return data == o.data && m == o.m && n == o.n && device == o.device && fingerprint == o.fingerprint;
    }
};

constexpr std::size_t kCacheEntries = 2;
inline std::mutex g_cache_mu;
inline std::list<std::pair<CacheKey, std::shared_ptr<Handle>>> g_cache;  // front = most recent

inline std::uint64_t mix64(std::uint64_t x) {  // splitmix64 finalizer
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ull;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

inline std::uint64_t fingerprint(const std::vector<double>& v) {
    const std::size_t count = v.size();
    const double* p = v.data();
    std::uint64_t acc = 0;
#pragma omp parallel for reduction(+ : acc) schedule(static)
    for (std::size_t i = 0; i < count; ++i) {
        std::uint64_t b;
        std::memcpy(&b, p + i, 8);
        acc += mix64(b ^ mix64(i + 0x9e3779b97f4a7c15ull));
    }
    return acc;
}

inline std::shared_ptr<Handle> device_dataset(const Dataset& d) {
    const CacheKey key{d.values().data(), d.m(), d.n(), device_of_thread(), fingerprint(d.values())};
    {
        std::lock_guard<std::mutex> lk(g_cache_mu);
        for (auto it = g_cache.begin(); it != g_cache.end(); ++it)
            if (it->first == key) {
                g_cache.splice(g_cache.begin(), g_cache, it);
                return g_cache.front().second;
            }
    }
    auto h = std::make_shared<Handle>();
    rethrow(bm_dataset_create(d.values().data(), d.m(), d.n(), BM_F64, key.device, &h->h));
    std::lock_guard<std::mutex> lk(g_cache_mu);
    g_cache.emplace_front(key, h);
    while (g_cache.size() > kCacheEntries) g_cache.pop_back();
    return h;
}


}  // namespace dropin
}  // namespace bigmeans
