#pragma once
// B200 drop-in for the reference's ebic/fitness.hpp
// (/root/reference/proj/include/ebic/fitness.hpp:1-145).
//
// Put this directory BEFORE the reference's include directory on the compiler's
// -I path and link libebic_b200.so: the reference's own evolution.hpp,
// expansion.hpp and io.hpp then compile against these declarations, and every
// generation's evaluate_population (evolution.hpp:484-485, :504-505) runs as one
// sm_100a kernel launch instead of a ThreadPool pass over row chunks.  Every
// symbol the other reference headers consume from fitness.hpp is provided with
// the reference's signature and semantics:
//   RowRange, ChunkPlan, make_chunk_plan, FitnessParams, default_sigma,
//   row_matches, count_matches, fitness_score, evaluate_population.
// Results are bit-identical (integer counts; Eq. 1 with the same libm).
//
// The reference passes the matrix by const& on every call and has no context
// object; the device copy is therefore cached per matrix, keyed by its buffer
// address, shape and a hash of its whole contents, and pinned without
// re-hashing inside a b200::MatrixScope (the drop-in run() and
// finalize_biclusters open one: the matrix is const there).  Devices: EBIC_GPUS="0,1,..." (default 0);
// rows are sharded over them and partial counts reduced exactly.

#include <algorithm>
#include <cassert>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <span>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "ebic/cbf.hpp"
#include "ebic/matrix.hpp"
#include "ebic_b200.h"

namespace ebic {

// fitness.hpp:20-39 -- the reference's row partition for its thread pool.
// The B200 path shards rows across devices instead; counts are partition
// invariant (fitness.hpp:17-19), so a plan is accepted for signature parity
// and never changes a result.  Same chunks as the reference: ceil(n / w)
// rows each, the last one short.
struct RowRange {
    std::size_t lo = 0;
    std::size_t hi = 0;
};

struct ChunkPlan {
    std::vector<RowRange> chunks;
    unsigned worker_count = 1;
};

inline ChunkPlan make_chunk_plan(std::size_t rows, unsigned workers = 0) {
    if (!rows) throw std::invalid_argument("matrix has no rows");
    const unsigned w = workers ? workers : std::max(1u, std::thread::hardware_concurrency());
    const std::size_t step = rows / w + (rows % w != 0);
    ChunkPlan out;
    out.worker_count = w;
    out.chunks.reserve((rows + step - 1) / step);
    for (std::size_t at = 0; at < rows; at += step) out.chunks.push_back(RowRange{at, std::min(rows, at + step)});
    return out;
}

// fitness.hpp:41-52 -- sigma: the expected-support scale of Eq. 1.
struct FitnessParams {
    std::uint64_t sigma = 4;
};

inline std::uint64_t default_sigma(std::size_t rows) { return ebic_default_sigma(rows); }

// fitness.hpp:57-67 -- one row, on the host (tests and single-row checks);
// the same fp64 add-then-compare over adjacent pairs, first failure ends it.
inline bool row_matches(const ExpressionMatrix& matrix, std::size_t row,
                        std::span<const ColumnIndex> cols, double eps = 0.0) {
    const double* r = matrix.row_ptr(row);
    for (std::size_t k = 1; k < cols.size(); ++k)
        if (!(r[cols[k - 1]] < r[cols[k]] + eps)) return false;
    return true;
}

namespace b200 {

[[noreturn]] inline void throw_status(int status) {
    const std::string msg = ebic_last_error();
    if (status == EBIC_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

inline void check(int status) {
    if (status != EBIC_OK) throw_status(status);
}

inline std::vector<int> devices_from_env() {
    std::vector<int> devs;
    if (const char* e = std::getenv("EBIC_GPUS")) {
        std::string s(e);
        std::size_t at = 0;
        while (at < s.size()) {
            std::size_t comma = s.find(',', at);
            if (comma == std::string::npos) comma = s.size();
            if (comma > at) devs.push_back(std::stoi(s.substr(at, comma - at)));
            at = comma + 1;
        }
    }
    if (devs.empty()) devs.push_back(0);
    return devs;
}

// Content hash of the whole matrix (4 independent multiply-xorshift lanes,
// ~10-20 GB/s): a cached device copy is reused only for a matrix with the same
// buffer, shape and contents.  A matrix edited in place, or a new matrix in a
// reused buffer, gets a fresh context.
inline std::uint64_t content_hash(const ExpressionMatrix& m) {
    const std::size_t n = m.values.size();
    const double* v = m.values.data();
    std::uint64_t h[4] = {0x9e3779b97f4a7c15ull ^ n, 0xc2b2ae3d27d4eb4full ^ m.n_rows,
                          0x165667b19e3779f9ull ^ m.n_cols, 0x27d4eb2f165667c5ull};
    auto mix = [](std::uint64_t x, std::uint64_t w) {
        x = (x ^ w) * 0xff51afd7ed558ccdull;
        return x ^ (x >> 29);
    };
    std::size_t i = 0;
    for (; i + 4 <= n; i += 4) {
        std::uint64_t w[4];
        std::memcpy(w, v + i, sizeof w);
        for (int k = 0; k < 4; ++k) h[k] = mix(h[k], w[k]);
    }
    for (; i < n; ++i) {
        std::uint64_t w;
        std::memcpy(&w, v + i, sizeof w);
        h[0] = mix(h[0], w);
    }
    return mix(mix(h[0], h[1]), mix(h[2], h[3]));
}

// One device context; destroyed when the last holder lets go (a cache
// eviction never frees a context a call or scope is still using).
struct DeviceMatrix {
    ebic_ctx* ctx = nullptr;
    explicit DeviceMatrix(const ExpressionMatrix& m) {
        const std::vector<int> devs = devices_from_env();
        check(ebic_ctx_create(m.values.data(), m.n_rows, m.n_cols, devs.data(),
                              static_cast<int>(devs.size()), &ctx));
    }
    ~DeviceMatrix() { ebic_ctx_destroy(ctx); }
    DeviceMatrix(const DeviceMatrix&) = delete;
    DeviceMatrix& operator=(const DeviceMatrix&) = delete;
};
using DeviceMatrixPtr = std::shared_ptr<DeviceMatrix>;

struct CachedContext {
    const double* data = nullptr;
    std::size_t rows = 0, cols = 0;
    std::uint64_t hash = 0;
    DeviceMatrixPtr dm;
};

struct ContextCache {
    std::mutex mu;
    std::vector<CachedContext> entries;  // most recently used last
};

inline ContextCache& cache() {
    static ContextCache c;
    return c;
}

// Matrices pinned by a live MatrixScope on this thread (innermost last).
struct PinnedMatrix {
    const double* data;
    std::size_t rows, cols;
    DeviceMatrixPtr dm;
};
inline std::vector<PinnedMatrix>& pinned() {
    thread_local std::vector<PinnedMatrix> p;
    return p;
}

// Device context holding `m`: the pinned one of an enclosing MatrixScope
// (no hashing: the matrix is const for the scope's duration, as in run()),
// else a cached context with the same buffer, shape and content hash, else a
// new one (uploaded once).
inline DeviceMatrixPtr context_for(const ExpressionMatrix& m) {
    for (auto it = pinned().rbegin(); it != pinned().rend(); ++it)
        if (it->data == m.values.data() && it->rows == m.n_rows && it->cols == m.n_cols) return it->dm;
    const std::uint64_t h = content_hash(m);
    ContextCache& c = cache();
    std::lock_guard<std::mutex> lock(c.mu);
    for (std::size_t i = 0; i < c.entries.size(); ++i) {
        CachedContext& e = c.entries[i];
        if (e.data == m.values.data() && e.rows == m.n_rows && e.cols == m.n_cols && e.hash == h) {
            std::rotate(c.entries.begin() + static_cast<std::ptrdiff_t>(i),
                        c.entries.begin() + static_cast<std::ptrdiff_t>(i) + 1, c.entries.end());
            return c.entries.back().dm;
        }
    }
    if (c.entries.size() >= 4) c.entries.erase(c.entries.begin());  // holders keep theirs alive
    auto dm = std::make_shared<DeviceMatrix>(m);
    c.entries.push_back({m.values.data(), m.n_rows, m.n_cols, h, dm});
    return dm;
}

// Pins the device copy of `m` for a block in which `m` does not change
// (the drop-in's run() and finalize_biclusters): every call inside reuses it
// without re-hashing the matrix.
class MatrixScope {
  public:
    explicit MatrixScope(const ExpressionMatrix& m) {
        pinned().push_back({m.values.data(), m.n_rows, m.n_cols, context_for(m)});
    }
    ~MatrixScope() { pinned().pop_back(); }
    MatrixScope(const MatrixScope&) = delete;
    MatrixScope& operator=(const MatrixScope&) = delete;
};

}  // namespace b200

// fitness.hpp:100-118 -- one sm_100a launch per device shard; exact integer sums.
inline std::vector<std::uint64_t> count_matches(const ExpressionMatrix& m, const CbfPopulation& pop,
                                                const ChunkPlan& plan, double epsilon = 0.0) {
    (void)plan;
    const std::size_t n = pop.size();
    std::vector<std::uint64_t> counts(n, 0);
    if (n == 0) return counts;
    const b200::DeviceMatrixPtr dm = b200::context_for(m);
    b200::check(ebic_count_matches(dm->ctx, pop.offsets.data(), pop.col_indices.data(), n, epsilon,
                                   counts.data()));
    return counts;
}

// fitness.hpp:124-133, verbatim arithmetic (host libm).
inline double fitness_score(std::uint64_t match_count, std::size_t series_len,
                            const FitnessParams& params) {
    assert(series_len >= kMinSeriesLength);
    return ebic_fitness_score(match_count, series_len, params.sigma);
}

// fitness.hpp:135-143 -- counts and Eq. 1 (fused into the count kernel's
// epilogue from host-glibc tables; bit-identical).
inline std::vector<double> evaluate_population(const ExpressionMatrix& m, const CbfPopulation& pop,
                                               const ChunkPlan& plan, const FitnessParams& params,
                                               double epsilon = 0.0) {
    (void)plan;
    const std::size_t n = pop.size();
    std::vector<double> fitness(n, 0.0);
    if (n == 0) return fitness;
    const b200::DeviceMatrixPtr dm = b200::context_for(m);
    b200::check(ebic_evaluate_population(dm->ctx, pop.offsets.data(), pop.col_indices.data(), n,
                                         params.sigma, epsilon, nullptr, fitness.data()));
    return fitness;
}

}  // namespace ebic
