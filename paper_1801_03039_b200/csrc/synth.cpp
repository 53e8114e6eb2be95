// synth.cpp -- deterministic synthetic scenario matrices (ebic_synth_generate).
//
// Restates the reference generator so the bench and tests can build the
// BASELINE.json inputs in-process with no reference code at run time:
//   Rng              /root/reference/proj/include/ebic/rng.hpp:13-77
//   place_blocks     /root/reference/proj/include/ebic/synthgen.hpp:70-96
//   generate         /root/reference/proj/include/ebic/synthgen.hpp:114-223
// The engine is the C++-standard std::mt19937_64 (bit-exact by specification);
// the draws and the Box-Muller transform use the same arithmetic and the same
// glibc libm calls, so matrices are bit-identical to ebic::generate for the same
// ScenarioSpec (pinned by tests/test_synth.py against oracle/_ref).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../../include/ebic_b200.h"

namespace {

class SynthRng {
  public:
    explicit SynthRng(uint64_t seed) : eng_(seed) {}

    // Unbiased integer in [0, bound) by rejection (rng.hpp:21-28).
    uint64_t below(uint64_t bound) {
        const uint64_t threshold = (0 - bound) % bound;
        for (;;) {
            const uint64_t r = eng_();
            if (r >= threshold) return r % bound;
        }
    }
    size_t index(size_t bound) { return static_cast<size_t>(below(bound)); }
    // 53-bit uniform in [0, 1) (rng.hpp:35).
    double real() { return static_cast<double>(eng_() >> 11) * 0x1.0p-53; }
    double real(double lo, double hi) { return lo + (hi - lo) * real(); }
    // Box-Muller with a cached spare (rng.hpp:43-58).
    double normal(double mean, double sd) {
        if (have_spare_) {
            have_spare_ = false;
            return mean + sd * spare_;
        }
        double u1;
        do {
            u1 = real();
        } while (u1 <= 0.0);
        const double u2 = real();
        const double radius = std::sqrt(-2.0 * std::log(u1));
        const double angle = 2.0 * kPi * u2;
        spare_ = radius * std::sin(angle);
        have_spare_ = true;
        return mean + sd * radius * std::cos(angle);
    }

    // m[i] = normal(0, 1) for i < n, in order -- the bulk of generate()'s draws
    // (the background of every cell).  Same values as the sequential loop:
    // the pairs' raw engine outputs are drawn in order (into m itself, two
    // slots per pair), then every pair's Box-Muller transform -- the same glibc
    // log/sqrt/sin/cos in the same expression order -- runs on all host
    // threads.  A rejected u1 (engine output < 2^11, p = 2^-53) switches the
    // rest to the sequential loop at exactly that point.
    void fill_standard_normals(double* m, size_t n) {
        size_t i = 0;
        if (n && have_spare_) m[i++] = normal(0.0, 1.0);
        const size_t pairs = (n - i) / 2;
        if (pairs < (size_t{1} << 16)) {
            for (; i < n; ++i) m[i] = normal(0.0, 1.0);
            return;
        }
        uint64_t* raw = reinterpret_cast<uint64_t*>(m + i);
        // Pipeline: this thread draws pairs in order and publishes how many
        // are ready; workers transform blocks as soon as they are drawn.
        constexpr size_t kBlock = size_t{1} << 14;
        std::atomic<size_t> drawn{0}, next{0}, limit{pairs};
        std::atomic<bool> done{false};
        const unsigned nt = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
        const double* const out0 = m + i;
        auto transform = [&] {
            for (;;) {
                const size_t b = next.fetch_add(kBlock);
                size_t e = std::min(b + kBlock, pairs);
                if (b >= pairs) return;
                for (;;) {  // wait until the block is drawn (or drawing stopped short)
                    const size_t lim = limit.load(std::memory_order_acquire);
                    e = std::min(e, lim);
                    if (b >= e) return;
                    if (drawn.load(std::memory_order_acquire) >= e) break;
                    if (done.load(std::memory_order_acquire) && drawn.load(std::memory_order_acquire) < e) {
                        e = std::min(e, drawn.load(std::memory_order_acquire));
                        break;
                    }
                    std::this_thread::yield();
                }
                double* out = const_cast<double*>(out0);
                for (size_t k = b; k < e; ++k) {
                    const double u1 = static_cast<double>(raw[2 * k] >> 11) * 0x1.0p-53;
                    const double u2 = static_cast<double>(raw[2 * k + 1] >> 11) * 0x1.0p-53;
                    const double radius = std::sqrt(-2.0 * std::log(u1));
                    const double angle = 2.0 * kPi * u2;
                    const double spare = radius * std::sin(angle);
                    out[2 * k] = 0.0 + 1.0 * radius * std::cos(angle);
                    out[2 * k + 1] = 0.0 + 1.0 * spare;
                }
            }
        };
        std::vector<std::thread> pool;
        for (unsigned t = 0; t + 1 < nt; ++t) pool.emplace_back(transform);
        size_t good = pairs;  // pairs whose u1 needs no redraw
        for (size_t k = 0; k < pairs; ++k) {
            const uint64_t a = eng_();
            if ((a >> 11) == 0) {  // normal() would redraw u1 here: finish sequentially
                good = k;
                limit.store(k, std::memory_order_release);
                break;
            }
            raw[2 * k] = a;
            raw[2 * k + 1] = eng_();
            if (((k + 1) & (kBlock - 1)) == 0) drawn.store(k + 1, std::memory_order_release);
        }
        drawn.store(good, std::memory_order_release);
        done.store(true, std::memory_order_release);
        transform();  // this thread helps with what is left
        for (std::thread& th : pool) th.join();
        // The rest in order: the odd tail, or everything from a rejected u1 on
        // (that draw is consumed; normal()'s do-while continues with the next).
        for (i += 2 * good; i < n; ++i) m[i] = normal(0.0, 1.0);
    }

  private:
    static constexpr double kPi = 3.141592653589793238462643383279502884;
    std::mt19937_64 eng_;
    double spare_ = 0.0;
    bool have_spare_ = false;
};

// Shuffled index pool; block i+1 reuses the trailing `overlap` indices of
// block i (synthgen.hpp:74-96).
std::vector<std::vector<size_t>> place(size_t n, size_t overlap, const std::vector<size_t>& sizes,
                                       SynthRng& rng) {
    size_t needed = 0;
    for (size_t i = 0; i < sizes.size(); ++i) needed += i == 0 ? sizes[i] : sizes[i] - overlap;
    if (needed > n) throw std::runtime_error("scenario infeasible");
    std::vector<size_t> pool(n);
    std::iota(pool.begin(), pool.end(), size_t{0});
    for (size_t i = pool.size(); i > 1; --i) std::swap(pool[i - 1], pool[rng.index(i)]);
    std::vector<std::vector<size_t>> out;
    size_t start = 0;
    for (size_t sz : sizes) {
        out.emplace_back(pool.begin() + static_cast<std::ptrdiff_t>(start),
                         pool.begin() + static_cast<std::ptrdiff_t>(start + sz));
        start += sz - overlap;
    }
    return out;
}

enum Pattern { kTrend = 0, kColConst, kRowConst, kShift, kScale, kShiftScale };

}  // namespace

extern "C" int ebic_synth_generate(size_t n_rows, size_t n_cols, size_t n_blocks,
                                   const size_t* block_rows, const size_t* block_cols, int pattern,
                                   size_t overlap_rows, size_t overlap_cols, double noise_sd,
                                   uint64_t seed, double* values_out) {
    try {
        if (n_rows == 0 || n_cols == 0) throw std::invalid_argument("matrix shape must be positive");
        if (noise_sd < 0.0) throw std::invalid_argument("noise_sd must be non-negative");
        if (pattern < kTrend || pattern > kShiftScale) throw std::invalid_argument("unknown pattern");
        if (!values_out || (n_blocks && (!block_rows || !block_cols)))
            throw std::invalid_argument("null argument");
        for (size_t i = 0; i < n_blocks; ++i) {
            if (block_rows[i] == 0 || block_cols[i] == 0 || block_rows[i] > n_rows ||
                block_cols[i] > n_cols)
                throw std::runtime_error("scenario infeasible");
            if (n_blocks > 1 && (overlap_rows >= block_rows[i] || overlap_cols >= block_cols[i]))
                throw std::runtime_error("scenario infeasible");
        }
        SynthRng rng(seed);
        const std::vector<size_t> rs(block_rows, block_rows + n_blocks), cs(block_cols, block_cols + n_blocks);
        const auto brows = place(n_rows, overlap_rows, rs, rng);
        const auto bcols = place(n_cols, overlap_cols, cs, rng);

        std::vector<uint8_t> implanted(n_rows * n_cols, 0);
        for (size_t i = 0; i < n_blocks; ++i)
            for (size_t r : brows[i])
                for (size_t c : bcols[i]) implanted[r * n_cols + c] = 1;

        std::vector<double> col_param(n_cols, 0.0), row_offset(n_rows, 0.0), row_mult(n_rows, 1.0);
        switch (pattern) {
            case kTrend:
                for (double& v : col_param) v = rng.real();
                break;
            case kColConst:
                for (double& v : col_param) v = rng.normal(0.0, 1.0);
                break;
            case kRowConst:
                for (double& v : row_offset) v = rng.normal(0.0, 1.0);
                break;
            case kShift:
                for (double& v : col_param) v = rng.normal(0.0, 1.0);
                for (double& v : row_offset) v = rng.normal(0.0, 2.0);
                break;
            case kScale:
                for (double& v : col_param) v = rng.normal(0.0, 1.0);
                for (double& v : row_mult) v = rng.real(0.5, 3.0);
                break;
            case kShiftScale:
                for (double& v : col_param) v = rng.normal(0.0, 1.0);
                for (double& v : row_offset) v = rng.normal(0.0, 2.0);
                for (double& v : row_mult) v = rng.real(0.5, 3.0);
                break;
        }

        double* m = values_out;
        rng.fill_standard_normals(m, n_rows * n_cols);

        if (pattern == kTrend) {
            std::vector<size_t> row_cols;
            std::vector<double> draws;
            for (size_t r = 0; r < n_rows; ++r) {
                row_cols.clear();
                for (size_t c = 0; c < n_cols; ++c)
                    if (implanted[r * n_cols + c]) row_cols.push_back(c);
                if (row_cols.empty()) continue;
                std::sort(row_cols.begin(), row_cols.end(), [&](size_t a, size_t b) {
                    if (col_param[a] != col_param[b]) return col_param[a] < col_param[b];
                    return a < b;
                });
                draws.resize(row_cols.size());
                for (double& v : draws) v = rng.normal(0.0, 1.0);
                std::sort(draws.begin(), draws.end());
                for (size_t i = 0; i < row_cols.size(); ++i) m[r * n_cols + row_cols[i]] = draws[i];
            }
        } else {
            for (size_t r = 0; r < n_rows; ++r)
                for (size_t c = 0; c < n_cols; ++c) {
                    if (!implanted[r * n_cols + c]) continue;
                    double value = 0.0;
                    switch (pattern) {
                        case kColConst: value = col_param[c]; break;
                        case kRowConst: value = row_offset[r]; break;
                        case kShift: value = col_param[c] + row_offset[r]; break;
                        case kScale: value = col_param[c] * row_mult[r]; break;
                        case kShiftScale: value = col_param[c] * row_mult[r] + row_offset[r]; break;
                        default: break;
                    }
                    m[r * n_cols + c] = value;
                }
        }
        if (noise_sd > 0.0)
            for (size_t r = 0; r < n_rows; ++r)
                for (size_t c = 0; c < n_cols; ++c)
                    if (implanted[r * n_cols + c]) m[r * n_cols + c] += rng.normal(0.0, noise_sd);
    } catch (const std::invalid_argument&) {
        return EBIC_ERR_INVALID_ARGUMENT;
    } catch (...) {
        return EBIC_ERR_RUNTIME;
    }
    return EBIC_OK;
}
