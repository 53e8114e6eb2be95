// toprank_time.cpp -- TEST INFRASTRUCTURE ONLY (§8f rank 1 measurement).
//
// Replays a recorded stream of whole populations (ref_run_population_trace
// file: repeated { u64 P; u64 offsets[P+1]; u16 cols[]; f64 fitness[P] })
// through ebic::TopRankList::update (evolution.hpp:168-206) and prints the
// mean wall time per update plus a digest of the final list.  Built twice
// from this one source by oracle/Makefile:
//   oracle/_ref/toprank_time_ref     reference evolution.hpp
//   oracle/_ref/toprank_time_dropin  include/ebic/evolution.hpp shadow
//                                    (ebic_top_rank_update in libebic_b200.so)
// usage: toprank_time <trace.bin> <reps> [threshold] [capacity]
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "ebic/evolution.hpp"

#ifndef EBIC_DRIVER_NAME
#define EBIC_DRIVER_NAME "reference"
#endif

int main(int argc, char** argv) {
    if (argc < 3) return 2;
    std::FILE* f = std::fopen(argv[1], "rb");
    if (!f) return 2;
    const int reps = std::atoi(argv[2]);
    ebic::EvolutionConfig cfg;
    if (argc > 3) cfg.overlap_threshold = std::atof(argv[3]);
    if (argc > 4) cfg.top_rank_capacity = std::strtoull(argv[4], nullptr, 10);
    std::vector<std::vector<ebic::ColumnSeries>> pops;
    std::vector<std::vector<double>> fits;
    std::size_t n_cols = 0;
    std::uint64_t P;
    while (std::fread(&P, 8, 1, f) == 1) {
        std::vector<std::uint64_t> off(P + 1);
        if (std::fread(off.data(), 8, P + 1, f) != P + 1) return 2;
        std::vector<std::uint16_t> cols(off[P]);
        if (std::fread(cols.data(), 2, off[P], f) != off[P]) return 2;
        std::vector<double> fit(P);
        if (std::fread(fit.data(), 8, P, f) != P) return 2;
        std::vector<ebic::ColumnSeries> pop(P);
        for (std::uint64_t i = 0; i < P; ++i) {
            pop[i].assign(cols.begin() + off[i], cols.begin() + off[i + 1]);
            for (auto c : pop[i]) n_cols = std::max<std::size_t>(n_cols, c + 1);
        }
        pops.push_back(std::move(pop));
        fits.push_back(std::move(fit));
    }
    std::fclose(f);
    double best_us = 1e300;
    std::uint64_t digest = 0;
    for (int r = 0; r < reps; ++r) {
        ebic::TopRankList top(n_cols);
        const auto t0 = std::chrono::steady_clock::now();
        for (std::size_t u = 0; u < pops.size(); ++u) top.update(pops[u], fits[u], cfg);
        const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
        best_us = std::min(best_us, us / double(pops.size()));
        digest = 1469598103934665603ull;
        for (const auto& e : top.entries()) {
            for (auto c : e.series) digest = (digest ^ c) * 1099511628211ull;
            digest = (digest ^ e.seq) * 1099511628211ull;
        }
    }
    std::printf("{\"impl\": \"%s\", \"updates\": %zu, \"us_per_update\": %.3f, \"digest\": \"%016llx\"}\n",
                EBIC_DRIVER_NAME, pops.size(), best_us, static_cast<unsigned long long>(digest));
    return 0;
}
