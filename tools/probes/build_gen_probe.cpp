// Splits build_generation (shadow evolution.hpp) into its parts on recorded
// GA populations: tournament selection, variation operators, tabu insert.
// build: g++ -std=c++20 -O2 -I include -I <ref include> -I <json> tools/probes/build_gen_probe.cpp \
//   -L paper_1801_03039_b200 -lebic_b200 -Wl,-rpath,'$ORIGIN/../../paper_1801_03039_b200'
// usage: build_gen_probe <population trace> [reps]
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <x86intrin.h>

#include "ebic/evolution.hpp"

using namespace ebic;

int main(int argc, char** argv) {
    std::FILE* f = std::fopen(argv[1], "rb");
    if (!f) return 2;
    const int reps = argc > 2 ? std::atoi(argv[2]) : 5;
    std::uint64_t P;
    std::vector<std::vector<ColumnSeries>> pops;
    std::vector<std::vector<double>> fits;
    std::size_t width = 0;
    while (std::fread(&P, 8, 1, f) == 1) {
        std::vector<std::uint64_t> o(P + 1);
        if (std::fread(o.data(), 8, P + 1, f) != P + 1) return 2;
        std::vector<std::uint16_t> c(o[P]);
        if (std::fread(c.data(), 2, o[P], f) != o[P]) return 2;
        std::vector<double> fi(P);
        if (std::fread(fi.data(), 8, P, f) != P) return 2;
        std::vector<ColumnSeries> pop(P);
        for (std::size_t i = 0; i < P; ++i) {
            pop[i].assign(c.begin() + o[i], c.begin() + o[i + 1]);
            for (auto x : pop[i]) width = std::max<std::size_t>(width, x + 1u);
        }
        pops.push_back(pop);
        fits.push_back(fi);
    }
    width = std::max<std::size_t>(width, 500);
    EvolutionConfig conf;
    conf.population_size = 600;
    unsigned long long cyc[4] = {0, 0, 0, 0};
    double wall = 0;
    std::size_t gens = 0;
    for (int r = 0; r < reps; ++r) {
        Rng gen(7);
        TabuList seen(width);
        TopRankList best(width);
        ColumnPenaltyTable crowding(width);
        for (std::size_t u = 0; u < pops.size(); ++u) {
            best.update(pops[u], fits[u], conf);
            const auto& parents = pops[u];
            const auto& pf = fits[u];
            const auto t0 = std::chrono::steady_clock::now();
            crowding.reset();
            std::vector<ColumnSeries> out;
            const std::size_t elites = std::min<std::size_t>(
                static_cast<std::size_t>(std::ceil(conf.elite_fraction * double(best.size()))), conf.population_size);
            for (std::size_t e = 0; e < elites; ++e) {
                crowding.add(best.entries()[e].series);
                out.push_back(best.entries()[e].series);
            }
            std::size_t misses = 0;
            while (out.size() < conf.population_size && misses <= conf.population_size) {
                unsigned long long a = __rdtsc();
                const OperatorKind kind = draw_operator(conf.probabilities, gen);
                const std::size_t pa = tournament_select(parents, pf, crowding, conf, gen);
                std::size_t pb = 0;
                if (kind == OperatorKind::kCrossover) pb = tournament_select(parents, pf, crowding, conf, gen);
                unsigned long long b = __rdtsc();
                ColumnSeries child;
                switch (kind) {
                    case OperatorKind::kInsertion: child = mutate_insertion(parents[pa], width, gen).series; break;
                    case OperatorKind::kDeletion: child = mutate_deletion(parents[pa], gen).series; break;
                    case OperatorKind::kSwap: child = mutate_swap(parents[pa], gen).series; break;
                    case OperatorKind::kSubstitution: child = mutate_substitution(parents[pa], width, gen).series; break;
                    case OperatorKind::kCrossover: child = crossover(parents[pa], parents[pb], pf[pa], pf[pb], gen); break;
                }
                unsigned long long c = __rdtsc();
                const bool fresh = seen.insert(child);
                unsigned long long d = __rdtsc();
                if (fresh) {
                    crowding.add(child);
                    out.push_back(std::move(child));
                } else {
                    ++misses;
                }
                unsigned long long e = __rdtsc();
                cyc[0] += b - a, cyc[1] += c - b, cyc[2] += d - c, cyc[3] += e - d;
            }
            wall += std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
            ++gens;
        }
    }
    const auto t0 = std::chrono::steady_clock::now();
    const unsigned long long c0 = __rdtsc();
    while (std::chrono::steady_clock::now() - t0 < std::chrono::milliseconds(50)) {}
    const double ghz = double(__rdtsc() - c0) / 50e6;
    std::printf("{\"us_per_generation\": %.1f, \"tsc_ghz\": %.2f, \"us_select\": %.1f, \"us_operator\": %.1f, "
                "\"us_tabu\": %.1f, \"us_admit\": %.1f}\n",
                wall / gens, ghz, cyc[0] / ghz / 1e3 / gens, cyc[1] / ghz / 1e3 / gens, cyc[2] / ghz / 1e3 / gens,
                cyc[3] / ghz / 1e3 / gens);
}
