// build_generation timing on a recorded population stream; compile against the shadow
// headers (drop-in) or the reference headers alone (reference).
// usage: build_gen_compare <population trace> [width]   (width: max column + 1 by default)
#include <chrono>
#include <cstdio>
#include "ebic/evolution.hpp"
using namespace ebic;
int main(int argc, char** argv) {
    FILE* f = fopen(argv[1], "rb"); uint64_t P;
    std::vector<std::vector<ColumnSeries>> pops; std::vector<std::vector<double>> fits;
    while (fread(&P, 8, 1, f) == 1) {
        std::vector<uint64_t> o(P + 1); if (fread(o.data(), 8, P + 1, f) != P + 1) return 2;
        std::vector<uint16_t> c(o[P]); if (fread(c.data(), 2, o[P], f) != o[P]) return 2;
        std::vector<double> fi(P); if (fread(fi.data(), 8, P, f) != P) return 2;
        std::vector<ColumnSeries> pop(P);
        for (size_t i = 0; i < P; ++i) pop[i].assign(c.begin() + o[i], c.begin() + o[i + 1]);
        pops.push_back(pop); fits.push_back(fi);
    }
    size_t width = 0;
    for (auto& pop : pops) for (auto& s : pop) for (auto c : s) width = std::max<size_t>(width, c + 1u);
    if (argc > 2) width = std::stoull(argv[2]);
    EvolutionConfig evo; evo.population_size = 600;
    double best = 1e30; uint64_t dig = 0;
    for (int rep = 0; rep < 5; ++rep) {
        Rng rng(7); TabuList tabu(width); TopRankList top(width); ColumnPenaltyTable pen(width);
        double tot = 0; dig = 1469598103934665603ull;
        for (size_t u = 0; u < pops.size(); ++u) {
            top.update(pops[u], fits[u], evo);
            auto t0 = std::chrono::steady_clock::now();
            GenerationResult g = build_generation(pops[u], fits[u], top, tabu, pen, evo, width, rng);
            tot += std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
            for (auto& s : g.individuals) for (auto c : s) dig = (dig ^ c) * 1099511628211ull;
        }
        best = std::min(best, tot / pops.size());
    }
    printf("build_generation us %.1f digest %016llx\n", best, (unsigned long long)dig);
}
