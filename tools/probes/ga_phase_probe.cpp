// Times the phases of the EBIC GA loop (evolution.hpp run()) when compiled
// against the shadow headers: build_generation, encode, evaluate, top-rank.
// build: g++ -std=c++20 -O2 -I include -I /root/reference/proj/include -I <json> \
//   tools/probes/ga_phase_probe.cpp -L paper_1801_03039_b200 -lebic_b200 -Wl,-rpath,...
#include <chrono>
#include <cstdio>

#include "ebic/evolution.hpp"
#include "ebic/synthgen.hpp"

using namespace ebic;
using clk = std::chrono::steady_clock;

int main(int argc, char** argv) {
    const std::size_t rows = argc > 1 ? std::stoull(argv[1]) : 20000;
    const std::size_t cols = argc > 2 ? std::stoull(argv[2]) : 500;
    const std::size_t gens = argc > 3 ? std::stoull(argv[3]) : 50;
    ScenarioSpec spec;
    spec.n_rows = rows;
    spec.n_cols = cols;
    for (int b = 0; b < 5; ++b) spec.blocks.push_back({rows / 40, 20});
    spec.seed = 2026;
    auto ms = [](clk::time_point a, clk::time_point b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    const auto g0 = clk::now();
    const GeneratedScenario data = generate(spec);
    std::printf("{\"generate_ms\": %.1f}\n", ms(g0, clk::now()));
    const ExpressionMatrix& m = data.matrix;
    EvolutionConfig evo;
    evo.population_size = 600;
    FitnessParams params;
    params.sigma = default_sigma(rows);
    const ChunkPlan plan = make_chunk_plan(rows, 1);
    Rng rng(1);
    TabuList tabu(cols);
    TopRankList top(cols);
    ColumnPenaltyTable pen(cols);
    double t_build = 0, t_enc = 0, t_eval = 0, t_top = 0;
    auto pop = init_population(cols, evo, rng, tabu);
    const auto s0 = clk::now();
    int ndev = 0;
    ebic_device_count(&ndev);
    const auto s1 = clk::now();
    ebic_ctx* probe_ctx = nullptr;
    int dev0 = 0;
    ebic_ctx_create(m.values.data(), m.n_rows, m.n_cols, &dev0, 1, &probe_ctx);
    const auto s2 = clk::now();
    auto fit = evaluate_population(m, encode_population(pop), plan, params, 1e-9);
    const auto s3 = clk::now();
    auto fit2 = evaluate_population(m, encode_population(pop), plan, params, 1e-9);
    const auto s4 = clk::now();
    ebic_ctx_destroy(probe_ctx);
    std::printf("{\"startup_ms\": {\"cuda_init\": %.2f, \"ctx_create\": %.2f, \"first_evaluate(ctx+ranks)\": %.2f, \"second_evaluate\": %.3f}}\n",
                ms(s0, s1), ms(s1, s2), ms(s2, s3), ms(s3, s4));
    top.update(pop, fit, evo);
    for (std::size_t g = 1; g <= gens; ++g) {
        auto t0 = clk::now();
        GenerationResult nx = build_generation(pop, fit, top, tabu, pen, evo, cols, rng);
        auto t1 = clk::now();
        std::vector<double> nf = nx.elite_fitness;
        nf.resize(nx.individuals.size());
        std::span<const ColumnSeries> novel(nx.individuals.data() + nx.elite_count, nx.individuals.size() - nx.elite_count);
        const CbfPopulation cbf = encode_population(novel);
        auto t2 = clk::now();
        auto f = evaluate_population(m, cbf, plan, params, 1e-9);
        auto t3 = clk::now();
        std::copy(f.begin(), f.end(), nf.begin() + nx.elite_count);
        pop = std::move(nx.individuals);
        fit = std::move(nf);
        top.update(pop, fit, evo);
        auto t4 = clk::now();
        t_build += ms(t0, t1); t_enc += ms(t1, t2); t_eval += ms(t2, t3); t_top += ms(t3, t4);
    }
    std::printf("{\"rows\": %zu, \"gens\": %zu, \"ms_per_gen\": {\"build_generation\": %.4f, \"encode\": %.4f, "
                "\"evaluate\": %.4f, \"top_rank\": %.4f}}\n", rows, gens, t_build / gens, t_enc / gens,
                t_eval / gens, t_top / gens);
}
