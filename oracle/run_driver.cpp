// run_driver.cpp -- TEST INFRASTRUCTURE ONLY (drop-in proof).
//
// One end-to-end EBIC run written purely against the reference's public API:
// generate a scenario (inc/synthgen.hpp:114), run the GA (inc/evolution.hpp:464),
// finalize Steps 6-7 (inc/io.hpp:164) and write the results JSON
// (inc/io.hpp:64-78), mirroring `ebic run` (proj/tools/ebic_main.cpp:151-197).
//
// oracle/Makefile compiles this file twice from the same source:
//   oracle/_ref/ebic_ref_run     -I /root/reference/proj/include only
//                                (pure reference CPU path)
//   oracle/_ref/ebic_dropin_run  -I include  -I /root/reference/proj/include
//                                i.e. the repo's include/ebic/{fitness,expansion,
//                                evolution}.hpp shadow the reference's, so the
//                                GA loop, top-rank list and the reference's own
//                                finalize_biclusters() run on the B200 library.
// tests/test_gpu_dropin.py requires the two JSON files to be byte-identical.
//
// Prints the phase wall times (generate / run / finalize / write, ms) on stderr.
// Usage: run_driver key=value ... out=<path>
//   rows cols blocks=RxC[,RxC...] pattern overlap seed population iterations
//   rng_seed epsilon overlap_threshold threads sigma
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <sstream>
#include <string>

#include "ebic/ebic.hpp"

#ifndef EBIC_DRIVER_NAME
#define EBIC_DRIVER_NAME "reference"
#endif

using namespace ebic;

int main(int argc, char** argv) {
    std::map<std::string, std::string> kv = {
        {"rows", "500"},        {"cols", "100"},          {"blocks", "50x10,50x10,50x10"},
        {"pattern", "trend_preserving"}, {"overlap", "0"}, {"seed", "1"},
        {"noise", "0"},         {"population", "600"},    {"iterations", "1000"},
        {"rng_seed", "1"},      {"epsilon", "0"},         {"overlap_threshold", "0.75"},
        {"threads", "1"},       {"sigma", "0"},           {"allow_negative", "1"},
        {"approx", "1"},        {"threshold", "auto"},    {"out", "out.json"}};
    for (int i = 1; i < argc; ++i) {
        std::string a = argv[i];
        auto eq = a.find('=');
        if (eq == std::string::npos) {
            std::fprintf(stderr, "bad argument %s\n", argv[i]);
            return 2;
        }
        kv[a.substr(0, eq)] = a.substr(eq + 1);
    }
    try {
        ScenarioSpec spec;
        spec.n_rows = std::stoull(kv["rows"]);
        spec.n_cols = std::stoull(kv["cols"]);
        std::stringstream bs(kv["blocks"]);
        std::string item;
        while (std::getline(bs, item, ',')) {
            auto x = item.find('x');
            spec.blocks.push_back({std::stoull(item.substr(0, x)), std::stoull(item.substr(x + 1))});
        }
        spec.pattern = pattern_from_name(kv["pattern"]);
        spec.overlap_rows = spec.overlap_cols = std::stoull(kv["overlap"]);
        spec.noise_sd = std::stod(kv["noise"]);
        spec.seed = std::stoull(kv["seed"]);
        using clk = std::chrono::steady_clock;
        auto ms = [](clk::time_point a, clk::time_point b) {
            return std::chrono::duration<double, std::milli>(b - a).count();
        };
        const auto t0 = clk::now();
        const GeneratedScenario data = generate(spec);
        const auto t1 = clk::now();

        RunConfig cfg;
        cfg.evo.population_size = std::stoull(kv["population"]);
        cfg.evo.max_iterations = std::stoull(kv["iterations"]);
        cfg.evo.rng_seed = std::stoull(kv["rng_seed"]);
        cfg.evo.overlap_threshold = std::stod(kv["overlap_threshold"]);
        cfg.epsilon = std::stod(kv["epsilon"]);
        cfg.threads = static_cast<unsigned>(std::stoul(kv["threads"]));
        cfg.sigma = std::stoull(kv["sigma"]);
        // Time of the first generation callback: start-up (the drop-in's CUDA
        // context + matrix upload) and the initial population's evaluation.
        clk::time_point first{};
        RunHooks hooks;
        hooks.on_generation = [&](std::size_t, const TopRankList&) {
            if (first == clk::time_point{}) first = clk::now();
        };
        const RunResult result = run(data.matrix, cfg, hooks);
        const auto t2 = clk::now();
        if (first == clk::time_point{}) first = t2;

        ExpansionOptions exp;
        exp.allow_negative = kv["allow_negative"] != "0";
        exp.approx_violations = std::stoull(kv["approx"]);
        OutputOptions out_opts;
        if (kv["threshold"] == "none") out_opts.threshold = OutputOptions::Threshold::kNone;
        const std::vector<Bicluster> biclusters = finalize_biclusters(
            result.top_rank, data.matrix, exp, cfg.epsilon, out_opts, result.sigma_used);
        const auto t3 = clk::now();

        RunSummary summary;
        summary.generations = result.generations;
        summary.series_evaluated = result.series_evaluated;
        summary.sigma = result.sigma_used;
        summary.tabu_terminated = result.tabu_terminated;
        write_biclusters_file(kv["out"], biclusters, &summary);
        const auto t4 = clk::now();
        std::fprintf(stderr, "[%s] timing_ms generate=%.3f run=%.3f finalize=%.3f write=%.3f\n",
                     EBIC_DRIVER_NAME, ms(t0, t1), ms(t1, t2), ms(t2, t3), ms(t3, t4));
        std::fprintf(stderr, "[%s] run_ms to_first_generation=%.3f after=%.3f\n", EBIC_DRIVER_NAME,
                     ms(t1, first), ms(first, t2));
        std::fprintf(stderr, "[%s] generations=%zu series_evaluated=%llu biclusters=%zu\n",
                     EBIC_DRIVER_NAME, result.generations,
                     static_cast<unsigned long long>(result.series_evaluated), biclusters.size());
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
    return 0;
}
