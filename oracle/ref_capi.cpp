// ref_capi.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" wrapper that compiles the UNMODIFIED reference headers
// (/root/reference/proj/include/ebic/*.hpp, included from where they lie; no
// reference source is copied into this repository) into
// oracle/_ref/libebic_ref.so.  tests/ use it to pin the C restatement
// (oracle/ebic_oracle.c) and to produce golden vectors; bench.py uses it as
// the reference CPU arm (`--impl reference`, cpu_baseline kind "reference").
// Built by oracle/Makefile only when /root/reference is present.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <span>
#include <string>
#include <vector>

#include "ebic/ebic.hpp"

using namespace ebic;

namespace {

CbfPopulation make_cbf(const std::size_t* offsets, const std::uint16_t* cols, std::size_t n) {
    CbfPopulation pop;
    pop.offsets.assign(offsets, offsets + n + 1);
    pop.col_indices.assign(cols, cols + offsets[n]);
    return pop;
}

}  // namespace

extern "C" {

// ExpressionMatrix (inc/matrix.hpp:21-44) built from a row-major buffer.
void* ref_matrix_create(const double* values, std::size_t n_rows, std::size_t n_cols) {
    auto* m = new ExpressionMatrix(ExpressionMatrix::with_shape(n_rows, n_cols));
    std::memcpy(m->values.data(), values, n_rows * n_cols * sizeof(double));
    return m;
}

void ref_matrix_destroy(void* h) { delete static_cast<ExpressionMatrix*>(h); }

// inc/fitness.hpp:100-118 with make_chunk_plan(n_rows, workers) (:30-39).
int ref_count_matches(void* h, const std::size_t* offsets, const std::uint16_t* cols,
                      std::size_t n, double eps, unsigned workers, std::uint64_t* out) {
    const auto& m = *static_cast<ExpressionMatrix*>(h);
    try {
        const ChunkPlan plan = make_chunk_plan(m.n_rows, workers);
        const auto counts = count_matches(m, make_cbf(offsets, cols, n), plan, eps);
        std::copy(counts.begin(), counts.end(), out);
    } catch (...) {
        return -1;
    }
    return 0;
}

// inc/fitness.hpp:135-143.
int ref_evaluate_population(void* h, const std::size_t* offsets, const std::uint16_t* cols,
                            std::size_t n, std::uint64_t sigma, double eps, unsigned workers,
                            double* out) {
    const auto& m = *static_cast<ExpressionMatrix*>(h);
    try {
        const ChunkPlan plan = make_chunk_plan(m.n_rows, workers);
        const auto fit =
            evaluate_population(m, make_cbf(offsets, cols, n), plan, FitnessParams{sigma}, eps);
        std::copy(fit.begin(), fit.end(), out);
    } catch (...) {
        return -1;
    }
    return 0;
}

double ref_fitness_score(std::uint64_t count, std::size_t len, std::uint64_t sigma) {
    return fitness_score(count, len, FitnessParams{sigma});
}

std::uint64_t ref_default_sigma(std::size_t n_rows) { return default_sigma(n_rows); }

// inc/expansion.hpp:16-23.
std::size_t ref_assign_rows(void* h, const std::uint16_t* series, std::size_t len, double eps,
                            std::uint64_t* rows_out) {
    const auto& m = *static_cast<ExpressionMatrix*>(h);
    const auto rows = assign_rows(m, std::span<const ColumnIndex>(series, len), eps);
    std::copy(rows.begin(), rows.end(), rows_out);
    return rows.size();
}

// inc/expansion.hpp:56-87 applied to an arbitrary (ascending) core.
std::size_t ref_expand_bicluster(void* h, const std::uint16_t* series, std::size_t len,
                                 const std::uint64_t* core_rows, const std::uint8_t* core_flags,
                                 std::size_t n_core, int allow_negative, std::size_t approx_k,
                                 double eps, std::uint64_t* rows_out, std::uint8_t* flags_out) {
    const auto& m = *static_cast<ExpressionMatrix*>(h);
    Bicluster core;
    core.series.assign(series, series + len);
    core.rows.assign(core_rows, core_rows + n_core);
    for (std::size_t i = 0; i < n_core; ++i) core.row_flags.push_back(RowFlag(core_flags[i]));
    ExpansionOptions opts;
    opts.allow_negative = allow_negative != 0;
    opts.approx_violations = approx_k;
    const Bicluster out = expand_bicluster(m, core, opts, eps);
    for (std::size_t i = 0; i < out.rows.size(); ++i) {
        rows_out[i] = out.rows[i];
        flags_out[i] = static_cast<std::uint8_t>(out.row_flags[i]);
    }
    return out.rows.size();
}

// inc/synthgen.hpp:114-223.  Writes the row-major values (n_rows * n_cols).
int ref_generate(std::size_t n_rows, std::size_t n_cols, std::size_t n_blocks,
                 const std::size_t* block_rows, const std::size_t* block_cols, int pattern,
                 std::size_t overlap_rows, std::size_t overlap_cols, double noise_sd,
                 std::uint64_t seed, double* values_out) {
    ScenarioSpec spec;
    spec.n_rows = n_rows;
    spec.n_cols = n_cols;
    for (std::size_t i = 0; i < n_blocks; ++i) spec.blocks.push_back({block_rows[i], block_cols[i]});
    spec.pattern = static_cast<Pattern>(pattern);
    spec.overlap_rows = overlap_rows;
    spec.overlap_cols = overlap_cols;
    spec.noise_sd = noise_sd;
    spec.seed = seed;
    try {
        const GeneratedScenario g = generate(spec);
        std::memcpy(values_out, g.matrix.values.data(), n_rows * n_cols * sizeof(double));
    } catch (...) {
        return -1;
    }
    return 0;
}

std::uint64_t ref_derive_seed(std::uint64_t master, std::uint64_t index) {
    return Rng::derive_seed(master, index);
}

// Runs the reference GA (inc/evolution.hpp:464-520) and records every
// evaluated batch through RunHooks::on_evaluate (:483, :503) together with
// the reference's own count_matches result for it.  Trace file layout
// (little endian):  repeated { u64 P; u64 offsets[P+1]; u16 cols[offsets[P]];
// u64 counts[P] }.  Stops recording after max_batches batches (0 = all).
// Returns the number of recorded batches, or -1 on error.
long ref_run_trace(void* h, std::size_t population, std::size_t iterations, std::uint64_t rng_seed,
                   double eps, std::uint64_t sigma, unsigned threads, std::size_t max_batches,
                   const char* path) {
    const auto& m = *static_cast<ExpressionMatrix*>(h);
    std::FILE* f = std::fopen(path, "wb");
    if (!f) return -1;
    RunConfig cfg;
    cfg.evo.population_size = population;
    cfg.evo.max_iterations = iterations;
    cfg.evo.rng_seed = rng_seed;
    cfg.epsilon = eps;
    cfg.sigma = sigma;
    cfg.threads = threads;
    const ChunkPlan plan = make_chunk_plan(m.n_rows, threads);
    long recorded = 0;
    RunHooks hooks;
    hooks.on_evaluate = [&](std::span<const ColumnSeries> novel) {
        if (max_batches != 0 && static_cast<std::size_t>(recorded) >= max_batches) return;
        const CbfPopulation cbf = encode_population(novel);
        const auto counts = count_matches(m, cbf, plan, eps);
        const std::uint64_t p = cbf.size();
        std::fwrite(&p, sizeof p, 1, f);
        std::vector<std::uint64_t> off(cbf.offsets.begin(), cbf.offsets.end());
        std::fwrite(off.data(), sizeof(std::uint64_t), off.size(), f);
        std::fwrite(cbf.col_indices.data(), sizeof(std::uint16_t), cbf.col_indices.size(), f);
        std::fwrite(counts.data(), sizeof(std::uint64_t), counts.size(), f);
        ++recorded;
    };
    try {
        (void)run(m, cfg, hooks);
    } catch (...) {
        std::fclose(f);
        return -1;
    }
    std::fclose(f);
    return recorded;
}


// Same run, recording only selected batches: batch k (k = 0 is the initial
// population, k = g the novel children of generation g) is recorded iff
// k < record_first or (record_every && k % record_every == 0) -- early
// generations plus a sparse sample of the steady state up to `iterations`.
// Layout: repeated { u64 k; u64 P; u64 offsets[P+1]; u16 cols[]; u64 counts[P] }.
long ref_run_trace_sel(void* h, std::size_t population, std::size_t iterations, std::uint64_t rng_seed,
                       double eps, std::uint64_t sigma, unsigned threads, std::size_t record_first,
                       std::size_t record_every, const char* path) {
    const auto& m = *static_cast<ExpressionMatrix*>(h);
    std::FILE* f = std::fopen(path, "wb");
    if (!f) return -1;
    RunConfig cfg;
    cfg.evo.population_size = population;
    cfg.evo.max_iterations = iterations;
    cfg.evo.rng_seed = rng_seed;
    cfg.epsilon = eps;
    cfg.sigma = sigma;
    cfg.threads = threads;
    const ChunkPlan plan = make_chunk_plan(m.n_rows, threads);
    long recorded = 0;
    std::uint64_t k = 0;
    RunHooks hooks;
    hooks.on_evaluate = [&](std::span<const ColumnSeries> novel) {
        const std::uint64_t batch = k++;
        if (!(batch < record_first || (record_every && batch % record_every == 0))) return;
        const CbfPopulation cbf = encode_population(novel);
        const auto counts = count_matches(m, cbf, plan, eps);
        const std::uint64_t p = cbf.size();
        std::fwrite(&batch, sizeof batch, 1, f);
        std::fwrite(&p, sizeof p, 1, f);
        std::vector<std::uint64_t> off(cbf.offsets.begin(), cbf.offsets.end());
        std::fwrite(off.data(), sizeof(std::uint64_t), off.size(), f);
        std::fwrite(cbf.col_indices.data(), sizeof(std::uint16_t), cbf.col_indices.size(), f);
        std::fwrite(counts.data(), sizeof(std::uint64_t), counts.size(), f);
        ++recorded;
    };
    try {
        (void)run(m, cfg, hooks);
    } catch (...) {
        std::fclose(f);
        return -1;
    }
    std::fclose(f);
    return recorded;
}

// ---- fixture generators: the input streams of the reference's own tests ----

// proj/tests/acceptance_main.cpp:233-251 (property_match_counts): a 300x30
// matrix filled from Rng(1002).normal and 500 series from Rng(1003).
// values_out: 9000 doubles; offsets_out: 501; cols_out: capacity 3500.
void ref_fixture_acceptance_match_counts(double* values_out, std::size_t* offsets_out,
                                         std::uint16_t* cols_out) {
    Rng fill(1002);
    for (std::size_t i = 0; i < 300 * 30; ++i) values_out[i] = fill.normal(0.0, 1.0);
    Rng rng(1003);
    std::size_t at = 0;
    offsets_out[0] = 0;
    for (int i = 0; i < 500; ++i) {
        const std::size_t len = 2 + rng.index(5);
        ColumnSeries s;
        while (s.size() < len) {
            const ColumnIndex c = static_cast<ColumnIndex>(rng.index(30));
            if (std::find(s.begin(), s.end(), c) == s.end()) s.push_back(c);
        }
        for (ColumnIndex c : s) cols_out[at++] = c;
        offsets_out[i + 1] = at;
    }
}

// proj/tests/test_fitness.cpp:111-126 (chunk invariance): trial `trial` of the
// Rng(4242) stream.  Writes rows/cols/eps/n_series and the data; buffers sized
// for the maxima (124 x 22 values, 10 series x 6 columns).
void ref_fixture_fitness_trial(int trial, std::size_t* rows_out, std::size_t* cols_out,
                               double* eps_out, std::size_t* n_series_out, double* values_out,
                               std::size_t* offsets_out, std::uint16_t* series_cols_out) {
    Rng rng(4242);
    for (int t = 0; t <= trial; ++t) {
        const std::size_t rows = 5 + rng.index(120);
        const std::size_t cols = 3 + rng.index(20);
        ExpressionMatrix m = ExpressionMatrix::with_shape(rows, cols);
        for (double& v : m.values) v = rng.normal();
        const double epsilon = rng.chance(0.3) ? rng.real(0.0, 0.5) : 0.0;
        std::vector<ColumnSeries> series(1 + rng.index(10));
        for (ColumnSeries& s : series) {
            const std::size_t len = 2 + rng.index(std::min<std::size_t>(cols, 6) - 1);
            while (s.size() < len) {
                const auto col = static_cast<ColumnIndex>(rng.index(cols));
                if (std::find(s.begin(), s.end(), col) == s.end()) s.push_back(col);
            }
        }
        if (t != trial) continue;
        *rows_out = rows;
        *cols_out = cols;
        *eps_out = epsilon;
        *n_series_out = series.size();
        std::memcpy(values_out, m.values.data(), rows * cols * sizeof(double));
        std::size_t at = 0;
        offsets_out[0] = 0;
        for (std::size_t i = 0; i < series.size(); ++i) {
            for (ColumnIndex c : series[i]) series_cols_out[at++] = c;
            offsets_out[i + 1] = at;
        }
    }
}

// Matrix of Rng(seed).normal() draws, row-major (test_expansion.cpp:21-26).
void ref_fixture_random_matrix(std::size_t rows, std::size_t cols, std::uint64_t seed,
                               double* values_out) {
    Rng rng(seed);
    for (std::size_t i = 0; i < rows * cols; ++i) values_out[i] = rng.normal(0.0, 1.0);
}

// Runs the reference GA and records, per generation, the whole population and
// fitness vector that TopRankList::update receives (evolution.hpp:487, :513):
// gen 0 = the initial population; gen g = the elite clones of the previous
// top-rank list (build_generation, :394-402) followed by the novel series
// (on_evaluate, :503) with their evaluated fitness.  File layout: repeated
// { u64 P; u64 offsets[P+1]; u16 cols[offsets[P]]; f64 fitness[P] }.
long ref_run_population_trace(void* h, std::size_t population, std::size_t iterations,
                              std::uint64_t rng_seed, double eps, std::uint64_t sigma,
                              unsigned threads, const char* path) {
    const auto& m = *static_cast<ExpressionMatrix*>(h);
    std::FILE* f = std::fopen(path, "wb");
    if (!f) return -1;
    RunConfig cfg;
    cfg.evo.population_size = population;
    cfg.evo.max_iterations = iterations;
    cfg.evo.rng_seed = rng_seed;
    cfg.epsilon = eps;
    cfg.sigma = sigma;
    cfg.threads = threads;
    const ChunkPlan plan = make_chunk_plan(m.n_rows, threads);
    FitnessParams params;
    params.sigma = sigma != 0 ? sigma : default_sigma(m.n_rows);
    std::vector<TopRankEntry> prev_top;
    std::vector<ColumnSeries> novel;
    long recorded = 0;
    RunHooks hooks;
    hooks.on_evaluate = [&](std::span<const ColumnSeries> s) { novel.assign(s.begin(), s.end()); };
    hooks.on_generation = [&](std::size_t gen, const TopRankList& top) {
        std::vector<ColumnSeries> pop;
        std::vector<double> fit;
        if (gen > 0) {
            const std::size_t elites = std::min<std::size_t>(
                static_cast<std::size_t>(std::ceil(cfg.evo.elite_fraction * double(prev_top.size()))),
                population);
            for (std::size_t e = 0; e < elites; ++e) {
                pop.push_back(prev_top[e].series);
                fit.push_back(prev_top[e].fitness);
            }
        }
        if (!novel.empty()) {
            const auto nf = evaluate_population(m, encode_population(novel), plan, params, eps);
            pop.insert(pop.end(), novel.begin(), novel.end());
            fit.insert(fit.end(), nf.begin(), nf.end());
        }
        novel.clear();
        const CbfPopulation cbf = encode_population(pop);
        const std::uint64_t p = cbf.size();
        std::fwrite(&p, sizeof p, 1, f);
        std::vector<std::uint64_t> off(cbf.offsets.begin(), cbf.offsets.end());
        std::fwrite(off.data(), sizeof(std::uint64_t), off.size(), f);
        std::fwrite(cbf.col_indices.data(), sizeof(std::uint16_t), cbf.col_indices.size(), f);
        std::fwrite(fit.data(), sizeof(double), fit.size(), f);
        prev_top = top.entries();
        ++recorded;
    };
    try {
        (void)run(m, cfg, hooks);
    } catch (...) {
        std::fclose(f);
        return -1;
    }
    std::fclose(f);
    return recorded;
}

// ---- TopRankList (inc/evolution.hpp:142-218), driven through its public API ----

void* ref_toprank_create(std::size_t n_cols) { return new TopRankList(n_cols); }
void ref_toprank_destroy(void* h) { delete static_cast<TopRankList*>(h); }

// One TopRankList::update (:168-206) over a CBF population.
int ref_toprank_update(void* h, const std::size_t* offsets, const std::uint16_t* cols, std::size_t n,
                       const double* fitness, double overlap_threshold, std::size_t capacity) {
    auto& t = *static_cast<TopRankList*>(h);
    std::vector<ColumnSeries> pop;
    pop.reserve(n);
    for (std::size_t i = 0; i < n; ++i) pop.emplace_back(cols + offsets[i], cols + offsets[i + 1]);
    EvolutionConfig cfg;
    cfg.overlap_threshold = overlap_threshold;
    cfg.top_rank_capacity = capacity;
    t.update(pop, std::span<const double>(fitness, n), cfg);
    return 0;
}

std::size_t ref_toprank_size(void* h) { return static_cast<TopRankList*>(h)->size(); }

// entries() (:148) as CBF + fitness + seq; offsets_out has size()+1 slots,
// cols_out capacity = total columns (query with cols_out == nullptr).
std::size_t ref_toprank_entries(void* h, std::size_t* offsets_out, std::uint16_t* cols_out,
                                double* fitness_out, std::uint64_t* seq_out) {
    const auto& es = static_cast<TopRankList*>(h)->entries();
    std::size_t total = 0;
    for (std::size_t i = 0; i < es.size(); ++i) {
        if (offsets_out) offsets_out[i] = total;
        if (cols_out) std::copy(es[i].series.begin(), es[i].series.end(), cols_out + total);
        if (fitness_out) fitness_out[i] = es[i].fitness;
        if (seq_out) seq_out[i] = es[i].seq;
        total += es[i].series.size();
    }
    if (offsets_out) offsets_out[es.size()] = total;
    return total;
}

// Times n_updates TopRankList::update calls replaying a recorded sequence
// (the reference arm of the top-rank microbenchmark).  Populations are CBF
// slices pop_offsets[u]..; returns mean microseconds per update.
double ref_toprank_time(std::size_t n_cols, std::size_t n_updates, const std::size_t* pop_sizes,
                        const std::size_t* offsets, const std::uint16_t* cols, const double* fitness,
                        double overlap_threshold, std::size_t capacity, int reps) {
    std::vector<std::vector<ColumnSeries>> pops(n_updates);
    std::size_t s = 0;
    for (std::size_t u = 0; u < n_updates; ++u)
        for (std::size_t i = 0; i < pop_sizes[u]; ++i, ++s)
            pops[u].emplace_back(cols + offsets[s], cols + offsets[s + 1]);
    EvolutionConfig cfg;
    cfg.overlap_threshold = overlap_threshold;
    cfg.top_rank_capacity = capacity;
    double total = 0.0;
    for (int r = 0; r < reps; ++r) {
        TopRankList t(n_cols);
        std::size_t f0 = 0;
        const auto t0 = std::chrono::steady_clock::now();
        for (std::size_t u = 0; u < n_updates; ++u) {
            t.update(pops[u], std::span<const double>(fitness + f0, pop_sizes[u]), cfg);
            f0 += pop_sizes[u];
        }
        total += std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
    }
    return total / (double(reps) * double(n_updates));
}

}  // extern "C"
