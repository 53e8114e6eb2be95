// io_check.cpp -- TEST INFRASTRUCTURE ONLY.
//
// Exercises the io.hpp API (reference: /root/reference/proj/include/ebic/io.hpp)
// on deterministic inputs and prints / writes everything it produces.  Built
// twice by oracle/Makefile: io_check_ref (reference headers) and
// io_check_dropin (include/ebic/io.hpp shadow first).  The two runs must
// produce identical stdout and identical files (tests/test_reference_unit.py).
// usage: io_check <output directory>
#include <cstdio>
#include <random>
#include <string>

#include "ebic/io.hpp"

using namespace ebic;

static void emit(const char* tag, const std::string& s) { std::printf("== %s\n%s\n", tag, s.c_str()); }

int main(int argc, char** argv) {
    if (argc < 2) return 2;
    const std::string dir = argv[1];
    std::mt19937_64 g(77);
    auto uni = [&](std::size_t n) { return static_cast<std::size_t>(g() % n); };
    for (int set = 0; set < 6; ++set) {
        std::vector<Bicluster> bs;
        const std::size_t n = set == 0 ? 0 : 1 + uni(set < 3 ? 4 : 40);
        for (std::size_t i = 0; i < n; ++i) {
            Bicluster b;
            const std::size_t len = 2 + uni(8);
            for (std::size_t k = 0; k < len; ++k) b.series.push_back(static_cast<ColumnIndex>(uni(60000)));
            const std::size_t rows = (i % 5 == 3) ? 0 : uni(set == 5 ? 200000 : 300);
            std::size_t r = uni(10);
            for (std::size_t k = 0; k < rows; ++k) {
                b.rows.push_back(r);
                b.row_flags.push_back(static_cast<RowFlag>(uni(3)));
                r += 1 + uni(4);
            }
            const double fits[] = {0.0, 1.0, 29.086815449, 1e-7, 123456.7890125, 0.1 + 0.2, 3.0000005, 1e20};
            b.fitness = (i % 3 == 0) ? fits[uni(8)] : std::ldexp(static_cast<double>(g() >> 11), -40);
            bs.push_back(std::move(b));
        }
        RunSummary sum{uni(6000), g() % 100000000, 1 + uni(5000), (set % 2) == 1};
        write_biclusters_file(dir + "/result_" + std::to_string(set) + ".json", bs, set == 2 ? nullptr : &sum);
        if (!bs.empty()) emit("bicluster_to_json", bicluster_to_json(bs[0]).dump(2));
    }
    std::vector<CellRect> truth = {make_rect({3, 1, 2}, {9, 4}), make_rect({}, {1}), make_rect({7}, {})};
    write_truth_file(dir + "/truth.json", truth);
    for (const char* f : {"/truth.json", "/result_3.json"}) {
        std::string line;
        for (const CellRect& r : read_rects_file(dir + f)) {
            line += "rows";
            for (auto x : r.rows) line += " " + std::to_string(x);
            line += " cols";
            for (auto x : r.cols) line += " " + std::to_string(x);
            line += ";";
        }
        emit(f, line);
    }
    ScoreReport rep;
    rep.recovery = 0.123456789;
    rep.relevance = 2.0 / 3.0;
    rep.per_expected = {0.5, 1.0 / 3.0, 0.0};
    rep.per_found = {};
    emit("score", score_to_json(rep).dump(2));
    write_score_file(dir + "/score.json", rep);
    for (std::size_t rows : {0, 1, 500, 1000, 20000, 200000, 1234567})
        for (std::uint64_t sigma : {4, 10, 400, 4000}) {
            char buf[96];
            std::snprintf(buf, sizeof buf, "%zu %llu %.17g %.17g", rows, static_cast<unsigned long long>(sigma),
                          null_fitness_plateau(rows, sigma),
                          resolve_min_fitness(OutputOptions{}, rows, sigma));
            emit("plateau", buf);
        }
    OutputOptions none;
    none.threshold = OutputOptions::Threshold::kNone;
    OutputOptions val;
    val.threshold = OutputOptions::Threshold::kValue;
    val.min_fitness = 3.25;
    emit("thresholds", std::to_string(resolve_min_fitness(none, 10, 4)) + " " +
                           std::to_string(resolve_min_fitness(val, 10, 4)));
    const char* configs[] = {
        "population = 600\n# comment\n  iterations=5000  \nepsilon = 1e-9 # trailing\n\nkey = a = b\n",
        "{\"population\": 600, \"name\": \"x\", \"flag\": true, \"list\": [1, 2]}",
        "   \n\t{\"a\": {\"b\": 1}}",
        "a = 1\nbad line\n",
        " = 3\n",
        "[1, 2]",
        "a = 1\r\nb = 2\r\n",
        "",
    };
    for (const char* c : configs) {
        std::string line;
        try {
            for (const auto& [k, v] : parse_config_text(c)) line += "[" + k + "]=[" + v + "] ";
        } catch (const std::exception& e) {
            line = std::string("error: ") + e.what();
        }
        emit("config", line);
    }
    for (const char* name : {"exact", "negative", "approximate", "other"}) {
        try {
            emit("flag", row_flag_name(row_flag_from_name(name)));
        } catch (const std::exception& e) {
            emit("flag", e.what());
        }
    }
    try {
        load_config_file(dir + "/missing.cfg");
    } catch (const std::exception& e) {
        emit("missing config", e.what());
    }
    try {
        read_rects_file(dir + "/missing.json");
    } catch (const std::exception& e) {
        emit("missing rects", e.what());
    }
    return 0;
}
