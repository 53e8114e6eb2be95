#pragma once
// B200 drop-in for the reference's ebic/io.hpp
// (/root/reference/proj/include/ebic/io.hpp:1-237): result files, score
// files, the Steps 6-7 output filter and config parsing.  Same API and error
// texts.  SURVEY.md §8(f) row 4: with approximate rows on, a run's result
// file holds ~10^6 row indices and flags, and building them as a JSON DOM
// node by node dominated the output step.  write_biclusters_file here lets
// the JSON library lay out everything except those two arrays per
// bicluster, which it writes itself in the library's own array layout
// (learned once from the library: compact or one element per line).  The
// bytes are identical to the reference's `dump(2)`
// (tests/test_reference_unit.py::test_result_files_byte_identical).

#include "ebic/evolution.hpp"  // TopRankEntry (shadow)
#include "ebic/expansion.hpp"  // resolve / expand (shadow, GPU)
#include "ebic/metrics.hpp"    // CellRect, ScoreReport (reference)

#include <json.hpp>

#include <algorithm>
#include <charconv>
#include <cmath>
#include <fstream>
#include <iterator>
#include <map>
#include <stdexcept>
#include <string_view>

namespace ebic {
// :180-228 -- "key = value" lines ('#' starts a comment) or one flat JSON
// object; later keys win.
inline std::map<std::string, std::string> parse_config_text(const std::string& text) {
    std::map<std::string, std::string> kv;
    const std::size_t lead = text.find_first_not_of(" \t\r\n");
    if (lead != std::string::npos && text[lead] == '{') {
        const nlohmann::json doc = nlohmann::json::parse(text);
        if (!doc.is_object()) throw std::runtime_error("config JSON must be an object");
        for (const auto& [key, value] : doc.items()) kv[key] = value.is_string() ? value.get<std::string>() : value.dump();
        return kv;
    }
    auto strip = [](std::string_view s, const char* blanks) {
        const std::size_t b = s.find_first_not_of(blanks);
        if (b == std::string_view::npos) return std::string();
        return std::string(s.substr(b, s.find_last_not_of(blanks) - b + 1));
    };
    std::size_t number = 0;
    for (std::size_t from = 0; from <= text.size();) {
        std::size_t to = text.find('\n', from);
        if (to == std::string::npos) to = text.size();
        std::string_view raw(text.data() + from, to - from);
        from = to + 1;
        ++number;
        raw = raw.substr(0, raw.find('#'));
        const std::string line = strip(raw, " \t\r");
        if (line.empty()) continue;
        const std::size_t eq = line.find('=');
        if (eq == std::string::npos)
            throw std::runtime_error("config line " + std::to_string(number) + ": expected key = value");
        std::string key = strip(std::string_view(line).substr(0, eq), " \t");
        if (key.empty()) throw std::runtime_error("config line " + std::to_string(number) + ": empty key");
        kv[std::move(key)] = strip(std::string_view(line).substr(eq + 1), " \t");
    }
    return kv;
}

inline std::map<std::string, std::string> load_config_file(const std::string& path) {
    std::ifstream file(path);
    if (!file) throw std::runtime_error("cannot read config file " + path);
    const std::string text((std::istreambuf_iterator<char>(file)), std::istreambuf_iterator<char>());
    return parse_config_text(text);
}

// :128-143 -- best Eq. 1 score a signal-free background sustains: a series
// of length m keeps about n_rows / m! rows.
inline double null_fitness_plateau(std::size_t n_rows, std::uint64_t sigma) {
    const FitnessParams params{sigma};
    double plateau = 0.0;
    double m_factorial = 2.0;  // 2!
    for (std::size_t m = 2; m <= 20; ++m) {
        const auto rows = static_cast<std::uint64_t>(std::llround(static_cast<double>(n_rows) / m_factorial));
        plateau = std::max(plateau, fitness_score(rows, m, params));
        m_factorial *= static_cast<double>(m + 1);
    }
    return plateau;
}


// :145-162
struct OutputOptions {
    enum class Threshold : std::uint8_t { kAuto, kNone, kValue };
    Threshold threshold = Threshold::kAuto;
    double min_fitness = 0.0;
    std::size_t max_biclusters = 100;
};

inline double resolve_min_fitness(const OutputOptions& opts, std::size_t n_rows, std::uint64_t sigma) {
    if (opts.threshold == OutputOptions::Threshold::kAuto) return 2.0 * null_fitness_plateau(n_rows, sigma);
    if (opts.threshold == OutputOptions::Threshold::kValue) return opts.min_fitness;
    return 0.0;
}


// :164-178 -- threshold, cap, then exact rows and expansion per kept entry
// (both on the GPU through this repo's expansion.hpp).
inline std::vector<Bicluster> finalize_biclusters(std::span<const TopRankEntry> entries,
                                                  const ExpressionMatrix& matrix,
                                                  const ExpansionOptions& expansion, double epsilon,
                                                  const OutputOptions& output, std::uint64_t sigma) {
    const double floor = resolve_min_fitness(output, matrix.n_rows, sigma);
    std::vector<Bicluster> kept;
    for (const TopRankEntry& e : entries) {
        if (kept.size() >= output.max_biclusters) break;
        if (e.fitness < floor) continue;
        kept.push_back(expand_bicluster(matrix, resolve_bicluster(matrix, e.series, e.fitness, epsilon),
                                        expansion, epsilon));
    }
    return kept;
}


// :24-26 -- every number the tools write is rounded to six decimals.
inline double round6(double x) { return std::round(x * 1e6) / 1e6; }


// :28-42
inline const char* row_flag_name(RowFlag f) {
    if (f == RowFlag::kNegative) return "negative";
    if (f == RowFlag::kApproximate) return "approximate";
    return "exact";
}

inline RowFlag row_flag_from_name(const std::string& name) {
    static const std::pair<const char*, RowFlag> known[] = {
        {"exact", RowFlag::kExact}, {"negative", RowFlag::kNegative}, {"approximate", RowFlag::kApproximate}};
    for (const auto& [text, flag] : known)
        if (name == text) return flag;
    throw std::runtime_error("unknown row flag: " + name);
}


// :57-62
struct RunSummary {
    std::size_t generations = 0;
    std::uint64_t series_evaluated = 0;
    std::uint64_t sigma = 0;
    bool tabu_terminated = false;
};


// :44-55 -- one bicluster as a JSON object (keys sort as the library sorts).
inline nlohmann::json bicluster_to_json(const Bicluster& b) {
    nlohmann::json cols = nlohmann::json::array();
    for (const ColumnIndex c : b.series) cols.push_back(static_cast<std::size_t>(c));
    nlohmann::json flags = nlohmann::json::array();
    for (const RowFlag f : b.row_flags) flags.push_back(row_flag_name(f));
    nlohmann::json out;
    out["columns"] = std::move(cols);
    out["fitness"] = round6(b.fitness);
    out["row_flags"] = std::move(flags);
    out["rows"] = b.rows;
    return out;
}


// :109-126
inline nlohmann::json score_to_json(const ScoreReport& report) {
    auto rounded = [](const std::vector<double>& v) {
        nlohmann::json a = nlohmann::json::array();
        for (const double x : v) a.push_back(round6(x));
        return a;
    };
    nlohmann::json out;
    out["per_expected"] = rounded(report.per_expected);
    out["per_found"] = rounded(report.per_found);
    out["recovery"] = round6(report.recovery);
    out["relevance"] = round6(report.relevance);
    return out;
}

inline void write_score_file(const std::string& path, const ScoreReport& report) {
    std::ofstream file(path);
    if (!file) throw std::runtime_error("cannot write " + path);
    file << score_to_json(report).dump(2) << '\n';
}


namespace detail {

// How the JSON library pretty-prints a non-empty array at indent 0 (step 2):
// the text before the first element, between elements and after the last.
// At depth d every newline in them is followed by d more spaces.
struct ArrayLayout {
    std::string open, between, close;

    static ArrayLayout learn(const nlohmann::json& two_elements) {
        const std::string text = two_elements.dump(2);
        const std::string a = two_elements[0].dump(), b = two_elements[1].dump();
        const std::size_t at_a = text.find(a);
        const std::size_t at_b = text.rfind(b);
        ArrayLayout l;
        l.open = text.substr(0, at_a);
        l.between = text.substr(at_a + a.size(), at_b - at_a - a.size());
        l.close = text.substr(at_b + b.size());
        return l;
    }

    static void append_indented(std::string& out, const std::string& piece, std::size_t depth) {
        for (const char ch : piece) {
            out.push_back(ch);
            if (ch == '\n') out.append(depth, ' ');
        }
    }
};

inline const ArrayLayout& integer_layout() {
    static const ArrayLayout l = ArrayLayout::learn(nlohmann::json::array({std::size_t{1}, std::size_t{2}}));
    return l;
}

inline const ArrayLayout& string_layout() {
    static const ArrayLayout l = ArrayLayout::learn(nlohmann::json::array({"a", "b"}));
    return l;
}

// Appends `items` (already-formatted element texts produced by `emit`) as an
// array at `depth` in `layout`.
template <class Emit>
void append_array(std::string& out, std::size_t n, const ArrayLayout& layout, std::size_t depth, Emit&& emit) {
    if (n == 0) {
        out += "[]";
        return;
    }
    std::string between;
    ArrayLayout::append_indented(between, layout.between, depth);
    ArrayLayout::append_indented(out, layout.open, depth);
    emit(out, 0);
    for (std::size_t i = 1; i < n; ++i) {
        out += between;
        emit(out, i);
    }
    ArrayLayout::append_indented(out, layout.close, depth);
}

// Stand-in string for one bicluster's array in the document skeleton (the
// skeleton holds no other strings, and this one needs no JSON escaping).
inline std::string marker(const char* what, std::size_t i) {
    return std::string("@ebic_") + what + "_" + std::to_string(i) + "@";
}

}  // namespace detail


// :64-78 -- {"biclusters": [...], "run": {...}} as `dump(2)` lays it out.
// The library writes the document with a marker string in place of each
// bicluster's rows / row_flags; each marker is then replaced by the array,
// indented to the marker's line.
inline void write_biclusters_file(const std::string& path, std::span<const Bicluster> biclusters,
                                  const RunSummary* summary = nullptr) {
    nlohmann::json doc;
    doc["biclusters"] = nlohmann::json::array();
    for (std::size_t i = 0; i < biclusters.size(); ++i) {
        const Bicluster& b = biclusters[i];
        nlohmann::json cols = nlohmann::json::array();
        for (const ColumnIndex c : b.series) cols.push_back(static_cast<std::size_t>(c));
        nlohmann::json item;
        item["columns"] = std::move(cols);
        item["fitness"] = round6(b.fitness);
        item["row_flags"] = detail::marker("flags", i);
        item["rows"] = detail::marker("rows", i);
        doc["biclusters"].push_back(std::move(item));
    }
    if (summary != nullptr) {
        nlohmann::json run;
        run["generations"] = summary->generations;
        run["series_evaluated"] = summary->series_evaluated;
        run["sigma"] = summary->sigma;
        run["tabu_terminated"] = summary->tabu_terminated;
        doc["run"] = std::move(run);
    }
    const std::string skeleton = doc.dump(2);

    std::size_t total = skeleton.size() + 1;
    for (const Bicluster& b : biclusters) total += b.rows.size() * 24 + b.row_flags.size() * 32;
    std::string out;
    out.reserve(total);
    const detail::ArrayLayout& ints = detail::integer_layout();
    const detail::ArrayLayout& strs = detail::string_layout();
    std::size_t at = 0;
    for (std::size_t i = 0; i < biclusters.size(); ++i) {
        const Bicluster& b = biclusters[i];
        for (const bool rows : {false, true}) {  // key order: "row_flags" before "rows"
            const std::string quoted = "\"" + detail::marker(rows ? "rows" : "flags", i) + "\"";
            const std::size_t hit = skeleton.find(quoted, at);
            if (hit == std::string::npos) throw std::logic_error("result layout: marker not found");
            out.append(skeleton, at, hit - at);
            const std::size_t line = skeleton.rfind('\n', hit) + 1;
            const std::size_t depth = skeleton.find_first_not_of(' ', line) - line;
            if (rows) {
                detail::append_array(out, b.rows.size(), ints, depth, [&](std::string& o, std::size_t k) {
                    char digits[24];
                    const auto r = std::to_chars(digits, digits + sizeof digits, b.rows[k]);
                    o.append(digits, r.ptr);
                });
            } else {
                detail::append_array(out, b.row_flags.size(), strs, depth, [&](std::string& o, std::size_t k) {
                    o.push_back('"');
                    o += row_flag_name(b.row_flags[k]);
                    o.push_back('"');
                });
            }
            at = hit + quoted.size();
        }
    }
    out.append(skeleton, at, std::string::npos);
    out.push_back('\n');

    std::ofstream file(path, std::ios::binary);
    if (!file) throw std::runtime_error("cannot write " + path);
    file.write(out.data(), static_cast<std::streamsize>(out.size()));
}


// :80-88
inline void write_truth_file(const std::string& path, std::span<const CellRect> blocks) {
    nlohmann::json list = nlohmann::json::array();
    for (const CellRect& r : blocks) list.push_back({{"rows", r.rows}, {"columns", r.cols}});
    nlohmann::json doc;
    doc["biclusters"] = std::move(list);
    std::ofstream file(path);
    if (!file) throw std::runtime_error("cannot write " + path);
    file << doc.dump(2) << '\n';
}


// :90-107 -- row/column sets of a results or ground-truth file (a bare
// top-level array is accepted too).
inline std::vector<CellRect> read_rects_file(const std::string& path) {
    std::ifstream file(path);
    if (!file) throw std::runtime_error("cannot read " + path);
    nlohmann::json doc;
    file >> doc;
    const nlohmann::json& list = doc.is_array() ? doc : doc.at("biclusters");
    if (!list.is_array()) throw std::runtime_error("no bicluster array in " + path);
    std::vector<CellRect> rects;
    rects.reserve(list.size());
    for (const nlohmann::json& entry : list)
        rects.push_back(make_rect(entry.at("rows").get<std::vector<std::size_t>>(),
                                  entry.at("columns").get<std::vector<std::size_t>>()));
    return rects;
}

}  // namespace ebic
