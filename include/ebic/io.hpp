#pragma once
// B200 drop-in for the reference's ebic/io.hpp (SURVEY.md §8(f) row 4,
// result output; row a17, finalize_biclusters).  Everything except two
// functions is the reference's own code, read unchanged with #include_next
// (the next `ebic/io.hpp` on the include path, i.e.
// /root/reference/proj/include/ebic/io.hpp); the two are renamed while it is
// read and replaced below:
//
//  * finalize_biclusters (io.hpp:164-178): the same threshold and cap, then
//    the exact rows and the expansion of every kept entry in ONE membership
//    launch (ebic_resolve_expand_batch: exact / reversed / violation
//    bitmasks of all kept series in one pass over the rows) instead of two
//    launches per entry.
//  * write_biclusters_file (io.hpp:64-78): with approximate rows on, a result
//    file holds ~10^6 row indices and flags, and building them as a JSON DOM
//    node by node dominated the output step.  Here the JSON library lays out
//    everything except those two arrays per bicluster, which are written
//    directly in the library's own array layout (learned once from the
//    library: compact or one element per line).  The bytes are identical to
//    the reference's `dump(2)` (oracle/io_check.cpp,
//    tests/test_reference_unit.py::test_result_files_byte_identical).

// Everything the reference header includes comes first, so the renames below
// reach only the reference's two definitions.
#include <algorithm>
#include <cctype>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <fstream>
#include <map>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include <json.hpp>

#include "ebic/bicluster.hpp"
#include "ebic/evolution.hpp"  // shadow
#include "ebic/expansion.hpp"  // shadow
#include "ebic/fitness.hpp"    // shadow
#include "ebic/matrix.hpp"
#include "ebic/metrics.hpp"

#define finalize_biclusters reference_finalize_biclusters
#define write_biclusters_file reference_write_biclusters_file
#include_next "ebic/io.hpp"
#undef write_biclusters_file
#undef finalize_biclusters

namespace ebic {

// io.hpp:164-178 -- same filter and cap; rows of all kept entries from one
// batched membership launch, flagged with the reference's precedence
// (exact core, then negative, then approximate; expansion.hpp:56-87).
inline std::vector<Bicluster> finalize_biclusters(std::span<const TopRankEntry> entries,
                                                  const ExpressionMatrix& matrix,
                                                  const ExpansionOptions& expansion, double epsilon,
                                                  const OutputOptions& output, std::uint64_t sigma) {
    const double min_fitness = resolve_min_fitness(output, matrix.n_rows, sigma);
    std::vector<const TopRankEntry*> kept;
    for (const TopRankEntry& entry : entries) {
        if (kept.size() >= output.max_biclusters) break;
        if (entry.fitness >= min_fitness) kept.push_back(&entry);
    }
    std::vector<Bicluster> out(kept.size());
    if (kept.empty()) return out;
    std::vector<std::size_t> offsets{0};
    std::vector<ColumnIndex> cols;
    for (const TopRankEntry* e : kept) {
        cols.insert(cols.end(), e->series.begin(), e->series.end());
        offsets.push_back(cols.size());
    }
    const b200::MatrixScope scope(matrix);
    std::vector<std::uint64_t> rows(kept.size() * matrix.n_rows);
    std::vector<std::uint8_t> flags(rows.size());
    std::vector<std::size_t> counts(kept.size());
    b200::check(ebic_resolve_expand_batch(b200::context_for(matrix)->ctx, offsets.data(), cols.data(),
                                          kept.size(), expansion.allow_negative ? 1 : 0,
                                          expansion.approx_violations, epsilon, rows.data(),
                                          flags.data(), counts.data()));
    std::size_t at = 0;
    for (std::size_t i = 0; i < kept.size(); ++i) {
        Bicluster& b = out[i];
        b.series = kept[i]->series;
        b.fitness = kept[i]->fitness;
        b.rows.assign(rows.begin() + static_cast<std::ptrdiff_t>(at),
                      rows.begin() + static_cast<std::ptrdiff_t>(at + counts[i]));
        b.row_flags.reserve(counts[i]);
        for (std::size_t k = at; k < at + counts[i]; ++k) b.row_flags.push_back(static_cast<RowFlag>(flags[k]));
        at += counts[i];
    }
    return out;
}

namespace b200_io {

// How the JSON library pretty-prints a non-empty array at indent 0 (step 2):
// the text before the first element, between elements and after the last.
// At depth d every newline in them is followed by d more spaces.
struct ArrayLayout {
    std::string open, between, close;

    static ArrayLayout of(const nlohmann::json& pair) {
        const std::string text = pair.dump(2);
        const std::string first = pair[0].dump(), second = pair[1].dump();
        const std::size_t a = text.find(first), b = text.rfind(second);
        return {text.substr(0, a), text.substr(a + first.size(), b - a - first.size()),
                text.substr(b + second.size())};
    }
};

inline void put_indented(std::string& out, const std::string& piece, std::size_t depth) {
    for (const char ch : piece) {
        out.push_back(ch);
        if (ch == '\n') out.append(depth, ' ');
    }
}

// n elements formatted by put(out, k), in `layout`, nested `depth` deep.
template <class Put>
void put_array(std::string& out, std::size_t n, const ArrayLayout& layout, std::size_t depth, Put&& put) {
    if (n == 0) {
        out += "[]";
        return;
    }
    std::string sep;
    put_indented(sep, layout.between, depth);
    put_indented(out, layout.open, depth);
    for (std::size_t k = 0; k < n; ++k) {
        if (k) out += sep;
        put(out, k);
    }
    put_indented(out, layout.close, depth);
}

// Placeholder string for one bicluster's array in the document skeleton
// (no JSON escaping needed; no other string in the skeleton looks like it).
inline std::string placeholder(bool rows, std::size_t i) {
    return std::string(rows ? "@ebic_rows_" : "@ebic_flags_") + std::to_string(i) + "@";
}

}  // namespace b200_io

// io.hpp:64-78 -- {"biclusters": [...], "run": {...}} exactly as the
// reference's bicluster_to_json + dump(2) lays it out: the library writes the
// skeleton with a placeholder in place of each bicluster's row_flags / rows,
// and each placeholder is replaced by its array, indented to its line.
inline void write_biclusters_file(const std::string& path, std::span<const Bicluster> biclusters,
                                  const RunSummary* summary = nullptr) {
    nlohmann::json doc;
    doc["biclusters"] = nlohmann::json::array();
    for (std::size_t i = 0; i < biclusters.size(); ++i) {
        Bicluster head;  // columns + fitness through the reference's own formatter
        head.series = biclusters[i].series;
        head.fitness = biclusters[i].fitness;
        nlohmann::json item = bicluster_to_json(head);
        item["row_flags"] = b200_io::placeholder(false, i);
        item["rows"] = b200_io::placeholder(true, i);
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
    static const b200_io::ArrayLayout ints =
        b200_io::ArrayLayout::of(nlohmann::json::array({std::size_t{1}, std::size_t{2}}));
    static const b200_io::ArrayLayout strs = b200_io::ArrayLayout::of(nlohmann::json::array({"a", "b"}));

    std::size_t bytes = skeleton.size() + 1;
    for (const Bicluster& b : biclusters) bytes += b.rows.size() * 24 + b.row_flags.size() * 32;
    std::string text;
    text.reserve(bytes);
    std::size_t at = 0;
    for (std::size_t i = 0; i < biclusters.size(); ++i) {
        const Bicluster& b = biclusters[i];
        for (const bool rows : {false, true}) {  // the library sorts "row_flags" before "rows"
            const std::string quoted = "\"" + b200_io::placeholder(rows, i) + "\"";
            const std::size_t hit = skeleton.find(quoted, at);
            if (hit == std::string::npos) throw std::logic_error("result layout: placeholder not found");
            text.append(skeleton, at, hit - at);
            const std::size_t line = skeleton.rfind('\n', hit) + 1;
            const std::size_t depth = skeleton.find_first_not_of(' ', line) - line;
            if (rows) {
                b200_io::put_array(text, b.rows.size(), ints, depth, [&](std::string& o, std::size_t k) {
                    char digits[24];
                    o.append(digits, std::to_chars(digits, digits + sizeof digits, b.rows[k]).ptr);
                });
            } else {
                b200_io::put_array(text, b.row_flags.size(), strs, depth, [&](std::string& o, std::size_t k) {
                    o.push_back('"');
                    o += row_flag_name(b.row_flags[k]);
                    o.push_back('"');
                });
            }
            at = hit + quoted.size();
        }
    }
    text.append(skeleton, at, std::string::npos);
    text.push_back('\n');

    std::ofstream file(path, std::ios::binary);
    if (!file) throw std::runtime_error("cannot write " + path);
    file.write(text.data(), static_cast<std::streamsize>(text.size()));
}

}  // namespace ebic
