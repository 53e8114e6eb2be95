#pragma once
// B200 drop-in for the reference's ebic/synthgen.hpp: SURVEY.md §8(f) row 3
// (matrix ingest).  Everything except `generate` is the reference's own code,
// pulled in unchanged with #include_next (the next `ebic/synthgen.hpp` on the
// include path, i.e. /root/reference/proj/include/ebic/synthgen.hpp); its
// `generate` is renamed while it is read, and stays in use for suite emission
// (emit_suite).  `generate` below draws the same matrix with
// ebic_synth_generate (paper_1801_03039_b200/csrc/synth.cpp: the background
// normals' engine outputs in order, the Box-Muller transforms on all host
// threads; bit-identical, checked by tests/test_capi_host.py and the
// reference's own test_synthgen.cpp) and the ground truth with the
// reference's block placement, which takes the first draws of the stream
// (synthgen.hpp:125-136).

// Everything the reference header includes comes first, so the rename below
// cannot reach a standard-library `generate`.
#include <algorithm>
#include <cstdint>
#include <filesystem>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

#include "ebic/io.hpp"
#include "ebic/matrix.hpp"
#include "ebic/metrics.hpp"
#include "ebic/rng.hpp"
#include "ebic_b200.h"

#define generate reference_generate
#include_next "ebic/synthgen.hpp"
#undef generate

namespace ebic {

// synthgen.hpp:114-223, same checks and messages, same bytes out.
inline GeneratedScenario generate(const ScenarioSpec& spec) {
    if (spec.n_rows == 0 || spec.n_cols == 0) throw std::invalid_argument("matrix shape must be positive");
    if (spec.noise_sd < 0.0) throw std::invalid_argument("noise_sd must be non-negative");
    const bool chained = spec.blocks.size() > 1;
    std::vector<std::size_t> heights, widths;
    for (const BlockShape& shape : spec.blocks) {
        const bool fits = shape.rows && shape.cols && shape.rows <= spec.n_rows && shape.cols <= spec.n_cols;
        if (!fits || (chained && (spec.overlap_rows >= shape.rows || spec.overlap_cols >= shape.cols)))
            throw std::runtime_error("scenario infeasible");
        heights.push_back(shape.rows);
        widths.push_back(shape.cols);
    }
    if (static_cast<int>(spec.pattern) > static_cast<int>(Pattern::kShiftScale))
        return reference_generate(spec);  // out-of-range enum value: whatever the reference does
    Rng placement(spec.seed);  // the stream's first draws: rows, then columns
    const auto rows = detail::place_blocks(spec.n_rows, spec.overlap_rows, heights, placement);
    const auto cols = detail::place_blocks(spec.n_cols, spec.overlap_cols, widths, placement);

    GeneratedScenario out;
    out.truth.reserve(spec.blocks.size());
    for (std::size_t b = 0; b < spec.blocks.size(); ++b) out.truth.push_back(make_rect(rows[b], cols[b]));
    out.matrix = ExpressionMatrix::with_shape(spec.n_rows, spec.n_cols);
    b200::check(ebic_synth_generate(spec.n_rows, spec.n_cols, spec.blocks.size(), heights.data(), widths.data(),
                                    static_cast<int>(spec.pattern), spec.overlap_rows, spec.overlap_cols,
                                    spec.noise_sd, spec.seed, out.matrix.values.data()));
    return out;
}

}  // namespace ebic
