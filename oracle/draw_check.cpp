// draw_check.cpp -- TEST INFRASTRUCTURE ONLY.
//
// The shadow evolution.hpp draws bounded indices with detail::draw_index (a
// cached reciprocal instead of Rng::below's two 64-bit divisions,
// rng.hpp:20-32).  This checks it against the reference's Rng::index draw for
// draw over a sweep of bounds (small, 16-bit, random 64-bit, powers of two
// +-1, near 2^64), including that both leave the engine at the same state.
// Built by `make -C oracle unit` as oracle/_ref/draw_check; exit 0 = equal.
#include <cstdio>
#include <random>

#include "ebic/evolution.hpp"

int main() {
    std::mt19937_64 meta(5);
    unsigned long long mismatches = 0, draws = 0;
    for (int t = 0; t < 20000; ++t) {
        std::uint64_t bound = 0;
        switch (t % 5) {
            case 0: bound = 2 + meta() % 1000; break;
            case 1: bound = 2 + meta() % 70000; break;
            case 2: bound = (meta() >> (meta() % 64)) | 2; break;
            case 3: bound = (std::uint64_t{1} << (1 + meta() % 63)) + (meta() % 3) - 1; break;
            default: bound = ~std::uint64_t{0} - meta() % 1000; break;
        }
        if (bound < 1) bound = 1;
        const std::uint64_t seed = meta();
        ebic::Rng reference(seed), shadow(seed);
        for (int k = 0; k < 50; ++k, ++draws)
            mismatches += reference.index(bound) != ebic::detail::draw_index(shadow, bound);
        mismatches += reference.next() != shadow.next();
    }
    std::printf("{\"draws\": %llu, \"mismatches\": %llu}\n", draws, mismatches);
    return mismatches != 0;
}
