// toprank.cpp -- exact top-rank admission (ebic_top_rank_update).
//
// Restates TopRankList::update (/root/reference/proj/include/ebic/evolution.hpp:168-206)
// with the same admission, eviction, sequence-number and tie semantics, but
// with no per-entry heap objects and no dense mask sweeps:
//
//   * an entry overlaps a candidate iff |cols(e) & cols(c)| / min(|e|, |c|) >
//     threshold (evolution.hpp:154-160).  For a threshold >= 0 (run() requires
//     (0, 1], evolution.hpp:48-49) an entry sharing no column never overlaps,
//     so only entries reachable through the candidate's columns need looking at.
//     Per-column posting lists (entry slots containing the column) give the
//     exact intersection sizes by counting, O(sum of posting lengths) per
//     candidate instead of O(entries x mask words);
//   * the "> threshold" test on the quotient is decided by a per-length integer
//     table need[m] = the least k with double(k)/double(m) > threshold,
//     evaluated with the very same double division, so the decision is
//     bit-for-bit the reference's;
//   * admission order (fitness desc, population index asc, :176-179), the
//     blocking test (>= fitness, :185-191), eviction (< fitness, :194-196),
//     sequence numbers (:197), the final (fitness desc, seq asc) order and the
//     truncation to capacity (:201-205) are kept exactly.  Every admitted
//     candidate consumes a sequence number even if truncated later, as in the
//     reference.
//
// The function is stateless: the caller passes the current entries and gets
// back the new list as references to old entries / candidates (see
// include/ebic_b200.h).  Host-only; never touches the GPU.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <vector>

#include "../../include/ebic_b200.h"

namespace ebic_b200_detail {
int set_error(int status, const char* msg);
}

namespace {

// Entry slots are held structure-of-arrays; posting lists are contiguous
// per-column arrays of slot ids (sequential scans, no pointer chasing).  Slots
// evicted during the update stay in the postings and are skipped by `alive`.
struct Workspace {
    std::vector<double> fit;
    std::vector<uint64_t> seq;
    std::vector<uint32_t> len;        // series length as stored (the reference's series.size())
    std::vector<int64_t> ref;         // >= 0: existing entry index; < 0: -(candidate + 1)
    std::vector<uint8_t> alive;
    std::vector<std::vector<int32_t>> post;  // per column: slots containing it
    std::vector<uint64_t> cnt;        // per slot: (visit << 32) | intersection with that candidate
    std::vector<int32_t> touched, all;
    std::vector<uint32_t> stamp;      // per column: last series that used it (dedupe)
    std::vector<uint32_t> need;       // per length: least overlapping intersection
    std::vector<uint16_t> distinct;
    std::vector<uint64_t> order, order_tmp;  // (high half of ~fitness bits, index)
};

Workspace& workspace() {
    static thread_local Workspace ws;
    return ws;
}

constexpr uint32_t kNever = std::numeric_limits<uint32_t>::max();

// Least k in [1, m] with double(k) / double(m) > thr (evolution.hpp:158-159);
// kNever if none (thr >= 1, or m == 0 where the reference divides 0 by 0).
uint32_t least_overlap(uint32_t m, double thr) {
    if (m == 0 || thr != thr) return kNever;  // 0/0 and "> NaN" are false
    const double dm = static_cast<double>(m);
    double guess = std::floor(thr * dm);
    uint32_t k = guess < 1.0 ? 1u : static_cast<uint32_t>(std::min(guess, dm));
    while (k > 1 && static_cast<double>(k - 1) / dm > thr) --k;
    while (k <= m && !(static_cast<double>(k) / dm > thr)) ++k;
    return k <= m ? k : kNever;
}

}  // namespace

extern "C" int ebic_top_rank_update(size_t n_cols, size_t n_entries, const size_t* entry_offsets,
                                    const uint16_t* entry_cols, const double* entry_fitness,
                                    const uint64_t* entry_seq, size_t n_cand, const size_t* cand_offsets,
                                    const uint16_t* cand_cols, const double* cand_fitness,
                                    double overlap_threshold, size_t capacity, uint64_t* next_seq,
                                    int64_t* out_ref, uint64_t* out_seq, size_t* out_count) {
    using ebic_b200_detail::set_error;
    if (!next_seq || !out_count || (capacity && n_entries + n_cand && (!out_ref || !out_seq)))
        return set_error(EBIC_ERR_INVALID_ARGUMENT, "ebic_top_rank_update: null output pointer");
    if (n_entries && (!entry_offsets || !entry_cols || !entry_fitness || !entry_seq))
        return set_error(EBIC_ERR_INVALID_ARGUMENT, "ebic_top_rank_update: null entry arrays");
    if (n_cand && (!cand_offsets || !cand_cols || !cand_fitness))
        return set_error(EBIC_ERR_INVALID_ARGUMENT, "ebic_top_rank_update: null candidate arrays");
    if (n_cols == 0 || n_cols > 65536) return set_error(EBIC_ERR_INVALID_ARGUMENT, "ebic_top_rank_update: bad n_cols");
    if (n_entries + n_cand > size_t(std::numeric_limits<int32_t>::max()))
        return set_error(EBIC_ERR_INVALID_ARGUMENT, "ebic_top_rank_update: too many series");
    for (int pass = 0; pass < 2; ++pass) {  // CBF sanity + column range (mask words, :210-213)
        const size_t n = pass ? n_cand : n_entries;
        const size_t* off = pass ? cand_offsets : entry_offsets;
        const uint16_t* cols = pass ? cand_cols : entry_cols;
        if (!n) continue;
        if (off[0] != 0) return set_error(EBIC_ERR_INVALID_ARGUMENT, "ebic_top_rank_update: offsets[0] != 0");
        for (size_t i = 0; i < n; ++i)
            if (off[i + 1] < off[i]) return set_error(EBIC_ERR_INVALID_ARGUMENT, "ebic_top_rank_update: offsets not monotone");
        for (size_t i = 0; i < off[n]; ++i)
            if (cols[i] >= n_cols) return set_error(EBIC_ERR_INVALID_ARGUMENT, "ebic_top_rank_update: column out of range");
    }

    Workspace& w = workspace();
    const size_t n_slots_max = n_entries + n_cand;
    w.fit.clear();
    w.seq.clear();
    w.len.clear();
    w.ref.clear();
    w.alive.clear();
    if (w.post.size() < n_cols) w.post.resize(n_cols);
    for (size_t c = 0; c < n_cols; ++c) w.post[c].clear();
    if (w.stamp.size() < n_cols) w.stamp.resize(n_cols);
    std::fill(w.stamp.begin(), w.stamp.begin() + n_cols, 0u);
    if (w.cnt.size() < n_slots_max) w.cnt.resize(n_slots_max);
    std::fill(w.cnt.begin(), w.cnt.begin() + n_slots_max, uint64_t{0});
    w.touched.resize(n_slots_max + 1);
    uint32_t stamp_id = 0;

    // need[m] for every length that can occur (min of two series lengths).
    size_t max_len = 0;
    for (size_t e = 0; e < n_entries; ++e) max_len = std::max(max_len, entry_offsets[e + 1] - entry_offsets[e]);
    for (size_t p = 0; p < n_cand; ++p) max_len = std::max(max_len, cand_offsets[p + 1] - cand_offsets[p]);
    w.need.resize(max_len + 1);
    for (size_t m = 0; m <= max_len; ++m) w.need[m] = least_overlap(uint32_t(m), overlap_threshold);

    // Distinct columns of one series, in first-occurrence order (mask semantics, :210-213).
    auto distinct_cols = [&](const uint16_t* c, size_t n) {
        ++stamp_id;
        w.distinct.clear();
        for (size_t i = 0; i < n; ++i)
            if (w.stamp[c[i]] != stamp_id) {
                w.stamp[c[i]] = stamp_id;
                w.distinct.push_back(c[i]);
            }
    };
    auto add_slot = [&](double f, uint64_t sq, uint32_t n, int64_t r) {
        const int32_t s = int32_t(w.fit.size());
        w.fit.push_back(f);
        w.seq.push_back(sq);
        w.len.push_back(n);
        w.ref.push_back(r);
        w.alive.push_back(1);
        for (uint16_t c : w.distinct) w.post[c].push_back(s);
    };

    for (size_t e = 0; e < n_entries; ++e) {
        const size_t n = entry_offsets[e + 1] - entry_offsets[e];
        distinct_cols(entry_cols + entry_offsets[e], n);
        add_slot(entry_fitness[e], entry_seq[e], uint32_t(n), int64_t(e));
    }

    // Visiting order: positive fitness only, fitness desc then index asc
    // (:172-179).  The bit pattern of a positive double orders like its value.
    // Keys are (high half of ~bits, index): a stable LSD radix sort over their
    // high 32 bits, then runs that tie there are finished by the full order
    // (equal fitness <=> equal bits for x > 0; such runs stay in index order).
    w.order.clear();
    for (size_t i = 0; i < n_cand; ++i)
        if (cand_fitness[i] > 0.0) {
            uint64_t bits;
            std::memcpy(&bits, &cand_fitness[i], sizeof bits);
            w.order.push_back(((~bits) & 0xffffffff00000000ull) | uint64_t(i));
        }
    w.order_tmp.resize(w.order.size());
    for (int shift = 32; shift < 64; shift += 8) {
        uint32_t hist[256] = {};
        for (const uint64_t o : w.order) ++hist[(o >> shift) & 0xff];
        if (hist[(w.order.empty() ? 0 : w.order[0] >> shift) & 0xff] == w.order.size()) continue;
        uint32_t at = 0;
        for (uint32_t& h : hist) {
            const uint32_t c = h;
            h = at;
            at += c;
        }
        for (const uint64_t o : w.order) w.order_tmp[hist[(o >> shift) & 0xff]++] = o;
        w.order.swap(w.order_tmp);
    }
    auto before = [&](uint64_t x, uint64_t y) {  // full visiting order
        const double fx = cand_fitness[uint32_t(x)], fy = cand_fitness[uint32_t(y)];
        return fx != fy ? fx > fy : uint32_t(x) < uint32_t(y);
    };
    for (size_t i = 1; i < w.order.size(); ++i) {  // insertion within tied runs
        const uint64_t x = w.order[i];
        size_t j = i;
        while (j > 0 && (w.order[j - 1] >> 32) == (x >> 32) && before(x, w.order[j - 1])) {
            w.order[j] = w.order[j - 1];
            --j;
        }
        w.order[j] = x;
    }

    // The reference does not validate the threshold here (run() does, :48-49).
    // For threshold >= 0 (or NaN) an entry sharing no column never overlaps
    // and the posting lists see every candidate pair that matters; a negative
    // threshold makes every pair of non-empty series overlap (0/m > thr), and
    // an empty series never does (0/0 is NaN).
    //
    // Intersection counts carry the candidate's visit number in their high
    // half, so they need no reset between candidates.  Entries that reach the
    // overlap bound with a lower fitness are noted as they are found and
    // evicted once the candidate is known to be admitted.
    const bool all_overlap = overlap_threshold < 0.0;
    const uint32_t* need = w.need.data();
    uint64_t next = *next_seq;
    uint64_t visit = 0;
    for (const uint64_t o : w.order) {
        const uint32_t p = uint32_t(o);
        const double f = cand_fitness[p];
        const size_t n = cand_offsets[p + 1] - cand_offsets[p];
        distinct_cols(cand_cols + cand_offsets[p], n);
        int32_t* lower = w.touched.data();  // overlapping entries of lower fitness
        size_t n_lower = 0;
        bool blocked = false;
        if (all_overlap) {
            const bool any = n > 0;
            for (size_t s = 0; s < w.fit.size() && any; ++s) {
                if (!w.alive[s] || w.len[s] == 0) continue;
                if (w.fit[s] >= f) {
                    blocked = true;
                    break;
                }
                lower[n_lower++] = int32_t(s);
            }
        } else {
            const uint64_t tag = ++visit << 32;
            uint64_t* cnt = w.cnt.data();
            const uint32_t* len = w.len.data();
            const uint8_t* alive = w.alive.data();
            const double* fit = w.fit.data();
            for (const uint16_t c : w.distinct) {
                for (const int32_t s : w.post[c]) {
                    const uint64_t v = cnt[s];
                    const uint64_t k = (v & 0xffffffff00000000ull) == tag ? v + 1 : tag + 1;
                    cnt[s] = k;
                    if (uint32_t(k) != need[std::min<size_t>(len[s], n)] || !alive[s]) continue;
                    if (fit[s] >= f) {
                        blocked = true;
                        break;
                    }
                    lower[n_lower++] = s;
                }
                if (blocked) break;
            }
        }
        if (!blocked) {  // evict overlapping lower-fitness entries (:194-196), admit (:197-198)
            for (size_t t = 0; t < n_lower; ++t) w.alive[lower[t]] = 0;
            add_slot(f, next++, uint32_t(n), -int64_t(p) - 1);
        }
    }
    *next_seq = next;

    // Final order (fitness desc, seq asc) and truncation (:201-205).  Slots
    // admitted here already come in that order with sequence numbers above
    // every entry's; when the entries do too (the list's own invariant) the
    // result is a merge, else a partial sort.
    auto first = [&](int32_t a, int32_t b) {
        if (w.fit[a] != w.fit[b]) return w.fit[a] > w.fit[b];
        return w.seq[a] < w.seq[b];
    };
    int32_t* old_alive = w.touched.data();
    int32_t* new_alive = old_alive + n_entries;
    size_t n_old = 0, n_new = 0;
    bool sorted = true;
    for (size_t s = 0; s < n_entries; ++s)
        if (w.alive[s]) {
            if (n_old && !first(old_alive[n_old - 1], int32_t(s))) sorted = false;
            old_alive[n_old++] = int32_t(s);
        }
    for (size_t s = n_entries; s < w.fit.size(); ++s)
        if (w.alive[s]) new_alive[n_new++] = int32_t(s);
    const size_t n_alive = n_old + n_new;
    const size_t keep = std::min(capacity, n_alive);
    if (sorted) {
        size_t i = 0, j = 0;
        for (size_t r = 0; r < keep; ++r) {
            const bool take_new = i == n_old || (j < n_new && first(new_alive[j], old_alive[i]));
            const int32_t s = take_new ? new_alive[j++] : old_alive[i++];
            out_ref[r] = w.ref[s];
            out_seq[r] = w.seq[s];
        }
    } else {
        std::vector<int32_t>& all = w.all;
        all.assign(old_alive, old_alive + n_old);
        all.insert(all.end(), new_alive, new_alive + n_new);
        std::partial_sort(all.begin(), all.begin() + keep, all.end(), first);
        for (size_t r = 0; r < keep; ++r) {
            out_ref[r] = w.ref[all[r]];
            out_seq[r] = w.seq[all[r]];
        }
    }
    *out_count = keep;
    return EBIC_OK;
}
