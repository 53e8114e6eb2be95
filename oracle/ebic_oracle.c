/*
 * ebic_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, single-threaded restatement of the reference EBIC fitness
 * evaluation hot path (/root/reference/proj/include/ebic/fitness.hpp and
 * expansion.hpp).  It is the parity checker for the CUDA product path and
 * the "port" CPU baseline; it is never linked into, called by, or shipped
 * with the product library (paper_1801_03039_b200/libebic_b200.so).  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg load it.
 *
 * Parity pinning: the restatement is checked against (a) the reference's own
 * known-answer tests restated in tests/test_oracle_golden.py and (b) golden
 * vectors produced by the reference headers themselves, compiled here into
 * oracle/_ref/ by oracle/Makefile (tests/golden/make_golden.py).
 *
 * Every function cites the reference lines it follows.
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_EXPORT __attribute__((visibility("default")))

/* fitness.hpp:48-52 -- sigma = max(ceil(n_rows / 50), 4). */
ORC_EXPORT uint64_t orc_default_sigma(size_t n_rows) {
    uint64_t scaled = (uint64_t)((n_rows + 49) / 50);
    return scaled < 4 ? 4 : scaled;
}

/* fitness.hpp:57-67 -- strict increase along the series with epsilon slack.
 * The predicate is kept in the reference's NaN-sensitive form
 * !(prev < cur + eps), evaluated in IEEE fp64 (no reassociation). */
ORC_EXPORT int orc_row_matches(const double* values, size_t n_cols, size_t row,
                               const uint16_t* series, size_t len, double eps) {
    const double* v = values + row * n_cols;
    double prev = v[series[0]];
    for (size_t i = 1; i < len; ++i) {
        const double cur = v[series[i]];
        if (!(prev < cur + eps)) return 0;
        prev = cur;
    }
    return 1;
}

/* fitness.hpp:71-93 (detail::count_chunk): rows outer, population inner,
 * early exit, out[p] += ok. */
static void count_chunk(const double* values, size_t n_cols, size_t lo, size_t hi,
                        const size_t* off, const uint16_t* cols, size_t n, double eps,
                        uint64_t* out) {
    for (size_t r = lo; r < hi; ++r) {
        const double* v = values + r * n_cols;
        for (size_t p = 0; p < n; ++p) {
            const size_t end = off[p + 1];
            double prev = v[cols[off[p]]];
            int ok = 1;
            for (size_t i = off[p] + 1; i < end; ++i) {
                const double cur = v[cols[i]];
                if (!(prev < cur + eps)) {
                    ok = 0;
                    break;
                }
                prev = cur;
            }
            out[p] += (uint64_t)ok;
        }
    }
}

/* fitness.hpp:30-39 (make_chunk_plan) + :100-118 (count_matches): contiguous
 * chunks of ceil(n_rows / workers) rows, private partial counts, summed in
 * chunk order.  Runs the chunks serially (integer sums make the result
 * partition invariant, fitness.hpp:17-19).  Returns -1 for n_rows == 0
 * ("matrix has no rows", fitness.hpp:31). */
ORC_EXPORT int orc_count_matches(const double* values, size_t n_rows, size_t n_cols,
                                 const size_t* offsets, const uint16_t* cols, size_t n_series,
                                 double eps, unsigned workers, uint64_t* counts_out) {
    if (n_rows == 0) return -1;
    if (workers == 0) workers = 1;
    for (size_t p = 0; p < n_series; ++p) counts_out[p] = 0;
    if (n_series == 0) return 0;
    const size_t chunk = (n_rows + workers - 1) / workers;
    uint64_t* partial = (uint64_t*)calloc(n_series, sizeof(uint64_t));
    if (!partial) return -2;
    for (size_t lo = 0; lo < n_rows; lo += chunk) {
        const size_t hi = lo + chunk < n_rows ? lo + chunk : n_rows;
        memset(partial, 0, n_series * sizeof(uint64_t));
        count_chunk(values, n_cols, lo, hi, offsets, cols, n_series, eps, partial);
        for (size_t p = 0; p < n_series; ++p) counts_out[p] += partial[p];
    }
    free(partial);
    return 0;
}

/* fitness.hpp:124-133 -- Eq. 1 with the same libm calls (glibc log, exp2). */
ORC_EXPORT double orc_fitness_score(uint64_t match_count, size_t series_len, uint64_t sigma) {
    if (match_count <= 1) return 0.0;
    double f = (double)series_len * log((double)(match_count - 1));
    if (match_count < sigma) f *= exp2((double)match_count - (double)sigma);
    return f > 0.0 ? f : 0.0;
}

/* fitness.hpp:135-143 -- counts, then Eq. 1 with len = off[p+1] - off[p]. */
ORC_EXPORT int orc_evaluate_population(const double* values, size_t n_rows, size_t n_cols,
                                       const size_t* offsets, const uint16_t* cols,
                                       size_t n_series, double eps, uint64_t sigma,
                                       unsigned workers, uint64_t* counts_out,
                                       double* fitness_out) {
    int rc = orc_count_matches(values, n_rows, n_cols, offsets, cols, n_series, eps, workers,
                               counts_out);
    if (rc != 0) return rc;
    for (size_t p = 0; p < n_series; ++p)
        fitness_out[p] = orc_fitness_score(counts_out[p], offsets[p + 1] - offsets[p], sigma);
    return 0;
}

/* expansion.hpp:26-33 -- failing adjacent pairs, no early exit. */
ORC_EXPORT size_t orc_trend_violations(const double* values, size_t n_cols, size_t row,
                                       const uint16_t* series, size_t len, double eps) {
    const double* v = values + row * n_cols;
    size_t violations = 0;
    for (size_t i = 1; i < len; ++i)
        if (!(v[series[i - 1]] < v[series[i]] + eps)) ++violations;
    return violations;
}

/* expansion.hpp:16-23 (assign_rows): ascending matching rows.  Returns the
 * number written to rows_out (capacity n_rows). */
ORC_EXPORT size_t orc_assign_rows(const double* values, size_t n_rows, size_t n_cols,
                                  const uint16_t* series, size_t len, double eps,
                                  uint64_t* rows_out) {
    size_t n = 0;
    for (size_t r = 0; r < n_rows; ++r)
        if (orc_row_matches(values, n_cols, r, series, len, eps)) rows_out[n++] = r;
    return n;
}

/* Per-row membership classes used by the product's membership kernel,
 * stated directly from expansion.hpp: bit r of word r/64 is set in
 *   exact_bits  iff row_matches(series)            (expansion.hpp:21)
 *   neg_bits    iff row_matches(reversed series)   (expansion.hpp:58,64)
 *   approx_bits iff trend_violations(series) <= k  (expansion.hpp:66-67)
 * Each bitmask holds ceil(n_rows / 64) words. */
ORC_EXPORT void orc_membership_bits(const double* values, size_t n_rows, size_t n_cols,
                                    const uint16_t* series, size_t len, double eps,
                                    size_t approx_k, uint64_t* exact_bits, uint64_t* neg_bits,
                                    uint64_t* approx_bits) {
    const size_t words = (n_rows + 63) / 64;
    uint16_t* rev = (uint16_t*)malloc((len ? len : 1) * sizeof(uint16_t));
    for (size_t i = 0; i < len; ++i) rev[i] = series[len - 1 - i];
    for (size_t w = 0; w < words; ++w) exact_bits[w] = neg_bits[w] = approx_bits[w] = 0;
    for (size_t r = 0; r < n_rows; ++r) {
        const uint64_t bit = (uint64_t)1 << (r % 64);
        if (orc_row_matches(values, n_cols, r, series, len, eps)) exact_bits[r / 64] |= bit;
        if (orc_row_matches(values, n_cols, r, rev, len, eps)) neg_bits[r / 64] |= bit;
        if (orc_trend_violations(values, n_cols, r, series, len, eps) <= approx_k)
            approx_bits[r / 64] |= bit;
    }
    free(rev);
}

static int find_sorted(const uint64_t* a, size_t n, uint64_t x) {
    size_t lo = 0, hi = n;
    while (lo < hi) {
        size_t mid = lo + (hi - lo) / 2;
        if (a[mid] < x) lo = mid + 1;
        else hi = mid;
    }
    return lo < n && a[lo] == x;
}

/* expansion.hpp:56-87 (expand_bicluster).  core_rows/core_flags: the input
 * bicluster's ascending rows and flags.  Rows not in the core get exactly one
 * flag: negative (1) if allow_negative and the reversed series matches,
 * else approximate (2) if approx_k > 0 and violations <= approx_k.  Output is
 * merged and ordered by row (rows_out/flags_out capacity n_rows + n_core);
 * returns the number of rows written. */
ORC_EXPORT size_t orc_expand_bicluster(const double* values, size_t n_rows, size_t n_cols,
                                       const uint16_t* series, size_t len,
                                       const uint64_t* core_rows, const uint8_t* core_flags,
                                       size_t n_core, int allow_negative, size_t approx_k,
                                       double eps, uint64_t* rows_out, uint8_t* flags_out) {
    uint16_t* rev = (uint16_t*)malloc((len ? len : 1) * sizeof(uint16_t));
    for (size_t i = 0; i < len; ++i) rev[i] = series[len - 1 - i];
    size_t n = 0, ci = 0;
    for (size_t r = 0; r < n_rows; ++r) {
        /* Merge the (already ordered) core rows in front of row r. */
        while (ci < n_core && core_rows[ci] <= r) {
            rows_out[n] = core_rows[ci];
            flags_out[n] = core_flags[ci];
            ++n;
            ++ci;
        }
        if (find_sorted(core_rows, n_core, r)) continue;
        if (allow_negative && orc_row_matches(values, n_cols, r, rev, len, eps)) {
            rows_out[n] = r;
            flags_out[n] = 1;
            ++n;
        } else if (approx_k > 0 &&
                   orc_trend_violations(values, n_cols, r, series, len, eps) <= approx_k) {
            rows_out[n] = r;
            flags_out[n] = 2;
            ++n;
        }
    }
    while (ci < n_core) {
        rows_out[n] = core_rows[ci];
        flags_out[n] = core_flags[ci];
        ++n;
        ++ci;
    }
    free(rev);
    return n;
}

/* ---- top-rank admission (evolution.hpp:132-218, TopRankList) ----------- */

typedef struct {
    int64_t ref;     /* >= 0 entry index, < 0 -(candidate + 1) */
    double fitness;
    uint64_t seq;
    size_t len;      /* series.size() */
    uint64_t* mask;  /* column mask, (n_cols + 63) / 64 words (:208-213) */
} orc_tr_entry;

static const double* g_tr_fit; /* qsort context (single-threaded oracle) */

/* :176-179 -- fitness desc, then population index asc. */
static int orc_tr_order_cmp(const void* a, const void* b) {
    size_t x = *(const size_t*)a, y = *(const size_t*)b;
    if (g_tr_fit[x] != g_tr_fit[y]) return g_tr_fit[x] > g_tr_fit[y] ? -1 : 1;
    return x < y ? -1 : (x > y);
}

/* :201-204 -- fitness desc, then seq asc. */
static int orc_tr_entry_cmp(const void* a, const void* b) {
    const orc_tr_entry* x = (const orc_tr_entry*)a;
    const orc_tr_entry* y = (const orc_tr_entry*)b;
    if (x->fitness != y->fitness) return x->fitness > y->fitness ? -1 : 1;
    return x->seq < y->seq ? -1 : (x->seq > y->seq);
}

/* :154-160 -- shared columns as a fraction of the smaller series. */
static double orc_tr_overlap(const orc_tr_entry* a, const orc_tr_entry* b, size_t words) {
    uint64_t inter = 0;
    for (size_t w = 0; w < words; ++w) inter += (uint64_t)__builtin_popcountll(a->mask[w] & b->mask[w]);
    size_t m = a->len < b->len ? a->len : b->len;
    return (double)inter / (double)m;
}

static void orc_tr_fill(orc_tr_entry* e, const uint16_t* cols, size_t len, size_t words) {
    e->len = len;
    e->mask = (uint64_t*)calloc(words ? words : 1, sizeof(uint64_t));
    for (size_t i = 0; i < len; ++i) e->mask[cols[i] / 64] |= (uint64_t)1 << (cols[i] % 64);
}

/* evolution.hpp:168-206 (TopRankList::update) in the stateless form of
 * ebic_top_rank_update (include/ebic_b200.h): the list starts as the given
 * entries in the given order; output out_ref/out_seq in final order. */
ORC_EXPORT int orc_top_rank_update(size_t n_cols, size_t n_entries, const size_t* eoff,
                                   const uint16_t* ecols, const double* efit, const uint64_t* eseq,
                                   size_t n_cand, const size_t* coff, const uint16_t* ccols,
                                   const double* cfit, double thr, size_t capacity,
                                   uint64_t* next_seq, int64_t* out_ref, uint64_t* out_seq,
                                   size_t* out_count) {
    size_t words = (n_cols + 63) / 64;
    orc_tr_entry* list = (orc_tr_entry*)malloc((n_entries + n_cand + 1) * sizeof(orc_tr_entry));
    size_t n = 0;
    for (size_t e = 0; e < n_entries; ++e, ++n) {
        list[n].ref = (int64_t)e;
        list[n].fitness = efit[e];
        list[n].seq = eseq[e];
        orc_tr_fill(&list[n], ecols + eoff[e], eoff[e + 1] - eoff[e], words);
    }
    size_t* order = (size_t*)malloc((n_cand + 1) * sizeof(size_t));
    size_t n_order = 0;
    for (size_t i = 0; i < n_cand; ++i)
        if (cfit[i] > 0.0) order[n_order++] = i; /* :172-175 */
    g_tr_fit = cfit;
    qsort(order, n_order, sizeof(size_t), orc_tr_order_cmp);

    for (size_t k = 0; k < n_order; ++k) {
        size_t i = order[k];
        orc_tr_entry cand;
        cand.ref = -(int64_t)i - 1;
        cand.fitness = cfit[i];
        orc_tr_fill(&cand, ccols + coff[i], coff[i + 1] - coff[i], words);
        int blocked = 0; /* :185-192 */
        for (size_t e = 0; e < n && !blocked; ++e)
            if (list[e].fitness >= cand.fitness && orc_tr_overlap(&list[e], &cand, words) > thr)
                blocked = 1;
        if (blocked) {
            free(cand.mask);
            continue;
        }
        size_t kept = 0; /* std::erase_if, order preserving (:194-196) */
        for (size_t e = 0; e < n; ++e) {
            if (list[e].fitness < cand.fitness && orc_tr_overlap(&list[e], &cand, words) > thr)
                free(list[e].mask);
            else
                list[kept++] = list[e];
        }
        n = kept;
        cand.seq = (*next_seq)++; /* :197-198 */
        list[n++] = cand;
    }
    qsort(list, n, sizeof(orc_tr_entry), orc_tr_entry_cmp); /* :201-204 */
    size_t keep = n < capacity ? n : capacity;              /* :205 */
    for (size_t e = 0; e < n; ++e) {
        if (e < keep) {
            out_ref[e] = list[e].ref;
            out_seq[e] = list[e].seq;
        }
        free(list[e].mask);
    }
    *out_count = keep;
    free(order);
    free(list);
    return 0;
}
