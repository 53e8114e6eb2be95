/*
 * ebic_b200.h -- C ABI of the B200-native EBIC fitness-evaluation hot path.
 *
 * The reference (arxiv/paper_1801_03039, header-only C++20) has no plugin
 * seam: its evolutionary loop calls inline free functions.  Each entry point
 * below replaces one of those functions (cited as reference file:line, paths
 * relative to /root/reference/proj/include/ebic/).  The repo's shadowing
 * headers include/ebic/{fitness,expansion,evolution,io,synthgen}.hpp bind these entry
 * points behind the reference's own C++ signatures.
 *
 * Conventions
 *  - Plain pointers and sizes only; no C++ or torch types cross the ABI.
 *  - Every function returns an ebic_status (0 = EBIC_OK).  On failure the
 *    thread-local message is available from ebic_last_error(); the texts for
 *    the reference's own error conditions are the reference's strings
 *    ("matrix has no rows", "empty population", "invalid series",
 *    "corrupt CBF").
 *  - Host buffers are caller-owned; the context owns every device copy.
 *  - A context is not thread-safe: calls on one context must be serialised
 *    (the reference evaluates one batch at a time, parallel.hpp:14-16).
 *    Device-pointer calls may use different streams: a launch on a stream
 *    other than the previous launch's first waits (on the device) for work
 *    already queued on that stream, since launches share the context's
 *    scratch.  The host-buffer calls use the context's own stream.
 *  - The matrix is copied into device memory when the context is created;
 *    later changes to the caller's host buffer are not seen (create a new
 *    context for a new matrix, as the drop-in headers do per run).
 *  - The population travels in CBF form exactly as the reference builds it
 *    (cbf.hpp:43-52): offsets[P+1] (size_t, offsets[0] == 0) and the
 *    concatenated uint16 column indices.
 *  - Results are bit-exact with the reference CPU path: counts are integer
 *    sums; fitness uses host-glibc log/exp2 (via host-built tables on the
 *    device), never device transcendental functions.
 */
#ifndef EBIC_B200_H
#define EBIC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* The library is built with -fvisibility=hidden; everything declared here is
 * exported. */
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

/* 2: ebic_ctx_info gained `kernel` (appended); callers built against version 1
 * pass a smaller struct to ebic_ctx_get_info and must be rebuilt. */
#define EBIC_B200_ABI_VERSION 2

typedef enum ebic_status {
    EBIC_OK = 0,
    EBIC_ERR_INVALID_ARGUMENT = 1, /* maps to std::invalid_argument */
    EBIC_ERR_RUNTIME = 2,          /* maps to std::runtime_error */
    EBIC_ERR_CUDA = 3,             /* CUDA runtime / driver failure */
    EBIC_ERR_NO_DEVICE = 4         /* no usable sm_100 device */
} ebic_status;

/* Row-membership flags, numerically identical to ebic::RowFlag
 * (bicluster.hpp:11-15). */
enum { EBIC_ROW_EXACT = 0, EBIC_ROW_NEGATIVE = 1, EBIC_ROW_APPROXIMATE = 2 };

typedef struct ebic_ctx ebic_ctx;

typedef struct ebic_ctx_info {
    size_t n_rows;        /* rows held by the context (all shards) */
    size_t n_cols;
    size_t row_begin;     /* first global row held (shard contexts) */
    size_t total_rows;    /* rows of the full matrix */
    int n_shards;         /* one per device */
    int rows_per_tile;    /* count-kernel row tile (0 = direct kernel) */
    int stages;           /* TMA pipeline depth of the count kernel */
    int grid;             /* CTAs per count launch on shard 0 */
    size_t device_bytes;  /* matrix bytes resident on shard 0 */
    int sm_count;         /* SMs of shard 0's device */
    int layout;           /* last count launch: 0 fp64 tile, 1/2 = exact rank tile (planes),
                             3 = one-plane collapsed rank tile (eps > 0), 4/5 = the one-plane
                             tile (strict / collapsed) packed three rows per 32-bit word,
                             6/7 = five rows per 64-bit word */
    int consumer_warps;   /* count-kernel consumer warps per CTA */
    int kernel;           /* last count launch: 1 = v1 tile or direct kernel, 2 = K1v2
                             (row tiles per CTA), 3 = K1s (series per CTA) */
} ebic_ctx_info;

/* Library / device queries. */
const char* ebic_last_error(void);
int ebic_abi_version(void);
int ebic_device_count(int* count_out);

/* ---- context ---------------------------------------------------------- */

/* Uploads a row-major fp64 matrix (ExpressionMatrix::values, matrix.hpp:24,
 * row_ptr :31) and re-lays it out column-major with a padded leading
 * dimension on each device.  Rows are split into contiguous shards (64-row
 * aligned) over devices[0..n_devices); devices == NULL means {0}.  This is
 * the one-time cost the reference pays implicitly by holding the matrix in
 * host memory; the context replaces make_chunk_plan/ThreadPool
 * (fitness.hpp:30-39, parallel.hpp:17-89).
 * Errors: n_rows == 0 -> "matrix has no rows" (fitness.hpp:31). */
int ebic_ctx_create(const double* row_major, size_t n_rows, size_t n_cols, const int* devices,
                    int n_devices, ebic_ctx** ctx_out);

/* Shard context for one-process-per-GPU deployments: holds global rows
 * [row_begin, row_begin + shard_rows) of a total_rows x n_cols matrix on one
 * device.  row_major_shard points at the shard's first row.  Counts produced
 * on a shard context are partial sums over its rows; the caller reduces them
 * (NCCL all-reduce of uint64) and then applies ebic_fitness_device. */
int ebic_ctx_create_shard(const double* row_major_shard, size_t shard_rows, size_t n_cols,
                          size_t total_rows, size_t row_begin, int device, ebic_ctx** ctx_out);

/* Device-resident variant of ebic_ctx_create_shard: d_row_major is a device
 * pointer (on `device`) to shard_rows x n_cols row-major doubles. */
int ebic_ctx_create_shard_device(const double* d_row_major, size_t shard_rows, size_t n_cols,
                                 size_t total_rows, size_t row_begin, int device,
                                 ebic_ctx** ctx_out);

int ebic_ctx_destroy(ebic_ctx* ctx);
int ebic_ctx_get_info(const ebic_ctx* ctx, ebic_ctx_info* info_out);

/* ---- fitness evaluation: the hot path ----------------------------------- */

/* count_matches (fitness.hpp:100-118): counts_out[p] = number of rows whose
 * values strictly increase along series p with slack eps, i.e. for every
 * adjacent pair !(v[prev] < v[cur] + eps) is false (fitness.hpp:63,84).
 * n_series == 0 is valid and writes nothing (fitness.hpp:104). */
int ebic_count_matches(ebic_ctx* ctx, const size_t* offsets, const uint16_t* cols,
                       size_t n_series, double eps, uint64_t* counts_out);

/* evaluate_population (fitness.hpp:135-143): counts followed by Eq. 1
 * fitness_score (fitness.hpp:124-133) with len = offsets[p+1]-offsets[p].
 * counts_out may be NULL. */
int ebic_evaluate_population(ebic_ctx* ctx, const size_t* offsets, const uint16_t* cols,
                             size_t n_series, uint64_t sigma, double eps, uint64_t* counts_out,
                             double* fitness_out);

/* fitness_score (fitness.hpp:124-133) and default_sigma (fitness.hpp:48-52),
 * host-side, same libm. */
double ebic_fitness_score(uint64_t match_count, size_t series_len, uint64_t sigma);
uint64_t ebic_default_sigma(size_t n_rows);

/* Eq. 1 for a whole population on the host: fitness_out[p] =
 * fitness_score(counts[p], offsets[p+1] - offsets[p], sigma).  Used after a
 * cross-process all-reduce of shard counts. */
int ebic_fitness_scores_host(const uint64_t* counts, const size_t* offsets, size_t n_series,
                             uint64_t sigma, double* fitness_out);

/* Device-pointer variants (single-shard contexts) for callers that keep the
 * CBF in HBM and own the stream (cudaStream_t passed as void*, used as is:
 * NULL is the legacy default stream, as everywhere in CUDA).  d_offsets: uint64[P+1]; d_cols: uint16[offsets[P]];
 * total_len == offsets[P] (host-known).  d_counts_out: uint64[P] (partial
 * counts on a shard context).  d_fitness_out may be NULL; when non-NULL on a
 * whole-matrix context the fitness epilogue is fused into the count kernel.
 * Returns without synchronising. */
int ebic_count_matches_device(ebic_ctx* ctx, const uint64_t* d_offsets, const uint16_t* d_cols,
                              size_t n_series, size_t total_len, double eps, uint64_t sigma,
                              uint64_t* d_counts_out, double* d_fitness_out, void* stream);

/* Eq. 1 over already-reduced device counts (after the all-reduce). */
int ebic_fitness_device(ebic_ctx* ctx, const uint64_t* d_counts, const uint64_t* d_offsets,
                        size_t n_series, uint64_t sigma, double* d_fitness_out, void* stream);

/* Diagnostics: per-CTA %globaltimer stamps (ns) of the last count launch on
 * shard 0 -- [start, work list built, tiles done, epilogue done, partial
 * counts flushed, arrival counted, -, -] per CTA -- recorded only when the
 * context was created with EBIC_PHASE_TIMING=1 in the environment.  Copies
 * min(grid, max_ctas) x 8 values; *n_ctas = grid. */
int ebic_ctx_phase_times(ebic_ctx* ctx, uint64_t* stamps_out, size_t max_ctas, size_t* n_ctas);

/* Diagnostics: mean host-side time (us) per ebic_count_matches /
 * ebic_evaluate_population call on this context, split into [validate CBF,
 * stage + H2D submit, kernel launch submit, wait for the completion flag,
 * copy-out]; *calls_out = number of calls. */
int ebic_ctx_host_timers(ebic_ctx* ctx, double* mean_us_out, uint64_t* calls_out);

/* ---- row membership (Steps 6-7) ----------------------------------------- */

/* Per-series row bitmasks over the context's rows (words = ceil(n_rows/64),
 * bit r%64 of word r/64; each output holds n_series * words uint64):
 *   exact_bits  : row_matches(series)                 (expansion.hpp:16-23)
 *   neg_bits    : row_matches(reversed series)        (expansion.hpp:58,64)
 *   approx_bits : trend_violations(series) <= approx_k (expansion.hpp:26-33,66-67)
 * Any output pointer may be NULL. */
int ebic_membership_bits(ebic_ctx* ctx, const size_t* offsets, const uint16_t* cols,
                         size_t n_series, double eps, size_t approx_k, uint64_t* exact_bits,
                         uint64_t* neg_bits, uint64_t* approx_bits);

/* assign_rows (expansion.hpp:16-23): ascending matching rows; rows_out has
 * capacity n_rows; *n_out receives the count. */
int ebic_assign_rows(ebic_ctx* ctx, const uint16_t* series, size_t len, double eps,
                     uint64_t* rows_out, size_t* n_out);

/* expand_bicluster (expansion.hpp:56-87): core rows (ascending) keep their
 * flags; other rows get NEGATIVE if allow_negative and the reversed series
 * matches, else APPROXIMATE if approx_k > 0 and violations <= approx_k.
 * Output merged by row; capacity n_rows + n_core. */
int ebic_expand_bicluster(ebic_ctx* ctx, const uint16_t* series, size_t len,
                          const uint64_t* core_rows, const uint8_t* core_flags, size_t n_core,
                          int allow_negative, size_t approx_k, double eps, uint64_t* rows_out,
                          uint8_t* flags_out, size_t* n_out);

/* Batched Steps 6-7 for finalize_biclusters (io.hpp:164-178): for each of
 * n_series series, the exact core (resolve_bicluster, expansion.hpp:36-44)
 * expanded by expand_bicluster.  Results are concatenated: row_counts[s]
 * rows for series s, rows_out/flags_out with capacity n_series * n_rows. */
int ebic_resolve_expand_batch(ebic_ctx* ctx, const size_t* offsets, const uint16_t* cols,
                              size_t n_series, int allow_negative, size_t approx_k, double eps,
                              uint64_t* rows_out, uint8_t* flags_out, size_t* row_counts);

/* ---- synthetic input (synthgen.hpp:114-223) ----------------------------- */

/* Deterministic scenario matrix, bit-identical to ebic::generate for the
 * same ScenarioSpec (pattern numbering as ebic::Pattern, synthgen.hpp:18-25).
 * Writes n_rows * n_cols row-major doubles. */
int ebic_synth_generate(size_t n_rows, size_t n_cols, size_t n_blocks, const size_t* block_rows,
                        const size_t* block_cols, int pattern, size_t overlap_rows,
                        size_t overlap_cols, double noise_sd, uint64_t seed, double* values_out);

/* ---- multi-process row shards: reduction inside the count kernels -------- */

/* One process per GPU, each holding a shard context (ebic_ctx_create_shard),
 * replaces count_matches' row-chunk partial sums (fitness.hpp:100-118) across
 * processes without a separate collective: every rank's count kernel adds its
 * shard's per-series totals into one accumulator on rank 0's GPU (CUDA IPC
 * peer memory, system-scope atomics) and takes a ticket; the last rank's
 * kernel writes the whole-matrix counts and Eq. 1 fitness into a POSIX
 * shared-memory block every rank has mapped, then raises its flag.  No
 * kernel waits for another (ranks may share a GPU).
 *   rank 0:     ebic_xgroup_create(ctx0, max_series, "/name", handle)
 *   broadcast:  handle (EBIC_XGROUP_HANDLE_BYTES) and the name to all ranks
 *   every rank: ebic_xgroup_join(ctx, handle, "/name", n_ranks, max_series, &g)
 *   per call (same increasing seq on every rank):
 *               ebic_xgroup_evaluate(g, offsets, cols, P, sigma, eps, seq, counts, fitness)
 *           or  ebic_xgroup_count(g, d_off, d_cols, P, L, eps, sigma, want_fit, seq, stream)
 *               + ebic_xgroup_wait(g, seq, P, counts, fitness)
 *   teardown:   ebic_xgroup_destroy on every rank (rank 0 last: it owns the memory). */
#define EBIC_XGROUP_HANDLE_BYTES 64
typedef struct ebic_xgroup ebic_xgroup;
int ebic_xgroup_create(ebic_ctx* ctx, size_t max_series, const char* shm_name, void* handle_out);
int ebic_xgroup_join(ebic_ctx* ctx, const void* handle, const char* shm_name, int n_ranks,
                     size_t max_series, ebic_xgroup** group_out);
int ebic_xgroup_evaluate(ebic_xgroup* g, const size_t* offsets, const uint16_t* cols, size_t n_series,
                         uint64_t sigma, double eps, uint64_t seq, uint64_t* counts_out,
                         double* fitness_out);
int ebic_xgroup_count(ebic_xgroup* g, const uint64_t* d_offsets, const uint16_t* d_cols,
                      size_t n_series, size_t total_len, double eps, uint64_t sigma, int want_fitness,
                      uint64_t seq, void* stream);
int ebic_xgroup_wait(ebic_xgroup* g, uint64_t seq, size_t n_series, uint64_t* counts_out,
                     double* fitness_out);
int ebic_xgroup_destroy(ebic_xgroup* g);

/* ---- top-rank admission (evolution.hpp:168-206) ------------------------- */

/* Replaces TopRankList::update (evolution.hpp:168-206), host only, stateless.
 * Current entries (n_entries series in CBF form with their fitness and seq)
 * are offered the n_cand candidates exactly as the reference does: positive
 * fitness only, visited by fitness desc / index asc; a candidate is blocked by
 * any entry of >= fitness overlapping it above overlap_threshold
 * (|a & b| / min(|a|, |b|), evolution.hpp:154-160), otherwise it evicts the
 * overlapping lower-fitness entries and is appended with seq = (*next_seq)++.
 * The survivors sorted by (fitness desc, seq asc) and truncated to capacity
 * are written as out_ref[i] (>= 0: entry index, < 0: candidate -(ref + 1))
 * and out_seq[i]; *out_count <= min(capacity, n_entries + n_cand) (size the
 * outputs for that).  Like the reference's update, threshold and capacity
 * are not validated (run() does that, evolution.hpp:45-49); columns must be
 * < n_cols. */
int ebic_top_rank_update(size_t n_cols, size_t n_entries, const size_t* entry_offsets,
                         const uint16_t* entry_cols, const double* entry_fitness,
                         const uint64_t* entry_seq, size_t n_cand, const size_t* cand_offsets,
                         const uint16_t* cand_cols, const double* cand_fitness,
                         double overlap_threshold, size_t capacity, uint64_t* next_seq,
                         int64_t* out_ref, uint64_t* out_seq, size_t* out_count);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
}
#endif

#endif /* EBIC_B200_H */
