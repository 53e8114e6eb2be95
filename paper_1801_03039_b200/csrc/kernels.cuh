// kernels.cuh -- sm_100a kernels of the EBIC fitness-evaluation hot path.
//
//   K0 transpose_pad_kernel   row-major fp64 -> column-major, leading dim padded
//   K1 count_tma_kernel       per-series match counts (+ fused Eq. 1 epilogue)
//      count_direct_kernel    same contract without TMA staging (very wide matrices)
//   K2 fitness_kernel         Eq. 1 over reduced counts (multi-shard path)
//   K3 membership_kernel      exact / negative / approximate row bitmasks
//
// Reference semantics: /root/reference/proj/include/ebic/fitness.hpp:57-143 and
// expansion.hpp:16-87.  The predicate is evaluated exactly as the reference does,
// !(prev < cur + eps) in IEEE fp64 round-to-nearest (no FMA can form: one add,
// one compare), over adjacent pairs only (fitness.hpp:63,84).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace ebic_b200 {

constexpr int kMaxStages = 8;
// Grid reduction tree of the count kernels: CTAs publish per-series partial
// counts into their own row; the last CTA of each group of kGroupMin+ CTAs
// sums its group; the last group reducer finalises.  No atomics on data (a
// 148-way atomic reduction into the same P addresses serialises in the L2
// atomic units), two atomic tickets per CTA at most.
constexpr int kMaxGroups = 64;
constexpr int kGroupMin = 16;
__host__ __device__ inline uint32_t reduce_group_size(uint32_t grid) {
    const uint32_t g = (grid + kMaxGroups - 1) / kMaxGroups;
    return g < kGroupMin ? kGroupMin : g;
}
constexpr int kLenBuckets = 64;  // length histogram buckets for the work sort

// ---------------------------------------------------------------------------
// small PTX helpers (mbarrier + TMA)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    // try_wait with a suspend-time hint: a waiting warp sleeps until the
    // phase completes (or the hint expires) instead of re-issuing the probe
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
        "@P1 bra DONE_%=;\n"
        "bra WAIT_%=;\n"
        "DONE_%=:\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(0x989680u)
        : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* smem_dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void named_bar_sync(int id, int threads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// The reference predicate (fitness.hpp:63): a row continues iff prev < cur + eps.
// For eps == +0.0 the add is the identity for comparison purposes (x + 0.0 only
// maps -0.0 to +0.0, which compare equal; NaN stays NaN), so it is skipped.
template <bool kEpsZero>
__device__ __forceinline__ bool step_ok(double prev, double cur, double eps) {
    if (kEpsZero) return prev < cur;
    return prev < __dadd_rn(cur, eps);
}

// Eq. 1 (fitness.hpp:124-133) from host-glibc tables:
//   logt[c] = log(double(c - 1))   (c >= 2)
//   expt[c] = exp2(double(c) - double(sigma))   (c < sigma)
// The two multiplies are performed in the reference's order with explicit
// round-to-nearest, so the result is bit-identical to the host computation.
__device__ __forceinline__ double fitness_from_tables(uint64_t c, uint64_t len, uint64_t sigma,
                                                      const double* __restrict__ logt,
                                                      const double* __restrict__ expt) {
    if (c <= 1) return 0.0;
    double f = __dmul_rn(static_cast<double>(len), logt[c]);
    if (c < sigma) f = __dmul_rn(f, expt[c]);
    return f > 0.0 ? f : 0.0;
}

// ---------------------------------------------------------------------------
// K0: row-major [rows x cols] (ld_in = cols) -> column-major [cols x ld_out].
// 32x32 tiles through shared memory; padded rows (>= rows, < ld_out) get NaN so
// they can never satisfy the trend predicate.
// ---------------------------------------------------------------------------
// `in` holds in_rows valid rows; out_rows >= in_rows rows are written (the
// surplus as NaN padding).  `out` points at the first output row.
__global__ void transpose_pad_kernel(const double* __restrict__ in, size_t rows, size_t cols,
                                     double* __restrict__ out, size_t ld_out, size_t pad_rows) {
    __shared__ double tile[32][33];
    const size_t c0 = static_cast<size_t>(blockIdx.x) * 32;
    const size_t r0 = static_cast<size_t>(blockIdx.y) * 32;
    const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
    for (int k = ty; k < 32; k += 8) {
        const size_t r = r0 + k, c = c0 + tx;
        double v = __longlong_as_double(0x7ff8000000000000ULL);
        if (r < rows && c < cols) v = in[r * cols + c];
        tile[k][tx] = v;
    }
    __syncthreads();
    for (int k = ty; k < 32; k += 8) {
        const size_t c = c0 + k, r = r0 + tx;
        if (c < cols && r < pad_rows) out[c * ld_out + r] = tile[tx][k];
    }
}

// ---------------------------------------------------------------------------
// Shared-memory plan of one count launch (host computes the same layout).
// ---------------------------------------------------------------------------
struct CountParams {
    const uint64_t* __restrict__ offsets;  // [P+1] (absolute positions into cols)
    const uint16_t* __restrict__ cols;     // whole column array
    // total_len == offsets[P] - offsets[0]
    uint32_t n_series;
    uint32_t total_len;
    uint32_t n_rows;        // valid rows of this shard
    uint32_t n_tiles;       // ceil(n_rows / RPG)
    uint32_t n_cols;
    uint32_t box_cols;      // TMA box width (columns)
    uint32_t n_boxes;       // boxes per stage
    uint32_t stage_bytes;   // RPG * 8 * box_cols * n_boxes
    uint32_t stages;
    double eps;
    uint64_t sigma;
    uint32_t* __restrict__ partial;        // [(grid + groups) * P] reduction scratch
    unsigned int* __restrict__ done;       // [kMaxGroups + 1] tickets (zero on entry and exit)
    uint64_t* __restrict__ counts_out;     // [P]
    double* __restrict__ fitness_out;      // [P] or nullptr
    const double* __restrict__ logt;       // fitness tables (nullptr if no fitness)
    const double* __restrict__ expt;
    const double* __restrict__ matrix;     // column-major (direct kernel only)
    uint32_t ld;                           // leading dimension (direct kernel only)
    uint64_t cols_base;                    // == offsets[0] (host-known; no dependent load)
    uint32_t sched_static;                 // debug: static chunk assignment
    uint32_t max_parts;                    // tail split of the last wave (1 = off)
    uint32_t reduce_striped;               // 1: striped-accumulator tail, 0: reduction tree
    uint32_t scratch_in_stage;             // prologue scratch lives in the last stage buffer
    uint32_t rank_k;                       // one-plane rank test constant (RankWalker::step)
    const unsigned long long* __restrict__ row_excl;  // [ceil(rows/64)] rows not in the layout
    const uint32_t* __restrict__ excl_rows;           // their indices (n_excl)
    const double* __restrict__ excl_vals;             // their values, row-major [n_excl][n_cols]
    uint32_t n_excl;
    // Optional completion signal for host callers: after the final CTA has
    // written counts/fitness (which may live in mapped host memory), it makes
    // them system-visible and stores done_seq to *done_flag.
    unsigned long long* done_flag;
    unsigned long long done_seq;
    // Optional host-resident CBF (mapped pinned memory, device-visible): CTA 0
    // copies cbf_bytes from host_cbf to dev_cbf (where offsets / cols point)
    // and publishes cbf_seq in *cbf_ready; the other CTAs wait for it.  This
    // replaces a host cudaMemcpyAsync (several us of API time per call).
    const uint4* __restrict__ host_cbf;
    uint4* __restrict__ dev_cbf;
    uint32_t cbf_words;                    // 16-byte words to copy
    unsigned int* __restrict__ cbf_ready;
    unsigned int cbf_seq;
    uint64_t table_n;                      // entries of logt/expt (prefetched into L2)
    // Cross-shard reduction (one process, several row shards / devices): the
    // final CTA of every shard's launch adds its per-series totals into
    // xacc (home device memory, peer-accessible) and takes a system-scope
    // ticket; the last shard to arrive writes counts + fitness for the whole
    // matrix and raises the done flag.  No launch waits for another.
    unsigned long long* __restrict__ xacc;  // [P] or nullptr (single shard)
    unsigned int* __restrict__ xticket;
    uint32_t n_xshards;
    unsigned long long* __restrict__ phase_ns;  // optional [grid][8] %globaltimer stamps
    // Measurement only (EBIC_DEBUG_MODE; results are wrong): 1 = consumers
    // skip the walk (pure TMA streaming time), 2 = the producer skips the
    // loads (pure walk time over stale stages), 3 (K1v2) = no ring at all:
    // consumers walk stage 0 item after item (intrinsic walk rate).
    uint32_t debug_mode;
    // K1v2 (kernels_v2.cuh): tile-major rank matrix, usable dynamic shared bytes
    const unsigned char* __restrict__ ranks;
    uint32_t smem_window;
    uint32_t gap;         // K1v2: stage gaps of <= gap unreferenced columns (0-2)
    uint32_t compact;     // K1v2: stage the referenced columns (1) or whole tiles (0)
    uint32_t prefetch;    // K1v2 compact: L2-prefetch the block this many items ahead (0 off)
};

__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// Shared-memory work list of one count launch (P series, L column entries).
// Persistent part (lives through the whole launch):
//   s_sl     u32[P]   slot -> series id (slots are length-sorted)
//   s_slen   u32[P]   slot -> series length
//   s_sstart u32[P]   slot -> first entry in s_pcols (multiple of 4)
//   s_cnt    u32[P]   slot -> per-CTA match count
//   s_pcols  u32[L + 3P] per series, the BYTE OFFSETS (column x column-slice
//                     bytes) of its columns inside a staged tile, padded to a
//                     multiple of 4 entries: one LDS.128 fetches 4 offsets and
//                     an element address is a single add.
// Prologue scratch (dead once the list is built; placed in the last TMA stage
// buffer, which the producer fills only after the prologue, when it fits):
//   s_rel u32[P+1], s_raw u16[L+16], s_wh u32[ceil(P/32)][kLenBuckets],
//   s_hist/s_hpad u32[kLenBuckets], s_wsum u32[32]
__host__ __device__ inline size_t count_persist_bytes(uint32_t P, uint32_t L) {
    return ((16ull * P + 15) & ~size_t(15)) + 4ull * (L + 3ull * P) + 16;
}
__host__ __device__ inline size_t count_scratch_bytes(uint32_t P, uint32_t L) {
    size_t b = (4ull * (P + 1) + 15) & ~size_t(15);
    b += (2ull * L + 32 + 15) & ~size_t(15);
    return b + 4ull * kLenBuckets * ((P + 31) / 32) + 4ull * kLenBuckets * 2 + 4ull * 32 + 16;
}
__host__ __device__ inline size_t count_meta_bytes(uint32_t P, uint32_t L, bool scratch_in_stage) {
    return count_persist_bytes(P, L) + (scratch_in_stage ? 0 : count_scratch_bytes(P, L) + 16);
}

struct WorkList {
    uint32_t* sl;
    uint32_t* slen;
    uint32_t* sstart;
    uint32_t* cnt;
    uint32_t* pcols;
    // prologue scratch
    uint32_t* rel;
    uint16_t* raw;
    uint32_t* wh;
    uint32_t* hist;
    uint32_t* hpad;
    uint32_t* wsum;
};

__device__ __forceinline__ unsigned char* align16(unsigned char* base, size_t off) {
    return base + ((off + 15) & ~size_t(15));
}

// Carves the work list: persistent part at `p`, scratch at `q` (both 16-byte
// aligned).  Pointer arithmetic on the shared window only (LDS/STS addressing).
__device__ __forceinline__ WorkList carve_work_list(unsigned char* p, unsigned char* q, uint32_t P,
                                                    uint32_t L) {
    WorkList w;
    w.sl = reinterpret_cast<uint32_t*>(p);
    w.slen = w.sl + P;
    w.sstart = w.slen + P;
    w.cnt = w.sstart + P;
    w.pcols = reinterpret_cast<uint32_t*>(align16(p, 16ull * P));
    w.rel = reinterpret_cast<uint32_t*>(q);
    q = align16(q, 4ull * (P + 1));
    w.raw = reinterpret_cast<uint16_t*>(q);
    q = align16(q, 2ull * L + 32);
    w.wh = reinterpret_cast<uint32_t*>(q);
    w.hist = w.wh + kLenBuckets * ((P + 31) / 32);
    w.hpad = w.hist + kLenBuckets;
    w.wsum = w.hpad + kLenBuckets;
    return w;
}

// Exclusive scan over P items by `nthreads` threads (blocked partition).
// vals(g) -> item g; writes out[g]; all threads of the group participate.
template <class F>
__device__ __forceinline__ void block_exclusive_scan(uint32_t P, F vals, uint32_t* out,
                                                     uint32_t* wsum, int tid, int nthreads,
                                                     int bar_id) {
    const uint32_t per = (P + nthreads - 1) / nthreads;
    const uint32_t lo = min(P, tid * per), hi = min(P, lo + per);
    uint32_t local = 0;
    for (uint32_t g = lo; g < hi; ++g) local += vals(g);
    const int lane = tid & 31, warp = tid >> 5;
    uint32_t incl = local;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[warp] = incl;
    named_bar_sync(bar_id, nthreads);
    if (warp == 0) {
        const int nw = nthreads >> 5;
        uint32_t x = lane < nw ? wsum[lane] : 0u, xi = x;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, xi, o);
            if (lane >= o) xi += y;
        }
        if (lane < nw) wsum[lane] = xi - x;
    }
    named_bar_sync(bar_id, nthreads);
    uint32_t run = wsum[warp] + incl - local;
    for (uint32_t g = lo; g < hi; ++g) {
        out[g] = run;
        run += vals(g);
    }
}

__device__ __forceinline__ uint32_t pad4(uint32_t len) { return (len + 3u) & ~3u; }

// Exclusive warp scan of two 64-entry arrays (a: counts, b: weights), lane l
// owning entries l and l + 32.  Returns the totals through *ta.
__device__ __forceinline__ void warp_scan64(uint32_t* a, uint32_t* b, int lane) {
    uint32_t a0 = a[lane], a1 = a[lane + 32], b0 = b[lane], b1 = b[lane + 32];
    uint32_t x0 = a0, x1 = a1, y0 = b0, y1 = b1;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u0 = __shfl_up_sync(0xffffffffu, x0, o), u1 = __shfl_up_sync(0xffffffffu, x1, o);
        const uint32_t v0 = __shfl_up_sync(0xffffffffu, y0, o), v1 = __shfl_up_sync(0xffffffffu, y1, o);
        if (lane >= o) x0 += u0, x1 += u1, y0 += v0, y1 += v1;
    }
    const uint32_t tx = __shfl_sync(0xffffffffu, x0, 31), ty = __shfl_sync(0xffffffffu, y0, 31);
    a[lane] = x0 - a0;
    a[lane + 32] = tx + x1 - a1;
    b[lane] = y0 - b0;
    b[lane + 32] = ty + y1 - b1;
}

// Cooperative construction of the work list by `nthreads` threads (5 barriers).
//  A  one round trip to global memory: offsets + column words, coalesced.
//  B  per 32-series block: bucket (= length, lengths >= 63 share bucket 63),
//     __match_any_sync peers; block-bucket counts and bucket totals.
//  C  warp 0: bucket starts and column-list starts (within buckets < 63 all
//     lists have the same padded length); 64 other threads: per-bucket
//     exclusive scan over blocks.
//  D  every series gets slot = bucket start + earlier blocks + rank in block
//     -- a stable counting sort, so every CTA derives the same slot order (a
//     chunk range names the same series on every CTA; tail-split tiles rely
//     on it) -- and copies its columns into its padded list.
//  E  (only if some series is >= 63 long) list starts of the overflow bucket.
// Runs while the producer's first TMA stages are in flight.
__device__ __forceinline__ void build_work_list(const CountParams& p, const WorkList& w, int tid,
                                                int nthreads, int bar_id, uint32_t col_bytes) {
    const uint32_t P = p.n_series, L = p.total_len;
    const uint32_t nblk = (P + 31) / 32;
    const int lane = tid & 31, nw = nthreads >> 5;
    // A launch may cover a slice of a larger population: column positions are
    // taken relative to offsets[0] (== cols_base, passed by value so the loads
    // below do not wait on it).  The column indices are fetched as whole
    // 16-byte words from the aligned word containing cols[base]; `shift`
    // re-bases positions inside w.raw.
    const uint64_t base = p.cols_base;
    const uint16_t* src = p.cols + base;
    const uint32_t shift = static_cast<uint32_t>((reinterpret_cast<uintptr_t>(src) & 15u) >> 1);
    const uint4* vsrc = reinterpret_cast<const uint4*>(src - shift);
    const uint32_t n_vec = (shift + L + 7u) >> 3;
    constexpr int kPer = 4;  // loads in flight per thread per pass
    for (uint32_t s0 = tid; s0 <= P || s0 < n_vec; s0 += kPer * nthreads) {
        uint64_t o[kPer];
        uint4 v[kPer];
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            const uint32_t i = s0 + k * nthreads;
            // L2-coherent loads: the CBF may have been staged by CTA 0 during
            // this launch (stage_host_cbf), which the read-only path may miss.
            if (i <= P) o[k] = __ldcg(p.offsets + i);
            if (i < n_vec) v[k] = __ldcg(vsrc + i);
        }
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            const uint32_t i = s0 + k * nthreads;
            if (i <= P) w.rel[i] = static_cast<uint32_t>(o[k] - base) + shift;
            if (i < n_vec) reinterpret_cast<uint4*>(w.raw)[i] = v[k];
        }
    }
    for (uint32_t i = tid; i < nblk * kLenBuckets; i += nthreads) w.wh[i] = 0;
    for (int b = tid; b < kLenBuckets; b += nthreads) w.hist[b] = 0;
    named_bar_sync(bar_id, nthreads);                                        // 1

    auto bucket_of = [&](uint32_t s, uint32_t& len) -> uint32_t {
        len = s < P ? w.rel[s + 1] - w.rel[s] : 0u;
        return s < P ? (len < kLenBuckets ? len : kLenBuckets - 1) : 0xffffu;
    };
    for (uint32_t blk = tid >> 5; blk < nblk; blk += nw) {
        uint32_t len;
        const uint32_t bkt = bucket_of(blk * 32 + lane, len);
        const uint32_t peers = __match_any_sync(0xffffffffu, bkt);
        if (bkt != 0xffffu && lane == __ffs(peers) - 1) {
            w.wh[blk * kLenBuckets + bkt] = __popc(peers);
            atomicAdd(&w.hist[bkt], static_cast<uint32_t>(__popc(peers)));
        }
    }
    named_bar_sync(bar_id, nthreads);                                        // 2

    if (tid < 32) {
        // bucket starts (slots) and list starts (pcols entries); bucket 63's
        // lists are sized in phase E
        for (int k = 0; k < 2; ++k) {
            const int b = tid + 32 * k;
            w.hpad[b] = b < kLenBuckets - 1 ? w.hist[b] * pad4(b) : 0u;
        }
        __syncwarp();
        warp_scan64(w.hist, w.hpad, tid);
    } else if (tid < 32 + kLenBuckets) {
        const int b = tid - 32;
        uint32_t run = 0;
        for (uint32_t blk = 0; blk < nblk; ++blk) {
            const uint32_t t = w.wh[blk * kLenBuckets + b];
            w.wh[blk * kLenBuckets + b] = run;
            run += t;
        }
    }
    named_bar_sync(bar_id, nthreads);                                        // 3

    const uint32_t lt = (1u << lane) - 1u;
    for (uint32_t blk = tid >> 5; blk < nblk; blk += nw) {
        uint32_t len;
        const uint32_t s = blk * 32 + lane;
        const uint32_t bkt = bucket_of(s, len);
        const uint32_t peers = __match_any_sync(0xffffffffu, bkt);
        if (bkt == 0xffffu) continue;
        const uint32_t r = w.wh[blk * kLenBuckets + bkt] + __popc(peers & lt);  // rank in bucket
        const uint32_t g = w.hist[bkt] + r;
        w.sl[g] = s;
        w.slen[g] = len;
        w.cnt[g] = 0;
        if (bkt < kLenBuckets - 1) {
            const uint32_t st = w.hpad[bkt] + r * pad4(len);
            w.sstart[g] = st;
            const uint16_t* from = w.raw + w.rel[s];
            for (uint32_t i = 0; i < pad4(len); ++i) w.pcols[st + i] = i < len ? from[i] * col_bytes : 0u;
        }
    }
    named_bar_sync(bar_id, nthreads);                                        // 4

    const uint32_t ovf = w.hist[kLenBuckets - 1];  // first overflow slot
    if (ovf < P) {                                                           // E (rare)
        if (tid == 0) {
            uint32_t run = w.hpad[kLenBuckets - 1];
            for (uint32_t g = ovf; g < P; ++g) {
                w.sstart[g] = run;
                run += pad4(w.slen[g]);
            }
        }
        named_bar_sync(bar_id, nthreads);
        for (uint32_t g = ovf + tid; g < P; g += nthreads) {
            const uint32_t len = w.slen[g], st = w.sstart[g];
            const uint16_t* from = w.raw + w.rel[w.sl[g]];
            for (uint32_t i = 0; i < pad4(len); ++i) w.pcols[st + i] = i < len ? from[i] * col_bytes : 0u;
        }
        named_bar_sync(bar_id, nthreads);
    }
}

// Ticket with release (publishes this CTA's prior writes, ordered before it
// by the preceding __syncthreads) and acquire (makes the other CTAs' published
// writes visible to the CTA that draws the last ticket) -- the
// bar.sync + red/atom.release.gpu pattern of CUTLASS's grid barrier.
__device__ __forceinline__ uint32_t ticket_acq_rel(unsigned int* ctr) {
    uint32_t old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(ctr) : "memory");
    return old;
}

// Sum of rows[r * P + s] for r in [lo, hi): loads issued 16 at a time so the
// L2 round trips overlap (L2-only loads: the rows were written by other SMs).
__device__ __forceinline__ uint64_t sum_rows(const uint32_t* rows, size_t P, uint32_t s,
                                             uint32_t lo, uint32_t hi) {
    uint64_t c = 0;
    for (uint32_t b = lo; b < hi; b += 16) {
        uint32_t v[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) v[k] = (b + k < hi) ? __ldcg(rows + size_t(b + k) * P + s) : 0u;
#pragma unroll
        for (int k = 0; k < 16; ++k) c += v[k];
    }
    return c;
}

// Grid-wide reduction tail shared by the count kernels (see kMaxGroups): the
// final CTA publishes counts (and Eq. 1 fitness when tables are given) and
// every ticket counter is left at zero for the next launch.  Integer sums:
// the result does not depend on arrival order (fitness.hpp:17-19).
// `slot_series` maps a counter slot to its series id (nullptr = identity).
// Striped-accumulator tail (default): every CTA adds its per-series partial
// counts with fire-and-forget reductions into stripe (blockIdx % kStripes) of
// a [P][kStripes] u32 accumulator (the eight stripes of a series share one
// 32-byte sector), so each address sees ~G/8 reductions instead of G; one
// acq_rel ticket per CTA; the last CTA sums the stripes (one 32-byte load per
// series), re-zeroes them for the next launch and writes counts + Eq. 1.
constexpr int kStripes = 8;

// Completion signal of the final CTA (see CountParams::done_flag): the
// barrier orders every thread's output stores before thread 0's system-scope
// fence, which makes them visible to the host before the flag.
__device__ __forceinline__ void signal_done(const CountParams& p) {
    if (!p.done_flag) return;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        *reinterpret_cast<volatile unsigned long long*>(p.done_flag) = p.done_seq;
    }
}

// Final CTA of one shard, after adding its totals into p.xacc: the system-
// scope ticket orders every shard's additions before the last arriver's
// reads; that CTA takes each total (and re-zeroes it) with one exchange,
// writes counts + Eq. 1 and signals completion.  The others just return.
__device__ __forceinline__ void cross_shard_finish(const CountParams& p) {
    __shared__ int s_xlast;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        s_xlast = atomicAdd_system(p.xticket, 1u) == p.n_xshards - 1;
        __threadfence_system();
    }
    __syncthreads();
    if (!s_xlast) return;
    const uint32_t P = p.n_series;
    for (uint32_t s = threadIdx.x; s < P; s += blockDim.x) {
        const uint64_t c = atomicExch_system(p.xacc + s, 0ull);
        p.counts_out[s] = c;
        if (p.fitness_out)
            p.fitness_out[s] = fitness_from_tables(c, p.offsets[s + 1] - p.offsets[s], p.sigma,
                                                   p.logt, p.expt);
    }
    if (threadIdx.x == 0) atomicExch_system(p.xticket, 0u);
    signal_done(p);
}

__device__ __forceinline__ void count_epilogue_striped(const CountParams& p, const uint32_t* s_cnt,
                                                       const uint32_t* slot_series) {
    const uint32_t P = p.n_series;
    uint32_t* acc = p.partial;  // [P][kStripes]
    const uint32_t stripe = blockIdx.x % kStripes;
    unsigned long long* stamp = p.phase_ns ? p.phase_ns + 8ull * blockIdx.x : nullptr;
    __shared__ int s_last;
    for (uint32_t g = threadIdx.x; g < P; g += blockDim.x) {
        const uint32_t c = s_cnt[g];
        const uint32_t s = slot_series ? slot_series[g] : g;
        if (c) atomicAdd(acc + size_t(s) * kStripes + stripe, c);
    }
    __syncthreads();
    if (stamp && threadIdx.x == 0) stamp[4] = global_ns();
    if (threadIdx.x == 0) s_last = ticket_acq_rel(&p.done[kMaxGroups]) == gridDim.x - 1;
    __syncthreads();
    if (stamp && threadIdx.x == 0) stamp[5] = global_ns();
    if (!s_last) return;
    if (stamp && threadIdx.x == 0) stamp[7] = global_ns();
    if (p.xacc) {
        for (uint32_t s = threadIdx.x; s < P; s += blockDim.x) {
            uint4* a = reinterpret_cast<uint4*>(acc + size_t(s) * kStripes);
            const uint4 x = __ldcg(a), y = __ldcg(a + 1);
            const uint64_t c = uint64_t(x.x) + x.y + x.z + x.w + y.x + y.y + y.z + y.w;
            a[0] = make_uint4(0, 0, 0, 0);
            a[1] = make_uint4(0, 0, 0, 0);
            if (c) atomicAdd_system(p.xacc + s, static_cast<unsigned long long>(c));
        }
        if (threadIdx.x == 0) p.done[kMaxGroups] = 0u;
        cross_shard_finish(p);
        return;
    }
    for (uint32_t s = threadIdx.x; s < P; s += blockDim.x) {
        uint4* a = reinterpret_cast<uint4*>(acc + size_t(s) * kStripes);
        const uint4 x = __ldcg(a), y = __ldcg(a + 1);
        const uint64_t c = uint64_t(x.x) + x.y + x.z + x.w + y.x + y.y + y.z + y.w;
        a[0] = make_uint4(0, 0, 0, 0);
        a[1] = make_uint4(0, 0, 0, 0);
        p.counts_out[s] = c;
        if (p.fitness_out)
            p.fitness_out[s] = fitness_from_tables(c, p.offsets[s + 1] - p.offsets[s], p.sigma,
                                                   p.logt, p.expt);
    }
    if (threadIdx.x == 0) p.done[kMaxGroups] = 0u;
    signal_done(p);
}

// Striped tail with 4-wide float reductions (reduce_striped == 2, K1v2):
// `by_series` holds this CTA's counts indexed by series.  Counts are integers
// below 2^24 (the host requires shard rows < 2^24), so fp32 adds are exact;
// one red.global.add.v4.f32 carries four series (a quarter of the L2 atomic
// operations of the u32 stripes).  Accumulator: [kStripes][P4] floats, P4 =
// P rounded up to 4, zero between launches.
__device__ __forceinline__ void count_epilogue_v4(const CountParams& p, const uint32_t* by_series) {
    const uint32_t P = p.n_series, P4 = (P + 3u) & ~3u;
    float* acc = reinterpret_cast<float*>(p.partial);
    const uint32_t stripe = blockIdx.x % kStripes;
    unsigned long long* stamp = p.phase_ns ? p.phase_ns + 8ull * blockIdx.x : nullptr;
    __shared__ int s_last;
    for (uint32_t i = threadIdx.x; i < P4 / 4; i += blockDim.x) {
        const uint4 c = *reinterpret_cast<const uint4*>(by_series + 4 * i);
        if (c.x | c.y | c.z | c.w)
            asm volatile("red.relaxed.gpu.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(
                             acc + size_t(stripe) * P4 + 4 * i),
                         "f"(static_cast<float>(c.x)), "f"(static_cast<float>(c.y)), "f"(static_cast<float>(c.z)),
                         "f"(static_cast<float>(c.w))
                         : "memory");
    }
    __syncthreads();
    if (stamp && threadIdx.x == 0) stamp[4] = global_ns();
    if (threadIdx.x == 0) s_last = ticket_acq_rel(&p.done[kMaxGroups]) == gridDim.x - 1;
    __syncthreads();
    if (stamp && threadIdx.x == 0) stamp[5] = global_ns();
    if (!s_last) return;
    if (stamp && threadIdx.x == 0) stamp[7] = global_ns();
    for (uint32_t s = threadIdx.x; s < P; s += blockDim.x) {
        float x[kStripes];
#pragma unroll
        for (int k = 0; k < kStripes; ++k) x[k] = __ldcg(acc + size_t(k) * P4 + s);
        double t = 0.0;
#pragma unroll
        for (int k = 0; k < kStripes; ++k) t += static_cast<double>(x[k]);
#pragma unroll
        for (int k = 0; k < kStripes; ++k) __stcg(acc + size_t(k) * P4 + s, 0.0f);
        const uint64_t c = static_cast<uint64_t>(t);
        if (p.xacc) {
            if (c) atomicAdd_system(p.xacc + s, static_cast<unsigned long long>(c));
            continue;
        }
        p.counts_out[s] = c;
        if (p.fitness_out)
            p.fitness_out[s] = fitness_from_tables(c, p.offsets[s + 1] - p.offsets[s], p.sigma, p.logt, p.expt);
    }
    if (threadIdx.x == 0) p.done[kMaxGroups] = 0u;
    if (p.xacc) {
        cross_shard_finish(p);
        return;
    }
    signal_done(p);
}

__device__ __forceinline__ void count_epilogue(const CountParams& p, const uint32_t* s_cnt,
                                               const uint32_t* slot_series) {
    if (p.reduce_striped) {
        count_epilogue_striped(p, s_cnt, slot_series);
        return;
    }
    const uint32_t P = p.n_series, G = gridDim.x;
    const uint32_t gsz = reduce_group_size(G);
    const uint32_t n_groups = (G + gsz - 1) / gsz;
    const uint32_t grp = blockIdx.x / gsz;
    const uint32_t g_lo = grp * gsz, g_hi = min(G, g_lo + gsz);
    uint32_t* rows = p.partial;                   // [G][P]
    uint32_t* grows = p.partial + size_t(G) * P;  // [n_groups][P]
    unsigned long long* stamp = p.phase_ns ? p.phase_ns + 8ull * blockIdx.x : nullptr;
    __shared__ int s_last;

    for (uint32_t g = threadIdx.x; g < P; g += blockDim.x)
        rows[size_t(blockIdx.x) * P + (slot_series ? slot_series[g] : g)] = s_cnt[g];
    __syncthreads();
    if (stamp && threadIdx.x == 0) stamp[4] = global_ns();
    if (threadIdx.x == 0) s_last = ticket_acq_rel(&p.done[grp]) == (g_hi - g_lo) - 1;
    __syncthreads();
    if (stamp && threadIdx.x == 0) stamp[5] = global_ns();
    if (!s_last) return;

    // last CTA of its group: sum the group's rows
    for (uint32_t s = threadIdx.x; s < P; s += blockDim.x)
        grows[size_t(grp) * P + s] = static_cast<uint32_t>(sum_rows(rows, P, s, g_lo, g_hi));
    __syncthreads();
    if (stamp && threadIdx.x == 0) stamp[6] = global_ns();
    if (threadIdx.x == 0) {
        p.done[grp] = 0u;
        s_last = ticket_acq_rel(&p.done[kMaxGroups]) == n_groups - 1;
    }
    __syncthreads();
    if (!s_last) return;
    if (stamp && threadIdx.x == 0) stamp[7] = global_ns();

    // last group reducer: final counts + fused Eq. 1
    if (p.xacc) {
        for (uint32_t s = threadIdx.x; s < P; s += blockDim.x) {
            const uint64_t c = sum_rows(grows, P, s, 0, n_groups);
            if (c) atomicAdd_system(p.xacc + s, static_cast<unsigned long long>(c));
        }
        if (threadIdx.x == 0) p.done[kMaxGroups] = 0u;
        cross_shard_finish(p);
        return;
    }
    for (uint32_t s = threadIdx.x; s < P; s += blockDim.x) {
        const uint64_t c = sum_rows(grows, P, s, 0, n_groups);
        p.counts_out[s] = c;
        if (p.fitness_out)
            p.fitness_out[s] = fitness_from_tables(c, p.offsets[s + 1] - p.offsets[s], p.sigma,
                                                   p.logt, p.expt);
    }
    if (threadIdx.x == 0) p.done[kMaxGroups] = 0u;
    signal_done(p);
}

// ---------------------------------------------------------------------------
// Series walkers over a staged fp64 tile: [col][RPG] doubles, one lane = RPL
// consecutive rows at byte offset gl*RPL*8.  Result: per-lane bit mask of
// matching rows (bit k = row k of the lane).  Branch-free AND over every
// adjacent pair: the same boolean as the reference's early-exit loop.
// ---------------------------------------------------------------------------
template <int RPG, int RPL, bool kEpsZero>
struct F64Walker {
    static constexpr int kShift = (RPG == 32) ? 8 : (RPG == 16) ? 7 : (RPG == 8) ? 6 : (RPG == 4) ? 5 : 4;
    static_assert((1 << kShift) == RPG * 8, "RPG must be a power of two in [2,32]");
    static constexpr uint32_t kAll = (1u << RPL) - 1u;
    // tile geometry (see count_tma_kernel)
    static constexpr int kRowsPerTile = RPG;
    static constexpr int kRowsPerLane = RPL;
    static constexpr int kLaneBytes = RPL * 8;
    static constexpr int kColBytes = RPG * 8;      // one column of a staged tile
    static constexpr int kDim0PerTile = RPG;       // TMA dim-0 extent of a tile (fp64 elements)
    static constexpr bool kTileMajor = false;      // column-major fp64 matrix
    using Mask = uint32_t;
    // excl: bit k set = the lane's row k is excluded (fixed up separately).
    __device__ __forceinline__ static Mask valid(uint32_t row0, uint32_t n_rows, uint32_t excl,
                                                 uint32_t) {
        uint32_t m = 0;
#pragma unroll
        for (int k = 0; k < RPL; ++k) m |= (row0 + k < n_rows) ? (1u << k) : 0u;
        return m & ~excl;
    }

    static constexpr int kSeriesPerGroup = 1;
    __device__ __forceinline__ static uint32_t count_group(const unsigned char* base,
                                                           const WorkList& wl, uint32_t g0,
                                                           uint32_t P, bool uniform, uint32_t ulen,
                                                           double eps, Mask vm) {
        if (g0 >= P) return 0u;
        const uint32_t len = uniform ? ulen : wl.slen[g0];
        return __popc(walk(base, wl.pcols + wl.sstart[g0], len, uniform, eps) & vm);
    }

    __device__ __forceinline__ static void load_offs(uint32_t* w, const uint32_t* pc, int L) {
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            if (4 * q < L) {
                const uint4 x = *reinterpret_cast<const uint4*>(pc + 4 * q);
                w[4 * q] = x.x;
                w[4 * q + 1] = x.y;
                w[4 * q + 2] = x.z;
                w[4 * q + 3] = x.w;
            }
        }
    }

    // All lane groups of the warp walk series of exactly L columns.
    template <int L>
    __device__ __forceinline__ static uint32_t walk_fixed(const unsigned char* base,
                                                          const uint32_t* pc, double eps) {
        uint32_t w[12];
        load_offs(w, pc, L);
        if (RPL == 1) {
            double prev = *reinterpret_cast<const double*>(base + w[0]);
            bool ok = true;
#pragma unroll
            for (int i = 1; i < L; ++i) {
                const double cur = *reinterpret_cast<const double*>(base + w[i]);
                ok = ok & step_ok<kEpsZero>(prev, cur, eps);
                prev = cur;
            }
            return ok ? 1u : 0u;
        } else {
            double2 prev = *reinterpret_cast<const double2*>(base + w[0]);
            bool a = true, b = true;
#pragma unroll
            for (int i = 1; i < L; ++i) {
                const double2 cur = *reinterpret_cast<const double2*>(base + w[i]);
                a = a & step_ok<kEpsZero>(prev.x, cur.x, eps);
                b = b & step_ok<kEpsZero>(prev.y, cur.y, eps);
                prev = cur;
            }
            return (a ? 1u : 0u) | (b ? 2u : 0u);
        }
    }

    // Any length, per-lane trip count (mixed-length warps, long series).
    __device__ __forceinline__ static uint32_t walk_any(const unsigned char* base,
                                                        const uint32_t* pc, uint32_t len,
                                                        double eps) {
        if (len <= 1) return kAll;  // no adjacent pair: the row matches (fitness.hpp:80-90)
        if (RPL == 1) {
            double prev = *reinterpret_cast<const double*>(base + pc[0]);
            bool ok = true;
            for (uint32_t i = 1; i < len; ++i) {
                const double cur = *reinterpret_cast<const double*>(base + pc[i]);
                ok = ok & step_ok<kEpsZero>(prev, cur, eps);
                prev = cur;
            }
            return ok ? 1u : 0u;
        } else {
            double2 prev = *reinterpret_cast<const double2*>(base + pc[0]);
            bool a = true, b = true;
            for (uint32_t i = 1; i < len; ++i) {
                const double2 cur = *reinterpret_cast<const double2*>(base + pc[i]);
                a = a & step_ok<kEpsZero>(prev.x, cur.x, eps);
                b = b & step_ok<kEpsZero>(prev.y, cur.y, eps);
                prev = cur;
            }
            return (a ? 1u : 0u) | (b ? 2u : 0u);
        }
    }

    __device__ __forceinline__ static uint32_t walk(const unsigned char* base, const uint32_t* pc,
                                                    uint32_t len, bool uniform, double eps) {
        if (uniform) {
            switch (len) {
                case 2: return walk_fixed<2>(base, pc, eps);
                case 3: return walk_fixed<3>(base, pc, eps);
                case 4: return walk_fixed<4>(base, pc, eps);
                case 5: return walk_fixed<5>(base, pc, eps);
                case 6: return walk_fixed<6>(base, pc, eps);
                case 7: return walk_fixed<7>(base, pc, eps);
                case 8: return walk_fixed<8>(base, pc, eps);
                case 9: return walk_fixed<9>(base, pc, eps);
                case 10: return walk_fixed<10>(base, pc, eps);
                case 11: return walk_fixed<11>(base, pc, eps);
                case 12: return walk_fixed<12>(base, pc, eps);
                default: break;
            }
        }
        return walk_any(base, pc, len, eps);
    }
};

// ---------------------------------------------------------------------------
// Series walker over a staged RANK tile (exact integer restatement of the fp64
// predicate; built by rank_build_kernel).  For every row, each cell's value v
// and its slack-shifted value fl(v + eps) are replaced by their dense ranks
// among the row's values {v_j} u {fl(v_j + eps)}; then
//     v_a < fl(v_b + eps)   <=>   lo(a) < hi(b)
// exactly (ranks preserve strict order; ties share a rank; NaN maps to
// sentinels that fail every test, as NaN compares false).  Ranks are stored
// with bit 15 set (r' = r | 0x8000, r <= 0x7fff), two rows per 32-bit word;
// for one word pair the test of both rows is one IADD3 + one LOP3:
//     ok &= hi'(cur) - lo'(prev) + 0x7fff7fff      (bit 15 / bit 31 = row test)
// since each 16-bit lane of the sum is hi - lo + 0x7fff in [0, 0xfffc] (no
// carry between lanes) and has bit 15 set iff hi > lo.
//   PLANES == 2 (eps != 0 or NaN present): a column slice holds, per 4 rows,
//     lo'[4] then hi'[4] (16 bytes); a lane owns 4 rows (one LDS.128).
//   PLANES == 1 (eps == 0, no NaN): lo == hi, one u16 per cell; a lane owns
//     8 rows (one LDS.128).
//   PLANES == 3 (K1v2 only; one plane whose ranks fit 9 bits, i.e. at most
//     510 distinct values per row): three rows per 32-bit word in 10-bit
//     fields (r' = r | 0x200, bits 0-9 / 10-19 / 20-29, row 3w + f of the
//     tile in field f of word w), so the same IADD3 + LOP3 tests three rows:
//         ok &= cur' - prev' + 0x1ff7fdff     (bits 9 / 19 / 29)
//     (each field of the sum is in [0, 0x3fe]: no carry between fields).
//     A lane owns 12 consecutive rows (one LDS.128), a tile 96 rows: a third
//     fewer bytes per row to stream, stage and test than one 16-bit plane.
//   PLANES == 4 (K1v2/K1s; one plane, ranks up to 2046 distinct values):
//     five rows per 64-bit word in 12-bit fields (r | 0x800, row 5w + f of an
//     80-row tile in bits 12f..12f+11 of word w), the test one 64-bit add
//     (IADD3 + IADD3.X) and AND per two words:
//         ok &= cur' - prev' + 0x07ff7ff7ff7ff7ff   (or + 0x0800800800800800)
//     a lane owns 10 rows (two words), a tile 80 rows: a fifth fewer bytes
//     per row than one 16-bit plane for matrices too wide for PLANES == 3.
// Tile: 128 bytes per column (32 rows x 2 planes, 64 rows x 1 plane, or 96 /
// 80 packed rows).
// ---------------------------------------------------------------------------
template <int PLANES, int SLICE, int SPG = 2>
struct RankWalker {
    static_assert(SLICE == 64 || SLICE == 128, "column slice of 64 or 128 bytes");
    static_assert(PLANES < 3 || SLICE == 128, "packed ranks: 128-byte slices");
    static constexpr bool kPacked = PLANES == 3;
    static constexpr bool kPacked64 = PLANES == 4;
    static constexpr int kRowsPerLane = kPacked ? 12 : kPacked64 ? 10 : PLANES == 2 ? 4 : 8;
    static constexpr int kRowsPerTile = kPacked ? 96 : kPacked64 ? 80 : SLICE / (2 * PLANES);
    static constexpr uint64_t kStrict64 = 0x07ff7ff7ff7ff7ffull, kCollapsed64 = 0x0800800800800800ull;
    static constexpr int kLaneBytes = 16;
    static constexpr int kColBytes = SLICE;
    static constexpr int kShift = SLICE == 128 ? 7 : 6;
    static constexpr int kDim0PerTile = kRowsPerTile * PLANES;  // u16 elements
    // The rank matrix is tile-major (rank_build_kernel): 128-byte blocks of
    // one column's rows, [block][column][64 u16]; a 64-byte slice is half a block.
    static constexpr bool kTileMajor = true;
    static constexpr int kSlicesPerBlock = 128 / SLICE;
    static constexpr int kWords = (kPacked || kPacked64) ? 4 : kRowsPerLane / 2;  // ok words per lane
    static constexpr int kSeriesPerGroup = SPG;               // independent walks per group
    static constexpr int kFieldBits = 32 / SPG;               // packed per-series counts
    static_assert(SPG == 2 || SPG == 4, "2 or 4 series per lane group");
    // Result bits: bit 15 / 31 of ok word k hold the lane's rows 2k / 2k+1.
    // tally() folds word k down by k bits (rows land on bits 15-k / 31-k)
    // and counts once; `m` is the lane's valid-row mask in that folded form.
    struct Mask {
        uint32_t m;     // folded valid-row mask
        uint32_t k;     // per-pair constant: 0x7fff7fff (strict <) or 0x80008000 (<=, collapsed)
        uint32_t m_hi;  // PLANES == 4: high half of the 64-bit folded mask
    };
    // excl: bit j set = the lane's row j is excluded (fixed up separately).
    __device__ __forceinline__ static Mask valid(uint32_t row0, uint32_t n_rows, uint32_t excl,
                                                 uint32_t kconst) {
        Mask v;
        v.m = 0;
        v.m_hi = 0;
        if constexpr (kPacked64) {  // row 5w + f: bit 11 + 12 f of 64-bit word w, folded down by w
            uint64_t m = 0;
#pragma unroll
            for (int w = 0; w < 2; ++w)
#pragma unroll
                for (int f = 0; f < 5; ++f)
                    if (row0 + 5 * w + f < n_rows && !((excl >> (5 * w + f)) & 1u)) m |= (1ull << (11 + 12 * f)) >> w;
            v.m = static_cast<uint32_t>(m);
            v.m_hi = static_cast<uint32_t>(m >> 32);
            v.k = kconst;
            return v;
        }
        if constexpr (kPacked) {  // row 3k + f: bit 9 + 10 f of word k, folded down by k
#pragma unroll
            for (int k = 0; k < 4; ++k)
#pragma unroll
                for (int f = 0; f < 3; ++f)
                    if (row0 + 3 * k + f < n_rows && !((excl >> (3 * k + f)) & 1u)) v.m |= (1u << (9 + 10 * f)) >> k;
            v.k = kconst;
            return v;
        }
#pragma unroll
        for (int k = 0; k < kWords; ++k)
            v.m |= (((row0 + 2 * k < n_rows && !((excl >> (2 * k)) & 1u)) ? 0x8000u : 0u) |
                    ((row0 + 2 * k + 1 < n_rows && !((excl >> (2 * k + 1)) & 1u)) ? 0x80000000u : 0u)) >> k;
        v.k = PLANES == 2 ? 0x7fff7fffu : kconst;
        return v;
    }
    // 32-bit shared-window address arithmetic: one add per element.
    __device__ __forceinline__ static uint4 ld(uint32_t base, uint32_t off) {
        uint4 v;
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                     : "r"(base + off));
        return v;
    }
    // Offset lists are 16-byte aligned (padded to 4 entries): LDS.128 per 4.
    __device__ __forceinline__ static void load_offs(uint32_t* w, const uint32_t* pc, int L) {
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            if (4 * q < L) {
                const uint4 x = *reinterpret_cast<const uint4*>(pc + 4 * q);
                w[4 * q] = x.x;
                w[4 * q + 1] = x.y;
                w[4 * q + 2] = x.z;
                w[4 * q + 3] = x.w;
            }
        }
    }
    // One adjacent pair: ok[k] accumulates bit 15/31 per row.  With one
    // plane, K = 0x7fff7fff tests r(prev) < r(cur) (eps == 0) and
    // K = 0x80008000 tests r(prev) <= r(cur) (collapsed eps > 0 layout).
    __device__ __forceinline__ static void step(uint32_t* ok, const uint4& prev, const uint4& cur,
                                                uint32_t K) {
        if constexpr (kPacked64) {
            // cur - prev + K per 64-bit word as two carry chains (4 integer
            // adds; the compiler's own lowering negates first and takes 5)
            const uint64_t K64 = (K & 1u) ? kStrict64 : kCollapsed64;  // from the 16-bit constants
            const uint32_t klo = static_cast<uint32_t>(K64), khi = static_cast<uint32_t>(K64 >> 32);
            uint32_t a0, a1, b0, b1;
            asm("sub.cc.u32 %0, %4, %6;\n\t"
                "subc.u32 %1, %5, %7;\n\t"
                "add.cc.u32 %0, %0, %8;\n\t"
                "addc.u32 %1, %1, %9;\n\t"
                "sub.cc.u32 %2, %10, %12;\n\t"
                "subc.u32 %3, %11, %13;\n\t"
                "add.cc.u32 %2, %2, %8;\n\t"
                "addc.u32 %3, %3, %9;"
                : "=&r"(a0), "=&r"(a1), "=&r"(b0), "=&r"(b1)
                : "r"(cur.x), "r"(cur.y), "r"(prev.x), "r"(prev.y), "r"(klo), "r"(khi), "r"(cur.z), "r"(cur.w),
                  "r"(prev.z), "r"(prev.w));
            ok[0] &= a0;
            ok[1] &= a1;
            ok[2] &= b0;
            ok[3] &= b1;
        } else if (PLANES == 2) {
            ok[0] &= cur.z - prev.x + 0x7fff7fffu;
            ok[1] &= cur.w - prev.y + 0x7fff7fffu;
        } else {
            ok[0] &= cur.x - prev.x + K;
            ok[1] &= cur.y - prev.y + K;
            ok[2] &= cur.z - prev.z + K;
            ok[3] &= cur.w - prev.w + K;
        }
    }
    // The packed 64-bit pair test with the constant known at compile time
    // (STRICT: kStrict64, else kCollapsed64): cur + ~prev + (K + 1) equals
    // cur - prev + K mod 2^64, which ptxas lowers, with K as immediates, to
    // a three-input IADD3 (two carry-outs, prev negated in the operand) for
    // the low half and IADD3.X + IMAD.IADD for the high half -- 2
    // integer-pipe instructions per 64-bit word (the IMAD issues on the FMA
    // pipe) instead of step()'s 3.  Same bits as step().
    template <bool STRICT>
    __device__ __forceinline__ static void step_k(uint32_t* ok, const uint4& prev, const uint4& cur) {
        static_assert(kPacked64, "64-bit packed layout only");
        constexpr uint64_t K1 = (STRICT ? kStrict64 : kCollapsed64) + 1ull;
        const uint64_t a = ((uint64_t(cur.y) << 32) | cur.x) + ~((uint64_t(prev.y) << 32) | prev.x) + K1;
        const uint64_t b = ((uint64_t(cur.w) << 32) | cur.z) + ~((uint64_t(prev.w) << 32) | prev.z) + K1;
        ok[0] &= static_cast<uint32_t>(a);
        ok[1] &= static_cast<uint32_t>(a >> 32);
        ok[2] &= static_cast<uint32_t>(b);
        ok[3] &= static_cast<uint32_t>(b >> 32);
    }
    __device__ __forceinline__ static uint32_t tally(const uint32_t* ok, const Mask& vm) {
        if constexpr (kPacked64) {
            // result bits 11 + 12 f of each 64-bit word: 11, 23 in its low
            // half, 3, 15, 27 in its high half -- disjoint, so both halves of
            // both words fold into one 32-bit word (the second word's one bit
            // down) and one POPC; the folded valid mask is m | m_hi.
            constexpr uint32_t kLo = static_cast<uint32_t>(kCollapsed64), kHi = static_cast<uint32_t>(kCollapsed64 >> 32);
            static_assert((kLo & kHi) == 0 && (((kLo | kHi) >> 1) & (kLo | kHi)) == 0, "disjoint result bits");
            const uint32_t f = (ok[0] & kLo) | (ok[1] & kHi) | (((ok[2] & kLo) | (ok[3] & kHi)) >> 1);
            return __popc(f & (vm.m | vm.m_hi));
        }
        constexpr uint32_t kRes = kPacked ? 0x20080200u : 0x80008000u;  // result bits of an ok word
        uint32_t f = ok[0] & kRes;
#pragma unroll
        for (int k = 1; k < kWords; ++k) f |= (ok[k] & kRes) >> k;
        return __popc(f & vm.m);
    }
    // Two series of exactly L columns, walked interleaved (independent chains).
    template <int L>
    __device__ __forceinline__ static uint32_t count2_fixed(uint32_t base, const uint32_t* pa,
                                                            const uint32_t* pb, const Mask& vm) {
        uint32_t wa[12], wb[12];
        load_offs(wa, pa, L);
        load_offs(wb, pb, L);
        uint32_t oka[kWords], okb[kWords];
#pragma unroll
        for (int k = 0; k < kWords; ++k) oka[k] = okb[k] = 0xffffffffu;
        uint4 preva = ld(base, wa[0]), prevb = ld(base, wb[0]);
#pragma unroll
        for (int i = 1; i < L; ++i) {
            const uint4 cura = ld(base, wa[i]);
            const uint4 curb = ld(base, wb[i]);
            step(oka, preva, cura, vm.k);
            step(okb, prevb, curb, vm.k);
            preva = cura;
            prevb = curb;
        }
        return tally(oka, vm) | (tally(okb, vm) << 16);
    }
    __device__ __forceinline__ static uint32_t count_any(uint32_t base, const uint32_t* pc,
                                                         uint32_t len, const Mask& vm) {
        uint32_t ok[kWords];
#pragma unroll
        for (int k = 0; k < kWords; ++k) ok[k] = 0xffffffffu;
        if (len > 1) {  // len <= 1: no adjacent pair, every row matches (fitness.hpp:80-90)
            uint4 prev = ld(base, pc[0]);
            for (uint32_t i = 1; i < len; ++i) {
                const uint4 cur = ld(base, pc[i]);
                step(ok, prev, cur, vm.k);
                prev = cur;
            }
        }
        return tally(ok, vm);
    }
    // SPG series of exactly L columns, walked interleaved (independent chains).
    // Column offsets are fetched 4 at a time (one LDS.128 per series) just
    // ahead of use, keeping 4 offset registers per series live instead of L.
    template <int L>
    __device__ __forceinline__ static uint32_t countN_fixed(uint32_t base, const WorkList& wl,
                                                            uint32_t g0, const Mask& vm) {
        const uint32_t* pc[SPG];
        uint4 w[SPG];
        uint32_t ok[SPG][kWords];
        uint4 prev[SPG];
#pragma unroll
        for (int q = 0; q < SPG; ++q) {
            pc[q] = wl.pcols + wl.sstart[g0 + q];
            w[q] = *reinterpret_cast<const uint4*>(pc[q]);
#pragma unroll
            for (int k = 0; k < kWords; ++k) ok[q][k] = 0xffffffffu;
            prev[q] = ld(base, w[q].x);
        }
#pragma unroll
        for (int i = 1; i < L; ++i) {
            if ((i & 3) == 0) {
#pragma unroll
                for (int q = 0; q < SPG; ++q) w[q] = *reinterpret_cast<const uint4*>(pc[q] + i);
            }
#pragma unroll
            for (int q = 0; q < SPG; ++q) {
                const uint32_t off = (i & 3) == 0 ? w[q].x : (i & 3) == 1 ? w[q].y : (i & 3) == 2 ? w[q].z : w[q].w;
                const uint4 cur = ld(base, off);
                step(ok[q], prev[q], cur, vm.k);
                prev[q] = cur;
            }
        }
        uint32_t c = 0;
#pragma unroll
        for (int q = 0; q < SPG; ++q) c |= tally(ok[q], vm) << (q * kFieldBits);
        return c;
    }

    // Counts of slots g0 .. g0+SPG-1 (packed kFieldBits-bit fields; a group
    // covers at most 64 rows, so 8 bits suffice).  `uniform`: every slot of
    // the warp's chunk exists and has length ulen.
    __device__ __forceinline__ static uint32_t count_group(const unsigned char* base_ptr,
                                                           const WorkList& wl, uint32_t g0,
                                                           uint32_t P, bool uniform, uint32_t ulen,
                                                           double, const Mask& vm) {
        const uint32_t base = smem_u32(base_ptr);
        if (uniform) {
            switch (ulen) {
                case 2: return countN_fixed<2>(base, wl, g0, vm);
                case 3: return countN_fixed<3>(base, wl, g0, vm);
                case 4: return countN_fixed<4>(base, wl, g0, vm);
                case 5: return countN_fixed<5>(base, wl, g0, vm);
                case 6: return countN_fixed<6>(base, wl, g0, vm);
                case 7: return countN_fixed<7>(base, wl, g0, vm);
                case 8: return countN_fixed<8>(base, wl, g0, vm);
                case 9: return countN_fixed<9>(base, wl, g0, vm);
                case 10: return countN_fixed<10>(base, wl, g0, vm);
                case 11: return countN_fixed<11>(base, wl, g0, vm);
                case 12: return countN_fixed<12>(base, wl, g0, vm);
                default: break;
            }
        }
        uint32_t c = 0;
#pragma unroll
        for (int q = 0; q < SPG; ++q)
            if (g0 + q < P)
                c |= count_any(base, wl.pcols + wl.sstart[g0 + q], wl.slen[g0 + q], vm) << (q * kFieldBits);
        return c;
    }
};

// Host-resident CBF (see CountParams::host_cbf): CTA 0's consumers copy it
// into device memory with one round of 16-byte PCIe reads and publish a
// release flag; every other CTA acquires it.  CTA 0 is normally resident
// first (CTAs start in index order), but nothing guarantees it -- with more
// CTAs than free SMs, or SMs held by another process -- so a CTA that has
// waited 20 us copies the (identical) bytes itself: forward progress never
// depends on another CTA being scheduled.
__device__ __forceinline__ void stage_host_cbf(const CountParams& p, int tid, int nthreads,
                                               int bar_id) {
    __shared__ int s_self;
    if (blockIdx.x == 0) {
        for (uint32_t i = tid; i < p.cbf_words; i += nthreads) p.dev_cbf[i] = p.host_cbf[i];
        __threadfence();
        named_bar_sync(bar_id, nthreads);
        // (EBIC_DEBUG_MODE=4, tests only: CTA 0 never publishes, so every
        // other CTA takes the self-copy path)
        if (tid == 0 && p.debug_mode != 4)
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p.cbf_ready), "r"(p.cbf_seq)
                         : "memory");
    } else {
        if (tid == 0) {
            const unsigned long long t0 = global_ns();
            uint32_t v;
            int self = 0;
            for (;;) {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p.cbf_ready) : "memory");
                if (v == p.cbf_seq) break;
                if (global_ns() - t0 > 20000ull) {
                    self = 1;
                    break;
                }
            }
            s_self = self;
        }
        named_bar_sync(bar_id, nthreads);
        if (s_self) {
            for (uint32_t i = tid; i < p.cbf_words; i += nthreads) p.dev_cbf[i] = p.host_cbf[i];
            __threadfence();
            named_bar_sync(bar_id, nthreads);
        }
    }
}

// ---------------------------------------------------------------------------
// K1: TMA-staged count kernel.
//
// Persistent CTAs (grid <= SMs) walk row tiles tile = blockIdx.x,
// blockIdx.x + gridDim.x, ...  A tile is RPG rows x all n_cols columns of the
// column-major matrix, brought into shared memory by one producer warp with 2D
// TMA boxes (RPG rows x box_cols columns, landing as [col][RPG] doubles) into a
// `stages`-deep mbarrier ring, so the matrix is read from HBM exactly once per
// launch.  NCW consumer warps evaluate EVERY series of the population against
// the staged tile.  A warp is split into GW lane groups of RPG/RPL lanes; a
// group walks one series, a lane RPL adjacent rows (RPL = 2: 16-byte LDS.128).
// Groups of one warp take consecutive slots of the length-sorted work list;
// when their lengths agree (the common case) the walk is fully unrolled with
// 8 column indices per LDS.128.  Row hits are reduced within the group with
// shuffles into per-CTA shared counters; the last CTA publishes counts and
// the fused Eq. 1 fitness.
// ---------------------------------------------------------------------------
template <class Walker, int NCW>
__global__ void __launch_bounds__((NCW + 1) * 32, 1)
    count_tma_kernel(const __grid_constant__ CUtensorMap tmap, const CountParams p) {
    constexpr int RPG = Walker::kRowsPerTile;
    constexpr int RPL = Walker::kRowsPerLane;
    constexpr int GL = RPG / RPL;    // lanes per group
    constexpr int GW = 32 / GL;      // groups per warp
    static_assert(GL >= 1 && GL <= 32 && (32 % GL) == 0, "bad lane grouping");

    extern __shared__ __align__(128) unsigned char smem_raw[];
    // TMA destinations need 128-byte alignment; static shared memory (the
    // epilogue flag) may precede the dynamic window, so align by offset
    // (pointer arithmetic on the shared array keeps LDS addressing).
    unsigned char* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
    const uint32_t P = p.n_series;
    unsigned char* stage_base = smem;
    uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + size_t(p.stages) * p.stage_bytes);
    uint64_t* empty_bar = full_bar + kMaxStages;
    uint64_t* prol_bar = empty_bar + kMaxStages;  // work list built (scratch stage released)
    unsigned char* persist = reinterpret_cast<unsigned char*>(prol_bar + 2);
    unsigned char* scratch = p.scratch_in_stage
                                 ? stage_base + size_t(p.stages - 1) * p.stage_bytes
                                 : align16(persist, count_persist_bytes(P, p.total_len));
    const WorkList wl = carve_work_list(persist, scratch, P, p.total_len);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    unsigned long long* stamp = p.phase_ns ? p.phase_ns + 8ull * blockIdx.x : nullptr;
    if (stamp && threadIdx.x == 0) stamp[0] = global_ns();

    if (threadIdx.x == 0) {
        for (uint32_t s = 0; s < p.stages; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], NCW);
        }
        mbar_init(prol_bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    // Work items.  Every full wave of tiles is one item per tile; the tiles of
    // a final partial wave are split into `parts` items by chunk range, so the
    // last wave keeps every CTA busy (each part re-loads its tile: a few MB of
    // extra traffic instead of one idle tile-time on most SMs).
    constexpr int SPG = Walker::kSeriesPerGroup;
    constexpr uint32_t CHUNK = GW * SPG;  // slots per warp-iteration
    const uint32_t n_chunks = (P + CHUNK - 1) / CHUNK;
    const uint32_t G = gridDim.x;
    const uint32_t full = (p.n_tiles / G) * G;
    const uint32_t rem = p.n_tiles - full;
    uint32_t parts = rem ? G / rem : 1u;
    parts = max(1u, min(parts, min(p.max_parts, n_chunks)));
    const uint32_t n_items = full + rem * parts;
    __shared__ uint32_t s_next[kMaxStages];  // per-stage chunk dispenser

    if (warp == NCW) {
        // ---------------- producer warp: TMA ring ----------------
        if (lane == 1 && p.fitness_out && p.table_n) {
            // Warm L2 with this CTA's slice of the Eq. 1 tables: the final CTA
            // looks entries up at arbitrary counts after the last tile.
            const uint64_t bytes = p.table_n * sizeof(double);
            const uint64_t per = ((bytes + gridDim.x - 1) / gridDim.x + 127) & ~uint64_t(127);
            const uint64_t lo = per * blockIdx.x;
            if (lo < bytes) {
                const uint32_t n = static_cast<uint32_t>(min(per, bytes - lo) & ~uint64_t(15));
                if (n) {
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(
                                     reinterpret_cast<const unsigned char*>(p.logt) + lo), "r"(n) : "memory");
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(
                                     reinterpret_cast<const unsigned char*>(p.expt) + lo), "r"(n) : "memory");
                }
            }
        }
        if (lane == 0) {
            uint32_t st = 0, phase = 0, issued = 0;
            for (uint32_t item = blockIdx.x; item < n_items; item += G, ++issued) {
                const uint32_t tile = item < full ? item : full + (item - full) / parts;
                // the last stage holds the prologue scratch until the work list is built
                if (p.scratch_in_stage && issued == p.stages - 1) mbar_wait(prol_bar, 0);
                mbar_wait(&empty_bar[st], phase ^ 1u);
                s_next[st] = 0;  // published to the consumers by the arrive below (release)
                if (p.debug_mode == 2) {
                    mbar_arrive(&full_bar[st]);
                } else {
                    mbar_arrive_expect_tx(&full_bar[st], p.stage_bytes);
                    unsigned char* dst = stage_base + size_t(st) * p.stage_bytes;
                    // fp64: column-major [cols][ld]; ranks: tile-major, the tensor
                    // viewed as [blocks * cols][64 u16] (one row per 128-byte block)
                    int c0, c1;
                    if constexpr (Walker::kTileMajor) {
                        c0 = static_cast<int>((tile % Walker::kSlicesPerBlock) * Walker::kDim0PerTile);
                        c1 = static_cast<int>((tile / Walker::kSlicesPerBlock) * p.n_cols);
                    } else {
                        c0 = static_cast<int>(tile * Walker::kDim0PerTile);
                        c1 = 0;
                    }
                    for (uint32_t b = 0; b < p.n_boxes; ++b)
                        tma_load_2d(dst + size_t(b) * p.box_cols * Walker::kColBytes, &tmap,
                                    &full_bar[st], c0, c1 + static_cast<int>(b * p.box_cols));
                }
                if (++st == p.stages) st = 0, phase ^= 1u;
            }
        }
    } else {
        // ---------------- consumer warps ----------------
        if (p.host_cbf) stage_host_cbf(p, threadIdx.x, NCW * 32, 1);
        build_work_list(p, wl, threadIdx.x, NCW * 32, 1, Walker::kColBytes);
        if (threadIdx.x == 0) mbar_arrive(prol_bar);
        if (stamp && threadIdx.x == 0) stamp[1] = global_ns();

        // Rows excluded from the layout (collapsed rank layout: two values
        // closer than eps, or NaN) are evaluated exactly in fp64 before the
        // first tile, while its TMA load is still in flight: one row per CTA
        // in turn (the last CTAs first: they carry no tail-split item), one
        // series per thread, reading a contiguous row copy (gathered once per
        // context) through L1.
        for (uint32_t i = G - 1 - blockIdx.x; i < p.n_excl; i += G) {
            const double* rowv = p.excl_vals + size_t(i) * p.n_cols;
            for (uint32_t g = threadIdx.x; g < P; g += NCW * 32) {
                const uint32_t len = wl.slen[g];
                const uint32_t* pc = wl.pcols + wl.sstart[g];
                bool ok = true;
                if (len > 1) {
                    double prev = __ldg(rowv + pc[0] / Walker::kColBytes);
                    for (uint32_t k = 1; k < len; ++k) {
                        const double cur = __ldg(rowv + pc[k] / Walker::kColBytes);
                        ok = ok & step_ok<false>(prev, cur, p.eps);
                        prev = cur;
                    }
                }
                if (ok) atomicAdd(&wl.cnt[g], 1u);
            }
        }

        const int grp = lane / GL;   // group within warp
        const int gl = lane % GL;    // lane within group
        const double eps = p.eps;
        const bool sched_static = p.sched_static != 0;

        uint32_t st = 0, phase = 0;
        for (uint32_t item = blockIdx.x; item < n_items; item += G) {
            uint32_t tile = item, c_lo = 0, c_hi = n_chunks;
            if (item >= full) {
                const uint32_t j = item - full, part = j % parts;
                tile = full + j / parts;
                c_lo = part * n_chunks / parts;
                c_hi = (part + 1) * n_chunks / parts;
            }
            // rows the layout cannot represent (fixed up below): the mask word is
            // fetched before the stage wait so its latency hides behind it
            uint32_t excl = 0;
            const uint32_t r0 = tile * RPG + gl * RPL;
            unsigned long long excl_word = 0ull;
            if (p.row_excl) excl_word = __ldg(p.row_excl + (r0 >> 6));
            mbar_wait(&full_bar[st], phase);
            const unsigned char* base = stage_base + size_t(st) * p.stage_bytes + gl * Walker::kLaneBytes;
            if (p.row_excl) excl = static_cast<uint32_t>(excl_word >> (r0 & 63)) & ((1u << RPL) - 1u);
            // rows of this tile that exist (the last tile may be partial)
            const typename Walker::Mask vmask = Walker::valid(r0, p.n_rows, excl, p.rank_k);

            // Chunks are handed out dynamically (longest first: slots are
            // sorted by ascending length) so the warps of the CTA finish a
            // tile together; the next index is fetched before the current
            // chunk is walked.
            const uint32_t n_here = c_hi - c_lo;
            uint32_t stat_k = warp;
            auto grab = [&]() {
                if (sched_static) {
                    const uint32_t v = stat_k;
                    stat_k += NCW;
                    return v;
                }
                uint32_t v = 0;
                if (lane == 0) v = atomicAdd(&s_next[st], 1u);
                return __shfl_sync(0xffffffffu, v, 0);
            };
            uint32_t k = p.debug_mode == 1 ? n_here : grab();
            while (k < n_here) {
                const uint32_t ch = c_hi - 1 - k;
                k = grab();
                const uint32_t first = ch * CHUNK;
                // Slots are sorted by length, so a full chunk is uniform iff its
                // first and last slots agree (lengths > 12 never take the
                // unrolled path, so the unsorted overflow bucket is harmless).
                const uint32_t ulen = wl.slen[first];
                const bool uniform = first + CHUNK <= P && wl.slen[first + CHUNK - 1] == ulen;
                const uint32_t g0 = first + grp * SPG;
                uint32_t c = Walker::count_group(base, wl, g0, P, uniform, ulen, eps, vmask);
#pragma unroll
                for (int o = GL / 2; o >= 1; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
                if (gl == 0) {
                    constexpr int kBits = 32 / SPG;
                    constexpr uint32_t kFieldMask = (kBits == 32) ? 0xffffffffu : ((1u << kBits) - 1u);
#pragma unroll
                    for (int q = 0; q < SPG; ++q) {
                        const uint32_t cq = (c >> (kBits * q)) & kFieldMask;
                        // warps on different tiles may hold the same chunk
                        if (g0 + q < P && cq) atomicAdd(&wl.cnt[g0 + q], cq);
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty_bar[st]);
            if (++st == p.stages) st = 0, phase ^= 1u;
        }
    }
    __syncthreads();
    if (stamp && threadIdx.x == 0) stamp[2] = global_ns();
    count_epilogue(p, wl.cnt, wl.sl);
    if (stamp && threadIdx.x == 0) stamp[3] = global_ns();
}

// ---------------------------------------------------------------------------
// K1 (direct): no staging; for matrices too wide for a shared-memory tile.
// Block = 8 warps over 256 consecutive rows (32 per warp); every warp walks
// every series for its rows; loads are coalesced 256-byte column slices of the
// column-major matrix (L1/L2 reuse across series).
// ---------------------------------------------------------------------------
template <bool kEpsZero>
__global__ void __launch_bounds__(256)
    count_direct_kernel(const CountParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    const uint32_t P = p.n_series;
    uint32_t* s_cnt = reinterpret_cast<uint32_t*>(smem);
    uint32_t* s_len = s_cnt + P;
    for (uint32_t s = threadIdx.x; s < P; s += blockDim.x) {
        s_cnt[s] = 0;
        s_len[s] = static_cast<uint32_t>(p.offsets[s + 1] - p.offsets[s]);
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t row = blockIdx.x * 256 + threadIdx.x;
    const bool valid = row < p.n_rows;
    const double* col0 = p.matrix + row;
    (void)warp;
    for (uint32_t s = 0; s < P; ++s) {
        const uint64_t a = p.offsets[s];
        const uint32_t len = s_len[s];
        bool ok = valid;
        if (valid && len > 1) {
            double prev = col0[size_t(p.cols[a]) * p.ld];
            for (uint32_t i = 1; i < len; ++i) {
                const double cur = col0[size_t(p.cols[a + i]) * p.ld];
                ok &= step_ok<kEpsZero>(prev, cur, p.eps);
                prev = cur;
            }
        }
        const uint32_t c = __popc(__ballot_sync(0xffffffffu, ok));
        if (lane == 0 && c) atomicAdd(&s_cnt[s], c);
    }
    __syncthreads();
    count_epilogue(p, s_cnt, nullptr);
}

// ---------------------------------------------------------------------------
// K4: rank layout builder (one CTA per row, rows [0, ld) incl. padding).
// Keys: the row's values v_j (plane 0) and, with PLANES == 2, fl(v_j + eps)
// computed exactly as the reference does (fitness.hpp:63, `cur + epsilon`).
// Bitonic sort in shared memory, dense ranks by a block scan of "new value"
// flags, scatter to the interleaved layout read by RankWalker.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t sortable_key(double x) {
    if (x != x) return ~0ull;  // NaN: not a value (fails every comparison)
    if (x == 0.0) x = 0.0;     // -0.0 and +0.0 compare equal
    const uint64_t u = static_cast<uint64_t>(__double_as_longlong(x));
    return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

__device__ __forceinline__ double key_value(uint64_t k) {
    const uint64_t u = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
    return __longlong_as_double(static_cast<long long>(u));
}

// PLANES == 1 && COLLAPSED (eps > 0): one plane of dense value ranks tested
// with <= ; valid for a row iff every distinct value s has fl(s + eps) > s and
// the next larger distinct value exceeds fl(s + eps) (then, for all a, b:
// v_a < fl(v_b + eps) <=> v_a <= v_b).  Rows failing that (or holding NaN)
// are flagged in dirty_out and evaluated exactly on the fp64 matrix.
template <int PLANES, bool COLLAPSED = false>
__global__ void __launch_bounds__(256)
    rank_build_kernel(const double* __restrict__ mat, uint32_t ld, uint32_t n_rows,
                      uint32_t n_cols, double eps, uint32_t Kp, uint16_t* __restrict__ out,
                      uint8_t* __restrict__ dirty_out = nullptr) {
    extern __shared__ __align__(16) unsigned char smem[];
    uint64_t* key = reinterpret_cast<uint64_t*>(smem);
    uint32_t* pay = reinterpret_cast<uint32_t*>(key + Kp);
    uint32_t* rk = pay + Kp;
    uint32_t* wsum = rk + Kp;
    const uint32_t r = blockIdx.x;
    const int tid = threadIdx.x, nt = blockDim.x;
    // Tile-major: 128-byte blocks [block][column][64 u16], a block holding 64
    // rows (one plane) or 32 rows as lo[4] hi[4] per 4 rows (two planes), so
    // a row tile is one contiguous n_cols * 128-byte range and any column
    // subset of it is a list of 128-byte slices.
    constexpr uint32_t kRowsPerBlock = PLANES == 2 ? 32 : 64;
    const size_t block_u16 = size_t(n_cols) * 64;
    auto at = [&](uint32_t c, uint32_t plane) -> size_t {
        const size_t b = size_t(r / kRowsPerBlock) * block_u16 + size_t(c) * 64;
        const uint32_t q = r % kRowsPerBlock;
        return PLANES == 2 ? b + (q >> 2) * 8 + plane * 4 + (q & 3) : b + q;
    };
    if (r >= n_rows) {  // padding rows: fail every test
        for (uint32_t c = tid; c < n_cols; c += nt) {
            if (PLANES == 2) {
                out[at(c, 0)] = 0xffff;
                out[at(c, 1)] = 0x8000;
            } else {
                out[at(c, 0)] = 0x8000;
            }
        }
        return;
    }
    const uint32_t K = PLANES * n_cols;
    __shared__ int s_dirty;
    if (tid == 0) s_dirty = 0;
    for (uint32_t i = tid; i < Kp; i += nt) {
        uint64_t k = ~0ull;
        uint32_t pl = 0xffffffffu;
        if (i < K) {
            const uint32_t plane = i >= n_cols ? 1u : 0u;
            const uint32_t c = i - plane * n_cols;
            double v = mat[size_t(c) * ld + r];
            if (plane) v = __dadd_rn(v, eps);
            k = sortable_key(v);
            pl = c | (plane << 16);
        }
        key[i] = k;
        pay[i] = pl;
    }
    __syncthreads();
    for (uint32_t size = 2; size <= Kp; size <<= 1) {
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            for (uint32_t i = tid; i < Kp / 2; i += nt) {
                const uint32_t lo = 2 * i - (i & (stride - 1));
                const uint32_t hi = lo + stride;
                const bool up = (lo & size) == 0;
                const uint64_t a = key[lo], b = key[hi];
                if ((a > b) == up) {
                    key[lo] = b;
                    key[hi] = a;
                    const uint32_t t = pay[lo];
                    pay[lo] = pay[hi];
                    pay[hi] = t;
                }
            }
            __syncthreads();
        }
    }
    auto is_new = [&](uint32_t i) -> uint32_t {
        return key[i] != ~0ull && (i == 0 || key[i] != key[i - 1]) ? 1u : 0u;
    };
    if (COLLAPSED) {
        for (uint32_t i = tid; i < K; i += nt) {
            if (key[i] == ~0ull) {  // NaN cell
                s_dirty = 1;
                continue;
            }
            const double x = key_value(key[i]);
            const double t = __dadd_rn(x, eps);
            bool bad = !(t > x);
            if (i + 1 < K && key[i + 1] != ~0ull && key[i + 1] != key[i])
                bad = bad || !(key_value(key[i + 1]) > t);
            if (bad) s_dirty = 1;
        }
        __syncthreads();
    }
    block_exclusive_scan(Kp, is_new, rk, wsum, tid, nt, 0);
    __syncthreads();
    for (uint32_t i = tid; i < Kp; i += nt) {
        const uint32_t pl = pay[i];
        if (pl == 0xffffffffu) continue;
        const uint32_t c = pl & 0xffffu, plane = pl >> 16;
        uint16_t v;
        if (key[i] == ~0ull) v = plane ? 0x8000 : 0xffff;  // NaN
        else v = static_cast<uint16_t>((rk[i] + is_new(i)) | 0x8000u);
        out[at(c, plane)] = v;
    }
    if (COLLAPSED && tid == 0) dirty_out[r] = static_cast<uint8_t>(s_dirty);
}

// One-plane 16-bit rank matrix (tile-major, 64-row blocks) -> the packed
// layout of RankWalker<3>: [tile][column][32 words], 96 rows per tile, row
// 3w + f in bits 10f..10f+9 of word w.  A cell r' = 0x8000 | r (r <= 0x1fe)
// becomes 0x200 | r, the NaN sentinel 0xffff becomes 0x3ff (above every
// rank, as 0xffff is), rows past the matrix 0x200 (masked by the kernel).
__global__ void rank_pack10_kernel(const uint16_t* __restrict__ in, uint32_t in_rows, uint32_t n_cols,
                                   uint32_t n_tiles, uint32_t* __restrict__ out) {
    const size_t n = size_t(n_tiles) * n_cols * 32;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
        const uint32_t w = static_cast<uint32_t>(i & 31);
        const size_t tc = i >> 5;
        const uint32_t c = static_cast<uint32_t>(tc % n_cols);
        const uint32_t t = static_cast<uint32_t>(tc / n_cols);
        uint32_t x = 0;
#pragma unroll
        for (int f = 0; f < 3; ++f) {
            const uint32_t r = t * 96 + 3 * w + f;
            uint32_t v = 0x200u;
            if (r < in_rows) {
                const uint32_t u = in[(size_t(r / 64) * n_cols + c) * 64 + (r % 64)];
                v = u == 0xffffu ? 0x3ffu : (0x200u | (u & 0x1ffu));
            }
            x |= v << (10 * f);
        }
        out[i] = x;
    }
}

// The same into RankWalker<4>: [tile][column][16 u64], 80 rows per tile, row
// 5w + f in bits 12f..12f+11 of word w; 0x800 | r (r <= 0x7fe), NaN 0xfff.
__global__ void rank_pack12_kernel(const uint16_t* __restrict__ in, uint32_t in_rows, uint32_t n_cols,
                                   uint32_t n_tiles, unsigned long long* __restrict__ out) {
    const size_t n = size_t(n_tiles) * n_cols * 16;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
        const uint32_t w = static_cast<uint32_t>(i & 15);
        const size_t tc = i >> 4;
        const uint32_t c = static_cast<uint32_t>(tc % n_cols);
        const uint32_t t = static_cast<uint32_t>(tc / n_cols);
        unsigned long long x = 0;
#pragma unroll
        for (int f = 0; f < 5; ++f) {
            const uint32_t r = t * 80 + 5 * w + f;
            unsigned long long v = 0x800u;
            if (r < in_rows) {
                const uint32_t u = in[(size_t(r / 64) * n_cols + c) * 64 + (r % 64)];
                v = u == 0xffffu ? 0xfffu : (0x800u | (u & 0x7ffu));
            }
            x |= v << (12 * f);
        }
        out[i] = x;
    }
}

// Row-major copy of selected rows of the column-major matrix (one CTA per row).
__global__ void gather_rows_kernel(const double* __restrict__ mat, size_t ld, uint32_t n_cols,
                                   const uint32_t* __restrict__ rows, double* __restrict__ out) {
    const uint32_t r = rows[blockIdx.x];
    for (uint32_t c = threadIdx.x; c < n_cols; c += blockDim.x)
        out[size_t(blockIdx.x) * n_cols + c] = mat[size_t(c) * ld + r];
}

// Sets *flag if any real (non-padding) cell of the column-major matrix is NaN.
__global__ void has_nan_kernel(const double* __restrict__ mat, size_t ld, size_t n_rows, size_t n,
                               int* __restrict__ flag) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
         i += size_t(gridDim.x) * blockDim.x)
        if ((i % ld) < n_rows && mat[i] != mat[i]) *flag = 1;
}

// ---------------------------------------------------------------------------
// K2: Eq. 1 over reduced counts (multi-shard path, after the all-reduce).
// ---------------------------------------------------------------------------
__global__ void fitness_kernel(const uint64_t* __restrict__ counts,
                               const uint64_t* __restrict__ offsets, uint32_t P, uint64_t sigma,
                               const double* __restrict__ logt, const double* __restrict__ expt,
                               double* __restrict__ fitness) {
    const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= P) return;
    fitness[s] = fitness_from_tables(counts[s], offsets[s + 1] - offsets[s], sigma, logt, expt);
}

// ---------------------------------------------------------------------------
// K3: membership bitmasks (Steps 6-7, expansion.hpp:16-87).  One thread per
// row; one warp writes half of a 64-row word per bitmask.  For every adjacent
// pair (a, b) = (v[s_{i-1}], v[s_i]):
//   forward  : a < b + eps        (fitness.hpp:63)
//   reversed : b < a + eps        (reversed series, expansion.hpp:58,64)
//   violation: !(a < b + eps)     (expansion.hpp:31)
// grid = (ceil(ld / 256), n_series); block = 256.
// ---------------------------------------------------------------------------
template <bool kEpsZero>
__global__ void __launch_bounds__(256)
    membership_kernel(const double* __restrict__ matrix, uint32_t ld, uint32_t n_rows,
                      const uint64_t* __restrict__ offsets, const uint16_t* __restrict__ cols,
                      double eps, uint64_t approx_k, uint32_t words,
                      uint64_t* __restrict__ exact_bits, uint64_t* __restrict__ neg_bits,
                      uint64_t* __restrict__ approx_bits) {
    const uint32_t s = blockIdx.y;
    const uint32_t row = blockIdx.x * 256 + threadIdx.x;
    const uint64_t a0 = offsets[s];
    const uint32_t len = static_cast<uint32_t>(offsets[s + 1] - a0);
    const bool valid = row < n_rows;
    bool fwd = true, rev = true;
    uint32_t viol = 0;
    if (valid) {
        const double* col0 = matrix + row;
        double prev = col0[size_t(cols[a0]) * ld];
        for (uint32_t i = 1; i < len; ++i) {
            const double cur = col0[size_t(cols[a0 + i]) * ld];
            const bool f = step_ok<kEpsZero>(prev, cur, eps);
            const bool r = step_ok<kEpsZero>(cur, prev, eps);
            fwd &= f;
            rev &= r;
            viol += f ? 0u : 1u;
            prev = cur;
        }
    }
    const uint32_t be = __ballot_sync(0xffffffffu, valid && fwd);
    const uint32_t bn = __ballot_sync(0xffffffffu, valid && rev);
    const uint32_t ba = __ballot_sync(0xffffffffu, valid && viol <= approx_k);
    if ((threadIdx.x & 31) == 0) {
        const uint32_t word = row >> 6;       // 64-row word
        const uint32_t half = (row >> 5) & 1;  // low/high 32 bits
        if (word < words) {
            const size_t idx = size_t(s) * words + word;
            if (exact_bits) reinterpret_cast<uint32_t*>(exact_bits + idx)[half] = be;
            if (neg_bits) reinterpret_cast<uint32_t*>(neg_bits + idx)[half] = bn;
            if (approx_bits) reinterpret_cast<uint32_t*>(approx_bits + idx)[half] = ba;
        }
    }
}

}  // namespace ebic_b200
