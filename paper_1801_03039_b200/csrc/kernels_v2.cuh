// kernels_v2.cuh -- K1v2: the count kernel over the tile-major rank matrix
// with column-compacted staging.
//
// Same contract as count_tma_kernel (per-series match counts of one
// population over one row shard + the fused Eq. 1 epilogue,
// /root/reference/proj/include/ebic/fitness.hpp:71-143); differences:
//
//  * Staging.  A launch references U of the matrix's C columns (GA batches:
//    U ~ 0.6 C at 200,000 x 1000, ~0.9 C at 20,000 x 500).  The rank matrix
//    is tile-major (rank_build_kernel: [block][column][128 B]), so the U
//    referenced slices of a row tile are the launch's runs of consecutive
//    referenced columns, each one contiguous range: the producer warps copy
//    one run per cp.async.bulk into consecutive slots of the stage.  HBM
//    moves rows x U x 2 B instead of rows x C x 2 B, and a stage of 64-row
//    tiles (128-byte slices: one whole bank row per lane group, no bank
//    conflicts) fits twice or more in shared memory where the full tile
//    fitted only with 32-row tiles.  The ring depth follows U at run time.
//  * Walk.  Slots are length-sorted; a chunk (8 consecutive slots, 4 lane
//    groups x 2 series) of one length <= kV2MaxUnroll is described by one word
//    (length, first list entry), so the walk loads no per-slot metadata:
//    slot lists are consecutive with stride pad4(length).  Chunks are
//    assigned to warps statically (longest first, rotated every tile), and
//    every lane adds its own partial counts into a private word of the chunk
//    (16-bit halves for the chunk's two series per group): no dispenser, no
//    per-chunk shuffles, no contended atomics; the words are summed once.
//
// Producer warps build the column bitmap, slots and runs from the CBF while
// the consumer warps sort the population; both meet at `cols_ready`.
#pragma once

#include "kernels.cuh"

namespace ebic_b200 {

constexpr int kV2MaxCols = 2048;    // bitmap of 64 words
constexpr int kV2Chunk = 8;         // slots per warp iteration (4 groups x 2 series)
constexpr int kV2MaxStages = 4;
#ifndef EBIC_V2_MAX_UNROLL
#define EBIC_V2_MAX_UNROLL 8
#endif
// longest series length with a fully unrolled chunk walk (longer: per-slot
// loop).  Fewer unrolled variants keep the walk's code in the instruction
// cache: C5 steady state 76.7 us at 12, 74.7 at 8, 74.1 at 6, 77.6 at 4
// (profiles/r02_kernel_variants.log); C4 unchanged.
constexpr uint32_t kV2MaxUnroll = EBIC_V2_MAX_UNROLL;
static_assert(kV2MaxUnroll >= 3 && kV2MaxUnroll <= 12, "unrolled chunk lengths 2..3+");
// The 10-bit packed layout (C <= 510: C1-C4) unrolls lengths 2..6 only: its
// launches walk one or two tiles per SM with a cold instruction cache (L2
// evicted between steps), so less walk code beats unrolled lengths 7-8 there
// (C4 19.9 -> 18.7 us per step, L2 evicted), while C5's long launches keep
// 2..8 (6: 61.8 -> 62.6 us back to back; profiles/r02_walk_ab.log, ab15).
#ifndef EBIC_V2_MAX_UNROLL_P10
#define EBIC_V2_MAX_UNROLL_P10 6
#endif
template <class W>
__host__ __device__ constexpr uint32_t v2_max_unroll() {
    return W::kPacked ? (EBIC_V2_MAX_UNROLL_P10 < kV2MaxUnroll ? EBIC_V2_MAX_UNROLL_P10 : kV2MaxUnroll) : kV2MaxUnroll;
}
constexpr uint32_t kV2ExclItems = 64;  // per-CTA items whose excl words are preloaded
// Stripes of the slot-order tail's fp32 accumulators.  One: 148 CTAs' 4-wide
// reductions per slot quad contend less than the final CTA's extra loads cost
// (same box, L2 evicted / warm / back to back, us: C4 20.71 / 18.46 / 15.62
// with 8 stripes, 20.59 / 18.35 / 15.18 with 4, 20.47 / 17.93 / 14.98 with 1;
// C5 68.1 -> 67.4 evicted; profiles/r02_walk_ab.log, ab12-ab14).
constexpr int kV2Stripes = 1;

// Byte offsets of the persistent work list inside the dynamic window.
struct V2Layout {
    uint32_t bars;      // full[kMaxStages], empty[kMaxStages], prol, cols  (u64)
    uint32_t misc;      // u32[16]: U, n_runs, stages, ...
    uint32_t next;      // u32[kMaxStages] chunk dispensers
    uint32_t sl, slen, sstart, cnt, cdesc;
    uint32_t pcols;     // u32[L + 3P], 16-byte aligned lists
    uint32_t bm, bases; // u32[64] each
    uint32_t ucols;     // u16[n_cols] slot -> column
    uint32_t runs, run_slot;  // u32[max_runs] each
    uint32_t acc;       // u32[n_chunks][32] per-lane partial counts
    uint32_t colw;      // u32[4][64] run-start / run-end word masks and prefix counts
    uint32_t excl;      // u64[2][kV2ExclItems] excl words of the CTA's items (a tile spans <= 2)
    uint32_t area;      // first byte of the stage area (128-aligned)
};

__host__ __device__ inline uint32_t v2_max_runs(uint32_t n_cols) { return (n_cols + 1) / 2 + 1; }

// Length buckets 2..kV2MaxUnroll are padded to whole chunks with dummy slots (so every
// chunk of those lengths is uniform), bucket 1 so that bucket 2 starts on a
// chunk: at most kV2Pad extra slots.
constexpr uint32_t kV2Pad = 7 * 12;

__host__ __device__ inline V2Layout v2_layout(uint32_t P0, uint32_t L0, uint32_t n_cols) {
    auto up16 = [](uint32_t x) { return (x + 15u) & ~15u; };
    const uint32_t P = P0 + kV2Pad;        // slots, dummies included
    const uint32_t L = L0 + kV2Pad * 12;  // list entries, dummies included
    V2Layout v;
    uint32_t at = 0;
    v.bars = at;     at += (2 * kMaxStages + 2) * 8;
    v.misc = at;     at += 16 * 4;
    v.next = at;     at += kMaxStages * 4;
    at = up16(at);
    // chunk descriptors first: their offset is a compile-time constant, so
    // the walk reads a chunk's descriptor at smem + imm instead of
    // re-deriving the P-dependent offset per chunk (ptxas rematerialised it:
    // ~18 instructions per chunk visit; C5 66.2 -> 64.2 us back to back)
    v.cdesc = at;    at = up16(at + 4 * ((P + kV2Chunk - 1) / kV2Chunk));
    v.sl = at;       at = up16(at + 4 * P);
    v.slen = at;     at = up16(at + 4 * P);
    v.sstart = at;   at = up16(at + 4 * P);
    v.cnt = at;      at = up16(at + 4 * (P + 4));  // + read as whole quads by the tail
    v.pcols = at;    at = up16(at + 4 * (L + 3 * P));
    v.bm = at;       at += 64 * 4;
    v.bases = at;    at += 64 * 4;
    v.ucols = at;    at = up16(at + 2 * n_cols);
    v.runs = at;     at = up16(at + 4 * v2_max_runs(n_cols));
    v.run_slot = at; at = up16(at + 4 * v2_max_runs(n_cols));
    v.acc = at;      at = up16(at + 4 * 32 * ((P + kV2Chunk - 1) / kV2Chunk));
    v.colw = at;     at = up16(at + 4 * 4 * 64);
    v.excl = at;     at = up16(at + 16 * kV2ExclItems);
    v.area = (at + 127u) & ~127u;
    return v;
}

// Prologue scratch (dead once the work list is built), at the END of the
// stage area: rel u32[P+1], raw u16[L+16], wh u32[ceil(P/32)*64], hist,
// hpad u32[64], wsum u32[32] -- the v1 builder's scratch.
__host__ __device__ inline uint32_t v2_scratch_bytes(uint32_t P, uint32_t L) {
    // + original bucket counts u32[64] + owner slot of each 4-entry quad of
    // the offset lists u16[(L + 3P + dummies) / 4]
    return static_cast<uint32_t>(count_scratch_bytes(P, L)) + 64 * 4 +
           ((2 * ((L + 3 * P + 12 * kV2Pad) / 4 + 16) + 15) & ~15u);
}

__device__ __forceinline__ uint32_t v2_slot_of(const uint32_t* bm, const uint32_t* bases, uint32_t c) {
    return bases[c >> 5] + __popc(bm[c >> 5] & ((1u << (c & 31)) - 1u));
}

// Producer warps: column bitmap, slots, runs (from the CBF).  NP warps mark
// the referenced columns; warp 0 turns the 64 bitmap words into slot bases
// and run-start / run-end word masks with their prefix counts; then every
// producer thread handles whole columns (slot -> column map, run starts and
// ends by rank in their word) and finally whole runs.  Four barriers, no
// serial per-bit loops.
template <int NP>
__device__ __forceinline__ void v2_build_columns(const CountParams& p, unsigned char* smem, const V2Layout& v,
                                                 int pw, int lane) {
    uint32_t* bm = reinterpret_cast<uint32_t*>(smem + v.bm);
    uint32_t* bases = reinterpret_cast<uint32_t*>(smem + v.bases);
    uint32_t* misc = reinterpret_cast<uint32_t*>(smem + v.misc);
    uint16_t* ucols = reinterpret_cast<uint16_t*>(smem + v.ucols);
    uint32_t* runs = reinterpret_cast<uint32_t*>(smem + v.runs);
    uint32_t* run_slot = reinterpret_cast<uint32_t*>(smem + v.run_slot);
    uint32_t* smask = reinterpret_cast<uint32_t*>(smem + v.colw);  // run-start bits [64]
    uint32_t* emask = smask + 64;                                  // run-end bits [64]
    uint32_t* sbase = emask + 64;                                  // starts before word w [64]
    uint32_t* ebase = sbase + 64;                                  // ends before word w [64]
    const int ptid = pw * 32 + lane;
    constexpr int nthr = NP * 32;
    for (int w = ptid; w < 64; w += nthr) bm[w] = 0;
    named_bar_sync(2, nthr);
    const uint32_t L = p.total_len;
    const uint16_t* src = p.cols + p.cols_base;
    const uint32_t shift = static_cast<uint32_t>((reinterpret_cast<uintptr_t>(src) & 15u) >> 1);
    const uint4* vsrc = reinterpret_cast<const uint4*>(src - shift);
    const uint32_t n_vec = (shift + L + 7u) >> 3;
    constexpr int kPer = 4;
    for (uint32_t i0 = ptid; i0 < n_vec; i0 += kPer * nthr) {
        uint4 x[kPer];
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            const uint32_t i = i0 + k * nthr;
            if (i < n_vec) x[k] = __ldcg(vsrc + i);
        }
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            const uint32_t i = i0 + k * nthr;
            if (i >= n_vec) continue;
#pragma unroll
            for (int h = 0; h < 8; ++h) {
                const uint32_t pos = i * 8 + h;  // position from the aligned word
                if (pos < shift || pos >= shift + L) continue;
                const uint32_t wv = h < 2 ? x[k].x : h < 4 ? x[k].y : h < 6 ? x[k].z : x[k].w;
                const uint32_t c = (wv >> (16 * (h & 1))) & 0xffffu;
                atomicOr(&bm[c >> 5], 1u << (c & 31));
            }
        }
    }
    named_bar_sync(2, nthr);
    if (pw == 0) {
        // word w = lane (low half) and lane + 32 (high half).  Gaps of <= p.gap
        // unreferenced columns between referenced ones are staged too (fewer,
        // longer copies); the staged set replaces the bitmap.
        uint32_t x0 = bm[lane], x1 = bm[lane + 32];
        const uint32_t w31 = __shfl_sync(0xffffffffu, x0, 31), w32 = __shfl_sync(0xffffffffu, x1, 0);
        if (p.gap) {
            const uint32_t a0 = __shfl_up_sync(0xffffffffu, x0, 1), a1 = __shfl_up_sync(0xffffffffu, x1, 1);
            const uint32_t n0 = __shfl_down_sync(0xffffffffu, x0, 1), n1 = __shfl_down_sync(0xffffffffu, x1, 1);
            const uint32_t pv0 = lane == 0 ? 0u : a0, pv1 = lane == 0 ? w31 : a1;
            const uint32_t nx0 = lane == 31 ? w32 : n0, nx1 = lane == 31 ? 0u : n1;
            auto fill = [&](uint32_t x, uint32_t prev, uint32_t next) {
                const uint32_t m1 = (x << 1) | (prev >> 31), m2 = (x << 2) | (prev >> 30);
                const uint32_t q1 = (x >> 1) | (next << 31), q2 = (x >> 2) | (next << 30);
                uint32_t f = m1 & q1;                        // gap of one column
                if (p.gap >= 2) f |= (m1 & q2) | (m2 & q1);  // gap of two
                return x | f;
            };
            const uint32_t c0 = fill(x0, pv0, nx0), c1 = fill(x1, pv1, nx1);
            x0 = c0;
            x1 = c1;
            bm[lane] = x0;
            bm[lane + 32] = x1;
        }
        auto excl_scan = [&](uint32_t a, uint32_t& total) {
            uint32_t incl = a;
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            total = __shfl_sync(0xffffffffu, incl, 31);
            return incl - a;
        };
        // neighbouring bits for run starts (previous column clear) and ends
        // (next column clear)
        const uint32_t g31 = __shfl_sync(0xffffffffu, x0, 31), g32 = __shfl_sync(0xffffffffu, x1, 0);
        const uint32_t up0 = __shfl_up_sync(0xffffffffu, x0 >> 31, 1), up1 = __shfl_up_sync(0xffffffffu, x1 >> 31, 1);
        const uint32_t dn0 = __shfl_down_sync(0xffffffffu, x0 & 1u, 1), dn1 = __shfl_down_sync(0xffffffffu, x1 & 1u, 1);
        const uint32_t pt0 = lane == 0 ? 0u : up0, pt1 = lane == 0 ? (g31 >> 31) : up1;
        const uint32_t nb0 = lane == 31 ? (g32 & 1u) : dn0, nb1 = lane == 31 ? 0u : dn1;
        const uint32_t s0 = x0 & ~((x0 << 1) | pt0), s1 = x1 & ~((x1 << 1) | pt1);
        const uint32_t e0 = x0 & ~((x0 >> 1) | (nb0 << 31)), e1 = x1 & ~((x1 >> 1) | (nb1 << 31));
        uint32_t t0, t1, ts0, ts1, te0, te1;
        const uint32_t b0 = excl_scan(__popc(x0), t0);
        const uint32_t b1 = t0 + excl_scan(__popc(x1), t1);
        const uint32_t rs0 = excl_scan(__popc(s0), ts0);
        const uint32_t rs1 = ts0 + excl_scan(__popc(s1), ts1);
        const uint32_t re0 = excl_scan(__popc(e0), te0);
        const uint32_t re1 = te0 + excl_scan(__popc(e1), te1);
        bases[lane] = b0;
        bases[lane + 32] = b1;
        smask[lane] = s0;
        smask[lane + 32] = s1;
        emask[lane] = e0;
        emask[lane + 32] = e1;
        sbase[lane] = rs0;
        sbase[lane + 32] = rs1;
        ebase[lane] = re0;
        ebase[lane + 32] = re1;
        if (lane == 0) {
            misc[0] = t0 + t1;    // U
            misc[1] = ts0 + ts1;  // runs
        }
    }
    named_bar_sync(2, nthr);
    // column-parallel: slot -> column map; run starts (into runs[]) and ends
    // (into run_slot[], temporarily), each at its rank
    for (uint32_t c = ptid; c < p.n_cols; c += nthr) {
        const uint32_t w = c >> 5, lt = (1u << (c & 31)) - 1u, bit = 1u << (c & 31);
        const uint32_t x = bm[w];
        if (x & bit) ucols[bases[w] + __popc(x & lt)] = static_cast<uint16_t>(c);
        const uint32_t sm = smask[w], em = emask[w];
        if (sm & bit) runs[sbase[w] + __popc(sm & lt)] = c;
        if (em & bit) run_slot[ebase[w] + __popc(em & lt)] = c;
    }
    named_bar_sync(2, nthr);
    const uint32_t n_runs = misc[1];
    for (uint32_t r = ptid; r < n_runs; r += nthr) {
        const uint32_t c0 = runs[r], c1 = run_slot[r];
        runs[r] = (c0 << 16) | (c1 - c0 + 1);
        run_slot[r] = v2_slot_of(bm, bases, c0);
    }
    named_bar_sync(2, nthr);
}

// Consumer-side work list (NCW warps): the v1 counting sort by length
// (build_work_list phases A-C), then lists of slot byte offsets (slot x 128)
// once the producer's column slots are ready, then chunk descriptors.
template <int CHUNK, uint32_t MAXU>
__device__ __forceinline__ void v2_build_work_list(const CountParams& p, unsigned char* smem, const V2Layout& v,
                                                   const WorkList& w, uint64_t* cols_ready, int tid, int nthreads,
                                                   int bar_id, uint32_t n_items, uint32_t full, uint32_t parts,
                                                   uint32_t rows_per_tile) {
    const uint32_t P = p.n_series, L = p.total_len;
    // excl words of this CTA's items (rows the layout cannot represent): the
    // loads ride along with the CBF's, no extra round trip before the walk
    unsigned long long* excl_items = reinterpret_cast<unsigned long long*>(smem + v.excl);
    if (p.row_excl && tid < kV2ExclItems) {
        const uint32_t item = blockIdx.x + tid * gridDim.x;
        unsigned long long x0 = 0ull, x1 = 0ull;
        if (item < n_items) {
            // the host pads the mask with two zero words past the last tile
            const uint32_t tile = item < full ? item : full + (item - full) / parts;
            const unsigned long long* w = p.row_excl + ((tile * rows_per_tile) >> 6);
            x0 = __ldg(w);
            x1 = __ldg(w + 1);
        }
        excl_items[2 * tid] = x0;
        excl_items[2 * tid + 1] = x1;
    }
    const uint32_t nblk = (P + 31) / 32;
    const int lane = tid & 31, nw = nthreads >> 5;
    const uint64_t base = p.cols_base;
    const uint16_t* src = p.cols + base;
    const uint32_t shift = static_cast<uint32_t>((reinterpret_cast<uintptr_t>(src) & 15u) >> 1);
    const uint4* vsrc = reinterpret_cast<const uint4*>(src - shift);
    const uint32_t n_vec = (shift + L + 7u) >> 3;
    constexpr int kPer = 4;
    for (uint32_t s0 = tid; s0 <= P || s0 < n_vec; s0 += kPer * nthreads) {
        uint64_t o[kPer];
        uint4 x[kPer];
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            const uint32_t i = s0 + k * nthreads;
            if (i <= P) o[k] = __ldcg(p.offsets + i);
            if (i < n_vec) x[k] = __ldcg(vsrc + i);
        }
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            const uint32_t i = s0 + k * nthreads;
            if (i <= P) w.rel[i] = static_cast<uint32_t>(o[k] - base) + shift;
            if (i < n_vec) reinterpret_cast<uint4*>(w.raw)[i] = x[k];
        }
    }
    for (uint32_t i = tid; i < nblk * kLenBuckets; i += nthreads) w.wh[i] = 0;
    for (int b = tid; b < kLenBuckets; b += nthreads) w.hist[b] = 0;
    for (uint32_t i = tid; i < P + kV2Pad + 4; i += nthreads) w.cnt[i] = 0;
    {
        uint32_t* acc = reinterpret_cast<uint32_t*>(smem + v.acc);
        const uint32_t n_acc = 32u * ((P + kV2Pad + CHUNK - 1) / CHUNK);
        for (uint32_t i = tid; i < n_acc; i += nthreads) acc[i] = 0;
    }
    named_bar_sync(bar_id, nthreads);  // 1
    if (p.phase_ns && blockIdx.x == 0 && tid == 0) p.phase_ns[8 * 600 + 1] = global_ns();

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
    named_bar_sync(bar_id, nthreads);  // 2
    if (p.phase_ns && blockIdx.x == 0 && tid == 0) p.phase_ns[8 * 600 + 2] = global_ns();

    uint32_t* orig = w.wsum + 32;  // original bucket counts
    uint16_t* owner = reinterpret_cast<uint16_t*>(orig + 64);  // quad -> slot
    if (tid < 32) {
        for (int k = 0; k < 2; ++k) orig[tid + 32 * k] = w.hist[tid + 32 * k];
        __syncwarp();
        for (int k = 0; k < 2; ++k) {
            const int b = tid + 32 * k;
            uint32_t c = orig[b];
            if (b >= 2 && b <= MAXU) c = (c + CHUNK - 1) / CHUNK * CHUNK;
            if (b == 1) c = (orig[0] + orig[1] + CHUNK - 1) / CHUNK * CHUNK - orig[0];
            w.hist[b] = c;
            w.hpad[b] = b < kLenBuckets - 1 ? c * pad4(b) : 0u;
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
    named_bar_sync(bar_id, nthreads);  // 3
    if (p.phase_ns && blockIdx.x == 0 && tid == 0) p.phase_ns[8 * 600 + 3] = global_ns();

    const uint32_t* bm = reinterpret_cast<const uint32_t*>(smem + v.bm);
    const uint32_t* bases = reinterpret_cast<const uint32_t*>(smem + v.bases);
    const bool compact = cols_ready != nullptr;
    auto slot_of = [&](uint32_t c) -> uint32_t { return compact ? v2_slot_of(bm, bases, c) : c; };
    const uint32_t lt = (1u << lane) - 1u;
    for (uint32_t blk = tid >> 5; blk < nblk; blk += nw) {
        uint32_t len;
        const uint32_t s = blk * 32 + lane;
        const uint32_t bkt = bucket_of(s, len);
        const uint32_t peers = __match_any_sync(0xffffffffu, bkt);
        if (bkt == 0xffffu) continue;
        const uint32_t r = w.wh[blk * kLenBuckets + bkt] + __popc(peers & lt);
        const uint32_t g = w.hist[bkt] + r;
        w.sl[g] = s;
        w.slen[g] = len;
        if (bkt < kLenBuckets - 1) {
            const uint32_t st = w.hpad[bkt] + r * pad4(len);
            w.sstart[g] = st;
            if (g % CHUNK == 0) {
                // chunk descriptor: (first list entry << 8) | length when the
                // whole chunk lies in this length's bucket (lists consecutive,
                // stride pad4(length)) and the length is unrolled (2..kV2MaxUnroll); else
                // 0 (per-slot path).  Bucket b ends where bucket b + 1 starts.
                const uint32_t end = w.hist[bkt + 1];
                const bool uni = g + CHUNK <= end && len >= 2 && len <= MAXU;
                reinterpret_cast<uint32_t*>(smem + v.cdesc)[g / CHUNK] = uni ? ((st << 8) | len) : 0u;
            }
            if (compact) {
                // owner of each 4-entry quad of the list (filled quad-parallel below)
                for (uint32_t q = 0; q < pad4(len) / 4; ++q) owner[st / 4 + q] = static_cast<uint16_t>(g);
            } else {
                // whole tiles: a column's slot is the column itself, so the
                // lane writes its series' list now (no second pass, no barrier)
                const uint16_t* from = w.raw + w.rel[s];
                for (uint32_t q = 0; q < pad4(len) / 4; ++q) {
                    uint4 o;
                    o.x = from[4 * q] * 128u;
                    o.y = 4 * q + 1 < len ? from[4 * q + 1] * 128u : 0u;
                    o.z = 4 * q + 2 < len ? from[4 * q + 2] * 128u : 0u;
                    o.w = 4 * q + 3 < len ? from[4 * q + 3] * 128u : 0u;
                    reinterpret_cast<uint4*>(w.pcols)[st / 4 + q] = o;
                }
            }
        }
    }
    if (p.phase_ns && blockIdx.x == 0 && tid == 0) p.phase_ns[8 * 601] = global_ns();
    // dummy slots of the padded buckets 1..12: no series (sl = ~0), a zero
    // offset list (slot 0's column); their counts are never read
    const uint32_t pslots = w.hist[kLenBuckets - 1] + orig[kLenBuckets - 1];  // slots incl. dummies
    for (uint32_t t = tid; t < 12 * CHUNK; t += nthreads) {
        const uint32_t b = 1 + t / CHUNK, j = t % CHUNK;
        const uint32_t bucket_slots = w.hist[b + 1] - w.hist[b];
        if (orig[b] + j >= bucket_slots) continue;
        const uint32_t r = orig[b] + j;
        const uint32_t g = w.hist[b] + r;
        const uint32_t st = w.hpad[b] + r * pad4(b);
        w.sl[g] = 0xffffffffu;
        w.slen[g] = b;
        w.sstart[g] = st;
        for (uint32_t q = 0; q < pad4(b) / 4; ++q) {
            if (compact) owner[st / 4 + q] = static_cast<uint16_t>(g);
            else reinterpret_cast<uint4*>(w.pcols)[st / 4 + q] = make_uint4(0u, 0u, 0u, 0u);
        }
        if (g % CHUNK == 0)
            reinterpret_cast<uint32_t*>(smem + v.cdesc)[g / CHUNK] = (b >= 2 && b <= MAXU) ? ((st << 8) | b) : 0u;
    }
    if (tid == 0) reinterpret_cast<uint32_t*>(smem + v.misc)[3] = pslots;
    if (p.phase_ns && blockIdx.x == 0 && tid == 0) p.phase_ns[8 * 601 + 1] = global_ns();
    // Compacted staging: the lists of buckets < 63, four entries per thread:
    // slot byte offsets of the series' columns, zero past its length (and for
    // dummies).  A series-per-thread fill would leave the longest series (and
    // its slot look-ups) on the critical path.
    if (compact) {
        // the producers' column set (bitmap + slot bases) is needed from
        // here on only: placement above ran while they built it
        mbar_wait(cols_ready, 0);
        named_bar_sync(bar_id, nthreads);  // 4a
        if (p.phase_ns && blockIdx.x == 0 && tid == 0) p.phase_ns[8 * 601 + 2] = global_ns();
        const uint32_t n_quads = w.hpad[kLenBuckets - 1] / 4;
        for (uint32_t j = tid; j < n_quads; j += nthreads) {
            const uint32_t g = owner[j];
            const uint32_t s = w.sl[g];
            uint4 o = make_uint4(0u, 0u, 0u, 0u);
            if (s != 0xffffffffu) {
                const uint32_t q = j - w.sstart[g] / 4, len = w.slen[g];
                const uint16_t* from = w.raw + w.rel[s] + 4 * q;
                const uint32_t n = min(4u, len - 4 * q);
                o.x = slot_of(from[0]) * 128u;
                if (n > 1) o.y = slot_of(from[1]) * 128u;
                if (n > 2) o.z = slot_of(from[2]) * 128u;
                if (n > 3) o.w = slot_of(from[3]) * 128u;
            }
            reinterpret_cast<uint4*>(w.pcols)[j] = o;
        }
    }
    named_bar_sync(bar_id, nthreads);  // 4
    if (p.phase_ns && blockIdx.x == 0 && tid == 0) p.phase_ns[8 * 600 + 4] = global_ns();

    const uint32_t ovf = w.hist[kLenBuckets - 1];
    const uint32_t P_slots = pslots;
    if (ovf < P_slots) {  // series of 63+ columns (uniform branch)
        if (tid == 0) {
            uint32_t run = w.hpad[kLenBuckets - 1];
            for (uint32_t g = ovf; g < P_slots; ++g) {
                w.sstart[g] = run;
                run += pad4(w.slen[g]);
            }
        }
        named_bar_sync(bar_id, nthreads);
        for (uint32_t g = ovf + tid; g < P_slots; g += nthreads) {
            const uint32_t len = w.slen[g], st = w.sstart[g];
            const uint16_t* from = w.raw + w.rel[w.sl[g]];
            for (uint32_t i = 0; i < pad4(len); ++i)
                w.pcols[st + i] = i < len ? slot_of(from[i]) * 128u : 0u;
        }
        // their chunks take the per-slot path (the chunk holding slot ovf - 1,
        // if shared, already has descriptor 0: it ends past its bucket)
        uint32_t* cdesc = reinterpret_cast<uint32_t*>(smem + v.cdesc);
        for (uint32_t ch = (ovf + CHUNK - 1) / CHUNK + tid; ch < (P_slots + CHUNK - 1) / CHUNK; ch += nthreads)
            cdesc[ch] = 0u;
        named_bar_sync(bar_id, nthreads);  // 5
    }
    if (p.phase_ns && blockIdx.x == 0 && tid == 0) p.phase_ns[8 * 600 + 5] = global_ns();
}

// Two series of exactly L columns per lane group; lists at pc and pc + stride.
// KS: 0 = the pair constant from vm.k at run time; 1 / 2 = the 64-bit packed
// layout's strict / collapsed constant at compile time (W::step_k).
template <class W, int L, int KS = 0>
__device__ __forceinline__ uint32_t v2_count2(uint32_t base, const uint32_t* pc, uint32_t stride,
                                              const typename W::Mask& vm) {
    constexpr int kWords = W::kWords;
    const uint32_t* pa = pc;
    const uint32_t* pb = pc + stride;
    uint4 wa = *reinterpret_cast<const uint4*>(pa);
    uint4 wb = *reinterpret_cast<const uint4*>(pb);
    uint32_t oka[kWords], okb[kWords];
#pragma unroll
    for (int k = 0; k < kWords; ++k) oka[k] = okb[k] = 0xffffffffu;
    uint4 preva = W::ld(base, wa.x), prevb = W::ld(base, wb.x);
#pragma unroll
    for (int i = 1; i < L; ++i) {
        if ((i & 3) == 0) {
            wa = *reinterpret_cast<const uint4*>(pa + i);
            wb = *reinterpret_cast<const uint4*>(pb + i);
        }
        const uint32_t oa = (i & 3) == 0 ? wa.x : (i & 3) == 1 ? wa.y : (i & 3) == 2 ? wa.z : wa.w;
        const uint32_t ob = (i & 3) == 0 ? wb.x : (i & 3) == 1 ? wb.y : (i & 3) == 2 ? wb.z : wb.w;
        const uint4 cura = W::ld(base, oa);
        const uint4 curb = W::ld(base, ob);
        if constexpr (KS == 0) {
            W::step(oka, preva, cura, vm.k);
            W::step(okb, prevb, curb, vm.k);
        } else {
            W::template step_k<KS == 1>(oka, preva, cura);
            W::template step_k<KS == 1>(okb, prevb, curb);
        }
        preva = cura;
        prevb = curb;
    }
    return W::tally(oka, vm) | (W::tally(okb, vm) << 16);
}

template <class W, int KS = 0>
__device__ __forceinline__ uint32_t v2_count_uniform(uint32_t L, uint32_t base, const uint32_t* pc, uint32_t stride,
                                                     const typename W::Mask& vm) {
    // (lengths above kV2MaxUnroll never get a uniform descriptor; their cases
    // alias the longest instantiation so no extra walk code is generated)
    constexpr uint32_t M = v2_max_unroll<W>();
    switch (L) {
        case 2: return v2_count2<W, 2, KS>(base, pc, stride, vm);
        case 3: return v2_count2<W, 3, KS>(base, pc, stride, vm);
        case 4: return v2_count2<W, (4 < M ? 4 : M), KS>(base, pc, stride, vm);
        case 5: return v2_count2<W, (5 < M ? 5 : M), KS>(base, pc, stride, vm);
        case 6: return v2_count2<W, (6 < M ? 6 : M), KS>(base, pc, stride, vm);
        case 7: return v2_count2<W, (7 < M ? 7 : M), KS>(base, pc, stride, vm);
        case 8: return v2_count2<W, (8 < M ? 8 : M), KS>(base, pc, stride, vm);
        case 9: return v2_count2<W, (9 < M ? 9 : M), KS>(base, pc, stride, vm);
        case 10: return v2_count2<W, (10 < M ? 10 : M), KS>(base, pc, stride, vm);
        case 11: return v2_count2<W, (11 < M ? 11 : M), KS>(base, pc, stride, vm);
        default: return v2_count2<W, M, KS>(base, pc, stride, vm);
    }
}

// The uniform chunk walk.  On the 64-bit packed layout the pair constant is
// a compile-time immediate (one walk per constant; a launch executes only one
// of them): 2 integer-pipe instructions per 64-bit word instead of 3.
#ifndef EBIC_V2_CONST_K
#define EBIC_V2_CONST_K 1
#endif
template <class W>
__device__ __forceinline__ uint32_t v2_count_chunk(uint32_t L, uint32_t base, const uint32_t* pc, uint32_t stride,
                                                   const typename W::Mask& vm) {
    if constexpr (W::kPacked64 && EBIC_V2_CONST_K) {
        return (vm.k & 1u) ? v2_count_uniform<W, 1>(L, base, pc, stride, vm)
                           : v2_count_uniform<W, 2>(L, base, pc, stride, vm);
    } else {
        return v2_count_uniform<W>(L, base, pc, stride, vm);
    }
}

// Cross-CTA tail in slot order (see the kernel).  Stripes [kV2Stripes][PS4]
// fp32, PS4 = the slot count rounded to a whole chunk (the host sizes them for P + kV2Pad
// slots); integer counts below 2^24 are exact in fp32.
template <int GL, int SPG, uint32_t CHUNK>
__device__ __forceinline__ void v2_tail_slots(const CountParams& p, const WorkList& wl, const uint32_t* acc,
                                              uint32_t P_slots, int warp, int lane) {
    static_assert(GL == 8 && SPG == 2 && CHUNK == 8, "chunk = 4 groups x 2 slots");
    const uint32_t PS4 = (p.n_series + kV2Pad + 7u) & ~7u;  // whole chunks
    float* stripes = reinterpret_cast<float*>(p.partial);
    const uint32_t stripe = blockIdx.x % kV2Stripes;
    unsigned long long* stamp = p.phase_ns ? p.phase_ns + 8ull * blockIdx.x : nullptr;
    // One thread per 4 consecutive slots: chunk q / 2, lane groups 2 (q % 2)
    // and 2 (q % 2) + 1 -- sixteen consecutive per-lane words (low / high
    // halves: the group's two slots), summed unpacked, plus the fp64 fix-up
    // rows, out as one 4-wide reduction.
    (void)warp, (void)lane;
    const uint32_t n_quads = (P_slots + 3) / 4;
    for (uint32_t q = threadIdx.x; q < n_quads; q += blockDim.x) {
        const uint4* a4 = reinterpret_cast<const uint4*>(acc + (q >> 1) * 32 + (q & 1) * 2 * GL);
        uint32_t c[4] = {0u, 0u, 0u, 0u};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const uint4 w = a4[i];
            const int h = 2 * (i >> 1);  // group 2 (q % 2) for words 0-7, the next for 8-15
            c[h] += (w.x & 0xffffu) + (w.y & 0xffffu) + (w.z & 0xffffu) + (w.w & 0xffffu);
            c[h + 1] += (w.x >> 16) + (w.y >> 16) + (w.z >> 16) + (w.w >> 16);
        }
        const uint32_t g = 4 * q;
        const uint4 f = *reinterpret_cast<const uint4*>(wl.cnt + g);  // zero past P_slots
        c[0] += f.x, c[1] += f.y, c[2] += f.z, c[3] += f.w;
        if ((c[0] | c[1] | c[2] | c[3]) && p.debug_mode != 5)
            asm volatile("red.relaxed.gpu.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(
                             stripes + size_t(stripe) * PS4 + g),
                         "f"(static_cast<float>(c[0])), "f"(static_cast<float>(c[1])), "f"(static_cast<float>(c[2])),
                         "f"(static_cast<float>(c[3]))
                         : "memory");
    }
    __shared__ int s_last;
    __syncthreads();
    if (stamp && threadIdx.x == 0) stamp[4] = global_ns();
    if (threadIdx.x == 0) s_last = ticket_acq_rel(&p.done[kMaxGroups]) == gridDim.x - 1;
    __syncthreads();
    if (stamp && threadIdx.x == 0) stamp[5] = global_ns();
    if (!s_last) return;
    if (stamp && threadIdx.x == 0) stamp[7] = global_ns();
    for (uint32_t g = threadIdx.x; g < P_slots; g += blockDim.x) {
        float v[kV2Stripes];
#pragma unroll
        for (int k = 0; k < kV2Stripes; ++k) v[k] = __ldcg(stripes + size_t(k) * PS4 + g);
        double t = 0.0;
#pragma unroll
        for (int k = 0; k < kV2Stripes; ++k) t += static_cast<double>(v[k]);
#pragma unroll
        for (int k = 0; k < kV2Stripes; ++k) __stcg(stripes + size_t(k) * PS4 + g, 0.0f);
        const uint32_t s = wl.sl[g];
        if (s == 0xffffffffu) continue;  // dummy slot
        const uint64_t c = static_cast<uint64_t>(t);
        if (p.xacc) {
            if (c) atomicAdd_system(p.xacc + s, static_cast<unsigned long long>(c));
            continue;
        }
        p.counts_out[s] = c;
        if (p.fitness_out) p.fitness_out[s] = fitness_from_tables(c, wl.slen[g], p.sigma, p.logt, p.expt);
    }
    if (threadIdx.x == 0) p.done[kMaxGroups] = 0u;
    if (p.xacc) {
        cross_shard_finish(p);
        return;
    }
    signal_done(p);
}

// ---------------------------------------------------------------------------
// K1v2.  PLANES: 1 (64-row tiles), 2 (32-row tiles) or 3 (one plane packed
// three rows per word, 96-row tiles); 128-byte slices.
// Grid: persistent, <= SMs; block: NCW consumer + NP producer warps.
// p.compact: stage the launch's referenced columns (runs); else whole tiles,
// one contiguous bulk copy each (short launches: no wait for the column set).
// ---------------------------------------------------------------------------
template <int PLANES, int NCW, int NP>
__global__ void __launch_bounds__((NCW + NP) * 32, 1)
    count_v2_kernel(const __grid_constant__ CountParams p) {
    using W = RankWalker<PLANES, 128, 2>;
    constexpr int RPG = W::kRowsPerTile;  // 64, 32 or 96
    constexpr int RPL = W::kRowsPerLane;
    constexpr int GL = RPG / RPL;         // 8 lanes per group
    constexpr int GW = 32 / GL;           // 4 groups per warp
    constexpr int SPG = 2;
    constexpr uint32_t CHUNK = GW * SPG;
    static_assert(CHUNK == kV2Chunk, "chunk geometry");

    extern __shared__ __align__(128) unsigned char smem_raw[];
    unsigned char* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
    const uint32_t P = p.n_series, Lt = p.total_len;
    const V2Layout v = v2_layout(P, Lt, p.n_cols);
    uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + v.bars);
    uint64_t* empty_bar = full_bar + kMaxStages;
    uint64_t* prol_bar = empty_bar + kMaxStages;
    uint64_t* cols_ready = prol_bar + 1;
    uint32_t* misc = reinterpret_cast<uint32_t*>(smem + v.misc);
    unsigned char* area = smem + v.area;
    const uint32_t area_bytes = p.smem_window - v.area;  // p.smem_window: usable dynamic bytes
    const uint32_t scratch_bytes = v2_scratch_bytes(P, Lt);
    unsigned char* scratch = area + ((area_bytes - scratch_bytes) & ~15u);
    const bool compact = p.compact != 0;

    WorkList wl;
    wl.sl = reinterpret_cast<uint32_t*>(smem + v.sl);
    wl.slen = reinterpret_cast<uint32_t*>(smem + v.slen);
    wl.sstart = reinterpret_cast<uint32_t*>(smem + v.sstart);
    wl.cnt = reinterpret_cast<uint32_t*>(smem + v.cnt);
    wl.pcols = reinterpret_cast<uint32_t*>(smem + v.pcols);
    {
        unsigned char* q = scratch;
        wl.rel = reinterpret_cast<uint32_t*>(q);
        q = align16(q, 4ull * (P + 1));
        wl.raw = reinterpret_cast<uint16_t*>(q);
        q = align16(q, 2ull * Lt + 32);
        wl.wh = reinterpret_cast<uint32_t*>(q);
        wl.hist = wl.wh + kLenBuckets * ((P + 31) / 32);
        wl.hpad = wl.hist + kLenBuckets;
        wl.wsum = wl.hpad + kLenBuckets;
    }
    const uint32_t* cdesc = reinterpret_cast<const uint32_t*>(smem + v.cdesc);
    const uint16_t* ucols = reinterpret_cast<const uint16_t*>(smem + v.ucols);
    uint32_t* acc = reinterpret_cast<uint32_t*>(smem + v.acc);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    // The parameter block is read from the constant bank; its first touch of
    // each line misses.  One lane per 32-byte line of it, in parallel, so the
    // prologue's (dependent) parameter reads hit.
    constexpr uint32_t kParamWords = sizeof(CountParams) / 4;
    if (warp == 1 && lane * 8 < kParamWords) {
        const uint32_t x = reinterpret_cast<const uint32_t*>(&p)[lane * 8];
        asm volatile("" ::"r"(x));
    }
    unsigned long long* stamp = p.phase_ns ? p.phase_ns + 8ull * blockIdx.x : nullptr;
    if (stamp && threadIdx.x == 0) stamp[0] = global_ns();
    if (threadIdx.x == 0) {
        for (int s = 0; s < kMaxStages; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], NCW);
        }
        mbar_init(prol_bar, 1);
        mbar_init(cols_ready, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    const uint32_t n_chunks = (P + CHUNK - 1) / CHUNK;
    const uint32_t G = gridDim.x;
    const uint32_t full = (p.n_tiles / G) * G;
    const uint32_t rem = p.n_tiles - full;
    uint32_t parts = rem ? G / rem : 1u;
    parts = max(1u, min(parts, min(p.max_parts, n_chunks)));
    const uint32_t n_items = full + rem * parts;

    if (warp >= NCW) {
        // ---------------- producer warps ----------------
        const int pw = warp - NCW;
        if (pw == 0 && lane == 1 && p.fitness_out && p.table_n) {
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
        if (pw == 0 && lane == 2 && p.reduce_striped == 2) {
            // this CTA's share of the slot stripes, so the tail's reductions
            // (and the release before its ticket) do not wait on DRAM fills
            const uint64_t bytes = uint64_t(kV2Stripes) * ((P + kV2Pad + 7u) & ~7u) * 4u;
            const uint64_t per = ((bytes + gridDim.x - 1) / gridDim.x + 127) & ~uint64_t(127);
            const uint64_t lo = per * blockIdx.x;
            if (lo < bytes) {
                const uint32_t n = static_cast<uint32_t>(min(per, bytes - lo) & ~uint64_t(15));
                if (n)
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(
                                     reinterpret_cast<const unsigned char*>(p.partial) + lo), "r"(n) : "memory");
            }
        }
        const unsigned char* ranks = p.ranks;
        const size_t block_bytes = size_t(p.n_cols) * 128u;
        const uint32_t scratch_at = static_cast<uint32_t>(scratch - area);
        const uint32_t full_addr0 = smem_u32(&full_bar[0]);
        const uint32_t area_addr = smem_u32(area);
        if (!compact) {
            // whole tiles: one contiguous block per tile, one thread
            if (pw == 0 && lane == 0 && p.debug_mode != 3) {
                const uint32_t stage_bytes = static_cast<uint32_t>(block_bytes), stages = p.stages;
                uint32_t st = 0, phase = 0, issued = 0;
                for (uint32_t item = blockIdx.x; item < n_items; item += G, ++issued) {
                    const uint32_t tile = item < full ? item : full + (item - full) / parts;
                    if (issued < stages && (st + 1) * stage_bytes > scratch_at) mbar_wait(prol_bar, 0);
                    mbar_wait(&empty_bar[st], phase ^ 1u);
                    if (p.debug_mode == 2) {
                        mbar_arrive(&full_bar[st]);
                    } else {
                        mbar_arrive_expect_tx(&full_bar[st], stage_bytes);
                        asm volatile(
                            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                                area_addr + st * stage_bytes),
                            "l"(ranks + size_t(tile) * block_bytes), "r"(stage_bytes), "r"(full_addr0 + st * 8u)
                            : "memory");
                    }
                    if (++st == stages) st = 0, phase ^= 1u;
                }
            }
        } else {
            // the host CBF is in device memory once this CTA's consumers are
            // past stage_host_cbf (barrier 3: consumers + producers)
            if (p.host_cbf) named_bar_sync(3, (NCW + NP) * 32);
            v2_build_columns<NP>(p, smem, v, pw, lane);
            if (pw == 0 && lane == 0) {
                const uint32_t sb = misc[0] * 128u;
                uint32_t n = sb ? min(static_cast<uint32_t>(kV2MaxStages), area_bytes / sb) : 1u;
                if (p.stages && p.stages < n) n = p.stages;  // EBIC_STAGES cap
                misc[2] = max(n, 1u);
                mbar_arrive(cols_ready);  // release: misc, runs, ucols, bm, bases
            }
            mbar_wait(cols_ready, 0);
            const uint32_t stage_bytes = misc[0] * 128u;
            const uint32_t stages = misc[2];
            const uint32_t n_runs = misc[1];
            const uint32_t* runs = reinterpret_cast<const uint32_t*>(smem + v.runs);
            const uint32_t* run_slot = reinterpret_cast<const uint32_t*>(smem + v.run_slot);
            // Copies issued by all producer lanes.  (A bulk copy takes uniform
            // operands, so a warp issues its lanes' copies one after another;
            // four warps keep enough in flight -- one thread alone is ~4x
            // slower, tools/probes/gather_probe.cu modes 8/9.)
            const uint32_t ptid = pw * 32 + lane;
            uint32_t st = 0, phase = 0, issued = 0;
            if (p.debug_mode != 3) {
                for (uint32_t item = blockIdx.x; item < n_items; item += G, ++issued) {
                    const uint32_t tile = item < full ? item : full + (item - full) / parts;
                    unsigned long long* is = (p.phase_ns && blockIdx.x == 0 && issued < 64)
                                                 ? p.phase_ns + 8ull * (512 + issued) : nullptr;
                    if (ptid == 0) {  // one thread waits; the others sleep in the named barrier
                        if (is) is[0] = global_ns();
                        if (issued < stages && (st + 1) * stage_bytes > scratch_at) mbar_wait(prol_bar, 0);
                        mbar_wait(&empty_bar[st], phase ^ 1u);
                        if (is) is[1] = global_ns();
                            if (p.debug_mode == 2) mbar_arrive(&full_bar[st]);
                        else mbar_arrive_expect_tx(&full_bar[st], stage_bytes);
                    }
                    named_bar_sync(2, NP * 32);
                    if (p.debug_mode != 2) {
                        const uint32_t dst = area_addr + st * stage_bytes;
                        const uint32_t bar = full_addr0 + st * 8u;
                        const unsigned char* srcb = ranks + size_t(tile) * block_bytes;
                        for (uint32_t r = ptid; r < n_runs; r += NP * 32) {
                            const uint32_t x = runs[r];
                            asm volatile(
                                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                                    dst + run_slot[r] * 128u),
                                "l"(srcb + size_t(x >> 16) * 128u), "r"((x & 0xffffu) * 128u), "r"(bar)
                                : "memory");
                        }
                        if (is && ptid == 0) is[2] = global_ns();
                        // Keep HBM busy beyond the ring: warm L2 with the
                        // block of the tile p.prefetch items ahead, so its
                        // copies into shared memory later come from L2.
                        if (p.prefetch && ptid == 32) {
                            const uint32_t ahead = item + p.prefetch * G;
                            if (ahead < n_items) {
                                const uint32_t ta = ahead < full ? ahead : full + (ahead - full) / parts;
                                const unsigned char* pb = ranks + size_t(ta) * block_bytes;
                                for (uint32_t o = 0; o < block_bytes; o += 65536u) {
                                    const uint32_t n = static_cast<uint32_t>(block_bytes - o < 65536u ? block_bytes - o : 65536u);
                                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(pb + o), "r"(n)
                                                 : "memory");
                                }
                            }
                        }
                    }
                    if (++st == stages) st = 0, phase ^= 1u;
                }
            }
        }
    } else {
        // ---------------- consumer warps ----------------
        if (p.host_cbf) {
            stage_host_cbf(p, threadIdx.x, NCW * 32, 1);
            if (compact) {
                __threadfence_block();
                named_bar_sync(3, (NCW + NP) * 32);  // releases the producers (column set)
            }
        }
        if (p.phase_ns && blockIdx.x == 0 && threadIdx.x == 0) p.phase_ns[8 * 600] = global_ns();
        v2_build_work_list<CHUNK, v2_max_unroll<W>()>(p, smem, v, wl, compact ? cols_ready : nullptr, threadIdx.x, NCW * 32, 1,
                                  n_items, full, parts, RPG);
        if (threadIdx.x == 0) mbar_arrive(prol_bar);
        if (stamp && threadIdx.x == 0) stamp[1] = global_ns();
        const uint32_t stages = compact ? misc[2] : p.stages;
        const uint32_t stage_bytes = compact ? misc[0] * 128u : p.n_cols * 128u;
        const uint32_t P_slots = misc[3];  // slots incl. the padded buckets' dummies
        const uint32_t n_chunks_s = (P_slots + CHUNK - 1) / CHUNK;

        // rows the collapsed layout cannot represent, evaluated in fp64 (see v1)
        for (uint32_t i = G - 1 - blockIdx.x; i < p.n_excl; i += G) {
            const double* rowv = p.excl_vals + size_t(i) * p.n_cols;
            for (uint32_t g = threadIdx.x; g < P_slots; g += NCW * 32) {
                const uint32_t len = wl.slen[g];
                const uint32_t* pc = wl.pcols + wl.sstart[g];
                auto col = [&](uint32_t off) -> uint32_t { return compact ? ucols[off >> 7] : (off >> 7); };
                bool ok = true;
                if (len > 1) {
                    double prev = __ldg(rowv + col(pc[0]));
                    for (uint32_t k = 1; k < len; ++k) {
                        const double cur = __ldg(rowv + col(pc[k]));
                        ok = ok & step_ok<false>(prev, cur, p.eps);
                        prev = cur;
                    }
                }
                if (ok) atomicAdd(&wl.cnt[g], 1u);
            }
        }

        const int grp = lane / GL;
        const int gl = lane % GL;
        const typename W::Mask all_valid = W::valid(0, 0xffffffffu, 0u, p.rank_k);
        const uint32_t area_addr = smem_u32(area) + gl * 16u;
        uint32_t st = 0, phase = 0;
        // excl words of this CTA's first kV2ExclItems items (rows the layout
        // cannot represent), loaded once instead of a dependent global load
        // per item right before its walk
        const unsigned long long* excl_items = reinterpret_cast<const unsigned long long*>(smem + v.excl);
        uint32_t it = 0;  // this CTA's item number
        uint32_t* const acc_lane = acc + lane;
        for (uint32_t item = blockIdx.x; item < n_items; item += G, ++it) {
            uint32_t tile = item, c_lo = 0, c_hi = n_chunks_s;
            if (item >= full) {  // a part of a last-wave tile: a chunk range
                const uint32_t j = item - full, part = j % parts;
                tile = full + j / parts;
                c_lo = part * n_chunks_s / parts;
                c_hi = (part + 1) * n_chunks_s / parts;
            }
            const uint32_t r0 = tile * RPG + gl * RPL;
            uint32_t excl = 0;
            if (p.row_excl) {
                // the lane's RPL rows within the tile's two mask words
                const uint32_t wb = (tile * RPG) >> 6, sh = r0 - 64u * wb;
                unsigned long long w0, w1;
                if (it < kV2ExclItems) {
                    w0 = excl_items[2 * it];
                    w1 = excl_items[2 * it + 1];
                } else {
                    w0 = __ldg(p.row_excl + wb);
                    w1 = __ldg(p.row_excl + wb + 1);
                }
                const unsigned long long win = sh >= 64 ? w1 >> (sh - 64) : sh ? (w0 >> sh) | (w1 << (64 - sh)) : w0;
                excl = static_cast<uint32_t>(win) & ((1u << RPL) - 1u);
            }
            if (p.debug_mode != 3) mbar_wait(&full_bar[st], phase);
            const uint32_t base = area_addr + st * stage_bytes;
            typename W::Mask vm = all_valid;
            if ((tile + 1) * RPG > p.n_rows || excl != 0u) vm = W::valid(r0, p.n_rows, excl, p.rank_k);

            if (p.debug_mode != 1) {
                // Chunks longest first, statically, in snake order: in round
                // j warp w takes the k-th longest for k = j NCW + w' (j even)
                // or j NCW + NCW - 1 - w' (j odd), w' = (w + 7 item) mod NCW;
                // the rotation evens each warp's share out over the tiles.
                // Each lane adds its own partial counts (16-bit halves: q = 0,
                // 1) to a private word of the chunk -- no shuffles, no
                // contended atomics.
                const uint32_t wr = (static_cast<uint32_t>(warp) + item * 7u) % NCW;
                // k-th longest chunk = chunk c_hi - 1 - k, walked by its index
                // directly (k steps alternate between dk and 2 NCW - dk)
                for (int ch = static_cast<int>(c_hi - 1u - wr), dk = 2 * (NCW - 1 - static_cast<int>(wr)) + 1;
                     ch >= static_cast<int>(c_lo); ch -= dk, dk = 2 * NCW - dk) {
                    const uint32_t d = cdesc[ch];
                    uint32_t c;
                    if (d) {
                        const uint32_t len = d & 0xffu;
                        const uint32_t stride = pad4(len);
                        c = v2_count_chunk<W>(len, base, wl.pcols + (d >> 8) + grp * SPG * stride, stride, vm);
                    } else {
                        const uint32_t g0 = ch * CHUNK + grp * SPG;
                        c = 0;
#pragma unroll
                        for (int q = 0; q < SPG; ++q)
                            if (g0 + q < P_slots)
                                c |= W::count_any(base, wl.pcols + wl.sstart[g0 + q], wl.slen[g0 + q], vm) << (16 * q);
                    }
                    atomicAdd(acc_lane + ch * 32, c);  // (no zero test: the branch costs more than the ATOMS)
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty_bar[st]);
            if (++st == stages) st = 0, phase ^= 1u;
        }
    }
    __syncthreads();
    if (stamp && threadIdx.x == 0) stamp[2] = global_ns();
    if (p.reduce_striped == 2) {
        // Slot-order tail: every CTA builds the same slot order, so the
        // stripes are indexed by slot ([kV2Stripes][whole chunks] fp32) and a
        // chunk's 8 slot counts go out as two 4-wide reductions straight
        // from the lane sums -- no series-order scatter; the last CTA maps
        // slots to series.
        v2_tail_slots<GL, SPG, CHUNK>(p, wl, acc, misc[3], warp, lane);
    } else {
        // Sum each chunk's per-lane words over its groups' lanes, add the fp64
        // fix-up rows, and store the CTA's counts by series (the stage area
        // is idle now) for the cross-CTA tail.
        uint32_t* by_series = reinterpret_cast<uint32_t*>(area);
        const int nwarps = blockDim.x >> 5;
        const int grp = lane / GL, gl = lane % GL;
        for (uint32_t i = threadIdx.x; i < ((P + 3u) & ~3u); i += blockDim.x) by_series[i] = 0;
        __syncthreads();
        const uint32_t P_slots = misc[3];
        for (uint32_t ch = warp; ch < (P_slots + CHUNK - 1) / CHUNK; ch += nwarps) {
            // the two 16-bit halves summed apart: a CTA's count may pass 2^16
            uint32_t x = acc[ch * 32 + lane], lo = x & 0xffffu, hi = x >> 16;
#pragma unroll
            for (int o = GL / 2; o >= 1; o >>= 1) {
                lo += __shfl_xor_sync(0xffffffffu, lo, o);
                hi += __shfl_xor_sync(0xffffffffu, hi, o);
            }
            const uint32_t g0 = ch * CHUNK + grp * SPG;
            if (gl == 0) {
#pragma unroll
                for (int q = 0; q < SPG; ++q) {
                    const uint32_t s = g0 + q < P_slots ? wl.sl[g0 + q] : 0xffffffffu;
                    if (s != 0xffffffffu) by_series[s] = wl.cnt[g0 + q] + (q ? hi : lo);
                }
            }
        }
        __syncthreads();
        count_epilogue(p, by_series, nullptr);
    }
    if (stamp && threadIdx.x == 0) stamp[3] = global_ns();
}

}  // namespace ebic_b200
