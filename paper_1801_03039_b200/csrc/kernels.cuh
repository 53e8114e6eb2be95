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
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@P1 bra DONE_%=;\n"
        "bra WAIT_%=;\n"
        "DONE_%=:\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
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
    unsigned long long* __restrict__ acc;  // [P] zero on entry; zero again on exit
    unsigned int* __restrict__ done;       // grid arrival counter (zero on entry and exit)
    uint64_t* __restrict__ counts_out;     // [P]
    double* __restrict__ fitness_out;      // [P] or nullptr
    const double* __restrict__ logt;       // fitness tables (nullptr if no fitness)
    const double* __restrict__ expt;
    const double* __restrict__ matrix;     // column-major (direct kernel only)
    uint32_t ld;                           // leading dimension (direct kernel only)
};

// Smem layout: [stages * stage_bytes][mbar full/empty][meta]; meta =
//   s_start  u32[P]  first column position of series (in s_cols)
//   s_len    u32[P]
//   s_order  u32[P]  series ids sorted by length bucket
//   s_cnt    u32[P]  per-CTA match counts
//   s_cols   u16[total_len]
//   s_hist   u32[kLenBuckets]
__host__ __device__ inline size_t count_meta_bytes(uint32_t P, uint32_t total_len) {
    size_t b = 4ull * P * 4 + 2ull * total_len;
    b = (b + 15) & ~size_t(15);
    return b + 4ull * kLenBuckets + 16;
}

// Cooperative (all `nthreads` threads of the group) construction of the work
// list: series lengths, a length-bucketed order (so the lane groups of one warp
// walk equally long series), zeroed counters and the column list in smem.
__device__ __forceinline__ void build_work_list(const CountParams& p, uint32_t* s_start,
                                                uint32_t* s_len, uint32_t* s_order,
                                                uint32_t* s_cnt, uint16_t* s_cols, uint32_t* s_hist,
                                                int tid, int nthreads, int bar_id) {
    const uint32_t P = p.n_series;
    for (int b = tid; b < kLenBuckets; b += nthreads) s_hist[b] = 0;
    named_bar_sync(bar_id, nthreads);
    // A launch may cover a slice of a larger population: positions are taken
    // relative to offsets[0].
    const uint64_t base = p.offsets[0];
    for (uint32_t s = tid; s < P; s += nthreads) {
        const uint64_t a = p.offsets[s], e = p.offsets[s + 1];
        const uint32_t len = static_cast<uint32_t>(e - a);
        s_start[s] = static_cast<uint32_t>(a - base);
        s_len[s] = len;
        s_cnt[s] = 0;
        atomicAdd(&s_hist[len < kLenBuckets ? len : kLenBuckets - 1], 1u);
    }
    for (uint32_t i = tid; i < p.total_len; i += nthreads) s_cols[i] = p.cols[base + i];
    named_bar_sync(bar_id, nthreads);
    if (tid < 32) {  // exclusive scan of 64 buckets by one warp
        uint32_t a = s_hist[tid], b = s_hist[tid + 32];
        uint32_t x = a;
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (tid >= o) x += y;
        }
        const uint32_t total_a = __shfl_sync(0xffffffffu, x, 31);
        uint32_t z = b;
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xffffffffu, z, o);
            if (tid >= o) z += y;
        }
        s_hist[tid] = x - a;
        s_hist[tid + 32] = total_a + z - b;
    }
    named_bar_sync(bar_id, nthreads);
    for (uint32_t s = tid; s < P; s += nthreads) {
        const uint32_t len = s_len[s];
        const uint32_t pos = atomicAdd(&s_hist[len < kLenBuckets ? len : kLenBuckets - 1], 1u);
        s_order[pos] = s;
    }
    named_bar_sync(bar_id, nthreads);
}

// Grid-wide reduction tail shared by both count kernels: per-CTA counts are
// added to the global accumulator; the last CTA to arrive publishes the final
// counts (and Eq. 1 fitness when tables are given) and re-zeroes the
// accumulator and arrival counter for the next launch.
__device__ __forceinline__ void count_epilogue(const CountParams& p, const uint32_t* s_cnt,
                                               const uint32_t* s_len) {
    const uint32_t P = p.n_series;
    for (uint32_t s = threadIdx.x; s < P; s += blockDim.x) {
        const uint32_t c = s_cnt[s];
        if (c) atomicAdd(&p.acc[s], static_cast<unsigned long long>(c));
    }
    __threadfence();
    __syncthreads();
    __shared__ int s_last;
    if (threadIdx.x == 0) s_last = (atomicAdd(p.done, 1u) == gridDim.x - 1);
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    for (uint32_t s = threadIdx.x; s < P; s += blockDim.x) {
        const uint64_t c = atomicExch(&p.acc[s], 0ull);
        p.counts_out[s] = c;
        if (p.fitness_out) p.fitness_out[s] = fitness_from_tables(c, s_len[s], p.sigma, p.logt, p.expt);
    }
    if (threadIdx.x == 0) *p.done = 0u;
}

// ---------------------------------------------------------------------------
// K1: TMA-staged count kernel.
//
// Persistent CTAs (grid <= SMs x occupancy) walk row tiles tile = blockIdx.x,
// blockIdx.x + gridDim.x, ...  A tile is RPG rows x all n_cols columns of the
// column-major matrix, brought into shared memory by one producer warp with 2D
// TMA boxes (RPG rows x box_cols columns, landing as [col][RPG] doubles) into a
// `stages`-deep mbarrier ring.  NCW consumer warps then evaluate EVERY series of
// the population against the staged tile, so the matrix is read from HBM once
// per launch.  A warp is split into lane groups of RPG/RPL lanes; each group
// walks one series, each lane RPL adjacent rows (RPL = 2 -> 16-byte LDS.128).
// The walk is branch-free (AND of every adjacent test; identical boolean to the
// reference's early exit), groups of a warp take consecutive entries of the
// length-sorted order so they rarely diverge, and row hits are counted with
// __ballot_sync + __popc into per-CTA shared counters.
// ---------------------------------------------------------------------------
template <int RPG, int RPL, int NCW, bool kEpsZero>
__global__ void __launch_bounds__((NCW + 1) * 32, 1)
    count_tma_kernel(const __grid_constant__ CUtensorMap tmap, const CountParams p) {
    constexpr int GL = RPG / RPL;    // lanes per group
    constexpr int GW = 32 / GL;      // groups per warp
    static_assert(GL >= 1 && GL <= 32 && (32 % GL) == 0, "bad lane grouping");
    constexpr int kColBytesShift = (RPG == 32) ? 8 : (RPG == 16) ? 7 : (RPG == 8) ? 6 : (RPG == 4) ? 5 : 4;
    static_assert((1 << kColBytesShift) == RPG * 8, "RPG must be a power of two in [2,32]");

    extern __shared__ __align__(128) unsigned char smem_raw[];
    // TMA destinations need 128-byte alignment; static shared memory (the
    // epilogue flag) may precede the dynamic window, so align explicitly.
    unsigned char* smem = reinterpret_cast<unsigned char*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
    const uint32_t P = p.n_series;
    unsigned char* stage_base = smem;
    uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + size_t(p.stages) * p.stage_bytes);
    uint64_t* empty_bar = full_bar + kMaxStages;
    uint32_t* s_start = reinterpret_cast<uint32_t*>(empty_bar + kMaxStages);
    uint32_t* s_len = s_start + P;
    uint32_t* s_order = s_len + P;
    uint32_t* s_cnt = s_order + P;
    uint16_t* s_cols = reinterpret_cast<uint16_t*>(s_cnt + P);
    uint32_t* s_hist = reinterpret_cast<uint32_t*>(
        reinterpret_cast<uintptr_t>(s_cols + p.total_len + 7) & ~uintptr_t(15));

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (uint32_t s = 0; s < p.stages; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], NCW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == NCW) {
        // ---------------- producer warp: TMA ring ----------------
        if (lane == 0) {
            uint32_t it = 0;
            for (uint32_t tile = blockIdx.x; tile < p.n_tiles; tile += gridDim.x, ++it) {
                const uint32_t st = it % p.stages;
                const uint32_t round = it / p.stages;
                mbar_wait(&empty_bar[st], (round & 1u) ^ 1u);
                mbar_arrive_expect_tx(&full_bar[st], p.stage_bytes);
                unsigned char* dst = stage_base + size_t(st) * p.stage_bytes;
                for (uint32_t b = 0; b < p.n_boxes; ++b)
                    tma_load_2d(dst + size_t(b) * p.box_cols * RPG * 8, &tmap, &full_bar[st],
                                static_cast<int>(tile * RPG), static_cast<int>(b * p.box_cols));
            }
        }
    } else {
        // ---------------- consumer warps ----------------
        build_work_list(p, s_start, s_len, s_order, s_cnt, s_cols, s_hist, threadIdx.x, NCW * 32, 1);

        const int grp = lane / GL;               // group within warp
        const int gl = lane % GL;                // lane within group
        const uint32_t gmask = (GL == 32) ? 0xffffffffu : (((1u << GL) - 1u) << (grp * GL));
        const uint32_t per_round = NCW * GW;
        const uint32_t n_rounds = (P + per_round - 1) / per_round;
        const double eps = p.eps;

        uint32_t it = 0;
        for (uint32_t tile = blockIdx.x; tile < p.n_tiles; tile += gridDim.x, ++it) {
            const uint32_t st = it % p.stages;
            mbar_wait(&full_bar[st], (it / p.stages) & 1u);
            const unsigned char* base = stage_base + size_t(st) * p.stage_bytes + gl * (RPL * 8);
            // rows of this tile that exist (the last tile may be partial)
            const uint32_t row0 = tile * RPG + gl * RPL;
            const bool v0 = row0 < p.n_rows;
            const bool v1 = (RPL == 2) && (row0 + 1 < p.n_rows);

            for (uint32_t r = 0; r < n_rounds; ++r) {
                const uint32_t g = (r * NCW + warp) * GW + grp;
                bool ok0 = false, ok1 = false;
                uint32_t s = 0;
                if (g < P) {
                    s = s_order[g];
                    const uint32_t a = s_start[s];
                    const uint32_t len = s_len[s];
                    if (len <= 1) {
                        // No adjacent pair: the reference's loop body never runs and
                        // the row matches (fitness.hpp:80-90).
                        ok0 = v0;
                        ok1 = v1;
                    } else if (RPL == 1) {
                        double prev = *reinterpret_cast<const double*>(
                            base + (uint32_t(s_cols[a]) << kColBytesShift));
                        bool ok = true;
                        for (uint32_t i = 1; i < len; ++i) {
                            const double cur = *reinterpret_cast<const double*>(
                                base + (uint32_t(s_cols[a + i]) << kColBytesShift));
                            ok &= step_ok<kEpsZero>(prev, cur, eps);
                            prev = cur;
                        }
                        ok0 = ok && v0;
                    } else {
                        double2 prev = *reinterpret_cast<const double2*>(
                            base + (uint32_t(s_cols[a]) << kColBytesShift));
                        bool oka = true, okb = true;
                        for (uint32_t i = 1; i < len; ++i) {
                            const double2 cur = *reinterpret_cast<const double2*>(
                                base + (uint32_t(s_cols[a + i]) << kColBytesShift));
                            oka &= step_ok<kEpsZero>(prev.x, cur.x, eps);
                            okb &= step_ok<kEpsZero>(prev.y, cur.y, eps);
                            prev = cur;
                        }
                        ok0 = oka && v0;
                        ok1 = okb && v1;
                    }
                }
                const uint32_t b0 = __ballot_sync(0xffffffffu, ok0);
                uint32_t c = __popc(b0 & gmask);
                if (RPL == 2) {
                    const uint32_t b1 = __ballot_sync(0xffffffffu, ok1);
                    c += __popc(b1 & gmask);
                }
                if (gl == 0 && g < P && c) s_cnt[s] += c;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty_bar[st]);
        }
    }
    __syncthreads();
    count_epilogue(p, s_cnt, s_len);
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
    count_epilogue(p, s_cnt, s_len);
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
