// K1s: series-split count kernel for short launches (included by ebic_b200.cu
// after kernels.cuh).
//
// Same contract as count_v2_kernel (counts + fused Eq. 1 per series of one
// CBF population over one shard's rank layout), organised the other way
// round.  K1v2 gives every CTA a slice of the rows and every series, which
// costs each CTA a length sort of the whole population before its walk and a
// cross-CTA sum of every series after it.  K1s gives every CTA a share of the
// work (series x row tiles, weighted by series length) and all the rows of
// its series:
//   * work unit = one series on one row tile, weight = its length; the units
//     are laid out series-major and CTA b takes those starting in
//     [ceil(b W / G), ceil((b + 1) W / G)), W = total length x tiles -- so a
//     CTA holds a few whole series plus at most one partial series at each
//     end, and no sort is needed;
//   * a lane group of 8 lanes tests one series on one tile: the column
//     slices (128 B per tile and column, the tile-major rank matrix) are read
//     straight from global memory / L2 into registers (no staging: a CTA's
//     few series share almost no columns), one 16-byte load per lane and
//     column, the same IADD3 + LOP3 pair tests and tally as RankWalker;
//   * whole series: the CTA writes count + Eq. 1 itself; a series split
//     between CTAs adds its part to a global accumulator and the last of its
//     parts (a per-series arrival counter) writes the result.
// Rows the collapsed layout cannot represent are tested in fp64 by the CTA
// that owns the row's tile for that series.  On the host path the population
// arrives as in K1v2 (stage_host_cbf) and a grid ticket raises the host flag.
// The trade: every CTA reads its columns' slices of all rows, so the bytes
// moved through L2 are rows x sum(len) x b instead of rows x U x b, and each
// lane group has only one series' loads in flight: the walk is bound by L2
// latency.  Measured (tools/kernel_probe.py): C1 (500 rows, 1.6 MB through
// L2) 16.6 us against K1v2's 18.5; C3 (5000 rows, 17 MB) 19.1 against 17.9;
// C4 (20,000 rows, 73 MB) 32 against 20.6 (ncu: L2 throughput 11 %, long-
// scoreboard stalls).  The host picks K1s below 4 MB of L2 reads.

namespace ebic_b200 {

constexpr int kSThreads = 512;     // 16 warps = 64 lane groups
// series of one CTA (the host keeps sum(len) <= kSMaxMine * grid, so a CTA's
// range of sum(len) x tiles / grid units holds at most ~sum(len) / (2 grid) + 2
// series of length >= 2)
constexpr int kSMaxMine = 256;

__device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

template <int PLANES>
__global__ void __launch_bounds__(kSThreads, 2) count_s_kernel(const __grid_constant__ CountParams p) {
    using W = RankWalker<PLANES, 128, 2>;
    constexpr uint32_t RPG = W::kRowsPerTile;
    constexpr uint32_t RPL = W::kRowsPerLane;
    constexpr uint32_t GL = 8;
    static_assert(RPG == GL * RPL, "8 lanes per tile");
    extern __shared__ __align__(16) unsigned char smem_s[];
    const uint32_t P = p.n_series, G = gridDim.x, T = p.n_tiles;
    const int tid = threadIdx.x, lane = tid & 31;
    uint32_t* rel = reinterpret_cast<uint32_t*>(smem_s);        // [P + 1] offsets - offsets[0]
    __shared__ uint32_t s_n_mine, s_tasks;
    __shared__ uint32_t m_s[kSMaxMine], m_tb[kSMaxMine], m_te[kSMaxMine], m_first[kSMaxMine + 1];
    __shared__ uint32_t m_cnt[kSMaxMine], m_cpos[kSMaxMine];
    unsigned long long* stamp = p.phase_ns ? p.phase_ns + 8ull * blockIdx.x : nullptr;
    if (stamp && tid == 0) stamp[0] = global_ns();

    if (p.host_cbf) stage_host_cbf(p, tid, kSThreads, 1);
    const uint64_t base = p.offsets[0];
    for (uint32_t i = tid; i <= P; i += kSThreads) rel[i] = static_cast<uint32_t>(__ldcg(p.offsets + i) - base);
    if (tid == 0) s_n_mine = 0;
    __syncthreads();

    // this CTA's units [lo, hi); W = total length x tiles
    const uint64_t Wt = uint64_t(rel[P]) * T;
    const uint64_t lo = (uint64_t(blockIdx.x) * Wt + G - 1) / G, hi = (uint64_t(blockIdx.x + 1) * Wt + G - 1) / G;
    auto owner = [&](uint64_t u) -> uint32_t {  // the CTA whose range holds unit u
        const uint64_t b = Wt ? u * G / Wt : 0;
        return static_cast<uint32_t>(b < G ? b : G - 1);
    };
    // my series: those with a task start in [lo, hi).  A series of length 0
    // or 1 has no adjacent pair -- every row matches -- and is written by the
    // owner of its first unit without a walk.
    for (uint32_t s = tid; s < P; s += kSThreads) {
        const uint32_t len = rel[s + 1] - rel[s];
        const uint64_t A = uint64_t(rel[s]) * T;
        if (len <= 1) {
            if (owner(A) == blockIdx.x) {
                p.counts_out[s] = p.n_rows;
                if (p.fitness_out) p.fitness_out[s] = fitness_from_tables(p.n_rows, len, p.sigma, p.logt, p.expt);
                if (p.done_flag) __threadfence_system();
            }
            continue;
        }
        const uint32_t tb = lo > A ? static_cast<uint32_t>(umin64(T, (lo - A + len - 1) / len)) : 0u;
        const uint32_t te = hi > A ? static_cast<uint32_t>(umin64(T, (hi - A + len - 1) / len)) : 0u;
        if (tb < te) {
            const uint32_t j = atomicAdd(&s_n_mine, 1u);
            if (j < kSMaxMine) {
                m_s[j] = s;
                m_tb[j] = tb;
                m_te[j] = te;
            }
        }
    }
    __syncthreads();
    const uint32_t n_mine = min(s_n_mine, static_cast<uint32_t>(kSMaxMine));
    if (tid < 32) {  // task prefix over my series (tasks of series j: [m_first[j], m_first[j+1]))
        uint32_t run = 0, crun = 0;  // and where each series' column list goes in shared memory
        for (uint32_t j0 = 0; j0 < n_mine; j0 += 32) {
            const uint32_t j = j0 + lane;
            const uint32_t n = j < n_mine ? m_te[j] - m_tb[j] : 0u;
            const uint32_t nc = j < n_mine ? rel[m_s[j] + 1] - rel[m_s[j]] : 0u;
            uint32_t x = n, y = nc;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t u = __shfl_up_sync(0xffffffffu, x, o), w = __shfl_up_sync(0xffffffffu, y, o);
                if (lane >= o) x += u, y += w;
            }
            if (j < n_mine) {
                m_first[j] = run + x - n;
                m_cpos[j] = crun + y - nc;
                m_cnt[j] = 0;
            }
            run += __shfl_sync(0xffffffffu, x, 31);
            crun += __shfl_sync(0xffffffffu, y, 31);
        }
        if (lane == 0) {
            m_first[n_mine] = run;
            s_tasks = run;
        }
    }
    __syncthreads();
    // my series' column lists as byte offsets of their 128-byte slices
    uint32_t* colb = rel + P + 1;
    for (uint32_t jj = tid / 32; jj < n_mine; jj += kSThreads / 32) {
        const uint32_t s = m_s[jj], len = rel[s + 1] - rel[s];
        for (uint32_t k = lane; k < len; k += 32) colb[m_cpos[jj] + k] = uint32_t(p.cols[base + rel[s] + k]) * 128u;
    }
    __syncthreads();
    if (stamp && tid == 0) stamp[1] = global_ns();

    // walk: lane group g takes tasks g, g + 64, ...; task -> (series j, tile)
    const uint32_t n_tasks = s_tasks;
    const uint32_t grp = tid / GL, gl = tid % GL, n_grp = kSThreads / GL;
    const typename W::Mask all_valid = W::valid(0, 0xffffffffu, 0u, p.rank_k);
    const size_t tile_bytes = size_t(p.n_cols) * 128u;
    const unsigned char* ranks = p.ranks + gl * 16u;
    uint32_t j = 0;
    for (uint32_t k = grp; k < n_tasks; k += n_grp) {
        while (m_first[j + 1] <= k) ++j;  // tasks ascend: j only moves forward
        const uint32_t s = m_s[j];
        const uint32_t tile = m_tb[j] + (k - m_first[j]);
        const uint32_t len = rel[s + 1] - rel[s];
        const uint32_t* cl = colb + m_cpos[j];
        const uint32_t r0 = tile * RPG + gl * RPL;
        typename W::Mask vm = all_valid;
        uint32_t excl = 0;
        if (p.row_excl) {
            const uint32_t wb = r0 >> 6, sh = r0 & 63u;
            const unsigned long long w0 = __ldg(p.row_excl + wb), w1 = __ldg(p.row_excl + wb + 1);
            excl = static_cast<uint32_t>(sh ? (w0 >> sh) | (w1 << (64 - sh)) : w0) & ((1u << RPL) - 1u);
        }
        if ((tile + 1) * RPG > p.n_rows || excl) vm = W::valid(r0, p.n_rows, excl, p.rank_k);
        const unsigned char* tb = ranks + size_t(tile) * tile_bytes;
        uint32_t ok[W::kWords];
#pragma unroll
        for (int q = 0; q < W::kWords; ++q) ok[q] = 0xffffffffu;
        if (len > 1) {
            // columns in batches of 8: loads issued together, then the chain
            uint4 prev = __ldcg(reinterpret_cast<const uint4*>(tb + cl[0]));
            for (uint32_t c0 = 1; c0 < len; c0 += 8) {
                uint4 v[8];
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    if (c0 + i < len) v[i] = __ldcg(reinterpret_cast<const uint4*>(tb + cl[c0 + i]));
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    if (c0 + i < len) {
                        W::step(ok, prev, v[i], vm.k);
                        prev = v[i];
                    }
            }
        }
        uint32_t c = W::tally(ok, vm);
        // the four groups of a warp may run different task counts: group mask
        const unsigned gmask = 0xffu << (lane & ~(GL - 1));
#pragma unroll
        for (int o = GL / 2; o >= 1; o >>= 1) c += __shfl_xor_sync(gmask, c, o, GL);
        if (gl == 0 && c) atomicAdd(&m_cnt[j], c);
    }
    __syncthreads();
    if (stamp && tid == 0) stamp[2] = global_ns();

    // rows the collapsed layout cannot represent: exact fp64 test, counted by
    // the CTA that owns the row's tile for the series
    for (uint32_t x = tid; x < n_mine * p.n_excl; x += kSThreads) {
        const uint32_t jj = x / p.n_excl, i = x % p.n_excl;
        const uint32_t tile = p.excl_rows[i] / RPG;
        if (tile < m_tb[jj] || tile >= m_te[jj]) continue;
        const uint32_t s = m_s[jj], len = rel[s + 1] - rel[s];
        const uint16_t* cl = p.cols + base + rel[s];
        const double* rowv = p.excl_vals + size_t(i) * p.n_cols;
        bool okr = true;
        if (len > 1) {
            double prev = __ldg(rowv + cl[0]);
            for (uint32_t k = 1; k < len; ++k) {
                const double cur = __ldg(rowv + cl[k]);
                okr = okr & step_ok<false>(prev, cur, p.eps);
                prev = cur;
            }
        }
        if (okr) atomicAdd(&m_cnt[jj], 1u);
    }
    __syncthreads();

    // results: whole series here; split ones through the accumulator
    uint32_t* g_cnt = p.partial;       // [P] partial counts (zero between launches)
    uint32_t* g_arrived = p.partial + P;  // [P] parts arrived
    for (uint32_t jj = tid; jj < n_mine; jj += kSThreads) {
        const uint32_t s = m_s[jj], len = rel[s + 1] - rel[s];
        uint64_t c = m_cnt[jj];
        const bool whole = m_tb[jj] == 0 && m_te[jj] == T;
        if (!whole) {
            // parts = CTAs holding at least one of the series' task starts (a
            // CTA range shorter than len may hold none)
            const uint64_t A = uint64_t(rel[s]) * T;
            uint32_t parts = 0;
            for (uint32_t b = owner(A), b1 = owner(A + uint64_t(T - 1) * len); b <= b1; ++b) {
                const uint64_t l = (uint64_t(b) * Wt + G - 1) / G, h = (uint64_t(b + 1) * Wt + G - 1) / G;
                const uint64_t t0 = l > A ? (l - A + len - 1) / len : 0, t1 = h > A ? (h - A + len - 1) / len : 0;
                parts += umin64(T, t0) < umin64(T, t1) ? 1u : 0u;
            }
            atomicAdd(g_cnt + s, static_cast<uint32_t>(c));
            uint32_t old;
            asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(g_arrived + s) : "memory");
            if (old + 1 != parts) continue;
            c = atomicExch(g_cnt + s, 0u);
            g_arrived[s] = 0;
        }
        p.counts_out[s] = c;
        if (p.fitness_out) p.fitness_out[s] = fitness_from_tables(c, len, p.sigma, p.logt, p.expt);
        if (p.done_flag) __threadfence_system();  // mapped host memory, before the ticket
    }
    if (stamp && tid == 0) stamp[3] = global_ns();
    if (p.done_flag) {
        // host path: every CTA's mapped writes, then one ticket; the last CTA
        // raises the flag
        __shared__ int s_last;
        __syncthreads();
        if (tid == 0) s_last = ticket_acq_rel(&p.done[kMaxGroups]) == G - 1;
        __syncthreads();
        if (!s_last) return;
        if (tid == 0) p.done[kMaxGroups] = 0u;
        signal_done(p);
    }
}

}  // namespace ebic_b200
