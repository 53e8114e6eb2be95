// ebic_b200.cu -- context management and the C ABI (include/ebic_b200.h).
//
// Replaces, B200-first, the reference's evaluation engine and its CPU runtime:
//   make_chunk_plan / ThreadPool / count_chunk / count_matches / evaluate_population
//     (/root/reference/proj/include/ebic/fitness.hpp:30-143, parallel.hpp:17-89)
//   assign_rows / trend_violations / expand_bicluster
//     (/root/reference/proj/include/ebic/expansion.hpp:16-87)
// Row chunks become per-device row shards held column-major in HBM; one kernel
// launch evaluates a whole generation against a shard.
#include <cuda.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <unistd.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <atomic>
#include <condition_variable>
#include <exception>
#include <functional>
#include <map>
#include <thread>
#include <string>
#include <vector>

#include "../../include/ebic_b200.h"
#include "kernels.cuh"
#include "kernels_v2.cuh"
#include "kernels_s.cuh"

using namespace ebic_b200;

namespace {

thread_local std::string g_last_error;

struct Error {
    int status;
    std::string msg;
};

[[noreturn]] void fail(int status, const std::string& msg) { throw Error{status, msg}; }

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        (void)cudaGetLastError();
        fail(EBIC_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
    }
}
#define CK(x) cuda_check((x), #x)

template <class F>
int guarded(F&& f) {
    try {
        f();
        return EBIC_OK;
    } catch (const Error& e) {
        g_last_error = e.msg;
        return e.status;
    } catch (const std::bad_alloc&) {
        g_last_error = "out of host memory";
        return EBIC_ERR_RUNTIME;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return EBIC_ERR_RUNTIME;
    }
}

}  // namespace

namespace ebic_b200_detail {
// Last-error hook for the host-only translation units (toprank.cpp).
int set_error(int status, const char* msg) {
    g_last_error = msg;
    return status;
}
}  // namespace ebic_b200_detail

namespace {

int env_int(const char* name, int dflt) {
    const char* v = std::getenv(name);
    return (v && *v) ? std::atoi(v) : dflt;
}

// Tuning / test overrides (EBIC_* environment variables), read once when a
// context is created so the per-generation launch path makes no getenv calls.
struct Knobs {
    int force_direct, rpg, rpl, stages, ncw, slice, layout_f64, no_collapse, sched_static,
        max_parts, reduce_tree, grid, phase_timing, spg, host_copy, xshard, graph, debug_mode, kernel,
        gap, compact, v2_np, prefetch, pack, split;
    static Knobs from_env() {
        Knobs k;
        k.force_direct = env_int("EBIC_FORCE_DIRECT", 0);
        k.rpg = env_int("EBIC_RPG", 0);
        k.rpl = env_int("EBIC_RPL", 0);
        k.stages = env_int("EBIC_STAGES", 0);
        k.ncw = env_int("EBIC_NCW", 0);
        k.slice = env_int("EBIC_SLICE", 0);
        k.layout_f64 = env_int("EBIC_LAYOUT_F64", 0);
        k.no_collapse = env_int("EBIC_NO_COLLAPSE", 0);
        k.sched_static = env_int("EBIC_SCHED_STATIC", 0);
        k.max_parts = env_int("EBIC_MAX_PARTS", 8);
        k.reduce_tree = env_int("EBIC_REDUCE_TREE", 0);
        k.grid = env_int("EBIC_GRID", 0);
        k.phase_timing = env_int("EBIC_PHASE_TIMING", 0);
        k.spg = env_int("EBIC_SPG", 0);
        k.host_copy = env_int("EBIC_HOST_COPY", 0);
        k.xshard = env_int("EBIC_XSHARD", 1);  // in-kernel cross-shard reduction
        k.graph = env_int("EBIC_GRAPH", 1);    // count launches through a cached one-node graph
        k.debug_mode = env_int("EBIC_DEBUG_MODE", 0);  // measurement only: wrong results
        // rank layouts: 2 = K1v2 (column-compacted staging, default), 1 = the
        // v1 TMA-tile kernel; the v1 tile knobs select v1 as well
        k.kernel = env_int("EBIC_KERNEL", 2);
        if (k.slice || k.rpg || k.rpl || k.spg || k.ncw) k.kernel = 1;
        k.gap = env_int("EBIC_GAP", 0);  // K1v2: unreferenced gap columns staged with their runs
        // K1v2 staging: -1 auto (referenced columns only for long launches), 0 whole tiles, 1 compact
        k.compact = env_int("EBIC_COMPACT", -1);
        k.v2_np = env_int("EBIC_V2_NP", 8);  // K1v2 producer warps (8: 20 consumers; 4: 24)
        k.prefetch = env_int("EBIC_PREFETCH", 0);  // K1v2 compact: L2 prefetch distance (items)
        // K1v2: one-plane ranks packed three rows per word when they fit 9 bits
        k.pack = env_int("EBIC_PACK", 1);
        // K1s (series-split kernel) for short single-shard launches: -1 auto, 0 off (default:
        // with its tiles split over idle SMs K1v2 is faster at every BASELINE size), 1 always
        k.split = env_int("EBIC_SPLIT", 0);
        return k;
    }
};

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !p)
            fail(EBIC_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
        fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

class DeviceGuard {
  public:
    explicit DeviceGuard(int dev) {
        CK(cudaGetDevice(&prev_));
        if (prev_ != dev) CK(cudaSetDevice(dev));
        dev_ = dev;
    }
    ~DeviceGuard() {
        if (prev_ != dev_) cudaSetDevice(prev_);
    }

  private:
    int prev_ = 0, dev_ = 0;
};

constexpr size_t kMaxSeriesPerLaunch = 2048;
constexpr size_t kMaxLenPerLaunch = 8192;

// Kernel configuration of the TMA count kernel for one shard.
struct CountConfig {
    int v2 = 0;         // 1: K1v2 (kernels_v2.cuh) over the tile-major rank matrix
    int layout = 0;     // 0 = fp64 tile, 1 = rank (1 plane), 2 = rank (2 planes)
    int rpg = 0;        // rows per tile (0 = direct kernel)
    int rpl = 1;        // rows per lane
    int ncw = 16;       // consumer warps per CTA
    int slice = 0;      // rank layout: bytes per staged column slice (64 or 128)
    int spg = 2;        // rank layout: series per lane group
    int stages = 0;
    uint32_t box_cols = 0, n_boxes = 0, stage_bytes = 0;
};

struct Tables {
    uint64_t sigma = 0;
    size_t n = 0;
    double* d_log = nullptr;
    double* d_exp = nullptr;
};

// Exact integer restatement of the matrix for one epsilon (RankWalker).
struct RankLayout {
    bool ok = false;
    uint64_t eps_bits = 0;
    int planes = 0;
    bool collapsed = false;            // one plane tested with <= (eps > 0)
    uint16_t* d = nullptr;
    // one plane repacked three rows per word (RankWalker<3>), when every rank
    // fits 9 bits (n_cols <= kPack10MaxCols); K1v2 streams this one
    uint32_t* d10 = nullptr;
    size_t d10_bytes = 0;
    int packed = 0;  // 0 none, 3 = 10-bit fields (RankWalker<3>), 4 = 12-bit fields (RankWalker<4>)
    // rows the collapsed layout cannot represent (evaluated exactly in fp64)
    unsigned long long* d_row_excl = nullptr;  // bitmask, ceil(ld / 64) words
    uint32_t* d_excl_rows = nullptr;
    double* d_excl_vals = nullptr;             // their values, row-major
    uint32_t n_excl = 0;
    CUtensorMap tmap;
    bool tmap_ok = false;
    int tmap_slice = 0;
    uint64_t last_use = 0;
};

struct Shard {
    int device = 0;
    Knobs knobs = Knobs::from_env();
    size_t row_begin = 0;  // global first row
    size_t rows = 0;
    size_t ld = 0;         // padded leading dimension (multiple of 64)
    double* d_mat = nullptr;
    cudaStream_t stream = nullptr;
    int sm_count = 0;
    int max_smem = 0;
    // TMA descriptors, one per row-tile height (index log2(rpg)).
    CUtensorMap tmap[6];
    bool tmap_ok[6] = {false, false, false, false, false, false};
    // scratch
    unsigned char* d_in = nullptr;
    size_t d_in_cap = 0;
    uint32_t* d_partial = nullptr;   // count-kernel reduction scratch
    size_t partial_cap = 0;          // u32 elements
    unsigned int* d_done = nullptr;
    unsigned char* d_out = nullptr;
    size_t d_out_cap = 0;
    unsigned char* h_pin = nullptr;
    size_t h_pin_cap = 0;
    // mapped pinned results of host-path launches: [flag (128 B)][counts P][fitness P]
    unsigned char* h_map = nullptr;
    size_t h_map_cap = 0;
    // mapped pinned staging of the host CBF (read by the device)
    unsigned char* h_in_map = nullptr;
    size_t h_in_map_cap = 0;
    unsigned long long seq = 0;
    uint64_t cbf_seq = 0;
    Tables tables;
    unsigned long long* d_phase = nullptr;  // EBIC_PHASE_TIMING: per-CTA phase stamps
    RankLayout ranks[2];
    uint64_t rank_clock = 0;
    int has_nan = -1;  // -1 unknown
    int last_grid = 0;
    // host-path phase timers (us, accumulated): validate, stage+H2D, launch, wait, copy-out
    double host_us[5] = {0, 0, 0, 0, 0};
    uint64_t host_calls = 0;
    int last_reduce = -1;  // reduction-tail mode of the last launch
    // Stream of the previous count launch.  Launches share this shard's
    // scratch (striped accumulators, tickets, Eq. 1 tables), so a launch on
    // another stream (device API on a caller's stream vs the host API on
    // `stream`) first waits for everything already queued on the previous one.
    cudaStream_t cur_stream = nullptr;
    cudaEvent_t switch_event = nullptr;
    bool last_collapsed = false;
    int last_kernel = 0;  // 1 v1 tile / direct, 2 K1v2, 3 K1s
    // choose_config memo (same P / L / layout as the previous launch)
    size_t memo_P = 0, memo_L = 0;
    int memo_planes = -1;
    CountConfig memo_cfg;
    CountConfig last_cfg;
    // One-node CUDA graphs of the count kernel, one per launch shape: a
    // parameter update + graph launch costs the host about 1.5 us against
    // about 3.5 us for a plain launch of this kernel.
    struct GraphSlot {
        const void* func = nullptr;
        cudaGraph_t g = nullptr;
        cudaGraphExec_t exec = nullptr;
        cudaGraphNode_t node = nullptr;
    };
    std::vector<GraphSlot> graphs;
};

void grow_device(unsigned char** p, size_t* cap, size_t need) {
    if (need <= *cap) return;
    if (*p) CK(cudaFree(*p));
    *p = nullptr;
    size_t n = std::max(need, *cap * 2);
    n = (n + 255) & ~size_t(255);
    CK(cudaMalloc(p, n));
    *cap = n;
}

// Host memory the device writes directly (zero-copy results + completion flag).
void grow_mapped(unsigned char** p, size_t* cap, size_t need) {
    if (need <= *cap) return;
    if (*p) CK(cudaFreeHost(*p));
    *p = nullptr;
    size_t n = std::max(need, *cap * 2);
    n = (n + 255) & ~size_t(255);
    // portable: with several shards, any device's final CTA may write results
    CK(cudaHostAlloc(reinterpret_cast<void**>(p), n, cudaHostAllocMapped | cudaHostAllocPortable));
    std::memset(*p, 0, n);
    *cap = n;
}

void grow_pinned(unsigned char** p, size_t* cap, size_t need) {
    if (need <= *cap) return;
    if (*p) CK(cudaFreeHost(*p));
    *p = nullptr;
    size_t n = std::max(need, *cap * 2);
    n = (n + 255) & ~size_t(255);
    CK(cudaMallocHost(p, n));
    *cap = n;
}

// Reduction scratch of one count launch: striped accumulators [P][kStripes]
// (zero between launches) or the tree's (grid + groups) rows of P counters.
// mode: 0 tree, 1 u32 stripes [P][8], 2 fp32 stripes [kV2Stripes][slots rounded to 8] (K1v2)
void ensure_partial(Shard& s, size_t P, int grid, int mode) {
    const size_t gsz = reduce_group_size((uint32_t)grid);
    const size_t need = mode == 3 ? 2 * P  // K1s: split-series counts + arrival counters
                        : mode == 2 ? ((P + kV2Pad + 7) & ~size_t(7)) * kV2Stripes  // slots incl. dummies, whole chunks
                        : mode == 1 ? P * kStripes : (size_t(grid) + (grid + gsz - 1) / gsz) * P;
    if (need <= s.partial_cap && mode == s.last_reduce) return;
    // a launch still queued on the previous stream may use the old scratch
    if (s.cur_stream) CK(cudaStreamSynchronize(s.cur_stream));
    s.last_reduce = mode;
    if (need <= s.partial_cap) {  // mode switch: the tree leaves non-zero rows behind
        CK(cudaMemsetAsync(s.d_partial, 0, s.partial_cap * sizeof(uint32_t), s.stream));
        CK(cudaStreamSynchronize(s.stream));
        return;
    }
    if (s.d_partial) CK(cudaFree(s.d_partial));
    s.d_partial = nullptr;
    const size_t n = std::max(need, s.partial_cap * 2);
    CK(cudaMalloc(&s.d_partial, n * sizeof(uint32_t)));
    // the striped tail expects zeros and leaves zeros behind
    CK(cudaMemsetAsync(s.d_partial, 0, n * sizeof(uint32_t), s.stream));
    CK(cudaStreamSynchronize(s.stream));
    s.partial_cap = n;
}

}  // namespace

// One host thread per extra row shard: the per-generation work of shard i
// (CBF staging + count launch) runs on its own thread with its device
// current, concurrently with the other shards, instead of a serial
// cudaSetDevice + launch loop on the caller's thread (the reference runs all
// row chunks at once on its ThreadPool, parallel.hpp:40-55).  Shard 0 runs on
// the caller's thread.  Workers spin on the job counter for EBIC_SPIN_US
// (default 2000 us: the GA's host work between generations) before
// sleeping, so a hand-off costs ~0.1-0.3 us instead of a futex wake.
class ShardPool {
  public:
    ShardPool(const std::vector<int>& devices, int spin_us) : spin_us_(spin_us) {
        const size_t n = devices.size();
        done_ = std::make_unique<std::atomic<uint64_t>[]>(n);
        errors_.resize(n);
        for (size_t i = 1; i < n; ++i) {
            done_[i].store(0);
            threads_.emplace_back([this, i, dev = devices[i]] { loop(i, dev); });
        }
    }
    ~ShardPool() {
        {
            std::lock_guard<std::mutex> lk(m_);
            stop_.store(true, std::memory_order_release);
        }
        cv_.notify_all();
        for (std::thread& t : threads_) t.join();
    }
    // Runs f(i) for every shard i (i >= 1 on the workers, 0 here) and
    // returns when all are done; the first exception is rethrown.
    void run(const std::function<void(size_t)>& f) {
        job_ = &f;
        for (auto& e : errors_) e = nullptr;
        uint64_t s;
        {
            std::lock_guard<std::mutex> lk(m_);  // pairs with the sleepers' predicate check
            s = seq_.fetch_add(1, std::memory_order_acq_rel) + 1;
        }
        cv_.notify_all();
        try {
            f(0);
        } catch (...) {
            errors_[0] = std::current_exception();
        }
        for (size_t i = 1; i <= threads_.size(); ++i)
            while (done_[i].load(std::memory_order_acquire) != s) {
            }
        job_ = nullptr;
        for (auto& e : errors_)
            if (e) std::rethrow_exception(e);
    }

  private:
    void loop(size_t i, int dev) {
        cudaSetDevice(dev);
        uint64_t seen = 0;
        for (;;) {
            const auto t0 = std::chrono::steady_clock::now();
            uint64_t s = seen;
            for (uint32_t k = 0;; ++k) {
                s = seq_.load(std::memory_order_acquire);
                if (s != seen || stop_.load(std::memory_order_acquire)) break;
                if ((k & 255) == 255 &&
                    std::chrono::steady_clock::now() - t0 > std::chrono::microseconds(spin_us_)) {
                    std::unique_lock<std::mutex> lk(m_);
                    cv_.wait(lk, [&] {
                        return seq_.load(std::memory_order_acquire) != seen ||
                               stop_.load(std::memory_order_acquire);
                    });
                }
            }
            if (stop_.load(std::memory_order_acquire)) return;
            seen = s;
            try {
                (*job_)(i);
            } catch (...) {
                errors_[i] = std::current_exception();
            }
            done_[i].store(s, std::memory_order_release);
        }
    }
    int spin_us_;
    std::vector<std::thread> threads_;
    std::unique_ptr<std::atomic<uint64_t>[]> done_;
    std::vector<std::exception_ptr> errors_;
    const std::function<void(size_t)>* job_ = nullptr;
    std::atomic<uint64_t> seq_{0};
    std::atomic<bool> stop_{false};
    std::mutex m_;
    std::condition_variable cv_;
};

struct ebic_ctx {
    size_t n_rows = 0;      // rows held
    size_t n_cols = 0;
    size_t row_begin = 0;   // global row of shards[0]
    size_t total_rows = 0;  // rows of the full matrix (fitness tables, sigma)
    std::vector<Shard> shards;
    // Cross-shard reduction state (several shards): per-series accumulator and
    // ticket on shards[0]'s device, reachable from every shard's device.
    int xshard = -1;  // -1 not set up, 0 unavailable, 1 ready
    unsigned long long* d_xacc = nullptr;
    size_t xacc_cap = 0;
    unsigned int* d_xticket = nullptr;
    std::unique_ptr<ShardPool> pool;  // several shards: one launch thread per extra shard
    // Runs f(shard) for every shard, concurrently when there are several.
    void for_shards(const std::function<void(Shard&)>& f) {
        if (shards.size() == 1) {
            DeviceGuard g(shards[0].device);
            f(shards[0]);
            return;
        }
        if (!pool) {
            std::vector<int> devs;
            for (const Shard& s : shards) devs.push_back(s.device);
            pool = std::make_unique<ShardPool>(devs, env_int("EBIC_SPIN_US", 2000));
        }
        pool->run([&](size_t i) {
            DeviceGuard g(shards[i].device);
            f(shards[i]);
        });
    }
};

namespace {

// ---------------------------------------------------------------------------
// matrix upload: row-major host/device buffer -> column-major padded shard
// ---------------------------------------------------------------------------
void upload_shard(Shard& s, const double* src_rows, size_t n_cols, bool src_on_device) {
    DeviceGuard g(s.device);
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, s.device));
    s.sm_count = prop.multiProcessorCount;
    CK(cudaDeviceGetAttribute(&s.max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, s.device));
    CK(cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking));
    s.ld = std::max<size_t>(64, (s.rows + 63) / 64 * 64);
    CK(cudaMalloc(&s.d_mat, s.ld * n_cols * sizeof(double)));
    CK(cudaMalloc(&s.d_done, (kMaxGroups + 2) * sizeof(unsigned int)));
    if (s.knobs.phase_timing) {
        CK(cudaMalloc(&s.d_phase, 4096 * 8 * sizeof(unsigned long long)));
        CK(cudaMemsetAsync(s.d_phase, 0, 4096 * 8 * sizeof(unsigned long long), s.stream));
    }
    CK(cudaMemsetAsync(s.d_done, 0, (kMaxGroups + 2) * sizeof(unsigned int), s.stream));

    // Stage <= 64 MB of rows at a time (and < 2^21 rows: grid.y limit).
    size_t chunk = std::max<size_t>(32, (64ull << 20) / (n_cols * sizeof(double)));
    chunk = std::min<size_t>(chunk, 1u << 20);
    chunk = (chunk + 31) / 32 * 32;
    double* staging = nullptr;
    if (!src_on_device) CK(cudaMalloc(&staging, std::min(chunk, s.rows) * n_cols * sizeof(double) + 8));
    for (size_t r0 = 0; r0 < s.ld; r0 += chunk) {
        const size_t out_rows = std::min(chunk, s.ld - r0);
        const size_t in_rows = r0 < s.rows ? std::min(out_rows, s.rows - r0) : 0;
        const double* in = nullptr;
        if (in_rows) {
            if (src_on_device) {
                in = src_rows + r0 * n_cols;
            } else {
                CK(cudaMemcpyAsync(staging, src_rows + r0 * n_cols, in_rows * n_cols * sizeof(double),
                                   cudaMemcpyHostToDevice, s.stream));
                in = staging;
            }
        }
        dim3 grid((unsigned)((n_cols + 31) / 32), (unsigned)((out_rows + 31) / 32));
        transpose_pad_kernel<<<grid, dim3(32, 8), 0, s.stream>>>(in, in_rows, n_cols, s.d_mat + r0,
                                                                 s.ld, out_rows);
        CK(cudaGetLastError());
    }
    CK(cudaStreamSynchronize(s.stream));
    if (staging) CK(cudaFree(staging));
}

int log2i(int x) {
    int l = 0;
    while ((1 << l) < x) ++l;
    return l;
}

const CUtensorMap& tensor_map(Shard& s, size_t n_cols, const CountConfig& cfg) {
    const int idx = log2i(cfg.rpg);
    if (!s.tmap_ok[idx]) {
        cuuint64_t dims[2] = {(cuuint64_t)s.ld, (cuuint64_t)n_cols};
        cuuint64_t strides[1] = {(cuuint64_t)(s.ld * sizeof(double))};
        cuuint32_t box[2] = {(cuuint32_t)cfg.rpg, cfg.box_cols};
        cuuint32_t estr[2] = {1, 1};
        CUresult r = tensor_map_encoder()(&s.tmap[idx], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, s.d_mat,
                                          dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                          CU_TENSOR_MAP_SWIZZLE_NONE,
                                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) fail(EBIC_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
        s.tmap_ok[idx] = true;
    }
    return s.tmap[idx];
}

// Shared-memory bytes of a TMA count launch.
bool scratch_in_stage(const CountConfig& c, size_t P, size_t L) {
    return c.stages >= 2 && count_scratch_bytes((uint32_t)P, (uint32_t)L) <= c.stage_bytes;
}

size_t tma_smem_bytes(const CountConfig& c, size_t P, size_t L) {
    return 128 + size_t(c.stages) * c.stage_bytes + (2 * kMaxStages + 2) * sizeof(uint64_t) +
           count_meta_bytes((uint32_t)P, (uint32_t)L, scratch_in_stage(c, P, L)) + 16;
}

// Fits a stage ring for a tile of `col_bytes` per column: the deepest ring
// (>= min_stages, <= 4 unless forced) whose shared memory fits the budget.
bool fit_ring(CountConfig& c, size_t n_cols, size_t col_bytes, size_t P, size_t L, size_t budget,
              int min_stages, int want_stages) {
    const uint32_t nb = (uint32_t)((n_cols + 255) / 256);
    uint32_t bc = (uint32_t)((n_cols + nb - 1) / nb);
    bc = (bc + 7) / 8 * 8;  // 128-byte aligned box destinations for every tile height
    c.n_boxes = nb;
    c.box_cols = bc;
    const size_t sb = col_bytes * bc * nb;
    if (sb >= (1u << 20)) return false;
    c.stage_bytes = (uint32_t)sb;
    int st = want_stages ? want_stages : kMaxStages;
    for (; st >= min_stages; --st) {
        c.stages = st;
        if (tma_smem_bytes(c, P, L) <= budget) break;
    }
    if (st < min_stages) return false;
    // Deep rings beyond 4 stages buy nothing once HBM is saturated.
    if (!want_stages) c.stages = std::min(c.stages, 4);
    return true;
}

// Chooses layout and tile.  Default: the exact rank layout (half the bytes of
// fp64 per cell with eps != 0, a quarter with eps == 0; integer tests) when the
// matrix is narrow enough for 16-bit ranks and the in-smem rank build; else the
// fp64 tile with the tallest row tile (coalesced 128-byte column slices at 16
// rows) that leaves a >= 3-deep TMA ring; else the unstaged direct kernel.
CountConfig choose_config(const Shard& s, size_t n_cols, size_t P, size_t L, int rank_planes) {
    CountConfig best;
    const Knobs& kn = s.knobs;
    if (kn.force_direct) return best;
    const int want_rpg = kn.rpg;
    const int want_rpl = kn.rpl;
    const int want_stages = kn.stages;
    const int want_ncw = kn.ncw;
    const size_t budget = (size_t)s.max_smem;
    if (rank_planes && kn.kernel == 2) {
        // K1v2: the whole opt-in window; one stage must fit even if the
        // launch referenced min(C, L) columns (the ring depth follows the
        // actual U at run time)
        const V2Layout v = v2_layout((uint32_t)P, (uint32_t)L, (uint32_t)n_cols);
        const size_t window = budget - 1024 - 128;  // static shared bytes + alignment
        const size_t worst = std::min(n_cols, L) * 128;
        if (v.area < window && window - v.area >= std::max<size_t>(worst, v2_scratch_bytes((uint32_t)P, (uint32_t)L))) {
            CountConfig c;
            c.v2 = 1;
            c.layout = rank_planes;
            c.slice = 128;
            c.rpg = rank_planes == 4 ? 80 : rank_planes == 3 ? 96 : rank_planes == 2 ? 32 : 64;
            c.rpl = rank_planes == 4 ? 10 : rank_planes == 3 ? 12 : rank_planes == 2 ? 4 : 8;
            c.ncw = 24;
            c.spg = 2;
            c.stages = kn.stages;  // 0: as many as fit (<= 4)
            // a lane's 16-bit partial counts grow by <= rpl rows per tile it walks
            const size_t tiles = (s.rows + c.rpg - 1) / c.rpg;
            if ((tiles / std::max(1, std::min<int>((int)tiles, s.sm_count)) + 2) * c.rpl <= 0xffff) return c;
        }
    }
    if (rank_planes >= 3) rank_planes = 1;  // v1: the 16-bit plane
    if (rank_planes) {
        const int want_slice = kn.slice;
        for (int min_stages : {3, 2}) {
            for (int slice : {128, 64}) {
                if (want_slice && slice != want_slice) continue;
                CountConfig c;
                c.layout = rank_planes;
                c.slice = slice;
                c.rpg = slice / (2 * rank_planes);
                c.rpl = rank_planes == 2 ? 4 : 8;
                // 24 warps (no spills under the 80-register cap) measured
                // fastest: one plane C5 103 us vs 107 at 16, 114 at 31 with
                // spills; two planes C5 154 us vs 169 at 16, 165 at 31.
                c.ncw = want_ncw == 16 ? 16 : want_ncw == 32 ? 32 : 24;
                c.spg = kn.spg == 4 ? 4 : 2;
                if (c.spg == 4) c.ncw = 16;  // 4 walks per group need the 16-warp register budget
                if (fit_ring(c, n_cols, slice, P, L, budget, min_stages, want_stages)) return c;
            }
        }
    }
    for (int min_stages : {3, 2}) {
        for (int rpg : {16, 32, 8, 4}) {
            if (want_rpg && rpg != want_rpg) continue;
            CountConfig c;
            c.rpg = rpg;
            c.rpl = want_rpl ? want_rpl : 2;
            if (c.rpl > 1 && rpg < 4) c.rpl = 1;
            // 16-row tiles: 24 warps (no spills; C4 47.0 us vs 47.2 at 31, 55 at 16).
            c.ncw = rpg == 16 ? (want_ncw == 32 ? 32 : 24) : 16;
            if (want_ncw == 16) c.ncw = 16;
            if (fit_ring(c, n_cols, size_t(rpg) * 8, P, L, budget, min_stages, want_stages)) return c;
        }
    }
    return best;  // rpg == 0 -> direct kernel
}

void launch_kernel(Shard* sh, const void* func, int grid, int block, size_t smem, cudaStream_t st,
                   void** args) {
    if (!sh || !sh->knobs.graph) {
        CK(cudaLaunchKernel(func, dim3(grid), dim3(block), args, smem, st));
        return;
    }
    cudaKernelNodeParams kp{};
    kp.func = const_cast<void*>(func);
    kp.gridDim = dim3(grid);
    kp.blockDim = dim3(block);
    kp.sharedMemBytes = static_cast<unsigned>(smem);
    kp.kernelParams = args;
    // One graph per kernel function: the parameter update re-points it at
    // this launch's grid, block and dynamic shared memory as well (the GA's
    // population and series lengths change the ring's size every generation).
    for (size_t i = 0; i < sh->graphs.size(); ++i) {
        Shard::GraphSlot& g = sh->graphs[i];
        if (g.func != func) continue;
        if (cudaGraphExecKernelNodeSetParams(g.exec, g.node, &kp) == cudaSuccess) {
            CK(cudaGraphLaunch(g.exec, st));
            return;
        }
        (void)cudaGetLastError();  // not updatable: rebuild below
        cudaGraphExecDestroy(g.exec);
        cudaGraphDestroy(g.g);
        sh->graphs.erase(sh->graphs.begin() + static_cast<std::ptrdiff_t>(i));
        break;
    }
    Shard::GraphSlot g;
    g.func = func;
    CK(cudaGraphCreate(&g.g, 0));
    CK(cudaGraphAddKernelNode(&g.node, g.g, nullptr, 0, &kp));
    CK(cudaGraphInstantiate(&g.exec, g.g, 0));
    if (sh->graphs.size() >= 16) {  // bounded: drop the oldest function
        cudaGraphExecDestroy(sh->graphs.front().exec);
        cudaGraphDestroy(sh->graphs.front().g);
        sh->graphs.erase(sh->graphs.begin());
    }
    sh->graphs.push_back(g);
    CK(cudaGraphLaunch(g.exec, st));
}

template <class W, int NCW>
void launch_tma_t(const CUtensorMap& tm, const CountParams& p, int grid, size_t smem,
                  cudaStream_t st, Shard* sh) {
    auto k = count_tma_kernel<W, NCW>;
    // The attribute is per function and device; set it only when it grows so
    // the per-generation launch path makes no extra driver calls.
    // (atomic: the shards of one context launch from their own host threads)
    static std::atomic<int> smem_set[64] = {};
    int dev = sh ? sh->device : 0;  // the caller's DeviceGuard made it current
    if (!sh) CK(cudaGetDevice(&dev));
    if (dev < 0 || dev >= 64 || (int)smem > smem_set[dev].load(std::memory_order_acquire)) {
        CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        if (dev >= 0 && dev < 64) {
            int cur = smem_set[dev].load(std::memory_order_relaxed);
            while ((int)smem > cur && !smem_set[dev].compare_exchange_weak(cur, (int)smem)) {
            }
        }
    }
    void* args[2] = {const_cast<CUtensorMap*>(&tm), const_cast<CountParams*>(&p)};
    launch_kernel(sh, reinterpret_cast<const void*>(k), grid, (NCW + 1) * 32, smem, st, args);
}

template <int RPG, int RPL, int NCW>
void launch_f64(bool e0, const CUtensorMap& tm, const CountParams& p, int grid, size_t smem,
                cudaStream_t st, Shard* sh) {
    if (e0) launch_tma_t<F64Walker<RPG, RPL, true>, NCW>(tm, p, grid, smem, st, sh);
    else launch_tma_t<F64Walker<RPG, RPL, false>, NCW>(tm, p, grid, smem, st, sh);
}

void launch_tma(const CountConfig& c, bool e0, const CUtensorMap& tm, const CountParams& p,
                int grid, size_t smem, cudaStream_t st, Shard* sh) {
    if (c.layout) {
        const bool n16 = c.ncw == 16, s64 = c.slice == 64;
        if (c.spg == 4) {
            if (c.layout == 2) {
                if (s64) launch_tma_t<RankWalker<2, 64, 4>, 16>(tm, p, grid, smem, st, sh);
                else launch_tma_t<RankWalker<2, 128, 4>, 16>(tm, p, grid, smem, st, sh);
            } else {
                if (s64) launch_tma_t<RankWalker<1, 64, 4>, 16>(tm, p, grid, smem, st, sh);
                else launch_tma_t<RankWalker<1, 128, 4>, 16>(tm, p, grid, smem, st, sh);
            }
            CK(cudaGetLastError());
            return;
        }
        const bool n24 = c.ncw == 24;
        if (c.layout == 2) {
            if (s64) {
                if (n16) launch_tma_t<RankWalker<2, 64>, 16>(tm, p, grid, smem, st, sh);
                else if (n24) launch_tma_t<RankWalker<2, 64>, 24>(tm, p, grid, smem, st, sh);
                else launch_tma_t<RankWalker<2, 64>, 31>(tm, p, grid, smem, st, sh);
            } else {
                if (n16) launch_tma_t<RankWalker<2, 128>, 16>(tm, p, grid, smem, st, sh);
                else if (n24) launch_tma_t<RankWalker<2, 128>, 24>(tm, p, grid, smem, st, sh);
                else launch_tma_t<RankWalker<2, 128>, 31>(tm, p, grid, smem, st, sh);
            }
        } else {
            if (s64) {
                if (n16) launch_tma_t<RankWalker<1, 64>, 16>(tm, p, grid, smem, st, sh);
                else if (n24) launch_tma_t<RankWalker<1, 64>, 24>(tm, p, grid, smem, st, sh);
                else launch_tma_t<RankWalker<1, 64>, 31>(tm, p, grid, smem, st, sh);
            } else {
                if (n16) launch_tma_t<RankWalker<1, 128>, 16>(tm, p, grid, smem, st, sh);
                else if (n24) launch_tma_t<RankWalker<1, 128>, 24>(tm, p, grid, smem, st, sh);
                else launch_tma_t<RankWalker<1, 128>, 31>(tm, p, grid, smem, st, sh);
            }
        }
        CK(cudaGetLastError());
        return;
    }
    switch (c.rpg * 1000 + c.rpl * 100 + c.ncw) {
        case 32116: launch_f64<32, 1, 16>(e0, tm, p, grid, smem, st, sh); break;
        case 32216: launch_f64<32, 2, 16>(e0, tm, p, grid, smem, st, sh); break;
        case 16116: launch_f64<16, 1, 16>(e0, tm, p, grid, smem, st, sh); break;
        case 16216: launch_f64<16, 2, 16>(e0, tm, p, grid, smem, st, sh); break;
        case 16124: launch_f64<16, 1, 24>(e0, tm, p, grid, smem, st, sh); break;
        case 16224: launch_f64<16, 2, 24>(e0, tm, p, grid, smem, st, sh); break;
        case 16132: launch_f64<16, 1, 31>(e0, tm, p, grid, smem, st, sh); break;
        case 16232: launch_f64<16, 2, 31>(e0, tm, p, grid, smem, st, sh); break;
        case 8116: launch_f64<8, 1, 16>(e0, tm, p, grid, smem, st, sh); break;
        case 8216: launch_f64<8, 2, 16>(e0, tm, p, grid, smem, st, sh); break;
        case 4116: launch_f64<4, 1, 16>(e0, tm, p, grid, smem, st, sh); break;
        case 4216: launch_f64<4, 2, 16>(e0, tm, p, grid, smem, st, sh); break;
        default: fail(EBIC_ERR_RUNTIME, "unsupported count-kernel configuration");
    }
    CK(cudaGetLastError());
}

constexpr size_t kRankMaxCols = 2048;  // 2C keys sorted in shared memory per row
constexpr size_t kPack10MaxCols = 510;   // ranks 1..510 + the NaN sentinel in 9 bits
constexpr size_t kPack12MaxCols = 2046;  // ranks 1..2046 + the NaN sentinel in 11 bits
constexpr double kSplitMaxL2Bytes = 4e6;  // K1s while rows x sum(len) x b stays below this (measured crossover: C1 1.6 MB K1s faster, C3 17 MB K1v2 faster)

uint64_t eps_key(double eps) {
    if (eps == 0.0) eps = 0.0;  // -0.0 and +0.0 give identical predicates
    uint64_t b;
    std::memcpy(&b, &eps, sizeof b);
    return b;
}

// The exact rank layout of this shard for `eps` (built on first use, two
// epsilons cached), or nullptr when the fp64 tile must be used.
template <int PLANES, bool COLLAPSED>
void launch_rank_build(Shard& s, size_t n_cols, double eps, uint16_t* out, uint8_t* dirty) {
    uint32_t Kp = 1;
    while (Kp < PLANES * n_cols) Kp <<= 1;
    const size_t smem = size_t(Kp) * 16 + 32 * 4 + 64;
    auto k = rank_build_kernel<PLANES, COLLAPSED>;
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k<<<(unsigned)s.ld, 256, smem, s.stream>>>(s.d_mat, (uint32_t)s.ld, (uint32_t)s.rows,
                                                (uint32_t)n_cols, eps, Kp, out, dirty);
    CK(cudaGetLastError());
}

// The exact rank layout of this shard for `eps` (built on first use, two
// epsilons cached), or nullptr when the fp64 tile must be used:
//   eps == 0, no NaN        one plane, strict test        (2 B/cell)
//   eps > 0, few dirty rows one plane, <= test (collapsed) (2 B/cell) + the
//                           dirty rows evaluated exactly in fp64 by the kernel
//   otherwise               two planes (lo, hi)            (4 B/cell)
RankLayout* ensure_ranks(Shard& s, size_t n_cols, double eps) {
    if (n_cols > kRankMaxCols || s.knobs.layout_f64) return nullptr;
    const uint64_t key = eps_key(eps);
    for (RankLayout& rl : s.ranks)
        if (rl.ok && rl.eps_bits == key) {
            rl.last_use = ++s.rank_clock;
            return &rl;
        }
    if (s.has_nan < 0) {
        int* d_flag = nullptr;
        CK(cudaMalloc(&d_flag, sizeof(int)));
        CK(cudaMemsetAsync(d_flag, 0, sizeof(int), s.stream));
        has_nan_kernel<<<s.sm_count * 4, 256, 0, s.stream>>>(s.d_mat, s.ld, s.rows, s.ld * n_cols, d_flag);
        CK(cudaGetLastError());
        int h = 0;
        CK(cudaMemcpyAsync(&h, d_flag, sizeof(int), cudaMemcpyDeviceToHost, s.stream));
        CK(cudaStreamSynchronize(s.stream));
        CK(cudaFree(d_flag));
        s.has_nan = h;
    }
    RankLayout& rl = s.ranks[0].last_use <= s.ranks[1].last_use ? s.ranks[0] : s.ranks[1];
    if (!rl.d) CK(cudaMalloc(&rl.d, 2 * s.ld * n_cols * sizeof(uint16_t)));  // room for 2 planes
    cudaFree(rl.d_row_excl);
    cudaFree(rl.d_excl_rows);
    cudaFree(rl.d_excl_vals);
    rl.d_row_excl = nullptr;
    rl.d_excl_rows = nullptr;
    rl.d_excl_vals = nullptr;
    rl.n_excl = 0;
    rl.ok = false;
    rl.tmap_ok = false;
    rl.eps_bits = key;
    rl.collapsed = false;
    bool done = false;
    if (eps == 0.0 && !s.has_nan) {
        rl.planes = 1;
        launch_rank_build<1, false>(s, n_cols, eps, rl.d, nullptr);
        done = true;
    } else if (eps > 0.0 && eps < INFINITY && !s.knobs.no_collapse) {
        uint8_t* d_dirty = nullptr;
        CK(cudaMalloc(&d_dirty, s.ld));
        launch_rank_build<1, true>(s, n_cols, eps, rl.d, d_dirty);
        std::vector<uint8_t> dirty(s.rows);
        CK(cudaMemcpyAsync(dirty.data(), d_dirty, s.rows, cudaMemcpyDeviceToHost, s.stream));
        CK(cudaStreamSynchronize(s.stream));
        CK(cudaFree(d_dirty));
        std::vector<uint32_t> rows;
        for (size_t r = 0; r < s.rows; ++r)
            if (dirty[r]) rows.push_back((uint32_t)r);
        // Exact fix-up costs ~P * len fp64 loads per dirty row: worth it while
        // dirty rows are rare.
        const size_t limit = std::max<size_t>(64, s.rows / 512);
        if (rows.size() <= limit) {
            rl.planes = 1;
            rl.collapsed = true;
            rl.n_excl = (uint32_t)rows.size();
            if (!rows.empty()) {
                const size_t words = (s.ld + 63) / 64 + 2;  // K1v2 reads a tile's two words
                std::vector<unsigned long long> mask(words, 0ull);
                for (uint32_t r : rows) mask[r / 64] |= 1ull << (r % 64);
                CK(cudaMalloc(&rl.d_row_excl, words * 8));
                CK(cudaMalloc(&rl.d_excl_rows, rows.size() * 4));
                CK(cudaMemcpy(rl.d_row_excl, mask.data(), words * 8, cudaMemcpyHostToDevice));
                CK(cudaMemcpy(rl.d_excl_rows, rows.data(), rows.size() * 4, cudaMemcpyHostToDevice));
                CK(cudaMalloc(&rl.d_excl_vals, rows.size() * n_cols * sizeof(double)));
                gather_rows_kernel<<<(unsigned)rows.size(), 256, 0, s.stream>>>(
                    s.d_mat, s.ld, (uint32_t)n_cols, rl.d_excl_rows, rl.d_excl_vals);
                CK(cudaGetLastError());
            }
            done = true;
        }
    }
    if (!done) {
        rl.planes = 2;
        launch_rank_build<2, false>(s, n_cols, eps, rl.d, nullptr);
    }
    rl.packed = 0;
    if (rl.planes == 1 && n_cols <= kPack12MaxCols && s.knobs.pack && s.knobs.kernel == 2) {
        // three rows per 32-bit word while ranks fit 9 bits, else five per 64-bit word
        const bool ten = n_cols <= kPack10MaxCols && s.knobs.pack != 12;
        const uint32_t rpt = ten ? 96 : 80;
        const uint32_t tiles = (uint32_t)((s.rows + rpt - 1) / rpt);
        const size_t bytes = size_t(tiles) * n_cols * 128;
        if (rl.d10_bytes < bytes) {
            if (rl.d10) CK(cudaFree(rl.d10));
            rl.d10 = nullptr;
            CK(cudaMalloc(&rl.d10, bytes));
            rl.d10_bytes = bytes;
        }
        if (ten)
            rank_pack10_kernel<<<s.sm_count * 8, 256, 0, s.stream>>>(rl.d, (uint32_t)s.ld, (uint32_t)n_cols, tiles,
                                                                   rl.d10);
        else
            rank_pack12_kernel<<<s.sm_count * 8, 256, 0, s.stream>>>(
                rl.d, (uint32_t)s.ld, (uint32_t)n_cols, tiles, reinterpret_cast<unsigned long long*>(rl.d10));
        CK(cudaGetLastError());
        rl.packed = ten ? 3 : 4;
    }
    CK(cudaStreamSynchronize(s.stream));
    rl.ok = true;
    rl.last_use = ++s.rank_clock;
    return &rl;
}

const CUtensorMap& rank_tensor_map(RankLayout& rl, const Shard& s, size_t n_cols, const CountConfig& cfg) {
    if (!rl.tmap_ok || rl.tmap_slice != cfg.slice) {
        rl.tmap_slice = cfg.slice;
        // tile-major rank matrix seen as [blocks * n_cols][64 u16] (one row
        // per 128-byte block of one column); a box is one slice of box_cols
        // consecutive columns of a block
        const size_t rows_per_block = rl.planes == 2 ? 32 : 64;
        cuuint64_t dims[2] = {64, (cuuint64_t)(s.ld / rows_per_block * n_cols)};
        cuuint64_t strides[1] = {128};
        cuuint32_t box[2] = {(cuuint32_t)(cfg.slice / 2), cfg.box_cols};  // one column slice
        cuuint32_t estr[2] = {1, 1};
        CUresult r = tensor_map_encoder()(&rl.tmap, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, rl.d, dims,
                                          strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                          CU_TENSOR_MAP_SWIZZLE_NONE,
                                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) fail(EBIC_ERR_CUDA, "cuTensorMapEncodeTiled (ranks) failed (" + std::to_string((int)r) + ")");
        rl.tmap_ok = true;
    }
    return rl.tmap;
}

// Host-built Eq. 1 tables (same glibc log/exp2 as fitness.hpp:129,131).
const Tables& ensure_tables(Shard& s, uint64_t sigma, size_t total_rows) {
    Tables& t = s.tables;
    if (t.d_log && t.sigma == sigma && t.n == total_rows + 1) return t;
    DeviceGuard g(s.device);
    // a launch still queued on the previous stream may read the old tables
    if (s.cur_stream) CK(cudaStreamSynchronize(s.cur_stream));
    const size_t n = total_rows + 1;
    std::vector<double> lg(n, 0.0), ex(n, 1.0);
    for (size_t c = 2; c < n; ++c) lg[c] = std::log(static_cast<double>(c - 1));
    for (size_t c = 0; c < n; ++c)
        if (c < sigma) ex[c] = std::exp2(static_cast<double>(c) - static_cast<double>(sigma));
    if (t.n != n) {
        if (t.d_log) CK(cudaFree(t.d_log));
        if (t.d_exp) CK(cudaFree(t.d_exp));
        t.d_log = t.d_exp = nullptr;
        CK(cudaMalloc(&t.d_log, n * sizeof(double)));
        CK(cudaMalloc(&t.d_exp, n * sizeof(double)));
    }
    CK(cudaMemcpyAsync(t.d_log, lg.data(), n * sizeof(double), cudaMemcpyHostToDevice, s.stream));
    CK(cudaMemcpyAsync(t.d_exp, ex.data(), n * sizeof(double), cudaMemcpyHostToDevice, s.stream));
    CK(cudaStreamSynchronize(s.stream));
    t.sigma = sigma;
    t.n = n;
    return t;
}

// Launches the count kernel for one shard.  All pointers are device pointers.
void launch_count(ebic_ctx& ctx, Shard& s, const uint64_t* d_off, const uint16_t* d_cols, size_t P,
                  size_t L, double eps, uint64_t* d_counts, double* d_fit, uint64_t sigma,
                  cudaStream_t st, uint64_t cols_base, unsigned long long* done_flag = nullptr,
                  unsigned long long done_seq = 0, const void* host_cbf = nullptr,
                  size_t cbf_bytes = 0, unsigned long long* xacc = nullptr,
                  unsigned int* xticket = nullptr, uint32_t n_xshards = 0) {
    if (P == 0) return;
    if (P > 0xffffffffull || L > 0xffffffffull || s.rows > 0xffffffffull)
        fail(EBIC_ERR_INVALID_ARGUMENT, "population or shard too large for one launch");
    if (s.cur_stream != st) {
        if (!s.switch_event) CK(cudaEventCreateWithFlags(&s.switch_event, cudaEventDisableTiming));
        CK(cudaEventRecord(s.switch_event, s.cur_stream ? s.cur_stream : s.stream));
        CK(cudaStreamWaitEvent(st, s.switch_event, 0));
        s.cur_stream = st;
    }
    CountParams p{};
    p.offsets = d_off;
    p.cols = d_cols;
    p.n_series = (uint32_t)P;
    p.total_len = (uint32_t)L;
    p.n_rows = (uint32_t)s.rows;
    p.n_cols = (uint32_t)ctx.n_cols;
    p.eps = eps;
    p.sigma = sigma;
    p.done = s.d_done;
    p.counts_out = d_counts;
    p.fitness_out = d_fit;
    p.matrix = s.d_mat;
    p.ld = (uint32_t)s.ld;
    p.cols_base = cols_base;
    p.sched_static = (uint32_t)s.knobs.sched_static;
    p.max_parts = (uint32_t)s.knobs.max_parts;
    p.reduce_striped = s.knobs.reduce_tree ? 0u : 1u;
    p.done_flag = done_flag;
    p.done_seq = done_seq;
    p.xacc = xacc;
    p.xticket = xticket;
    p.n_xshards = n_xshards;
    if (host_cbf) {
        p.host_cbf = static_cast<const uint4*>(host_cbf);
        p.dev_cbf = reinterpret_cast<uint4*>(s.d_in);
        p.cbf_words = (uint32_t)((cbf_bytes + 15) / 16);
        p.cbf_ready = s.d_done + kMaxGroups + 1;
        p.cbf_seq = (unsigned int)++s.cbf_seq;
    }
    p.phase_ns = s.d_phase;
    p.debug_mode = (uint32_t)s.knobs.debug_mode;
    if (d_fit) {
        const Tables& t = ensure_tables(s, sigma, ctx.total_rows);
        p.logt = t.d_log;
        p.expt = t.d_exp;
        p.table_n = t.n;
    }
    const bool e0 = (eps == 0.0);
    RankLayout* rl = ensure_ranks(s, ctx.n_cols, eps);
    const int planes = rl ? (rl->packed ? rl->packed : rl->planes) : 0;
    if (!(s.memo_P == P && s.memo_L == L && s.memo_planes == planes)) {
        s.memo_cfg = choose_config(s, ctx.n_cols, P, L, planes);
        s.memo_P = P, s.memo_L = L, s.memo_planes = planes;
    }
    const CountConfig c = s.memo_cfg;
    if (c.v2) {
        p.ranks = c.layout >= 3 ? reinterpret_cast<const unsigned char*>(rl->d10)
                                : reinterpret_cast<const unsigned char*>(rl->d);
        p.stages = (uint32_t)c.stages;
        p.n_tiles = (uint32_t)((s.rows + c.rpg - 1) / c.rpg);
        const size_t smem = (size_t)s.max_smem - 1024;  // leaves room for the static shared bytes
        p.smem_window = (uint32_t)(smem - 128);
        // fewer tiles than SMs: split every tile's chunks over up to
        // max_parts CTAs (the kernel's last-wave split) instead of leaving
        // SMs idle
        int grid = std::min<int>((int)p.n_tiles, s.sm_count);
        if ((int)p.n_tiles < s.sm_count)
            grid = std::min<int>(s.sm_count, (int)p.n_tiles * std::max(1, s.knobs.max_parts));
        if (s.knobs.grid > 0) grid = s.knobs.grid;
        p.gap = (uint32_t)std::min(std::max(s.knobs.gap, 0), 2);
        // 4-wide fp32 stripe reductions while every count is exact in fp32
        if (p.reduce_striped && s.rows < (1u << 24)) p.reduce_striped = 2;
        // Whole tiles (one contiguous copy each, issued at once) for short
        // launches; the referenced columns only once a CTA walks enough tiles
        // to amortise building the column set first, or when two whole-tile
        // stages do not fit.
        const V2Layout vl = v2_layout((uint32_t)P, (uint32_t)L, (uint32_t)ctx.n_cols);
        const size_t area = p.smem_window - vl.area;
        const size_t block = ctx.n_cols * 128;
        uint32_t full_stages = (uint32_t)std::min<size_t>(kV2MaxStages, area / block);
        if (c.stages > 0) full_stages = std::min<uint32_t>(full_stages, (uint32_t)c.stages);
        const bool long_launch = p.n_tiles >= 6u * (uint32_t)grid;
        bool compact = long_launch || full_stages < 2;
        if (s.knobs.compact == 0 && full_stages >= 1) compact = false;
        if (s.knobs.compact == 1) compact = true;
        p.compact = compact ? 1u : 0u;
        if (!compact) p.stages = full_stages;
        p.prefetch = compact ? (uint32_t)std::max(0, s.knobs.prefetch) : 0u;
        // K1s (kernels_s.cuh) for short single-shard launches: every CTA takes
        // whole series over all rows, reading its columns' slices through L2
        // (rows x sum(len) x b bytes) -- no length sort, no cross-CTA sum
        const int sgrid = s.knobs.grid > 0 ? s.knobs.grid : 2 * s.sm_count;
        const double cell = c.layout == 4 ? 1.6 : c.layout == 3 ? 4.0 / 3.0 : c.layout == 2 ? 4.0 : 2.0;
        // (auto: device-pointer calls only -- on the host path every CTA's
        // results cross PCIe behind its own system fence, C1 e2e 32.5 us
        // against K1v2's single final CTA)
        const bool use_s = !xacc && L <= size_t(kSMaxMine) * (size_t)sgrid &&
                           (s.knobs.split == 1 ||
                            (s.knobs.split < 0 && !done_flag && !long_launch &&
                             double(s.rows) * L * cell <= kSplitMaxL2Bytes));
        s.last_grid = use_s ? sgrid : grid;
        s.last_cfg = c;
        s.last_collapsed = rl->collapsed;
        s.last_kernel = use_s ? 3 : 2;
        ensure_partial(s, P, use_s ? sgrid : grid, use_s ? 3 : (int)p.reduce_striped);
        p.partial = s.d_partial;
        if (c.layout >= 3) {
            // packed fields: + 0x1ff (strict <) or + 0x200 (<=, collapsed) per
            // 10-bit field; the 12-bit walker derives its 64-bit constant from
            // the 16-bit codes
            p.rank_k = c.layout == 4 ? (rl->collapsed ? 0x80008000u : 0x7fff7fffu)
                                     : (rl->collapsed ? 0x20080200u : 0x1ff7fdffu);
            p.row_excl = rl->d_row_excl;
            p.excl_rows = rl->d_excl_rows;
            p.excl_vals = rl->d_excl_vals;
            p.n_excl = rl->n_excl;
        } else if (rl->collapsed) {
            p.rank_k = 0x80008000u;
            p.row_excl = rl->d_row_excl;
            p.excl_rows = rl->d_excl_rows;
            p.excl_vals = rl->d_excl_vals;
            p.n_excl = rl->n_excl;
        } else {
            p.rank_k = 0x7fff7fffu;
        }
        if (use_s) {
            const void* fs = c.layout == 4   ? reinterpret_cast<const void*>(count_s_kernel<4>)
                             : c.layout == 3 ? reinterpret_cast<const void*>(count_s_kernel<3>)
                             : c.layout == 2 ? reinterpret_cast<const void*>(count_s_kernel<2>)
                                             : reinterpret_cast<const void*>(count_s_kernel<1>);
            s.last_cfg.ncw = kSThreads / 32;
            s.last_cfg.stages = 0;
            void* args[1] = {const_cast<CountParams*>(&p)};
            const size_t ssmem = (P + 1 + L) * sizeof(uint32_t);  // offsets + my column lists (<= L)
            static std::atomic<int> s_smem_set[4][64] = {};
            std::atomic<int>& sflag = s_smem_set[c.layout - 1][s.device & 63];
            if (ssmem > 48 * 1024 && sflag.load(std::memory_order_acquire) < (int)ssmem) {
                CK(cudaFuncSetAttribute(fs, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssmem));
                sflag.store((int)ssmem, std::memory_order_release);
            }
            launch_kernel(&s, fs, sgrid, kSThreads, ssmem, st, args);
            CK(cudaGetLastError());
            return;
        }
        // warps: 20 consumers + 8 producers (default: eight warps' lanes issue
        // the compacted runs' bulk copies, 1.7 us per C5 tile against 2.9 us
        // with four); EBIC_V2_NP=4: 24 + 4
        const int np = s.knobs.v2_np == 4 ? 4 : 8;
        const int ncw = np == 8 ? 20 : 24;
        const void* fn;
        if (c.layout == 4)
            fn = np == 8 ? reinterpret_cast<const void*>(count_v2_kernel<4, 20, 8>)
                         : reinterpret_cast<const void*>(count_v2_kernel<4, 24, 4>);
        else if (c.layout == 3)
            fn = np == 8 ? reinterpret_cast<const void*>(count_v2_kernel<3, 20, 8>)
                         : reinterpret_cast<const void*>(count_v2_kernel<3, 24, 4>);
        else if (c.layout == 2)
            fn = np == 8 ? reinterpret_cast<const void*>(count_v2_kernel<2, 20, 8>)
                         : reinterpret_cast<const void*>(count_v2_kernel<2, 24, 4>);
        else
            fn = np == 8 ? reinterpret_cast<const void*>(count_v2_kernel<1, 20, 8>)
                         : reinterpret_cast<const void*>(count_v2_kernel<1, 24, 4>);
        static std::atomic<int> v2_smem_set[4][2][64] = {};
        std::atomic<int>& flag = v2_smem_set[c.layout - 1][np == 8 ? 1 : 0][s.device & 63];
        if (flag.load(std::memory_order_acquire) < (int)smem) {
            CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            flag.store((int)smem, std::memory_order_release);
        }
        s.last_cfg.ncw = ncw;                     // reported by ebic_ctx_get_info
        s.last_cfg.stages = compact ? 0 : (int)p.stages;  // compacted: chosen in-kernel from U
        void* args[1] = {const_cast<CountParams*>(&p)};
        launch_kernel(&s, fn, grid, (ncw + np) * 32, smem, st, args);
        CK(cudaGetLastError());
        return;
    }
    if (c.rpg) {
        p.box_cols = c.box_cols;
        p.n_boxes = c.n_boxes;
        p.stage_bytes = c.stage_bytes;
        p.stages = (uint32_t)c.stages;
        p.n_tiles = (uint32_t)((s.rows + c.rpg - 1) / c.rpg);
        p.scratch_in_stage = scratch_in_stage(c, P, L) ? 1u : 0u;
        const size_t smem = tma_smem_bytes(c, P, L);
        int grid = std::min<int>((int)p.n_tiles, s.sm_count);
        const int g_env = s.knobs.grid;
        if (g_env > 0) grid = std::min<int>(g_env, (int)p.n_tiles);
        s.last_grid = grid;
        s.last_kernel = 1;
        s.last_cfg = c;
        s.last_collapsed = c.layout && rl->collapsed;
        ensure_partial(s, P, grid, (int)p.reduce_striped);
        p.partial = s.d_partial;
        if (c.layout && rl->collapsed) {
            p.rank_k = 0x80008000u;
            p.row_excl = rl->d_row_excl;
            p.excl_rows = rl->d_excl_rows;
            p.excl_vals = rl->d_excl_vals;
            p.n_excl = rl->n_excl;
        } else {
            p.rank_k = 0x7fff7fffu;
        }
        const CUtensorMap& tm = c.layout ? rank_tensor_map(*rl, s, ctx.n_cols, c) : tensor_map(s, ctx.n_cols, c);
        launch_tma(c, e0, tm, p, grid, smem, st, &s);
    } else {
        const size_t smem = 8 * P + 16;
        if (smem > (size_t)s.max_smem) fail(EBIC_ERR_INVALID_ARGUMENT, "population too large for one launch");
        if (p.host_cbf) {  // the direct kernel reads the CBF straight from device memory
            CK(cudaMemcpyAsync(s.d_in, host_cbf, cbf_bytes, cudaMemcpyHostToDevice, st));
            p.host_cbf = nullptr;
        }
        const int grid = (int)((s.rows + 255) / 256);
        s.last_grid = grid;
        s.last_kernel = 1;
        s.last_cfg = c;
        s.last_collapsed = false;
        ensure_partial(s, P, grid, (int)p.reduce_striped);
        p.partial = s.d_partial;
        if (e0) {
            CK(cudaFuncSetAttribute(count_direct_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            count_direct_kernel<true><<<grid, 256, smem, st>>>(p);
        } else {
            CK(cudaFuncSetAttribute(count_direct_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            count_direct_kernel<false><<<grid, 256, smem, st>>>(p);
        }
        CK(cudaGetLastError());
    }
}

// Reference-side validation of a host CBF before it reaches the device:
// offsets start at 0 and never decrease (cbf.hpp:70-79) and every column index
// addresses the matrix (cbf.hpp:32-37).  count_matches itself does not check
// (its caller guarantees validity); the device must not read out of bounds, so
// the C ABI rejects what would be undefined behaviour in the reference.
void validate_cbf(const size_t* off, const uint16_t* cols, size_t P, size_t n_cols) {
    if (!off) fail(EBIC_ERR_INVALID_ARGUMENT, "corrupt CBF");
    if (off[0] != 0) fail(EBIC_ERR_RUNTIME, "corrupt CBF");
    // Branch-free reductions (vectorised by the compiler); the error paths
    // are taken only after the scan.
    size_t descending = 0;
    for (size_t p = 0; p < P; ++p) descending |= static_cast<size_t>(off[p + 1] < off[p]);
    if (descending) fail(EBIC_ERR_RUNTIME, "corrupt CBF");
    const size_t L = off[P];
    if (L && !cols) fail(EBIC_ERR_INVALID_ARGUMENT, "corrupt CBF");
    uint16_t hi = 0;
    for (size_t i = 0; i < L; ++i) hi = std::max(hi, cols[i]);
    if (L && hi >= n_cols) fail(EBIC_ERR_INVALID_ARGUMENT, "invalid series");
}

// Packs the CBF into pinned memory, copies it to every shard, launches the
// count kernel per shard; the kernel's final CTA writes counts (and fitness)
// straight into mapped pinned host memory and raises a completion flag, which
// the host polls -- no device-to-host copy and no stream synchronisation on
// the per-generation path (cudaStreamQuery is consulted while polling so a
// failed launch surfaces as an error instead of a hang).
void wait_flag(Shard& s, unsigned long long seq) {
    volatile unsigned long long* flag = reinterpret_cast<volatile unsigned long long*>(s.h_map);
    for (uint64_t spin = 0;; ++spin) {
        if (*flag == seq) return;
        if ((spin & 1023) == 1023) {
            const cudaError_t e = cudaStreamQuery(s.stream);
            if (e == cudaSuccess) {
                if (*flag == seq) return;
                fail(EBIC_ERR_CUDA, "count kernel finished without its completion flag");
            }
            if (e != cudaErrorNotReady) cuda_check(e, "count kernel");
        }
    }
}

using HostClock = std::chrono::steady_clock;
inline double us_since(HostClock::time_point& t) {
    const auto n = HostClock::now();
    const double d = std::chrono::duration<double, std::micro>(n - t).count();
    t = n;
    return d;
}

// The host CBF staged in a shard's mapped pinned buffer (read by the device:
// CTA 0 copies it into d_in inside the count kernel): offsets at byte 0,
// columns from the next 16-byte boundary.  Returns where the columns start and
// the staged size.
struct StagedCbf {
    size_t cols_at = 0;
    size_t bytes = 0;
};

StagedCbf stage_cbf(Shard& s, const size_t* off, const uint16_t* cols, size_t P) {
    static_assert(sizeof(size_t) == sizeof(uint64_t), "size_t must be 64-bit");
    const size_t L = off[P];
    StagedCbf st;
    st.cols_at = ((P + 1) * sizeof(uint64_t) + 15) & ~size_t(15);
    st.bytes = st.cols_at + L * sizeof(uint16_t);
    grow_mapped(&s.h_in_map, &s.h_in_map_cap, st.bytes + 64);
    grow_device(&s.d_in, &s.d_in_cap, st.bytes + 64);
    std::memcpy(s.h_in_map, off, (P + 1) * sizeof(uint64_t));
    if (L) std::memcpy(s.h_in_map + st.cols_at, cols, L * sizeof(uint16_t));
    return st;
}

// Cross-shard reduction setup: peer access from every shard's device to
// shards[0]'s, and the accumulator (zeroed; the last arriver of each launch
// re-zeroes what it consumes).  Returns false when unavailable.
bool setup_xshard(ebic_ctx& ctx, size_t P) {
    if (ctx.xshard == 0 || !ctx.shards[0].knobs.xshard) return false;
    const int home = ctx.shards[0].device;
    if (ctx.xshard < 0) {
        for (const Shard& s : ctx.shards) {
            if (s.device == home) continue;
            int can = 0;
            if (cudaDeviceCanAccessPeer(&can, s.device, home) != cudaSuccess || !can) {
                (void)cudaGetLastError();
                ctx.xshard = 0;
                return false;
            }
            DeviceGuard g(s.device);
            const cudaError_t e = cudaDeviceEnablePeerAccess(home, 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
                (void)cudaGetLastError();
                ctx.xshard = 0;
                return false;
            }
            (void)cudaGetLastError();
        }
        DeviceGuard g(home);
        CK(cudaMalloc(&ctx.d_xticket, sizeof(unsigned int)));
        CK(cudaMemset(ctx.d_xticket, 0, sizeof(unsigned int)));
        ctx.xshard = 1;
    }
    if (P > ctx.xacc_cap) {
        DeviceGuard g(home);
        for (const Shard& s : ctx.shards) CK(cudaStreamSynchronize(s.stream));
        if (ctx.d_xacc) CK(cudaFree(ctx.d_xacc));
        ctx.d_xacc = nullptr;
        const size_t n = std::max<size_t>(P, 2 * ctx.xacc_cap);
        CK(cudaMalloc(&ctx.d_xacc, n * sizeof(unsigned long long)));
        CK(cudaMemset(ctx.d_xacc, 0, n * sizeof(unsigned long long)));
        ctx.xacc_cap = n;
    }
    return true;
}

// Several shards, one launch each: every shard's kernel adds its totals into
// the home accumulator; the last one to finish writes counts + fitness for
// the whole matrix into shards[0]'s mapped buffer and raises its flag.
void host_evaluate_xshard(ebic_ctx& ctx, const size_t* off, const uint16_t* cols, size_t P, size_t L,
                          double eps, bool want_fit, uint64_t sigma, uint64_t* counts_out,
                          double* fit_out, HostClock::time_point& tp) {
    Shard& s0 = ctx.shards[0];
    {
        DeviceGuard g(s0.device);
        grow_mapped(&s0.h_map, &s0.h_map_cap, 128 + P * 16);
    }
    uint64_t* m_counts = reinterpret_cast<uint64_t*>(s0.h_map + 128);
    double* m_fit = want_fit ? reinterpret_cast<double*>(s0.h_map + 128 + P * 8) : nullptr;
    const unsigned long long seq = ++s0.seq;
    // A failure after some shards launched would leave partial sums in the
    // accumulator and the ticket short: drain and re-zero both, then rethrow.
    auto reset_partial = [&] {
        for (Shard& s : ctx.shards) {
            cudaSetDevice(s.device);
            cudaStreamSynchronize(s.stream);
        }
        cudaSetDevice(s0.device);
        cudaMemset(ctx.d_xacc, 0, ctx.xacc_cap * sizeof(unsigned long long));
        cudaMemset(ctx.d_xticket, 0, sizeof(unsigned int));
        cudaDeviceSynchronize();
        (void)cudaGetLastError();
    };
    try {
    // every shard stages and launches on its own host thread (ShardPool)
    ctx.for_shards([&](Shard& s) {
        const StagedCbf in = stage_cbf(s, off, cols, P);
        if (s.knobs.host_copy)
            CK(cudaMemcpyAsync(s.d_in, s.h_in_map, in.bytes, cudaMemcpyHostToDevice, s.stream));
        if (&s == &s0) s0.host_us[1] += us_since(tp);
        const auto* d_off = reinterpret_cast<const uint64_t*>(s.d_in);
        const auto* d_cols = reinterpret_cast<const uint16_t*>(s.d_in + in.cols_at);
        launch_count(ctx, s, d_off, d_cols, P, L, eps, m_counts, m_fit, sigma, s.stream, 0,
                     reinterpret_cast<unsigned long long*>(s0.h_map), seq,
                     s.knobs.host_copy ? nullptr : s.h_in_map, in.bytes, ctx.d_xacc, ctx.d_xticket,
                     static_cast<uint32_t>(ctx.shards.size()));
        if (&s == &s0) s0.host_us[2] += us_since(tp);
    });
    volatile unsigned long long* flag = reinterpret_cast<volatile unsigned long long*>(s0.h_map);
    for (uint64_t spin = 0;; ++spin) {
        if (*flag == seq) break;
        if ((spin & 1023) == 1023) {
            bool idle = true;
            for (Shard& s : ctx.shards) {
                DeviceGuard g(s.device);
                const cudaError_t e = cudaStreamQuery(s.stream);
                if (e == cudaErrorNotReady) idle = false;
                else if (e != cudaSuccess) cuda_check(e, "count kernel");
            }
            if (idle) {
                if (*flag == seq) break;
                fail(EBIC_ERR_CUDA, "cross-shard count finished without its completion flag");
            }
        }
    }
    } catch (...) {
        reset_partial();
        throw;
    }
    s0.host_us[3] += us_since(tp);
    if (counts_out) std::memcpy(counts_out, m_counts, P * 8);
    if (want_fit) std::memcpy(fit_out, m_fit, P * 8);
    s0.host_us[4] += us_since(tp);
    ++s0.host_calls;
}

void host_evaluate(ebic_ctx& ctx, const size_t* off, const uint16_t* cols, size_t P, double eps,
                   bool want_fit, uint64_t sigma, uint64_t* counts_out, double* fit_out) {
    if (P == 0) return;
    Shard& s0 = ctx.shards[0];
    auto tp = HostClock::now();
    validate_cbf(off, cols, P, ctx.n_cols);
    s0.host_us[0] += us_since(tp);
    const size_t L = off[P];
    const bool single = ctx.shards.size() == 1;
    if (!single && P <= kMaxSeriesPerLaunch && L <= kMaxLenPerLaunch && setup_xshard(ctx, P)) {
        host_evaluate_xshard(ctx, off, cols, P, L, eps, want_fit, sigma, counts_out, fit_out, tp);
        return;
    }
    ctx.for_shards([&](Shard& s) {
        grow_mapped(&s.h_map, &s.h_map_cap, 128 + P * 16);
        // A single TMA launch copies the staged CBF to the device itself (CTA
        // 0, stage_host_cbf): no cudaMemcpyAsync on the per-generation path.
        // Otherwise one async copy.
        const StagedCbf in = stage_cbf(s, off, cols, P);
        const size_t cols_at = in.cols_at, in_bytes = in.bytes;
        const bool one_launch = P <= kMaxSeriesPerLaunch && L <= kMaxLenPerLaunch &&
                                !s.knobs.host_copy;
        if (!one_launch)
            CK(cudaMemcpyAsync(s.d_in, s.h_in_map, in_bytes, cudaMemcpyHostToDevice, s.stream));
        if (&s == &s0) s0.host_us[1] += us_since(tp);
        uint64_t* m_counts = reinterpret_cast<uint64_t*>(s.h_map + 128);
        double* m_fit = (single && want_fit) ? reinterpret_cast<double*>(s.h_map + 128 + P * 8) : nullptr;
        const auto* d_off = reinterpret_cast<const uint64_t*>(s.d_in);
        const auto* d_cols = reinterpret_cast<const uint16_t*>(s.d_in + cols_at);
        const unsigned long long seq = ++s.seq;
        // One launch per slice of at most kMaxSeriesPerLaunch series /
        // kMaxLenPerLaunch columns (the per-CTA work list lives in shared
        // memory); a generation (P ~ 600) is always a single launch.  Only
        // the last launch raises the flag (launches are stream-ordered).
        for (size_t a = 0; a < P;) {
            size_t b = a;
            while (b < P && b - a < kMaxSeriesPerLaunch && off[b + 1] - off[a] <= kMaxLenPerLaunch) ++b;
            if (b == a) b = a + 1;  // a single over-long series still gets its own launch
            const bool last = b == P;
            launch_count(ctx, s, d_off + a, d_cols, b - a, off[b] - off[a], eps, m_counts + a,
                         m_fit ? m_fit + a : nullptr, sigma, s.stream, off[a],
                         last ? reinterpret_cast<unsigned long long*>(s.h_map) : nullptr, seq,
                         one_launch ? s.h_in_map : nullptr, in_bytes);
            a = b;
        }
        if (&s == &s0) s0.host_us[2] += us_since(tp);
    });
    std::vector<uint64_t> total;
    if (!single) total.assign(P, 0);
    for (Shard& s : ctx.shards) {
        DeviceGuard g(s.device);
        wait_flag(s, s.seq);
        if (&s == &s0) s0.host_us[3] += us_since(tp);
        const uint64_t* c = reinterpret_cast<const uint64_t*>(s.h_map + 128);
        if (single) {
            if (counts_out) std::memcpy(counts_out, c, P * 8);
            if (want_fit) std::memcpy(fit_out, s.h_map + 128 + P * 8, P * 8);
        } else {
            for (size_t p = 0; p < P; ++p) total[p] += c[p];  // exact integer reduction
        }
    }
    if (!single) {
        if (counts_out) std::memcpy(counts_out, total.data(), P * 8);
        if (want_fit)
            for (size_t p = 0; p < P; ++p)
                fit_out[p] = ebic_fitness_score(total[p], off[p + 1] - off[p], sigma);
    }
    s0.host_us[4] += us_since(tp);
    ++s0.host_calls;
}

// Membership bitmasks of every shard gathered into global word order.
void host_membership(ebic_ctx& ctx, const size_t* off, const uint16_t* cols, size_t S, double eps,
                     size_t k, uint64_t* ex, uint64_t* ng, uint64_t* ap) {
    if (S == 0) return;
    validate_cbf(off, cols, S, ctx.n_cols);
    if (S > 65535) fail(EBIC_ERR_INVALID_ARGUMENT, "too many series for one membership launch");
    const size_t L = off[S];
    const size_t words_total = (ctx.n_rows + 63) / 64;
    const size_t off_bytes = (S + 1) * 8, cols_at = (off_bytes + 15) & ~size_t(15);
    const size_t in_bytes = cols_at + L * 2;
    uint64_t* outs[3] = {ex, ng, ap};
    for (Shard& s : ctx.shards) {
        DeviceGuard g(s.device);
        const size_t words = (s.rows + 63) / 64;
        const size_t bits_bytes = S * words * 8;
        grow_pinned(&s.h_pin, &s.h_pin_cap, in_bytes);
        grow_device(&s.d_in, &s.d_in_cap, in_bytes);
        grow_device(&s.d_out, &s.d_out_cap, 3 * bits_bytes);
        std::memcpy(s.h_pin, off, off_bytes);
        if (L) std::memcpy(s.h_pin + cols_at, cols, L * 2);
        CK(cudaMemcpyAsync(s.d_in, s.h_pin, in_bytes, cudaMemcpyHostToDevice, s.stream));
        uint64_t* d_bits[3];
        for (int i = 0; i < 3; ++i)
            d_bits[i] = outs[i] ? reinterpret_cast<uint64_t*>(s.d_out + i * bits_bytes) : nullptr;
        dim3 grid((unsigned)((s.rows + 255) / 256), (unsigned)S);
        const auto* d_off = reinterpret_cast<const uint64_t*>(s.d_in);
        const auto* d_cols = reinterpret_cast<const uint16_t*>(s.d_in + cols_at);
        if (eps == 0.0)
            membership_kernel<true><<<grid, 256, 0, s.stream>>>(s.d_mat, (uint32_t)s.ld, (uint32_t)s.rows, d_off, d_cols, eps, (uint64_t)k, (uint32_t)words, d_bits[0], d_bits[1], d_bits[2]);
        else
            membership_kernel<false><<<grid, 256, 0, s.stream>>>(s.d_mat, (uint32_t)s.ld, (uint32_t)s.rows, d_off, d_cols, eps, (uint64_t)k, (uint32_t)words, d_bits[0], d_bits[1], d_bits[2]);
        CK(cudaGetLastError());
        const size_t word0 = (s.row_begin - ctx.row_begin) / 64;
        for (int i = 0; i < 3; ++i) {
            if (!outs[i]) continue;
            CK(cudaMemcpy2DAsync(outs[i] + word0, words_total * 8, d_bits[i], words * 8, words * 8, S,
                                 cudaMemcpyDeviceToHost, s.stream));
        }
    }
    for (Shard& s : ctx.shards) {
        DeviceGuard g(s.device);
        CK(cudaStreamSynchronize(s.stream));
    }
}

Shard& single_shard(ebic_ctx* ctx) {
    if (!ctx) fail(EBIC_ERR_INVALID_ARGUMENT, "null context");
    if (ctx->shards.size() != 1) fail(EBIC_ERR_INVALID_ARGUMENT, "device-pointer API needs a single-shard context");
    return ctx->shards[0];
}

void free_shard(Shard& s) {
    cudaSetDevice(s.device);
    for (Shard::GraphSlot& g : s.graphs) {
        cudaGraphExecDestroy(g.exec);
        cudaGraphDestroy(g.g);
    }
    s.graphs.clear();
    if (s.stream) cudaStreamSynchronize(s.stream);
    cudaFree(s.d_mat);
    cudaFree(s.d_in);
    cudaFree(s.d_partial);
    cudaFree(s.d_done);
    cudaFree(s.d_out);
    if (s.h_pin) cudaFreeHost(s.h_pin);
    if (s.h_map) cudaFreeHost(s.h_map);
    if (s.h_in_map) cudaFreeHost(s.h_in_map);
    cudaFree(s.tables.d_log);
    cudaFree(s.tables.d_exp);
    for (RankLayout& rl : s.ranks) {
        cudaFree(rl.d);
        cudaFree(rl.d10);
        cudaFree(rl.d_row_excl);
        cudaFree(rl.d_excl_rows);
        cudaFree(rl.d_excl_vals);
    }
    cudaFree(s.d_phase);
    if (s.switch_event) cudaEventDestroy(s.switch_event);
    if (s.stream) cudaStreamDestroy(s.stream);
}

ebic_ctx* make_ctx(const double* rows_ptr, size_t n_rows, size_t n_cols, size_t total_rows,
                   size_t row_begin, const int* devices, int n_devices, bool on_device) {
    if (n_rows == 0 || total_rows == 0) fail(EBIC_ERR_INVALID_ARGUMENT, "matrix has no rows");
    if (n_cols == 0) fail(EBIC_ERR_INVALID_ARGUMENT, "matrix has no columns");
    if (n_cols > 65535) fail(EBIC_ERR_INVALID_ARGUMENT, "too many columns (at most 65535 supported)");
    if (!rows_ptr) fail(EBIC_ERR_INVALID_ARGUMENT, "null matrix");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        (void)cudaGetLastError();
        fail(EBIC_ERR_NO_DEVICE, "no CUDA device available");
    }
    std::vector<int> devs;
    if (!devices || n_devices <= 0) devs.push_back(0);
    else devs.assign(devices, devices + n_devices);
    for (int d : devs)
        if (d < 0 || d >= ndev) fail(EBIC_ERR_INVALID_ARGUMENT, "invalid device id");
    auto ctx = std::make_unique<ebic_ctx>();
    ctx->n_rows = n_rows;
    ctx->n_cols = n_cols;
    ctx->row_begin = row_begin;
    ctx->total_rows = total_rows;
    // 64-row aligned contiguous shards (bitmask words concatenate across shards).
    size_t per = (n_rows + devs.size() - 1) / devs.size();
    per = (per + 63) / 64 * 64;
    size_t r = 0;
    for (size_t i = 0; i < devs.size() && r < n_rows; ++i) {
        Shard s;
        s.device = devs[i];
        s.row_begin = row_begin + r;
        s.rows = std::min(per, n_rows - r);
        ctx->shards.push_back(s);
        r += s.rows;
    }
    try {
        for (Shard& s : ctx->shards)
            upload_shard(s, rows_ptr + (s.row_begin - row_begin) * n_cols, n_cols, on_device);
    } catch (...) {
        for (Shard& s : ctx->shards) free_shard(s);
        throw;
    }
    return ctx.release();
}

// Row list of the set bits of `bits` (ctx-local rows) as global row ids.
template <class F>
void for_each_bit(const uint64_t* bits, size_t words, F&& f) {
    for (size_t w = 0; w < words; ++w) {
        uint64_t x = bits[w];
        while (x) {
            const int b = __builtin_ctzll(x);
            f(w * 64 + b);
            x &= x - 1;
        }
    }
}

}  // namespace

// ---------------------------------------------------------------------------
// Multi-process row shards (one process per GPU): the count kernels reduce
// across processes themselves.  Rank 0 owns one device allocation
// [ticket | 256 B pad | accumulator u64[max_series]] shared through a CUDA IPC
// handle, and a POSIX shared-memory result block [flag (128 B) | counts |
// fitness] that every rank maps and registers with its CUDA context.  Each
// rank's final CTA adds its shard's totals into the accumulator and takes the
// ticket; the last rank's final CTA writes counts + Eq. 1 for the whole matrix
// into the shared block and raises its flag, which every rank's host polls.
// No kernel ever waits for another, so ranks may even share one GPU.
// ---------------------------------------------------------------------------
namespace {

constexpr size_t kXAccOffset = 256;

// Rank 0's accumulator between ebic_xgroup_create and its own join.
std::mutex& xgroup_owned_mu() {
    static std::mutex m;
    return m;
}
std::map<std::string, unsigned char*>& xgroup_owned() {
    static std::map<std::string, unsigned char*> t;
    return t;
}

}  // namespace

struct ebic_xgroup {
    ebic_ctx* ctx = nullptr;
    int n_ranks = 0;
    bool owner = false;          // rank 0: allocated the accumulator, unlinks the shm
    size_t max_series = 0;
    unsigned char* d_base = nullptr;  // accumulator allocation (own or IPC-opened)
    unsigned char* shm = nullptr;     // mapped result block
    unsigned char* dev_shm = nullptr; // its device address
    cudaStream_t launch_stream = nullptr;  // stream of the last launch (polled while waiting)
    size_t shm_bytes = 0;
    std::string shm_name;
    unsigned long long last_seq = 0;
};

namespace {

size_t xgroup_shm_bytes(size_t max_series) {
    const size_t b = 128 + 16 * max_series;
    return (b + 4095) & ~size_t(4095);
}

unsigned char* map_shm(const char* name, size_t bytes, bool create) {
    const int fd = shm_open(name, create ? (O_CREAT | O_RDWR | O_EXCL) : O_RDWR, 0600);
    if (fd < 0) fail(EBIC_ERR_RUNTIME, std::string("shm_open failed for ") + name);
    if (create && ftruncate(fd, static_cast<off_t>(bytes)) != 0) {
        close(fd);
        fail(EBIC_ERR_RUNTIME, "ftruncate of the shared result block failed");
    }
    void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (p == MAP_FAILED) fail(EBIC_ERR_RUNTIME, "mmap of the shared result block failed");
    if (create) std::memset(p, 0, bytes);
    return static_cast<unsigned char*>(p);
}

}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

const char* ebic_last_error(void) { return g_last_error.c_str(); }

int ebic_abi_version(void) { return EBIC_B200_ABI_VERSION; }

int ebic_device_count(int* count_out) {
    return guarded([&] {
        if (!count_out) fail(EBIC_ERR_INVALID_ARGUMENT, "null output");
        int n = 0;
        if (cudaGetDeviceCount(&n) != cudaSuccess) {
            (void)cudaGetLastError();
            n = 0;
        }
        *count_out = n;
    });
}

int ebic_ctx_create(const double* row_major, size_t n_rows, size_t n_cols, const int* devices,
                    int n_devices, ebic_ctx** ctx_out) {
    return guarded([&] {
        if (!ctx_out) fail(EBIC_ERR_INVALID_ARGUMENT, "null output");
        *ctx_out = make_ctx(row_major, n_rows, n_cols, n_rows, 0, devices, n_devices, false);
    });
}

int ebic_ctx_create_shard(const double* row_major_shard, size_t shard_rows, size_t n_cols,
                          size_t total_rows, size_t row_begin, int device, ebic_ctx** ctx_out) {
    return guarded([&] {
        if (!ctx_out) fail(EBIC_ERR_INVALID_ARGUMENT, "null output");
        if (row_begin + shard_rows > total_rows) fail(EBIC_ERR_INVALID_ARGUMENT, "shard outside matrix");
        *ctx_out = make_ctx(row_major_shard, shard_rows, n_cols, total_rows, row_begin, &device, 1, false);
    });
}

int ebic_ctx_create_shard_device(const double* d_row_major, size_t shard_rows, size_t n_cols,
                                 size_t total_rows, size_t row_begin, int device,
                                 ebic_ctx** ctx_out) {
    return guarded([&] {
        if (!ctx_out) fail(EBIC_ERR_INVALID_ARGUMENT, "null output");
        if (row_begin + shard_rows > total_rows) fail(EBIC_ERR_INVALID_ARGUMENT, "shard outside matrix");
        *ctx_out = make_ctx(d_row_major, shard_rows, n_cols, total_rows, row_begin, &device, 1, true);
    });
}

int ebic_ctx_destroy(ebic_ctx* ctx) {
    return guarded([&] {
        if (!ctx) return;
        ctx->pool.reset();  // join the launch threads before their shards go away
        for (Shard& s : ctx->shards) free_shard(s);
        if (ctx->d_xacc || ctx->d_xticket) {
            cudaSetDevice(ctx->shards[0].device);
            cudaFree(ctx->d_xacc);
            cudaFree(ctx->d_xticket);
        }
        delete ctx;
    });
}

int ebic_ctx_get_info(const ebic_ctx* ctx, ebic_ctx_info* info) {
    return guarded([&] {
        if (!ctx || !info) fail(EBIC_ERR_INVALID_ARGUMENT, "null argument");
        std::memset(info, 0, sizeof(*info));
        info->n_rows = ctx->n_rows;
        info->n_cols = ctx->n_cols;
        info->row_begin = ctx->row_begin;
        info->total_rows = ctx->total_rows;
        info->n_shards = (int)ctx->shards.size();
        const Shard& s = ctx->shards[0];
        info->rows_per_tile = s.last_cfg.rpg;
        info->stages = s.last_cfg.stages;
        info->grid = s.last_grid;
        info->device_bytes = s.ld * ctx->n_cols * sizeof(double);
        info->sm_count = s.sm_count;
        info->layout = s.last_cfg.layout;
        if (s.last_cfg.layout == 1 && s.last_collapsed) info->layout = 3;
        if (s.last_cfg.layout == 3) info->layout = s.last_collapsed ? 5 : 4;  // packed 10-bit fields
        if (s.last_cfg.layout == 4) info->layout = s.last_collapsed ? 7 : 6;  // packed 12-bit fields
        info->consumer_warps = s.last_cfg.ncw == 32 ? 31 : s.last_cfg.ncw;
        info->kernel = s.last_kernel;
    });
}

int ebic_count_matches(ebic_ctx* ctx, const size_t* offsets, const uint16_t* cols,
                       size_t n_series, double eps, uint64_t* counts_out) {
    return guarded([&] {
        if (!ctx) fail(EBIC_ERR_INVALID_ARGUMENT, "null context");
        if (n_series && !counts_out) fail(EBIC_ERR_INVALID_ARGUMENT, "null output");
        host_evaluate(*ctx, offsets, cols, n_series, eps, false, 0, counts_out, nullptr);
    });
}

int ebic_evaluate_population(ebic_ctx* ctx, const size_t* offsets, const uint16_t* cols,
                             size_t n_series, uint64_t sigma, double eps, uint64_t* counts_out,
                             double* fitness_out) {
    return guarded([&] {
        if (!ctx) fail(EBIC_ERR_INVALID_ARGUMENT, "null context");
        if (n_series && !fitness_out) fail(EBIC_ERR_INVALID_ARGUMENT, "null output");
        host_evaluate(*ctx, offsets, cols, n_series, eps, true, sigma, counts_out, fitness_out);
    });
}

double ebic_fitness_score(uint64_t match_count, size_t series_len, uint64_t sigma) {
    // fitness.hpp:124-133, verbatim arithmetic.
    if (match_count <= 1) return 0.0;
    double f = static_cast<double>(series_len) * std::log(static_cast<double>(match_count - 1));
    if (match_count < sigma)
        f *= std::exp2(static_cast<double>(match_count) - static_cast<double>(sigma));
    return f > 0.0 ? f : 0.0;
}

int ebic_fitness_scores_host(const uint64_t* counts, const size_t* offsets, size_t n_series,
                             uint64_t sigma, double* fitness_out) {
    return guarded([&] {
        if (n_series && (!counts || !offsets || !fitness_out)) fail(EBIC_ERR_INVALID_ARGUMENT, "null argument");
        for (size_t p = 0; p < n_series; ++p)
            fitness_out[p] = ebic_fitness_score(counts[p], offsets[p + 1] - offsets[p], sigma);
    });
}

uint64_t ebic_default_sigma(size_t n_rows) {
    const uint64_t scaled = static_cast<uint64_t>((n_rows + 49) / 50);  // fitness.hpp:48-52
    return scaled < 4 ? 4 : scaled;
}

int ebic_count_matches_device(ebic_ctx* ctx, const uint64_t* d_offsets, const uint16_t* d_cols,
                              size_t n_series, size_t total_len, double eps, uint64_t sigma,
                              uint64_t* d_counts_out, double* d_fitness_out, void* stream) {
    return guarded([&] {
        Shard& s = single_shard(ctx);
        DeviceGuard g(s.device);
        if (n_series && (!d_offsets || !d_counts_out)) fail(EBIC_ERR_INVALID_ARGUMENT, "null argument");
        // Fused Eq. 1 only when the counts are final (whole-matrix context).
        const bool whole = ctx->row_begin == 0 && ctx->n_rows == ctx->total_rows;
        if (d_fitness_out && !whole) fail(EBIC_ERR_INVALID_ARGUMENT, "fitness needs reduced counts on a shard context");
        if (n_series > kMaxSeriesPerLaunch || total_len > kMaxLenPerLaunch)
            fail(EBIC_ERR_INVALID_ARGUMENT, "device batch exceeds 2048 series / 8192 columns; split it");
        cudaStream_t st = static_cast<cudaStream_t>(stream);  // 0 = legacy default stream
        launch_count(*ctx, s, d_offsets, d_cols, n_series, total_len, eps, d_counts_out, d_fitness_out,
                     sigma, st, 0);  // device CBF: offsets[0] == 0 (cbf.hpp:43-52)
    });
}

int ebic_fitness_device(ebic_ctx* ctx, const uint64_t* d_counts, const uint64_t* d_offsets,
                        size_t n_series, uint64_t sigma, double* d_fitness_out, void* stream) {
    return guarded([&] {
        Shard& s = single_shard(ctx);
        DeviceGuard g(s.device);
        if (n_series == 0) return;
        const Tables& t = ensure_tables(s, sigma, ctx->total_rows);
        cudaStream_t st = static_cast<cudaStream_t>(stream);  // 0 = legacy default stream
        fitness_kernel<<<(unsigned)((n_series + 255) / 256), 256, 0, st>>>(
            d_counts, d_offsets, (uint32_t)n_series, sigma, t.d_log, t.d_exp, d_fitness_out);
        CK(cudaGetLastError());
    });
}

int ebic_ctx_phase_times(ebic_ctx* ctx, uint64_t* stamps_out, size_t max_ctas, size_t* n_ctas) {
    return guarded([&] {
        Shard& s = single_shard(ctx);
        DeviceGuard g(s.device);
        if (!n_ctas) fail(EBIC_ERR_INVALID_ARGUMENT, "null argument");
        *n_ctas = s.d_phase ? (size_t)s.last_grid : 0;
        if (!s.d_phase || !stamps_out) return;
        // rows beyond the grid: K1v2's per-item stamps of CTA 0 (rows 512+)
        const size_t n = std::min<size_t>(max_ctas, 4096);
        CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(stamps_out, s.d_phase, n * 8 * sizeof(uint64_t), cudaMemcpyDeviceToHost));
    });
}

int ebic_ctx_host_timers(ebic_ctx* ctx, double* mean_us_out, uint64_t* calls_out) {
    return guarded([&] {
        if (!ctx || !mean_us_out) fail(EBIC_ERR_INVALID_ARGUMENT, "null argument");
        const Shard& s = ctx->shards[0];
        for (int i = 0; i < 5; ++i) mean_us_out[i] = s.host_calls ? s.host_us[i] / s.host_calls : 0.0;
        if (calls_out) *calls_out = s.host_calls;
    });
}

int ebic_membership_bits(ebic_ctx* ctx, const size_t* offsets, const uint16_t* cols,
                         size_t n_series, double eps, size_t approx_k, uint64_t* exact_bits,
                         uint64_t* neg_bits, uint64_t* approx_bits) {
    return guarded([&] {
        if (!ctx) fail(EBIC_ERR_INVALID_ARGUMENT, "null context");
        host_membership(*ctx, offsets, cols, n_series, eps, approx_k, exact_bits, neg_bits, approx_bits);
    });
}

int ebic_assign_rows(ebic_ctx* ctx, const uint16_t* series, size_t len, double eps,
                     uint64_t* rows_out, size_t* n_out) {
    return guarded([&] {
        if (!ctx || !n_out) fail(EBIC_ERR_INVALID_ARGUMENT, "null argument");
        if (len == 0) fail(EBIC_ERR_INVALID_ARGUMENT, "invalid series");
        const size_t off[2] = {0, len};
        const size_t words = (ctx->n_rows + 63) / 64;
        std::vector<uint64_t> ex(words);
        host_membership(*ctx, off, series, 1, eps, 0, ex.data(), nullptr, nullptr);
        size_t n = 0;
        for_each_bit(ex.data(), words, [&](size_t r) { rows_out[n++] = ctx->row_begin + r; });
        *n_out = n;
    });
}

int ebic_expand_bicluster(ebic_ctx* ctx, const uint16_t* series, size_t len,
                          const uint64_t* core_rows, const uint8_t* core_flags, size_t n_core,
                          int allow_negative, size_t approx_k, double eps, uint64_t* rows_out,
                          uint8_t* flags_out, size_t* n_out) {
    return guarded([&] {
        if (!ctx || !n_out) fail(EBIC_ERR_INVALID_ARGUMENT, "null argument");
        if (len == 0) fail(EBIC_ERR_INVALID_ARGUMENT, "invalid series");
        const size_t off[2] = {0, len};
        const size_t words = (ctx->n_rows + 63) / 64;
        std::vector<uint64_t> ng(words, 0), ap(words, 0);
        const bool want_neg = allow_negative != 0, want_ap = approx_k > 0;
        if (want_neg || want_ap)
            host_membership(*ctx, off, series, 1, eps, approx_k, nullptr, want_neg ? ng.data() : nullptr,
                            want_ap ? ap.data() : nullptr);
        // Candidate rows (ctx-local): negative first, then approximate; drop core rows.
        std::vector<uint64_t> cand(words);
        for (size_t w = 0; w < words; ++w) cand[w] = ng[w] | ap[w];
        for (size_t i = 0; i < n_core; ++i) {
            const uint64_t r = core_rows[i];
            if (r >= ctx->row_begin && r < ctx->row_begin + ctx->n_rows) {
                const uint64_t l = r - ctx->row_begin;
                cand[l / 64] &= ~(uint64_t(1) << (l % 64));
            }
        }
        // Merge ascending core rows with the added rows (expansion.hpp:73-86).
        size_t n = 0, ci = 0;
        auto emit_core_upto = [&](uint64_t row) {
            while (ci < n_core && core_rows[ci] < row) {
                rows_out[n] = core_rows[ci];
                flags_out[n] = core_flags[ci];
                ++n, ++ci;
            }
        };
        for_each_bit(cand.data(), words, [&](size_t l) {
            const uint64_t row = ctx->row_begin + l;
            emit_core_upto(row);
            const bool neg = (ng[l / 64] >> (l % 64)) & 1;
            rows_out[n] = row;
            flags_out[n] = neg ? EBIC_ROW_NEGATIVE : EBIC_ROW_APPROXIMATE;
            ++n;
        });
        emit_core_upto(~uint64_t(0));
        while (ci < n_core) {
            rows_out[n] = core_rows[ci];
            flags_out[n] = core_flags[ci];
            ++n, ++ci;
        }
        *n_out = n;
    });
}

int ebic_resolve_expand_batch(ebic_ctx* ctx, const size_t* offsets, const uint16_t* cols,
                              size_t n_series, int allow_negative, size_t approx_k, double eps,
                              uint64_t* rows_out, uint8_t* flags_out, size_t* row_counts) {
    return guarded([&] {
        if (!ctx) fail(EBIC_ERR_INVALID_ARGUMENT, "null context");
        if (n_series == 0) return;
        const size_t words = (ctx->n_rows + 63) / 64;
        std::vector<uint64_t> ex(n_series * words), ng(n_series * words, 0), ap(n_series * words, 0);
        const bool want_neg = allow_negative != 0, want_ap = approx_k > 0;
        host_membership(*ctx, offsets, cols, n_series, eps, approx_k, ex.data(),
                        want_neg ? ng.data() : nullptr, want_ap ? ap.data() : nullptr);
        size_t n = 0;
        for (size_t s = 0; s < n_series; ++s) {
            const size_t start = n;
            const uint64_t* e = ex.data() + s * words;
            const uint64_t* g = ng.data() + s * words;
            const uint64_t* a = ap.data() + s * words;
            for (size_t w = 0; w < words; ++w) {
                uint64_t x = e[w] | g[w] | a[w];
                while (x) {
                    const int b = __builtin_ctzll(x);
                    const uint64_t bit = uint64_t(1) << b;
                    rows_out[n] = ctx->row_begin + w * 64 + b;
                    flags_out[n] = (e[w] & bit) ? EBIC_ROW_EXACT
                                   : (g[w] & bit) ? EBIC_ROW_NEGATIVE
                                                  : EBIC_ROW_APPROXIMATE;
                    ++n;
                    x &= x - 1;
                }
            }
            row_counts[s] = n - start;
        }
    });
}


// ---- multi-process row shards: in-kernel reduction over peer memory --------

int ebic_xgroup_create(ebic_ctx* ctx, size_t max_series, const char* shm_name, void* handle_out) {
    return guarded([&] {
        Shard& s = single_shard(ctx);
        if (!shm_name || !handle_out || max_series == 0) fail(EBIC_ERR_INVALID_ARGUMENT, "null argument");
        DeviceGuard g(s.device);
        unsigned char* d = nullptr;
        CK(cudaMalloc(&d, kXAccOffset + max_series * sizeof(unsigned long long)));
        CK(cudaMemset(d, 0, kXAccOffset + max_series * sizeof(unsigned long long)));
        cudaIpcMemHandle_t h;
        const cudaError_t e = cudaIpcGetMemHandle(&h, d);
        if (e != cudaSuccess) {
            cudaFree(d);
            cuda_check(e, "cudaIpcGetMemHandle");
        }
        unsigned char* shm = nullptr;
        try {
            shm = map_shm(shm_name, xgroup_shm_bytes(max_series), true);
        } catch (...) {
            cudaFree(d);
            throw;
        }
        munmap(shm, xgroup_shm_bytes(max_series));  // each rank (rank 0 too) maps it in join
        // Stash the allocation for rank 0's join: the handle's first bytes are
        // opaque; keep the pointer in a process-local table keyed by the name.
        std::memcpy(handle_out, &h, sizeof h);
        static_assert(sizeof(cudaIpcMemHandle_t) <= EBIC_XGROUP_HANDLE_BYTES, "handle size");
        std::lock_guard<std::mutex> lock(xgroup_owned_mu());
        xgroup_owned()[shm_name] = d;
    });
}

int ebic_xgroup_join(ebic_ctx* ctx, const void* handle, const char* shm_name, int n_ranks,
                     size_t max_series, ebic_xgroup** group_out) {
    return guarded([&] {
        Shard& s = single_shard(ctx);
        if (!handle || !shm_name || !group_out || n_ranks < 1 || max_series == 0)
            fail(EBIC_ERR_INVALID_ARGUMENT, "null argument");
        DeviceGuard g(s.device);
        auto grp = std::make_unique<ebic_xgroup>();
        grp->ctx = ctx;
        grp->n_ranks = n_ranks;
        grp->max_series = max_series;
        grp->shm_name = shm_name;
        {
            std::lock_guard<std::mutex> lock(xgroup_owned_mu());
            auto it = xgroup_owned().find(shm_name);
            if (it != xgroup_owned().end()) {
                grp->owner = true;
                grp->d_base = it->second;
                xgroup_owned().erase(it);
            }
        }
        if (!grp->owner) {
            cudaIpcMemHandle_t h;
            std::memcpy(&h, handle, sizeof h);
            void* p = nullptr;
            CK(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
            grp->d_base = static_cast<unsigned char*>(p);
        }
        grp->shm_bytes = xgroup_shm_bytes(max_series);
        // Undo what this join acquired if a later step fails.
        auto release = [&] {
            if (grp->shm) {
                cudaHostUnregister(grp->shm);
                munmap(grp->shm, grp->shm_bytes);
            }
            if (grp->owner) cudaFree(grp->d_base);
            else cudaIpcCloseMemHandle(grp->d_base);
            (void)cudaGetLastError();
        };
        try {
            grp->shm = map_shm(shm_name, grp->shm_bytes, false);
            CK(cudaHostRegister(grp->shm, grp->shm_bytes, cudaHostRegisterMapped | cudaHostRegisterPortable));
            CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&grp->dev_shm), grp->shm, 0));
        } catch (...) {
            release();
            throw;
        }
        grp->last_seq = *reinterpret_cast<volatile unsigned long long*>(grp->shm);
        *group_out = grp.release();
    });
}

namespace {

void xgroup_launch(ebic_xgroup* g, const uint64_t* d_off, const uint16_t* d_cols, size_t P, size_t L,
                   double eps, uint64_t sigma, bool want_fit, uint64_t seq, cudaStream_t st,
                   const void* host_cbf, size_t cbf_bytes) {
    ebic_ctx& ctx = *g->ctx;
    Shard& s = ctx.shards[0];
    if (P > g->max_series) fail(EBIC_ERR_INVALID_ARGUMENT, "population larger than the group's max_series");
    if (P > kMaxSeriesPerLaunch || L > kMaxLenPerLaunch)
        fail(EBIC_ERR_INVALID_ARGUMENT, "batch exceeds 2048 series / 8192 columns; split it");
    unsigned char* dev_shm = g->dev_shm;
    auto* counts = reinterpret_cast<uint64_t*>(dev_shm + 128);
    auto* fit = want_fit ? reinterpret_cast<double*>(dev_shm + 128 + 8 * g->max_series) : nullptr;
    auto* ticket = reinterpret_cast<unsigned int*>(g->d_base);
    auto* acc = reinterpret_cast<unsigned long long*>(g->d_base + kXAccOffset);
    launch_count(ctx, s, d_off, d_cols, P, L, eps, counts, fit, sigma, st, 0,
                 reinterpret_cast<unsigned long long*>(dev_shm), seq, host_cbf, cbf_bytes, acc, ticket,
                 static_cast<uint32_t>(g->n_ranks));
    g->launch_stream = st;
}

void xgroup_wait(ebic_xgroup* g, uint64_t seq, size_t P, uint64_t* counts_out, double* fit_out,
                 cudaStream_t st) {
    volatile unsigned long long* flag = reinterpret_cast<volatile unsigned long long*>(g->shm);
    const auto t0 = std::chrono::steady_clock::now();
    for (uint64_t spin = 0;; ++spin) {
        if (*flag >= seq) break;
        if ((spin & 4095) == 4095) {
            const cudaError_t e = cudaStreamQuery(st);
            if (e != cudaSuccess && e != cudaErrorNotReady) cuda_check(e, "count kernel");
            if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(60))
                fail(EBIC_ERR_RUNTIME, "cross-rank reduction timed out (did every rank launch this call?)");
        }
    }
    std::atomic_thread_fence(std::memory_order_acquire);
    if (counts_out) std::memcpy(counts_out, g->shm + 128, P * 8);
    if (fit_out) std::memcpy(fit_out, g->shm + 128 + 8 * g->max_series, P * 8);
    g->last_seq = seq;
}

}  // namespace

int ebic_xgroup_count(ebic_xgroup* g, const uint64_t* d_offsets, const uint16_t* d_cols, size_t n_series,
                      size_t total_len, double eps, uint64_t sigma, int want_fitness, uint64_t seq,
                      void* stream) {
    return guarded([&] {
        if (!g) fail(EBIC_ERR_INVALID_ARGUMENT, "null group");
        if (seq <= g->last_seq) fail(EBIC_ERR_INVALID_ARGUMENT, "call numbers must increase");
        if (n_series == 0) return;
        if (!d_offsets) fail(EBIC_ERR_INVALID_ARGUMENT, "null argument");
        DeviceGuard dg(g->ctx->shards[0].device);
        xgroup_launch(g, d_offsets, d_cols, n_series, total_len, eps, sigma, want_fitness != 0, seq,
                      static_cast<cudaStream_t>(stream), nullptr, 0);
    });
}

int ebic_xgroup_wait(ebic_xgroup* g, uint64_t seq, size_t n_series, uint64_t* counts_out,
                     double* fitness_out) {
    return guarded([&] {
        if (!g) fail(EBIC_ERR_INVALID_ARGUMENT, "null group");
        if (n_series > g->max_series) fail(EBIC_ERR_INVALID_ARGUMENT, "n_series above max_series");
        // poll the stream the count kernel was launched on, so a failed
        // launch surfaces at once instead of after the timeout
        xgroup_wait(g, seq, n_series, counts_out, fitness_out,
                    g->launch_stream ? g->launch_stream : g->ctx->shards[0].stream);
    });
}

int ebic_xgroup_evaluate(ebic_xgroup* g, const size_t* offsets, const uint16_t* cols, size_t n_series,
                         uint64_t sigma, double eps, uint64_t seq, uint64_t* counts_out,
                         double* fitness_out) {
    return guarded([&] {
        if (!g) fail(EBIC_ERR_INVALID_ARGUMENT, "null group");
        if (seq <= g->last_seq) fail(EBIC_ERR_INVALID_ARGUMENT, "call numbers must increase");
        if (n_series == 0) return;
        ebic_ctx& ctx = *g->ctx;
        Shard& s = ctx.shards[0];
        validate_cbf(offsets, cols, n_series, ctx.n_cols);
        const size_t L = offsets[n_series];
        DeviceGuard dg(s.device);
        const StagedCbf in = stage_cbf(s, offsets, cols, n_series);
        xgroup_launch(g, reinterpret_cast<const uint64_t*>(s.d_in),
                      reinterpret_cast<const uint16_t*>(s.d_in + in.cols_at), n_series, L, eps, sigma,
                      fitness_out != nullptr, seq, s.stream, s.h_in_map, in.bytes);
        xgroup_wait(g, seq, n_series, counts_out, fitness_out, s.stream);
    });
}

int ebic_xgroup_destroy(ebic_xgroup* g) {
    return guarded([&] {
        if (!g) return;
        DeviceGuard dg(g->ctx->shards[0].device);
        cudaStreamSynchronize(g->ctx->shards[0].stream);
        cudaHostUnregister(g->shm);
        munmap(g->shm, g->shm_bytes);
        if (g->owner) {
            cudaFree(g->d_base);
            shm_unlink(g->shm_name.c_str());
        } else {
            cudaIpcCloseMemHandle(g->d_base);
        }
        delete g;
    });
}

}  // extern "C"
