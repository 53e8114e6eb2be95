// Streaming rate of the ways to stage a row tile of the 16-bit rank matrix
// into shared memory (no walk; one consumer warp just releases stages).
//
//   mode 0  TMA 2D boxes, every column (production: 32-row tiles, 64-B slices)
//   mode 1  TMA 2D boxes, every column, 64-row tiles (128-B slices)
//   mode 2  cp.async.bulk per referenced column (128-B slice of a 64-row tile),
//           issued by the 32 lanes of one producer warp
//   mode 3  the same issued by 4 producer warps
//   mode 4  cp.async (LDGSTS 16 B) per referenced column, 4 producer warps
//   mode 5  tile-major layout ([tile][col][64 rows]): one cp.async.bulk per tile
//   mode 6  tile-major layout: LDGSTS per referenced column, 4 producer warps
//   mode 7  as 4 with 8 producer warps
//   mode 8  tile-major: one cp.async.bulk per run of consecutive referenced
//           columns (runs x 128 B), issued by the lanes of one warp
//   mode 9  as 8, issued by 4 warps
//
// usage: gather_probe ROWS COLS U [iters]   (U = referenced columns, random)
// Prints useful GB/s = rows * U * 2 B / time (full-tile modes move all COLS).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { std::printf("%s: %s\n", #x, cudaGetErrorString(e)); std::exit(1); } } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mb_expect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t ph) {
    asm volatile("{\n.reg .pred P;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@P bra D;\nbra W;\nD:\n}\n" ::"r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* m, uint64_t* b, int c0, int c1) {
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 ::"r"(su32(dst)), "l"((uint64_t)m), "r"(c0), "r"(c1), "r"(su32(b)) : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t n, uint64_t* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(su32(dst)), "l"(src), "r"(n), "r"(su32(b)) : "memory");
}

struct P {
    const uint16_t* mat;  // column-major [cols][ld]
    uint32_t ld, cols, n_tiles, U, stages, stage_bytes, mode, rpt;
    const uint16_t* ucols;
    const uint32_t* runs;  // (first column << 16) | length
    uint32_t n_runs;
};

__global__ void __launch_bounds__(288, 1) probe(const __grid_constant__ CUtensorMap tm, const P p) {
    extern __shared__ __align__(128) unsigned char sm[];
    unsigned char* base = sm + ((128u - (su32(sm) & 127u)) & 127u);
    uint64_t* full = reinterpret_cast<uint64_t*>(base + p.stages * p.stage_bytes);
    uint64_t* empty = full + 8;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool ldgsts = p.mode == 4 || p.mode == 6 || p.mode == 7;
    const int nprod = p.mode == 7 ? 8 : (p.mode == 3 || p.mode == 4 || p.mode == 6 || p.mode == 9) ? 4 : 1;
    const uint32_t nthr = 32 * nprod;
    const bool tile_major = p.mode == 5 || p.mode == 6;
    if (threadIdx.x == 0) {
        for (uint32_t s = 0; s < p.stages; ++s) {
            mb_init(&full[s], ldgsts ? nthr : 1);
            mb_init(&empty[s], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp < nprod) {
        uint32_t st = 0, ph = 0;
        for (uint32_t t = blockIdx.x; t < p.n_tiles; t += gridDim.x) {
            mb_wait(&empty[st], ph ^ 1u);
            unsigned char* dst = base + st * p.stage_bytes;
            if (p.mode <= 1) {
                if (threadIdx.x == 0) {
                    const uint32_t nb = (p.cols + 249) / 250;
                    mb_expect(&full[st], p.stage_bytes);
                    for (uint32_t b = 0; b < nb; ++b)
                        tma2d(dst + b * 250 * (p.rpt * 2), &tm, &full[st], (int)(t * p.rpt), (int)(b * 250));
                }
            } else if (p.mode == 5) {
                if (threadIdx.x == 0) {
                    mb_expect(&full[st], p.cols * 128);
                    bulk(dst, p.mat + (size_t)t * p.cols * 64, p.cols * 128, &full[st]);
                }
            } else if (p.mode == 8 || p.mode == 9) {
                if (threadIdx.x == 0) mb_expect(&full[st], p.U * 128);
                if (nprod > 1) asm volatile("bar.sync 1, 128;" ::: "memory");
                else __syncwarp();
                // destination slot of run r = prefix of the run lengths (precomputed: low 16 bits of slot table)
                for (uint32_t r = threadIdx.x; r < p.n_runs; r += 32 * nprod) {
                    const uint32_t x = p.runs[r], c0 = x >> 16, len = x & 0xffffu;
                    const uint32_t slot = p.runs[p.n_runs + r];
                    bulk(dst + slot * 128, p.mat + ((size_t)t * p.cols + c0) * 64, len * 128, &full[st]);
                }
            } else if (p.mode == 2 || p.mode == 3) {
                if (threadIdx.x == 0) mb_expect(&full[st], p.U * 128);
                if (nprod > 1) asm volatile("bar.sync 1, 128;" ::: "memory");
                else __syncwarp();
                for (uint32_t i = threadIdx.x; i < p.U; i += 32 * nprod)
                    bulk(dst + i * 128, p.mat + (size_t)p.ucols[i] * p.ld + (size_t)t * 64, 128, &full[st]);
            } else {
                // 8 lanes x 16 B per column
                for (uint32_t i = threadIdx.x; i < p.U * 8; i += nthr) {
                    const uint32_t c = i >> 3, q = i & 7;
                    const uint16_t* src = tile_major ? p.mat + ((size_t)t * p.cols + p.ucols[c]) * 64 + q * 8
                                                     : p.mat + (size_t)p.ucols[c] * p.ld + (size_t)t * 64 + q * 8;
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(dst + c * 128 + q * 16)), "l"(src) : "memory");
                }
                asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su32(&full[st])) : "memory");
            }
            if (++st == p.stages) st = 0, ph ^= 1u;
        }
    } else if (warp == nprod) {
        uint32_t st = 0, ph = 0;
        for (uint32_t t = blockIdx.x; t < p.n_tiles; t += gridDim.x) {
            mb_wait(&full[st], ph);
            __syncwarp();
            if (lane == 0) mb_arrive(&empty[st]);
            if (++st == p.stages) st = 0, ph ^= 1u;
        }
    }
}

int main(int argc, char** argv) {
    const uint32_t rows = argc > 1 ? atoi(argv[1]) : 200000;
    const uint32_t cols = argc > 2 ? atoi(argv[2]) : 1000;
    const uint32_t U = argc > 3 ? atoi(argv[3]) : 620;
    const int iters = argc > 4 ? atoi(argv[4]) : 20;
    const uint32_t ld = (rows + 63) / 64 * 64;
    uint16_t* mat;
    CK(cudaMalloc(&mat, (size_t)ld * cols * 2));
    CK(cudaMemset(mat, 0x11, (size_t)ld * cols * 2));
    std::vector<uint16_t> uc(cols);
    for (uint32_t i = 0; i < cols; ++i) uc[i] = i;
    std::mt19937 rng(7);
    std::shuffle(uc.begin(), uc.end(), rng);
    uc.resize(U);
    std::sort(uc.begin(), uc.end());
    uint16_t* d_uc;
    CK(cudaMalloc(&d_uc, U * 2));
    CK(cudaMemcpy(d_uc, uc.data(), U * 2, cudaMemcpyHostToDevice));
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    float* flush;
    CK(cudaMalloc(&flush, 512 << 20));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    int dev_smem = 0;
    CK(cudaDeviceGetAttribute(&dev_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0));
    std::vector<uint32_t> runs, slots;
    for (uint32_t i = 0; i < U;) {
        uint32_t j = i + 1;
        while (j < U && uc[j] == uc[j - 1] + 1) ++j;
        runs.push_back((uint32_t(uc[i]) << 16) | (j - i));
        slots.push_back(i);
        i = j;
    }
    const uint32_t n_runs = (uint32_t)runs.size();
    runs.insert(runs.end(), slots.begin(), slots.end());
    uint32_t* d_runs;
    CK(cudaMalloc(&d_runs, runs.size() * 4));
    CK(cudaMemcpy(d_runs, runs.data(), runs.size() * 4, cudaMemcpyHostToDevice));
    std::printf("U %u runs %u\n", U, n_runs);
    for (uint32_t mode = 0; mode <= 9; ++mode) {
        P p{};
        p.mat = mat; p.ld = ld; p.cols = cols; p.U = U; p.mode = mode; p.ucols = d_uc;
        p.runs = d_runs; p.n_runs = n_runs;
        p.rpt = mode == 0 ? 32 : 64;
        p.n_tiles = (rows + p.rpt - 1) / p.rpt;
        p.stage_bytes = (mode <= 1 || mode == 5) ? cols * p.rpt * 2 : U * 128;
        p.stages = std::min<uint32_t>(4, (dev_smem - 1024) / p.stage_bytes);
        if (p.stages < 1) { std::printf("mode %u: stage does not fit\n", mode); continue; }
        CUtensorMap tm{};
        cuuint64_t dims[2] = {ld, cols};
        cuuint64_t str[1] = {(cuuint64_t)ld * 2};
        cuuint32_t box[2] = {p.rpt, 250};
        cuuint32_t es[2] = {1, 1};
        if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, mat, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
            std::printf("encode failed\n");
            return 1;
        }
        const size_t smem = p.stages * p.stage_bytes + 256;
        CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        float best = 1e30f, sum = 0;
        for (int it = 0; it < iters; ++it) {
            CK(cudaMemsetAsync(flush, it, 512 << 20));
            CK(cudaEventRecord(e0));
            probe<<<148, 32 * (mode == 7 ? 9 : 5), smem>>>(tm, p);
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            CK(cudaGetLastError());
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            best = std::min(best, ms);
            sum += ms;
        }
        const bool full_tile = mode <= 1 || mode == 5;
        const double useful = (double)rows * (full_tile ? cols : U) * 2;
        const double moved = (double)rows * (full_tile ? cols : U) * 2;
        std::printf("mode %u stages %u stage_kb %.1f: best %.1f us mean %.1f us  %.0f GB/s moved, %.0f GB/s of the U columns\n",
                    mode, p.stages, p.stage_bytes / 1024.0, best * 1e3, sum / iters * 1e3, moved / (best * 1e-3) / 1e9,
                    (double)rows * U * 2 / (best * 1e-3) / 1e9);
        (void)useful;
    }
    return 0;
}
