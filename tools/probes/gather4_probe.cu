// Validates TMA tile::gather4 on sm_100a for the count kernel's compact column
// staging: a column-major uint16 matrix [cols][ld], tensor map box {64, 1};
// one gather4 = 4 arbitrary columns x 64 rows -> 512 contiguous smem bytes.
// Also times N gather4 per tile vs one 2D box load of all columns.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__global__ void probe(const __grid_constant__ CUtensorMap tm, const int* cols, int n_cols_g, int row0, uint16_t* out) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t bytes = n_cols_g * 128;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(bytes) : "memory");
        for (int g = 0; g < n_cols_g / 4; ++g) {
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                :: "r"(smem_u32(smem + g * 512)), "l"(reinterpret_cast<uint64_t>(&tm)), "r"(row0),
                   "r"(cols[4 * g]), "r"(cols[4 * g + 1]), "r"(cols[4 * g + 2]), "r"(cols[4 * g + 3]),
                   "r"(smem_u32(&bar))
                : "memory");
        }
    }
    uint32_t done = 0;
    while (!done) {
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(smem_u32(&bar)), "r"(0) : "memory");
    }
    for (int i = threadIdx.x; i < n_cols_g * 64; i += blockDim.x) out[i] = reinterpret_cast<uint16_t*>(smem)[i];
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    const int ld = 256, ncols = 1000;
    std::vector<uint16_t> h(size_t(ld) * ncols);
    for (int c = 0; c < ncols; ++c)
        for (int r = 0; r < ld; ++r) h[size_t(c) * ld + r] = uint16_t((c * 7 + r * 131) & 0xffff);
    uint16_t* d;
    cudaMalloc(&d, h.size() * 2);
    cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
    EncodeFn enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q);
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)ld, (cuuint64_t)ncols};
    cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
    cuuint32_t box[2] = {64, 1};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode rc %d\n", (int)r);
    const int ng = 12;
    std::vector<int> cols = {5, 999, 0, 17, 17, 300, 301, 2, 640, 641, 642, 9};
    int* dc;
    cudaMalloc(&dc, ng * 4);
    cudaMemcpy(dc, cols.data(), ng * 4, cudaMemcpyHostToDevice);
    uint16_t* dout;
    cudaMalloc(&dout, ng * 64 * 2);
    const int row0 = 128;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    probe<<<1, 128, 64 * 1024>>>(tm, dc, ng, row0, dout);
    cudaError_t e = cudaDeviceSynchronize();
    printf("kernel: %s\n", cudaGetErrorString(e));
    std::vector<uint16_t> o(ng * 64);
    cudaMemcpy(o.data(), dout, o.size() * 2, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int g = 0; g < ng; ++g)
        for (int rr = 0; rr < 64; ++rr)
            if (o[g * 64 + rr] != h[size_t(cols[g]) * ld + row0 + rr]) ++bad;
    printf("gather4 layout [col][64 rows]: %s (%d mismatches)\n", bad ? "MISMATCH" : "ok", bad);
    if (bad) {
        for (int i = 0; i < 8; ++i) printf("o[%d]=%u expect col%d row%d=%u\n", i, o[i], cols[0], row0 + i, h[size_t(cols[0]) * ld + row0 + i]);
    }
    return bad ? 1 : 0;
}
