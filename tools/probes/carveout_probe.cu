// Does the L2-eviction kernel between timed steps cost the next (223 KB
// shared-memory) launch an L1/shared carve-out switch?  Times an empty
// persistent-shaped kernel with CUDA events after (a) nothing, (b) a read
// kernel with the default carve-out, (c) the same read kernel with the
// carve-out preference set to maximum shared memory.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void big_smem(int* out) {
    extern __shared__ int sm[];
    if (threadIdx.x == 0) sm[0] = blockIdx.x;
    __syncthreads();
    if (threadIdx.x == 0 && sm[0] < 0) out[0] = 1;
}
__global__ void evict_default(const float4* p, size_t n, float* sink) {
    float a = 0;
    for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
        float4 v = __ldcs(p + i);
        a += v.x + v.y + v.z + v.w;
    }
    if (a == 1234.5f) sink[0] = a;
}
__global__ void evict_maxsmem(const float4* p, size_t n, float* sink) {
    float a = 0;
    for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
        float4 v = __ldcs(p + i);
        a += v.x + v.y + v.z + v.w;
    }
    if (a == 1234.5f) sink[0] = a;
}
__global__ void spin(long long ns) {
    long long t0 = clock64();
    while (clock64() - t0 < ns) {}
}

int main() {
    const size_t smem = 223 * 1024;
    cudaFuncSetAttribute(big_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(evict_maxsmem, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    int* d; cudaMalloc(&d, 4);
    float* sink; cudaMalloc(&sink, 4);
    const size_t n = (512ull << 20) / 16;
    float4* buf; cudaMalloc(&buf, n * 16); cudaMemset(buf, 0, n * 16);
    cudaStream_t st; cudaStreamCreate(&st);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const char* names[3] = {"no kernel before", "eviction, default carve-out", "eviction, max-shared carve-out"};
    for (int mode = 0; mode < 3; ++mode) {
        float tot = 0; int reps = 200;
        for (int r = 0; r < reps + 5; ++r) {
            if (mode == 1) evict_default<<<148 * 4, 512, 0, st>>>(buf, n, sink);
            if (mode == 2) evict_maxsmem<<<148 * 4, 512, 0, st>>>(buf, n, sink);
            spin<<<1, 32, 0, st>>>(100000);
            cudaEventRecord(a, st);
            big_smem<<<148, 800, smem, st>>>(d);
            cudaEventRecord(b, st);
            cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            if (r >= 5) tot += ms;
        }
        printf("%-34s empty 148x800 kernel, 223 KB smem: %.2f us\n", names[mode], tot / reps * 1e3);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
