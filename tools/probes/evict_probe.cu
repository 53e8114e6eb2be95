// Eviction kernels for tools/probes/evict_probe.py: a read-reduction over a
// buffer, launched with (a) no dynamic shared memory or (b) the count kernel's
// ~223 KB, and (c) an empty kernel with the default carve-out.
#include <cuda_runtime.h>
#include <cstdint>
__global__ void rd(const float4* __restrict__ p, size_t n, float* sink) {
    extern __shared__ float sm[];
    float acc = 0.f;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
        const float4 v = p[i];
        acc += v.x + v.y + v.z + v.w;
    }
    if (acc == 12345.f) *sink = acc + sm[0];
}
__global__ void empty_k(float* sink) { if (threadIdx.x == 1234) *sink = 1.f; }
extern "C" int evict(const void* buf, size_t bytes, float* sink, int big_smem, void* stream) {
    size_t smem = big_smem ? 223 * 1024 : 0;
    if (big_smem) cudaFuncSetAttribute(rd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    rd<<<148, 1024, smem, (cudaStream_t)stream>>>((const float4*)buf, bytes / 16, sink);
    return (int)cudaGetLastError();
}
extern "C" int empty(float* sink, void* stream) {
    empty_k<<<148, 256, 0, (cudaStream_t)stream>>>(sink);
    return (int)cudaGetLastError();
}
