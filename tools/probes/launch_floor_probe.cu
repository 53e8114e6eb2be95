// Event-timed duration of an empty 148-CTA kernel as a function of its
// dynamic shared memory and block size (what sets the per-launch floor?).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* out) {
    extern __shared__ int sm[];
    if (threadIdx.x == 0) sm[0] = blockIdx.x;
    __syncthreads();
    if (threadIdx.x == 0 && sm[0] < 0) out[0] = 1;
}
__global__ void spin(long long c) { long long t0 = clock64(); while (clock64() - t0 < c) {} }
int main() {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    int* d; cudaMalloc(&d, 4);
    cudaStream_t st; cudaStreamCreate(&st);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const int smems[] = {1, 48, 100, 160, 200, 223};
    const int threads[] = {128, 256, 800, 1024};
    for (int carve = 0; carve < 2; ++carve) {
        cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, carve ? 100 : -1);
        for (int s : smems) for (int t : threads) {
            float tot = 0; const int reps = 300;
            for (int r = 0; r < reps + 5; ++r) {
                spin<<<1, 32, 0, st>>>(100000);
                cudaEventRecord(a, st);
                k<<<148, t, size_t(s) * 1024, st>>>(d);
                cudaEventRecord(b, st);
                cudaEventSynchronize(b);
                float ms; cudaEventElapsedTime(&ms, a, b);
                if (r >= 5) tot += ms;
            }
            printf("carveout %-4s smem %3d KB threads %4d: %.2f us\n", carve ? "max" : "def", s, t, tot / reps * 1e3);
        }
    }
    // two events back to back (the event floor itself)
    float tot = 0;
    for (int r = 0; r < 300; ++r) {
        spin<<<1, 32, 0, st>>>(100000);
        cudaEventRecord(a, st); cudaEventRecord(b, st); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); tot += ms;
    }
    printf("event pair, nothing between: %.2f us\n", tot / 300 * 1e3);
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
