// Event-timed floor of an empty 148-CTA, 896-thread, 231 KB kernel (the
// count kernel's launch shape, with a 512-byte parameter block) as a function
// of what ran on the stream just before the first event:
//   idle    : nothing queued (host waits 200 us after a sync)
//   spin0   : a 1-CTA spin kernel with no shared memory (bench.py's
//             torch.cuda._sleep)
//   spinbig : the same spin kernel launched with 231 KB of dynamic shared
//             memory (the count kernel's carve-out)
//   empty   : the empty kernel itself, back to back
// plus the bare event pair.  Does a shared-memory carve-out change between
// the preceding kernel and the count kernel sit inside the timed events?
#include <chrono>
#include <cstdio>
#include <thread>
#include <cuda_runtime.h>
struct Big { unsigned long long w[64]; };
__global__ void __launch_bounds__(896, 1) k(const __grid_constant__ Big p, int* out) {
    extern __shared__ int sm[];
    if (threadIdx.x == 0) sm[0] = blockIdx.x + (int)p.w[blockIdx.x & 63];
    __syncthreads();
    if (threadIdx.x == 0 && sm[0] < -5) out[0] = 1;
}
__global__ void spin(long long c) { long long t0 = clock64(); while (clock64() - t0 < c) {} }
int main() {
    const int smem = 231420;  // ncu: 231.42 KB (decimal) per block
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(spin, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int* d; cudaMalloc(&d, 4);
    cudaStream_t st; cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    Big p{};
    const char* names[] = {"idle", "spin0", "spinbig", "empty", "eventpair"};
    for (int mode = 0; mode < 5; ++mode) {
        float tot = 0, mn = 1e9; const int reps = 400;
        for (int r = 0; r < reps + 10; ++r) {
            if (mode == 0 || mode == 4) {
                cudaStreamSynchronize(st);
                std::this_thread::sleep_for(std::chrono::microseconds(200));
            } else if (mode == 1) {
                spin<<<1, 32, 0, st>>>(100000);
            } else if (mode == 2) {
                spin<<<1, 32, smem, st>>>(100000);
            } else {
                k<<<148, 896, smem, st>>>(p, d);
            }
            cudaEventRecord(a, st);
            if (mode != 4) k<<<148, 896, smem, st>>>(p, d);
            cudaEventRecord(b, st);
            cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            if (r >= 10) { tot += ms; mn = ms < mn ? ms : mn; }
        }
        printf("%-9s mean %.2f us  min %.2f us\n", names[mode], tot / reps * 1e3, mn * 1e3);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
