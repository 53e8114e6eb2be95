// Host-side cost of one cudaLaunchKernel vs kernel parameter size (and the
// 148 x 800-thread, 200 KB shared-memory shape of the count kernel).
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
template <int N> struct Blob { unsigned char b[N]; };
template <int N> __global__ void k(const __grid_constant__ Blob<N> p, int* out) {
    if (threadIdx.x == 0 && blockIdx.x == 0 && p.b[0] == 123) *out = 1;
}
template <int N> double time_launch(int grid, int block, size_t smem, cudaStream_t st, int* d) {
    Blob<N> p{};
    cudaFuncSetAttribute(k<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int i = 0; i < 50; ++i) k<N><<<grid, block, smem, st>>>(p, d);
    cudaStreamSynchronize(st);
    double tot = 0;
    for (int i = 0; i < 2000; ++i) {
        auto a = std::chrono::steady_clock::now();
        k<N><<<grid, block, smem, st>>>(p, d);
        auto b = std::chrono::steady_clock::now();
        tot += std::chrono::duration<double, std::micro>(b - a).count();
        cudaStreamSynchronize(st);
    }
    return tot / 2000;
}
int main() {
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    int* d;
    cudaMalloc(&d, 4);
    printf("params 16B   : %.2f us\n", time_launch<16>(148, 800, 200 * 1024, st, d));
    printf("params 128B  : %.2f us\n", time_launch<128>(148, 800, 200 * 1024, st, d));
    printf("params 512B  : %.2f us\n", time_launch<512>(148, 800, 200 * 1024, st, d));
    printf("params 2048B : %.2f us\n", time_launch<2048>(148, 800, 200 * 1024, st, d));
    printf("params 512B small grid: %.2f us\n", time_launch<512>(1, 32, 0, st, d));
    return 0;
}
