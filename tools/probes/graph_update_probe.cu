// Can one instantiated one-node graph be re-pointed at a launch with another
// grid / dynamic shared-memory size via cudaGraphExecKernelNodeSetParams?
// Times set+launch for changing shapes against a plain launch.
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* out, int v) {
    extern __shared__ int sm[];
    if (threadIdx.x == 0) sm[0] = v;
    __syncthreads();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = sm[0];
}
int main() {
    int* d; cudaMalloc(&d, 4);
    cudaStream_t st; cudaStreamCreate(&st);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    int v = 1; void* args[2] = {&d, &v};
    cudaKernelNodeParams kp{}; kp.func = (void*)k; kp.gridDim = dim3(148); kp.blockDim = dim3(800);
    kp.sharedMemBytes = 100 * 1024; kp.kernelParams = args;
    cudaGraph_t g; cudaGraphNode_t n; cudaGraphExec_t ex;
    cudaGraphCreate(&g, 0); cudaGraphAddKernelNode(&n, g, nullptr, 0, &kp); cudaGraphInstantiate(&ex, g, 0);
    int ok = 0, fails = 0;
    for (int i = 0; i < 2000; ++i) {
        kp.sharedMemBytes = (100 + (i * 37) % 100) * 1024; kp.gridDim = dim3(100 + i % 48); v = i;
        cudaError_t e = cudaGraphExecKernelNodeSetParams(ex, n, &kp);
        if (e != cudaSuccess) { ++fails; if (fails < 3) printf("set failed: %s\n", cudaGetErrorString(e)); cudaGetLastError(); continue; }
        cudaGraphLaunch(ex, st);
        int h = 0; cudaMemcpyAsync(&h, d, 4, cudaMemcpyDeviceToHost, st); cudaStreamSynchronize(st);
        ok += h == i;
    }
    printf("changing shapes: %d correct, %d set failures\n", ok, fails);
    for (int mode = 0; mode < 2; ++mode) {
        cudaStreamSynchronize(st);
        auto t0 = std::chrono::steady_clock::now();
        for (int i = 0; i < 2000; ++i) {
            kp.sharedMemBytes = (100 + (i * 37) % 100) * 1024; kp.gridDim = dim3(148);
            if (mode == 0) { cudaGraphExecKernelNodeSetParams(ex, n, &kp); cudaGraphLaunch(ex, st); }
            else cudaLaunchKernel((void*)k, kp.gridDim, kp.blockDim, args, kp.sharedMemBytes, st);
        }
        double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count() / 2000;
        cudaStreamSynchronize(st);
        printf("%s: host %.2f us per call\n", mode == 0 ? "graph set(smem changes)+launch" : "plain launch", us);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
