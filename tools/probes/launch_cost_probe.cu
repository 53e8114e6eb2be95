// Host cost of one launch of a kernel with a ~400-byte parameter block
// (CountParams-sized): plain launch, graph launch after a parameter update,
// graph launch with unchanged parameters.  (GPU box; diagnostics.)
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>
struct Big { unsigned long long w[50]; };
__global__ void k(const __grid_constant__ Big p, unsigned long long* out) {
    if (threadIdx.x == 0 && blockIdx.x == 0 && p.w[0] == 12345678ull) out[0] = p.w[1];
}
int main() {
    unsigned long long* d; cudaMalloc(&d, 8);
    cudaStream_t st; cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    Big p{}; void* args[2] = {&p, &d};
    cudaKernelNodeParams kp{}; kp.func = (void*)k; kp.gridDim = dim3(148); kp.blockDim = dim3(896);
    kp.kernelParams = args;
    cudaGraph_t g; cudaGraphNode_t n; cudaGraphExec_t ge;
    cudaGraphCreate(&g, 0); cudaGraphAddKernelNode(&n, g, nullptr, 0, &kp); cudaGraphInstantiate(&ge, g, 0);
    for (int mode = 0; mode < 3; ++mode) {
        double tot = 0; const int reps = 2000;
        for (int r = 0; r < reps + 100; ++r) {
            p.w[3] = r;
            auto t0 = std::chrono::steady_clock::now();
            if (mode == 0) cudaLaunchKernel((void*)k, dim3(148), dim3(896), args, 0, st);
            else if (mode == 1) { cudaGraphExecKernelNodeSetParams(ge, n, &kp); cudaGraphLaunch(ge, st); }
            else cudaGraphLaunch(ge, st);
            auto t1 = std::chrono::steady_clock::now();
            cudaStreamSynchronize(st);
            if (r >= 100) tot += std::chrono::duration<double, std::micro>(t1 - t0).count();
        }
        printf("%s: %.2f us host per launch\n", mode == 0 ? "plain launch" : mode == 1 ? "graph set + launch" : "graph launch (unchanged)", tot / reps);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
