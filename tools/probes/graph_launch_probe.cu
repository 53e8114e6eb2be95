// Host cost of a kernel launch vs a one-node CUDA graph whose kernel
// parameters are updated per launch (cudaGraphExecKernelNodeSetParams).
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
struct Blob { unsigned char b[512]; };
__global__ void k(const __grid_constant__ Blob p, int* out) {
    if (threadIdx.x == 0 && blockIdx.x == 0 && p.b[0] == 123) *out = 1;
}
int main() {
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    int* d;
    cudaMalloc(&d, 4);
    const int smem = 200 * 1024;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    Blob p{};
    // plain launches
    double t_launch = 0;
    for (int i = 0; i < 2050; ++i) {
        p.b[1] = (unsigned char)i;
        auto a = std::chrono::steady_clock::now();
        k<<<148, 800, smem, st>>>(p, d);
        auto b = std::chrono::steady_clock::now();
        if (i >= 50) t_launch += std::chrono::duration<double, std::micro>(b - a).count();
        cudaStreamSynchronize(st);
    }
    // graph with per-launch parameter update
    cudaGraph_t g;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
    k<<<148, 800, smem, st>>>(p, d);
    cudaStreamEndCapture(st, &g);
    cudaGraphExec_t ge;
    cudaGraphInstantiate(&ge, g, 0);
    size_t n = 1;
    cudaGraphNode_t node;
    cudaGraphGetNodes(g, &node, &n);
    cudaKernelNodeParams kp;
    cudaGraphKernelNodeGetParams(node, &kp);
    void* args[2] = {&p, &d};
    kp.kernelParams = args;
    double t_graph = 0, t_set = 0;
    for (int i = 0; i < 2050; ++i) {
        p.b[1] = (unsigned char)i;
        auto a = std::chrono::steady_clock::now();
        cudaGraphExecKernelNodeSetParams(ge, node, &kp);
        auto m = std::chrono::steady_clock::now();
        cudaGraphLaunch(ge, st);
        auto b = std::chrono::steady_clock::now();
        if (i >= 50) {
            t_graph += std::chrono::duration<double, std::micro>(b - a).count();
            t_set += std::chrono::duration<double, std::micro>(m - a).count();
        }
        cudaStreamSynchronize(st);
    }
    // graph without update
    double t_plain_graph = 0;
    for (int i = 0; i < 2050; ++i) {
        auto a = std::chrono::steady_clock::now();
        cudaGraphLaunch(ge, st);
        auto b = std::chrono::steady_clock::now();
        if (i >= 50) t_plain_graph += std::chrono::duration<double, std::micro>(b - a).count();
        cudaStreamSynchronize(st);
    }
    printf("launch %.2f us | graph set+launch %.2f us (set %.2f) | graph launch only %.2f us | %s\n",
           t_launch / 2000, t_graph / 2000, t_set / 2000, t_plain_graph / 2000, cudaGetErrorString(cudaGetLastError()));
}
