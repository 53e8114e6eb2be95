// Host round trip for getting a ~10 KB CBF to all 148 CTAs (GPU box).
// Each mode: host writes the payload, launches, spins on a mapped flag that
// the last CTA raises after every CTA has summed the payload; mean over runs.
//  mode 0  CTA 0 pulls the payload from mapped host memory into global, then
//          publishes a flag the other CTAs poll (the product's staging)
//  mode 1  payload inside the kernel parameters (cudaLaunchKernel, 32 KB max)
//  mode 2  payload inside the kernel parameters of a one-node graph
//          (cudaGraphExecKernelNodeSetParams + cudaGraphLaunch)
//  mode 3  cudaMemcpyAsync to device, then the kernel (graph launch)
// usage: param_probe [bytes=9906] [runs=2000]
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>

constexpr int kMaxWords = 7900;  // 31.6 KB of uint32 payload
struct BigParams {
    unsigned n_words;
    unsigned seq;
    unsigned* done;                 // device ticket
    volatile unsigned* host_flag;   // mapped
    unsigned* out;                  // device sums (one per CTA)
    const uint4* host_src;          // mode 0
    uint4* dev_buf;                 // mode 0/3
    unsigned* ready;                // mode 0 flag
    unsigned words[kMaxWords];
};
struct SmallParams {
    unsigned n_words, seq;
    unsigned* done;
    volatile unsigned* host_flag;
    unsigned* out;
    const uint4* host_src;
    uint4* dev_buf;
    unsigned* ready;
};

__device__ void finish(unsigned* done, volatile unsigned* host_flag, unsigned seq, unsigned* out, unsigned sum) {
    __shared__ unsigned s;
    __syncthreads();
    if (threadIdx.x == 0) {
        out[blockIdx.x] = sum;
        __threadfence();
        s = atomicAdd(done, 1u);
    }
    __syncthreads();
    if (threadIdx.x == 0 && s == gridDim.x - 1) {
        *done = 0;
        __threadfence_system();
        *host_flag = seq;
    }
}

__global__ void k_params(const __grid_constant__ BigParams p) {
    unsigned sum = 0;
    for (unsigned i = threadIdx.x; i < p.n_words; i += blockDim.x) sum += p.words[i];
    for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(~0u, sum, o);
    finish(p.done, p.host_flag, p.seq, p.out, sum);
}

__global__ void k_pull(const __grid_constant__ SmallParams p) {
    const unsigned n16 = (p.n_words + 3) / 4;
    if (blockIdx.x == 0) {
        for (unsigned i = threadIdx.x; i < n16; i += blockDim.x) p.dev_buf[i] = p.host_src[i];
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            atomicExch(p.ready, p.seq);
        }
    } else if (threadIdx.x == 0) {
        while (atomicAdd(p.ready, 0u) != p.seq) __nanosleep(32);
    }
    __syncthreads();
    unsigned sum = 0;
    const unsigned* w = reinterpret_cast<const unsigned*>(p.dev_buf);
    for (unsigned i = threadIdx.x; i < p.n_words; i += blockDim.x) sum += __ldcg(w + i);
    for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(~0u, sum, o);
    finish(p.done, p.host_flag, p.seq, p.out, sum);
}

__global__ void k_dev(const __grid_constant__ SmallParams p) {
    unsigned sum = 0;
    const unsigned* w = reinterpret_cast<const unsigned*>(p.dev_buf);
    for (unsigned i = threadIdx.x; i < p.n_words; i += blockDim.x) sum += __ldcg(w + i);
    for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(~0u, sum, o);
    finish(p.done, p.host_flag, p.seq, p.out, sum);
}

int main(int argc, char** argv) {
    const size_t bytes = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 9906;
    const int runs = argc > 2 ? std::atoi(argv[2]) : 2000;
    const unsigned n_words = unsigned((bytes + 3) / 4);
    if (n_words > kMaxWords) return 1;
    unsigned char* hmap;
    cudaHostAlloc(&hmap, 1 << 16, cudaHostAllocMapped);
    std::memset(hmap, 0, 1 << 16);
    volatile unsigned* flag = reinterpret_cast<volatile unsigned*>(hmap);
    uint4* hsrc = reinterpret_cast<uint4*>(hmap + 4096);
    unsigned *done, *out, *ready;
    uint4* dbuf;
    cudaMalloc(&done, 4);
    cudaMemset(done, 0, 4);
    cudaMalloc(&ready, 4);
    cudaMemset(ready, 0, 4);
    cudaMalloc(&out, 4096);
    cudaMalloc(&dbuf, 1 << 16);
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    static BigParams bp;
    SmallParams sp{n_words, 0, done, flag, out, hsrc, dbuf, ready};
    bp.n_words = n_words, bp.done = done, bp.host_flag = flag, bp.out = out;
    bp.host_src = hsrc, bp.dev_buf = dbuf, bp.ready = ready;
    cudaGraph_t g[3];
    cudaGraphExec_t ge[3];
    cudaGraphNode_t node[3];
    for (int m = 0; m < 4; ++m) {
        double total = 0;
        unsigned seq = 0;
        for (int r = 0; r < runs + 50; ++r) {
            ++seq;
            const auto t0 = std::chrono::steady_clock::now();
            for (unsigned i = 0; i < n_words; ++i) {  // the payload the host produces each call
                reinterpret_cast<unsigned*>(hsrc)[i] = i + seq;
                if (m == 1 || m == 2) bp.words[i] = i + seq;
            }
            sp.seq = bp.seq = seq;
            if (m == 0 || m == 3) {
                if (m == 3) cudaMemcpyAsync(dbuf, hsrc, n_words * 4, cudaMemcpyHostToDevice, st);
                cudaKernelNodeParams kp{};
                kp.func = m == 0 ? (void*)k_pull : (void*)k_dev;
                kp.gridDim = dim3(148);
                kp.blockDim = dim3(640);
                void* args[1] = {&sp};
                kp.kernelParams = args;
                const int gi = m == 0 ? 0 : 2;
                if (r == 0) {
                    cudaGraphCreate(&g[gi], 0);
                    cudaGraphAddKernelNode(&node[gi], g[gi], nullptr, 0, &kp);
                    cudaGraphInstantiate(&ge[gi], g[gi], 0);
                } else {
                    cudaGraphExecKernelNodeSetParams(ge[gi], node[gi], &kp);
                }
                cudaGraphLaunch(ge[gi], st);
            } else if (m == 1) {
                void* args[1] = {&bp};
                cudaLaunchKernel((void*)k_params, dim3(148), dim3(640), args, 0, st);
            } else {
                cudaKernelNodeParams kp{};
                kp.func = (void*)k_params;
                kp.gridDim = dim3(148);
                kp.blockDim = dim3(640);
                void* args[1] = {&bp};
                kp.kernelParams = args;
                if (r == 0) {
                    cudaGraphCreate(&g[1], 0);
                    cudaGraphAddKernelNode(&node[1], g[1], nullptr, 0, &kp);
                    cudaGraphInstantiate(&ge[1], g[1], 0);
                } else {
                    cudaGraphExecKernelNodeSetParams(ge[1], node[1], &kp);
                }
                cudaGraphLaunch(ge[1], st);
            }
            while (*flag != seq) {
            }
            const auto t1 = std::chrono::steady_clock::now();
            if (r >= 50) total += std::chrono::duration<double, std::micro>(t1 - t0).count();
        }
        cudaStreamSynchronize(st);
        const cudaError_t e = cudaGetLastError();
        std::printf("mode %d bytes %zu: %.2f us per round trip (%s)\n", m, bytes, total / runs, cudaGetErrorString(e));
    }
    return 0;
}
