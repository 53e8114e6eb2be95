// e2e_driver.cu -- end-to-end timing of the public C ABI from a C++ caller.
//
// This is the view of the reference's own GA loop, which reaches the library
// through include/ebic/fitness.hpp -> ebic_evaluate_population with host
// std::vector buffers (inc/evolution.hpp:504-505).  Each timed step is one
// ebic_evaluate_population call on a host CBF batch: pinned staging + H2D of
// the CBF, the count kernel, counts/fitness written back to host memory, and
// the wait for them.  Between steps (outside the timed region) L2 is evicted
// by reading 512 MB on another stream.
//
// usage: ebic_e2e_driver <batches.bin> rows cols n_blocks brows bcols pattern
//                        overlap noise seed eps sigma steps warmup
// batches.bin: repeated { u64 P; u64 offsets[P+1]; u16 cols[offsets[P]];
//                         u64 expected_counts[P]; f64 expected_fitness[P] }
// Prints one JSON object; exits 3 on any count/fitness mismatch.
#include <cuda_runtime.h>

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../../include/ebic_b200.h"

namespace {

struct Batch {
    std::vector<size_t> off;
    std::vector<uint16_t> cols;
    std::vector<uint64_t> counts;
    std::vector<double> fit;
};

__global__ void evict_l2(const float4* __restrict__ p, size_t n, float* sink) {
    float acc = 0.f;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
        const float4 v = p[i];
        acc += v.x + v.y + v.z + v.w;
    }
    if (acc == 12345.f) *sink = acc;
}

bool read_batches(const char* path, std::vector<Batch>& out) {
    FILE* f = std::fopen(path, "rb");
    if (!f) return false;
    uint64_t P;
    while (std::fread(&P, 8, 1, f) == 1) {
        Batch b;
        b.off.resize(P + 1);
        if (std::fread(b.off.data(), 8, P + 1, f) != P + 1) return false;
        b.cols.resize(b.off[P]);
        if (std::fread(b.cols.data(), 2, b.off[P], f) != b.off[P]) return false;
        b.counts.resize(P);
        b.fit.resize(P);
        if (std::fread(b.counts.data(), 8, P, f) != P) return false;
        if (std::fread(b.fit.data(), 8, P, f) != P) return false;
        out.push_back(std::move(b));
    }
    std::fclose(f);
    return !out.empty();
}

}  // namespace

int main(int argc, char** argv) {
    if (argc != 15) {
        std::fprintf(stderr, "usage: %s batches rows cols n_blocks brows bcols pattern overlap noise seed eps sigma steps warmup\n", argv[0]);
        return 2;
    }
    std::vector<Batch> batches;
    if (!read_batches(argv[1], batches)) {
        std::fprintf(stderr, "cannot read batches\n");
        return 2;
    }
    const size_t rows = std::strtoull(argv[2], nullptr, 10), cols = std::strtoull(argv[3], nullptr, 10);
    const size_t nb = std::strtoull(argv[4], nullptr, 10);
    std::vector<size_t> brows(nb, std::strtoull(argv[5], nullptr, 10)), bcols(nb, std::strtoull(argv[6], nullptr, 10));
    const int pattern = std::atoi(argv[7]);
    const size_t overlap = std::strtoull(argv[8], nullptr, 10);
    const double noise = std::atof(argv[9]);
    const uint64_t seed = std::strtoull(argv[10], nullptr, 10);
    const double eps = std::atof(argv[11]);
    const uint64_t sigma = std::strtoull(argv[12], nullptr, 10);
    const int steps = std::atoi(argv[13]), warmup = std::atoi(argv[14]);

    std::vector<double> values(rows * cols);
    if (ebic_synth_generate(rows, cols, nb, brows.data(), bcols.data(), pattern, overlap, overlap, noise,
                            seed, values.data()) != EBIC_OK) {
        std::fprintf(stderr, "generate failed\n");
        return 2;
    }
    ebic_ctx* ctx = nullptr;
    std::vector<int> devs;  // EBIC_GPUS="0,1,..." as in include/ebic/fitness.hpp (default 0)
    if (const char* e = std::getenv("EBIC_GPUS"))
        for (const char* q = e; *q;) {
            devs.push_back(std::atoi(q));
            while (*q && *q != ',') ++q;
            if (*q == ',') ++q;
        }
    if (devs.empty()) devs.push_back(0);
    if (ebic_ctx_create(values.data(), rows, cols, devs.data(), (int)devs.size(), &ctx) != EBIC_OK) {
        std::fprintf(stderr, "ctx: %s\n", ebic_last_error());
        return 2;
    }
    const size_t evict_bytes = 512ull << 20;
    float4* evict = nullptr;
    float* sink = nullptr;
    cudaStream_t es;
    cudaMalloc(&evict, evict_bytes);
    cudaMemset(evict, 0, evict_bytes);
    cudaMalloc(&sink, 4);
    cudaStreamCreateWithFlags(&es, cudaStreamNonBlocking);

    std::vector<double> fit;
    std::vector<uint64_t> cnt;
    double total_s = 0.0;
    uint64_t series = 0, h2d = 0, d2h = 0;
    int bad = 0;
    double ht0[5] = {0, 0, 0, 0, 0};
    uint64_t calls0 = 0;
    for (int k = 0; k < warmup + steps; ++k) {
        if (k == warmup) ebic_ctx_host_timers(ctx, ht0, &calls0);
        const Batch& b = batches[k % batches.size()];
        const size_t P = b.off.size() - 1;
        fit.assign(P, 0.0);
        cnt.assign(P, 0);
        evict_l2<<<148 * 4, 512, 0, es>>>(evict, evict_bytes / 16, sink);
        cudaStreamSynchronize(es);
        const auto t0 = std::chrono::steady_clock::now();
        const int rc = ebic_evaluate_population(ctx, b.off.data(), b.cols.data(), P, sigma, eps, cnt.data(),
                                                fit.data());
        const auto t1 = std::chrono::steady_clock::now();
        if (rc != EBIC_OK) {
            std::fprintf(stderr, "evaluate: %s\n", ebic_last_error());
            return 2;
        }
        if (std::memcmp(cnt.data(), b.counts.data(), P * 8) || std::memcmp(fit.data(), b.fit.data(), P * 8)) ++bad;
        if (k >= warmup) {
            total_s += std::chrono::duration<double>(t1 - t0).count();
            series += P;
            h2d += (P + 1) * 8 + b.off[P] * 2;
            d2h += P * 16;
        }
    }
    double ht[5] = {0, 0, 0, 0, 0};
    uint64_t calls = 0;
    ebic_ctx_host_timers(ctx, ht, &calls);
    for (int i = 0; i < 5; ++i)  // means over the timed calls only
        ht[i] = calls > calls0 ? (ht[i] * calls - ht0[i] * calls0) / double(calls - calls0) : 0.0;
    std::printf("{\"e2e_biclusters_per_s\": %.6e, \"us_per_step\": %.3f, \"steps\": %d, \"series\": %llu, "
                "\"h2d_bytes_per_step\": %llu, \"d2h_bytes_per_step\": %llu, \"mismatched_steps\": %d, "
                "\"host_us\": {\"validate\": %.2f, \"stage_h2d\": %.2f, \"launch\": %.2f, \"wait\": %.2f, \"copy_out\": %.2f}}\n",
                series / total_s, total_s / steps * 1e6, steps, (unsigned long long)series,
                (unsigned long long)(h2d / steps), (unsigned long long)(d2h / steps), bad,
                ht[0], ht[1], ht[2], ht[3], ht[4]);
    ebic_ctx_destroy(ctx);
    return bad ? 3 : 0;
}
