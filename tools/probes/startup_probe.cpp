// Start-up split of the drop-in (GPU box): how long each one-time step takes
// before the first generation is evaluated, in process order.
//   load      dlopen(libebic_b200.so): fat-binary registration of the library
//   cuInit    driver initialisation
//   context   primary context on device 0 (cudaFree(0) equivalent: cuDevicePrimaryCtxRetain + SetCurrent)
//   create    ebic_ctx_create: matrix upload + column-major transpose + tables
//   first     first ebic_evaluate_population: rank layout build for this eps,
//             lazy module load of the count kernel, graph instantiation
//   second    steady-state call
// usage: startup_probe ROWS COLS [repeat]   (N(0,1) matrix, 600 series of 4 columns)
#include <dlfcn.h>

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

using clk = std::chrono::steady_clock;
static double ms(clk::time_point a, clk::time_point b) { return std::chrono::duration<double, std::milli>(b - a).count(); }

typedef int (*cuInit_t)(unsigned);
typedef int (*cuDeviceGet_t)(int*, int);
typedef int (*cuRetain_t)(void**, int);
typedef int (*cuSetCurrent_t)(void*);
typedef int (*create_t)(const double*, size_t, size_t, const int*, int, void**);
typedef int (*eval_t)(void*, const size_t*, const uint16_t*, size_t, uint64_t, double, uint64_t*, double*);
typedef int (*destroy_t)(void*);
typedef const char* (*err_t)();

int main(int argc, char** argv) {
    const size_t rows = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 500;
    const size_t cols = argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 100;
    std::mt19937_64 g(7);
    std::normal_distribution<double> nd;
    std::vector<double> m(rows * cols);
    for (double& x : m) x = nd(g);
    const size_t P = 600, L = 4;
    std::vector<size_t> off(P + 1);
    std::vector<uint16_t> cl(P * L);
    for (size_t s = 0; s <= P; ++s) off[s] = s * L;
    for (size_t i = 0; i < P * L; ++i) cl[i] = static_cast<uint16_t>(g() % cols);
    std::vector<uint64_t> counts(P);
    std::vector<double> fit(P);

    const auto t0 = clk::now();
    void* cu = dlopen("libcuda.so.1", RTLD_NOW | RTLD_GLOBAL);
    const char* lib = std::getenv("EBIC_LIB") ? std::getenv("EBIC_LIB") : "paper_1801_03039_b200/libebic_b200.so";
    void* h = dlopen(lib, RTLD_NOW);
    if (!cu || !h) {
        std::fprintf(stderr, "dlopen: %s\n", dlerror());
        return 1;
    }
    const auto t1 = clk::now();
    auto cuInit = reinterpret_cast<cuInit_t>(dlsym(cu, "cuInit"));
    auto cuDeviceGet = reinterpret_cast<cuDeviceGet_t>(dlsym(cu, "cuDeviceGet"));
    auto cuRetain = reinterpret_cast<cuRetain_t>(dlsym(cu, "cuDevicePrimaryCtxRetain"));
    auto cuSet = reinterpret_cast<cuSetCurrent_t>(dlsym(cu, "cuCtxSetCurrent"));
    auto create = reinterpret_cast<create_t>(dlsym(h, "ebic_ctx_create"));
    auto eval = reinterpret_cast<eval_t>(dlsym(h, "ebic_evaluate_population"));
    auto destroy = reinterpret_cast<destroy_t>(dlsym(h, "ebic_ctx_destroy"));
    auto last_error = reinterpret_cast<err_t>(dlsym(h, "ebic_last_error"));
    if (cuInit(0)) return 2;
    const auto t2 = clk::now();
    int dev = 0;
    void* pctx = nullptr;
    if (cuDeviceGet(&dev, 0) || cuRetain(&pctx, dev) || cuSet(pctx)) return 3;
    const auto t3 = clk::now();
    void* ctx = nullptr;
    const int d0 = 0;
    if (create(m.data(), rows, cols, &d0, 1, &ctx)) {
        std::fprintf(stderr, "create: %s\n", last_error());
        return 4;
    }
    const auto t4 = clk::now();
    const uint64_t sigma = rows / 50 > 4 ? rows / 50 : 4;
    if (eval(ctx, off.data(), cl.data(), P, sigma, 1e-9, counts.data(), fit.data())) {
        std::fprintf(stderr, "eval: %s\n", last_error());
        return 5;
    }
    const auto t5 = clk::now();
    eval(ctx, off.data(), cl.data(), P, sigma, 1e-9, counts.data(), fit.data());
    const auto t6 = clk::now();
    destroy(ctx);
    const auto t7 = clk::now();
    std::printf("startup_ms rows=%zu cols=%zu load=%.2f cuInit=%.2f context=%.2f create=%.2f first=%.2f second=%.4f destroy=%.2f total_to_first=%.2f\n",
                rows, cols, ms(t0, t1), ms(t1, t2), ms(t2, t3), ms(t3, t4), ms(t4, t5), ms(t5, t6), ms(t6, t7),
                ms(t0, t5));
    return 0;
}
