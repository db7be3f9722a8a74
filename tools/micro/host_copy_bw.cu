// host_copy_bw.cu — how fast can the host-buffer drop-in move C and A?
// Measures (2 GiB, the size of config 5's int16 C):
//   D2H / H2D with cudaMemcpyAsync to/from pinned, pre-touched pageable and
//   freshly malloc'd (untouched) pageable memory; host memcpy bandwidth with
//   1..T threads; cudaHostRegister + Unregister cost.
//   nvcc -O3 -std=c++17 -o tools/micro/host_copy_bw tools/micro/host_copy_bw.cu -lpthread
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

static double now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
#define CK(x)                                                                   \
    do {                                                                        \
        cudaError_t e = (x);                                                    \
        if (e != cudaSuccess) {                                                 \
            std::printf("%s: %s\n", #x, cudaGetErrorString(e));                 \
            std::exit(1);                                                       \
        }                                                                       \
    } while (0)

static void par_memcpy(char* dst, const char* src, size_t n, int threads) {
    std::vector<std::thread> ts;
    for (int t = 0; t < threads; ++t) {
        size_t a = n * t / threads, b = n * (t + 1) / threads;
        ts.emplace_back([=] { std::memcpy(dst + a, src + a, b - a); });
    }
    for (auto& t : ts) t.join();
}

int main(int argc, char** argv) {
    const size_t N = (argc > 1 ? std::atoll(argv[1]) : 2048) << 20;
    const int maxt = std::thread::hardware_concurrency();
    std::printf("bytes %zu  hw threads %d\n", N, maxt);
    void* d;
    CK(cudaMalloc(&d, N));
    CK(cudaMemset(d, 1, N));
    char* pinned;
    CK(cudaMallocHost(&pinned, N));
    std::memset(pinned, 0, N);
    char* page = (char*)std::malloc(N);
    std::memset(page, 0, N);
    cudaStream_t s;
    CK(cudaStreamCreate(&s));
    auto rate = [&](const char* what, auto fn) {
        fn();
        CK(cudaDeviceSynchronize());
        double t0 = now();
        fn();
        CK(cudaDeviceSynchronize());
        double t = now() - t0;
        std::printf("%-44s %8.2f ms  %7.2f GB/s\n", what, t * 1e3, N / t / 1e9);
    };
    rate("D2H -> pinned", [&] { CK(cudaMemcpyAsync(pinned, d, N, cudaMemcpyDeviceToHost, s)); });
    rate("H2D <- pinned", [&] { CK(cudaMemcpyAsync(d, pinned, N, cudaMemcpyHostToDevice, s)); });
    rate("D2H -> pageable (touched)", [&] { CK(cudaMemcpyAsync(page, d, N, cudaMemcpyDeviceToHost, s)); });
    rate("H2D <- pageable (touched)", [&] { CK(cudaMemcpyAsync(d, page, N, cudaMemcpyHostToDevice, s)); });
    {
        char* fresh = (char*)std::malloc(N);
        double t0 = now();
        CK(cudaMemcpy(fresh, d, N, cudaMemcpyDeviceToHost));
        double t = now() - t0;
        std::printf("%-44s %8.2f ms  %7.2f GB/s\n", "D2H -> fresh malloc (page faults)", t * 1e3, N / t / 1e9);
        std::free(fresh);
    }
    for (int t = 1; t <= maxt; t *= 2) {
        char buf[64];
        std::snprintf(buf, sizeof buf, "host memcpy pinned->pageable, %d thr", t);
        double t0 = now();
        par_memcpy(page, pinned, N, t);
        double dt = now() - t0;
        std::printf("%-44s %8.2f ms  %7.2f GB/s\n", buf, dt * 1e3, N / dt / 1e9);
    }
    {
        double t0 = now();
        CK(cudaHostRegister(page, N, cudaHostRegisterDefault));
        double t1 = now();
        CK(cudaMemcpyAsync(page, d, N, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        double t2 = now();
        CK(cudaHostUnregister(page));
        double t3 = now();
        std::printf("cudaHostRegister %.2f ms, D2H into registered %.2f ms (%.2f GB/s), unregister %.2f ms\n",
                    (t1 - t0) * 1e3, (t2 - t1) * 1e3, N / (t2 - t1) / 1e9, (t3 - t2) * 1e3);
    }
    return 0;
}
