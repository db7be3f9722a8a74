// Launch-cost probe: a kernel that returns at entry (or spins ~W cycles), launched 10x back to back in a CUDA graph,
// with the launch shape of K7 varied one property at a time: dynamic smem, threads, cluster dims, PDL attribute
// (trigger early / none).   nvcc -arch=sm_100a -o launch_cost launch_cost.cu
#include <cstdio>
#include <cuda_runtime.h>
template <int CL>
__global__ void probe(int spin, int early, unsigned long long* sink) {
    if (early) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (spin) {
        const long long t0 = clock64();
        while (clock64() - t0 < spin) {}
        if (threadIdx.x == 0 && blockIdx.x == 0) *sink = t0;
    }
}
__global__ void __cluster_dims__(2, 1, 1) probe_cl(int spin, int early, unsigned long long* sink) {
    if (early) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (spin) {
        const long long t0 = clock64();
        while (clock64() - t0 < spin) {}
        if (threadIdx.x == 0 && blockIdx.x == 0) *sink = t0;
    }
}
static float run(bool cluster, int threads, int smem, bool pdl, int early, int spin, unsigned long long* sink) {
    cudaStream_t st;
    cudaStreamCreate(&st);
    void (*k)(int, int, unsigned long long*) = cluster ? probe_cl : probe<1>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(148);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < 10; ++i) cudaLaunchKernelEx(&cfg, k, spin, early, sink);
    cudaStreamEndCapture(st, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int i = 0; i < 3; ++i) cudaGraphLaunch(ge, st);
    cudaStreamSynchronize(st);
    float best = 1e9f;
    for (int r = 0; r < 10; ++r) {
        cudaEventRecord(a, st);
        cudaGraphLaunch(ge, st);
        cudaEventRecord(b, st);
        cudaStreamSynchronize(st);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("error: %s\n", cudaGetErrorString(e));
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
    cudaStreamDestroy(st);
    return best * 100.f;  // us per kernel
}
int main() {
    unsigned long long* sink;
    cudaMalloc(&sink, 8);
    const int S = 227 * 1024;
    for (int spin : {0, 20000}) {
        printf("spin %d cycles per kernel: us per kernel in a graph of 10\n", spin);
        printf("  128 thr, no smem, no pdl      %.2f\n", run(false, 128, 0, false, 0, spin, sink));
        printf("  128 thr, no smem, pdl late    %.2f\n", run(false, 128, 0, true, 0, spin, sink));
        printf("  128 thr, no smem, pdl early   %.2f\n", run(false, 128, 0, true, 1, spin, sink));
        printf("  864 thr, no smem, no pdl      %.2f\n", run(false, 864, 0, false, 0, spin, sink));
        printf("  128 thr, 227K smem, no pdl    %.2f\n", run(false, 128, S, false, 0, spin, sink));
        printf("  864 thr, 227K smem, no pdl    %.2f\n", run(false, 864, S, false, 0, spin, sink));
        printf("  864 thr, 227K, cluster, no pdl %.2f\n", run(true, 864, S, false, 0, spin, sink));
        printf("  864 thr, 227K, cluster, pdl late  %.2f\n", run(true, 864, S, true, 0, spin, sink));
        printf("  864 thr, 227K, cluster, pdl early %.2f\n", run(true, 864, S, true, 1, spin, sink));
        printf("  608 thr, 227K, cluster, pdl early %.2f\n", run(true, 608, S, true, 1, spin, sink));
        printf("  864 thr, 100K, cluster, pdl early %.2f\n", run(true, 864, 100 * 1024, true, 1, spin, sink));
    }
    return 0;
}
