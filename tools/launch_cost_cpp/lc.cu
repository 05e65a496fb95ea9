#include <cuda_runtime.h>
#include <dlfcn.h>
#include <chrono>
#include <cstdio>
#include <cstdint>
__global__ void empty_kernel(int* p) { if (p && threadIdx.x == 9999) *p = 1; }
typedef int (*AsyncFn)(int, const void*, size_t, uint64_t*, int, uint32_t, int, int, void*);
int main(int argc, char** argv) {
    void* h = dlopen(argv[1], RTLD_NOW);
    if (!h) { printf("dlopen failed %s\n", dlerror()); return 1; }
    AsyncFn fn = (AsyncFn)dlsym(h, "pospopcnt_async");
    cudaStream_t s; cudaStreamCreate(&s);
    void* d; cudaMalloc(&d, 1 << 20); cudaMemset(d, 0, 1 << 20);
    uint64_t* out; cudaMalloc(&out, 512);
    const int N = 20000;
    for (int i = 0; i < 100; ++i) fn(16, d, 2048, out, 0, 65535, 0, 0, s);
    cudaStreamSynchronize(s);
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < N; ++i) fn(16, d, 2048, out, 0, 65535, 0, 0, s);
    auto t1 = std::chrono::steady_clock::now();
    cudaStreamSynchronize(s);
    printf("pospopcnt_async host %.2f us/call\n", std::chrono::duration<double, std::micro>(t1 - t0).count() / N);
    cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(1); cfg.blockDim = dim3(256); cfg.stream = s;
    cudaLaunchAttribute attr[1]; attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1; cfg.attrs = attr; cfg.numAttrs = 1;
    for (int i = 0; i < 100; ++i) cudaLaunchKernelEx(&cfg, empty_kernel, (int*)nullptr);
    cudaStreamSynchronize(s);
    t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < N; ++i) cudaLaunchKernelEx(&cfg, empty_kernel, (int*)nullptr);
    t1 = std::chrono::steady_clock::now();
    cudaStreamSynchronize(s);
    printf("cudaLaunchKernelEx(PDL) empty host %.2f us/call\n", std::chrono::duration<double, std::micro>(t1 - t0).count() / N);
    cfg.numAttrs = 0;
    t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < N; ++i) cudaLaunchKernelEx(&cfg, empty_kernel, (int*)nullptr);
    t1 = std::chrono::steady_clock::now();
    cudaStreamSynchronize(s);
    printf("cudaLaunchKernelEx empty host %.2f us/call\n", std::chrono::duration<double, std::micro>(t1 - t0).count() / N);
    t0 = std::chrono::steady_clock::now();
    int dev; cudaPointerAttributes pa;
    for (int i = 0; i < N; ++i) { cudaGetDevice(&dev); }
    t1 = std::chrono::steady_clock::now();
    printf("cudaGetDevice %.3f us\n", std::chrono::duration<double, std::micro>(t1 - t0).count() / N);
    t0 = std::chrono::steady_clock::now();
    int nd;
    for (int i = 0; i < N; ++i) { cudaGetDeviceCount(&nd); }
    t1 = std::chrono::steady_clock::now();
    printf("cudaGetDeviceCount %.3f us\n", std::chrono::duration<double, std::micro>(t1 - t0).count() / N);
    t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < N; ++i) { cudaPointerGetAttributes(&pa, d); }
    t1 = std::chrono::steady_clock::now();
    printf("cudaPointerGetAttributes %.3f us\n", std::chrono::duration<double, std::micro>(t1 - t0).count() / N);
    return 0;
}
