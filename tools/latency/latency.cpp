// latency.cpp -- small-call latency of the C ABI, timed
// from C so no interpreter overhead is included.  For each size: the median
// wall time of
//   sync_dev   pospopcnt_u16(device ptr)           (launch + 128 B D2H + sync)
//   async      pospopcnt_async(...) + cudaStreamSynchronize
//   graph      pospopcnt_graph_launch(...) + cudaStreamSynchronize
//   sync_host  pospopcnt_u16(pinned host ptr)      (H2D + launch + D2H + sync)
// Output: CSV on stdout.  Build: make -C tools/latency
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "pospopcnt_b200.h"

static double now_us() {
    return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

template <class F>
static double median_us(F f, int reps) {
    std::vector<double> t;
    for (int i = 0; i < 5; ++i) f();
    for (int i = 0; i < reps; ++i) {
        const double a = now_us();
        f();
        t.push_back(now_us() - a);
    }
    std::sort(t.begin(), t.end());
    return t[t.size() / 2];
}

#define OK(x)                                                                              \
    do {                                                                                   \
        if ((x) != 0) {                                                                    \
            std::fprintf(stderr, "%s failed: %s\n", #x, pospop_last_error());              \
            std::exit(1);                                                                  \
        }                                                                                  \
    } while (0)

int main(int argc, char** argv) {
    const int reps = argc > 1 ? std::atoi(argv[1]) : 200;
    const size_t sizes[] = {1,       64,      1024,    4096,    16384,    32768,    65536,   131072,
                            262144,  524288,  1048576, 2097152, 4194304, 8388608, 16777216, 33554432};
    const size_t maxn = 33554432;
    uint16_t* h = nullptr;
    cudaMallocHost(&h, maxn * 2);
    for (size_t i = 0; i < maxn; ++i) h[i] = (uint16_t)(i * 2654435761u >> 7);
    uint16_t* d = nullptr;
    uint64_t* d_out = nullptr;
    cudaMalloc(&d, maxn * 2);
    cudaMalloc(&d_out, 64 * 8);
    cudaMemcpy(d, h, maxn * 2, cudaMemcpyHostToDevice);
    cudaStream_t s;
    cudaStreamCreate(&s);
    std::printf("len_words,sync_dev_us,async_us,graph_us,sync_host_us\n");
    for (size_t n : sizes) {
        uint64_t c[16], ch[16];
        OK(pospopcnt_u16(d, n, c));
        OK(pospopcnt_u16(h, n, ch));
        for (int p = 0; p < 16; ++p)
            if (c[p] != ch[p]) {
                std::fprintf(stderr, "device/host mismatch at n=%zu\n", n);
                return 1;
            }
        pospop_graph g = nullptr;
        OK(pospopcnt_graph_create(16, d, n, d_out, &g));
        const double t_sync = median_us([&] { OK(pospopcnt_u16(d, n, c)); }, reps);
        const double t_async = median_us([&] {
            OK(pospopcnt_async(16, d, n, d_out, 0, 65535, 0, 0, s));
            cudaStreamSynchronize(s);
        }, reps);
        const double t_graph = median_us([&] {
            OK(pospopcnt_graph_launch(g, s));
            cudaStreamSynchronize(s);
        }, reps);
        const double t_host = median_us([&] { OK(pospopcnt_u16(h, n, ch)); }, reps);
        pospopcnt_graph_destroy(g);
        std::printf("%zu,%.2f,%.2f,%.2f,%.2f\n", n, t_sync, t_async, t_graph, t_host);
    }
    return 0;
}
