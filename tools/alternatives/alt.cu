// alt.cu -- the counter schemes north_star names, measured side by side on the
// same device-resident u16 stream (measurement tool, not product code):
//   csa     the product kernel (Harley-Seal carry-save tree, libpospopcnt_b200)
//   swar    per-position SWAR: counter[p] += (x >> p) & 0x00010001 for every
//           32-bit register (two 16-bit lanes per counter), no tree
//   ballot  warp ballot per bit position: count += popc(ballot(bit p)) per
//           register, 32 ballots per register per warp
// All three must produce identical counts (checked); the output is one CSV
// row per scheme with device time (CUDA events, median of reps) and GB/s.
//   make -C tools/alternatives && tools/alternatives/alt [log2_words=32] [reps=10]
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "pospopcnt_b200.h"

#define CK(x)                                                                               \
    do {                                                                                    \
        cudaError_t e_ = (x);                                                               \
        if (e_ != cudaSuccess) {                                                            \
            std::fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));                   \
            std::exit(1);                                                                   \
        }                                                                                   \
    } while (0)

constexpr int kBlock = 256;

// Per-position SWAR: 16 counters, each holding positions p (low lane) and
// p + 16 (high lane) of the 32-bit register = positions p of both words.
__global__ void __launch_bounds__(kBlock) swar_kernel(const uint4* v, size_t nvec, unsigned long long* out) {
    uint32_t c[16] = {};
    uint32_t since = 0;
    __shared__ unsigned long long s[16];
    if (threadIdx.x < 16) s[threadIdx.x] = 0;
    __syncthreads();
    auto flush = [&] {
#pragma unroll
        for (int p = 0; p < 16; ++p) {
            atomicAdd(&s[p], (unsigned long long)((c[p] & 0xFFFFu) + (c[p] >> 16)));
            c[p] = 0;
        }
    };
    for (size_t i = blockIdx.x * (size_t)kBlock + threadIdx.x; i < nvec; i += (size_t)gridDim.x * kBlock) {
        uint4 x;
        asm("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
            : "=r"(x.x), "=r"(x.y), "=r"(x.z), "=r"(x.w) : "l"(v + i));
        const uint32_t r[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int p = 0; p < 16; ++p) c[p] += (r[j] >> p) & 0x00010001u;
        if (++since == 16383) {  // 4 registers per vector: lanes stay <= 65532
            flush();
            since = 0;
        }
    }
    flush();
    __syncthreads();
    if (threadIdx.x < 16) atomicAdd(&out[threadIdx.x], s[threadIdx.x]);
}

// Ballot: for every register and bit position, one warp vote + popc.  Every
// lane accumulates all 32 channel totals of its warp; lane c keeps channel c.
__global__ void __launch_bounds__(kBlock) ballot_kernel(const uint4* v, size_t nvec, unsigned long long* out) {
    const uint32_t lane = threadIdx.x & 31u;
    uint32_t c = 0;  // channel `lane` (bit `lane` of a 32-bit register), this warp
    __shared__ unsigned long long s[32];
    if (threadIdx.x < 32) s[threadIdx.x] = 0;
    __syncthreads();
    const size_t stride = (size_t)gridDim.x * kBlock;
    const size_t n_iter = (nvec + stride - 1) / stride;  // uniform trip count: ballots need full warps
    for (size_t it = 0; it < n_iter; ++it) {
        const size_t i = it * stride + blockIdx.x * (size_t)kBlock + threadIdx.x;
        uint4 x = make_uint4(0, 0, 0, 0);
        if (i < nvec)
            asm("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                : "=r"(x.x), "=r"(x.y), "=r"(x.z), "=r"(x.w) : "l"(v + i));
        const uint32_t r[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int p = 0; p < 32; ++p) {
                const uint32_t b = __popc(__ballot_sync(0xFFFFFFFFu, (r[j] >> p) & 1u));
                c += lane == (uint32_t)p ? b : 0u;
            }
        if ((it & 0x3FFFF) == 0x3FFFF) {  // <= 2^18 * 128 per lane between flushes
            atomicAdd(&s[lane], (unsigned long long)c);
            c = 0;
        }
    }
    atomicAdd(&s[lane], (unsigned long long)c);
    __syncthreads();
    if (threadIdx.x < 32) atomicAdd(&out[threadIdx.x & 15], s[threadIdx.x]);  // fold p, p + 16
}

template <class F>
static float median_ms(F launch, int reps) {
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    std::vector<float> t;
    launch();
    CK(cudaDeviceSynchronize());
    for (int i = 0; i < reps; ++i) {
        CK(cudaEventRecord(a));
        launch();
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, a, b));
        t.push_back(ms);
    }
    std::sort(t.begin(), t.end());
    return t[t.size() / 2];
}

int main(int argc, char** argv) {
    const int lg = argc > 1 ? std::atoi(argv[1]) : 32;
    const int reps = argc > 2 ? std::atoi(argv[2]) : 10;
    const size_t n = (size_t)1 << lg;  // u16 words
    const size_t bytes = n * 2;
    uint16_t* d = nullptr;
    CK(cudaMalloc(&d, bytes));
    if (pospop_generate(4, 1, 0, n, d, nullptr) != POSPOP_OK) {  // cfg4 Bernoulli(0.1) bits
        std::fprintf(stderr, "generate: %s\n", pospop_last_error());
        return 1;
    }
    unsigned long long* d_out = nullptr;
    CK(cudaMalloc(&d_out, 64 * 8));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const size_t nvec = bytes / 16;

    uint64_t want[16];
    if (pospopcnt_u16(d, n, want) != POSPOP_OK) return 1;
    std::printf("scheme,bytes,ms,gbs,ok\n");
    const float t_csa = median_ms([&] { pospopcnt_async(16, d, n, reinterpret_cast<uint64_t*>(d_out), 0, 65535, 0, 0, nullptr); }, reps);
    std::printf("csa,%zu,%.4f,%.1f,1\n", bytes, t_csa, bytes / (t_csa * 1e-3) / 1e9);

    struct Alt {
        const char* name;
        void (*fn)(const uint4*, size_t, unsigned long long*);
        int per_sm;
    } alts[] = {{"swar", swar_kernel, 8}, {"ballot", ballot_kernel, 8}};
    for (const Alt& a : alts) {
        const int grid = sms * a.per_sm;
        auto launch = [&] {
            cudaMemsetAsync(d_out, 0, 16 * 8);
            a.fn<<<grid, kBlock>>>(reinterpret_cast<const uint4*>(d), nvec, d_out);
        };
        const float t = median_ms(launch, reps);
        uint64_t got[16];
        CK(cudaMemcpy(got, d_out, sizeof got, cudaMemcpyDeviceToHost));
        bool ok = true;
        for (int p = 0; p < 16; ++p) ok = ok && got[p] == want[p];
        std::printf("%s,%zu,%.4f,%.1f,%d\n", a.name, bytes, t, bytes / (t * 1e-3) / 1e9, ok ? 1 : 0);
        if (!ok) return 2;
    }
    return 0;
}
