// probe.cu -- measurement tool (not product): the achievable HBM read
// bandwidth on this B200 for a pure streaming read with the same access
// pattern as the pospopcnt stream kernel (persistent grid, per-CTA 1 KiB-
// aligned group ranges, VB-byte vectors, VPT vectors per thread per step),
// so the roofline denominator for a READ-ONLY stream can be compared with
// the driver's copy-based MEASURED_PEAKS.json.
#include <cuda_runtime.h>
#include <cstdint>

template <int VB, int HINT>
__device__ __forceinline__ void ld(const uint8_t* p, uint32_t (&r)[VB / 4]) {
    if constexpr (VB == 16) {
        if constexpr (HINT == 2)
            asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "l"(p));
        else
            asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "l"(p));
    } else {
        if constexpr (HINT == 1)
            asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                         : "l"(p));
        else
            asm volatile("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                         : "l"(p));
    }
}

template <int VB, int HINT, int VPT>
__global__ void read_kernel(const uint8_t* base, unsigned long long nvec, unsigned long long* sink) {
    const unsigned long long ng = nvec / 32;
    const unsigned long long S = (ng * blockIdx.x / gridDim.x) * 32;
    const unsigned long long E = (ng * (blockIdx.x + 1) / gridDim.x) * 32;
    const unsigned long long tile = (unsigned long long)VPT * blockDim.x;
    uint32_t acc = 0;
    unsigned long long t = S;
    for (; t + tile <= E; t += tile) {
#pragma unroll
        for (int v = 0; v < VPT; ++v) {
            uint32_t x[VB / 4];
            ld<VB, HINT>(base + (t + v * blockDim.x + threadIdx.x) * VB, x);
#pragma unroll
            for (int j = 0; j < VB / 4; ++j) acc ^= x[j];
        }
    }
    for (unsigned long long i = t + threadIdx.x; i < E; i += blockDim.x) {
        uint32_t x[VB / 4];
        ld<VB, HINT>(base + i * VB, x);
#pragma unroll
        for (int j = 0; j < VB / 4; ++j) acc ^= x[j];
    }
    if (acc == 0x12345678u) atomicAdd(sink, 1ull);  // keeps the loads alive
}

template <int VB, int HINT, int VPT>
static int launch(const void* p, size_t nbytes, int block, int per_sm, cudaStream_t s, unsigned long long* sink) {
    int sms = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (per_sm <= 0) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, read_kernel<VB, HINT, VPT>, block, 0);
    read_kernel<VB, HINT, VPT><<<sms * per_sm, block, 0, s>>>((const uint8_t*)p, nbytes / VB, sink);
    return (int)cudaGetLastError();
}

extern "C" int probe_read(const void* p, size_t nbytes, int vb, int hint, int vpt, int block, int per_sm,
                          void* stream, unsigned long long* sink) {
    cudaStream_t s = (cudaStream_t)stream;
#define CASE(VB, H, V) if (vb == VB && hint == H && vpt == V) return launch<VB, H, V>(p, nbytes, block, per_sm, s, sink);
    CASE(16, 0, 4) CASE(16, 0, 8) CASE(16, 0, 16) CASE(16, 2, 8) CASE(16, 2, 16)
    CASE(32, 0, 2) CASE(32, 0, 4) CASE(32, 0, 8) CASE(32, 1, 4) CASE(32, 1, 8)
#undef CASE
    return -1;
}
