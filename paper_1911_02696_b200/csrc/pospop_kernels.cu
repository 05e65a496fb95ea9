// pospop_kernels.cu -- sm_100a kernels for positional population count.
//
// Hot path (BASELINE.json north_star; reference run_csa, proj/core/src/
// detail/csa_engine.hpp:100-132):
//
//   stream_kernel<NBANK, L>
//     persistent grid (SMs x resident CTAs), each CTA owns a contiguous,
//     16 B-aligned slice of the stream and walks it in tiles of
//     blockDim x (NBANK * 2^L / 4) 128-bit vectors (coalesced LDG.128,
//     read-only / no-L1-allocate / L2 evict-first);
//     per thread a Harley-Seal tree of depth L over 2^L 32-bit registers
//     (2 LOP3 per CSA), lane-counter extraction of the emitted plane,
//     an overflow-safe flush every `flush_threshold` tree blocks,
//     then residual-carry drain, warp transpose-reduce, shared-memory
//     atomics, one 64-bit global atomic per channel per CTA, and a
//     last-CTA ticket that folds channels to the k positions, adds the
//     unaligned head/tail words and writes (or accumulates) the result.
//     One launch, no memset, no second reduction kernel.
//
//   segmented_kernel<NBANK, L>
//     one warp per array (persistent warp-stride over arrays); the same
//     tree per lane; the warp transpose-reduce leaves channel c on lane c
//     and the row is written with one coalesced store per lane.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdlib>

#include "pospop_device.cuh"
#include "pospop_launch.h"

namespace pospop_b200 {

namespace {

std::atomic<unsigned long long> g_launches{0};

struct StreamArgs {
    const uint4* body;        // 16 B aligned
    unsigned long long nvec;  // 16 B vectors in the body
    const uint8_t* head;      // words before the body
    const uint8_t* tail;      // words after the body
    uint32_t head_bytes;
    uint32_t tail_bytes;
    int k;
    uint32_t flush_threshold;
    unsigned long long* acc;
    unsigned int* ticket;
    unsigned long long* out;
    int accumulate;
};

// Bit `pos` of every little-endian wb-byte word in [p, p + nbytes).
__device__ __forceinline__ unsigned long long count_pos_words(const uint8_t* p, uint32_t nbytes,
                                                             int wb, int pos) {
    unsigned long long c = 0;
    for (uint32_t i = 0; i + wb <= nbytes; i += wb) c += (p[i + (pos >> 3)] >> (pos & 7)) & 1u;
    return c;
}

// Channel -> position fold: the channels (of 32 * NBANK) that count position
// p are p + m * k for m = 0 .. 32/k - 1 (k <= 32), or channel p (k = 64).
__device__ __forceinline__ int channels_per_position(int k) { return k >= 32 ? 1 : 32 / k; }

template <int NBANK, int L>
__device__ __forceinline__ void tree_block(const uint32_t (&r)[NBANK << L], uint32_t (&carries)[NBANK][L],
                                           uint32_t (&counter)[NBANK][16]) {
    if constexpr (NBANK == 1) {
        extract(counter[0], Tree<L, 1>::run(carries[0], r));
    } else {
        extract(counter[0], Tree<L, 2>::run(carries[0], r));
        extract(counter[1], Tree<L, 2>::run(carries[1], r + 1));
    }
}

template <int NBANK>
__device__ __forceinline__ void zero_bank(uint32_t (&counter)[NBANK][16]) {
#pragma unroll
    for (int b = 0; b < NBANK; ++b)
#pragma unroll
        for (int p = 0; p < 16; ++p) counter[b][p] = 0;
}

template <int NBANK, int L>
__global__ void __launch_bounds__(256) stream_kernel(const StreamArgs a) {
    constexpr int REGS = NBANK << L;  // 32-bit input registers per tree block
    constexpr int V = REGS / 4;       // 128-bit vectors per tree block
    static_assert(V >= 1, "tree must consume at least one 128-bit vector");

    __shared__ unsigned long long s_acc[32 * NBANK];
    __shared__ int s_last;
    for (int i = threadIdx.x; i < 32 * NBANK; i += blockDim.x) s_acc[i] = 0;
    __syncthreads();

    const unsigned long long tile = (unsigned long long)V * blockDim.x;
    const unsigned long long begin = a.nvec * blockIdx.x / gridDim.x;
    const unsigned long long end = a.nvec * (blockIdx.x + 1) / gridDim.x;
    const uint32_t lane = threadIdx.x & 31u;

    uint32_t carries[NBANK][L];
    uint32_t counter[NBANK][16];
#pragma unroll
    for (int b = 0; b < NBANK; ++b)
#pragma unroll
        for (int j = 0; j < L; ++j) carries[b][j] = 0;
    zero_bank<NBANK>(counter);
    uint32_t nb = 0;

    auto flush = [&](int shift) {
        uint32_t d[16];
#pragma unroll
        for (int p = 0; p < 16; ++p) d[p] = 0;
#pragma unroll
        for (int b = 0; b < NBANK; ++b) {
            const uint32_t t = bank_warp_total(counter[b], shift, d);
            if (t) atomicAdd(&s_acc[b * 32 + lane], (unsigned long long)t);
        }
        zero_bank<NBANK>(counter);
        nb = 0;
    };

    unsigned long long base = begin;
    const uint4* p = a.body + threadIdx.x;
    for (; base + tile <= end; base += tile) {
        uint32_t r[REGS];
#pragma unroll
        for (int v = 0; v < V; ++v) {
            const uint4 x = ldg_stream(p + base + (unsigned long long)v * blockDim.x);
            r[4 * v + 0] = x.x;
            r[4 * v + 1] = x.y;
            r[4 * v + 2] = x.z;
            r[4 * v + 3] = x.w;
        }
        tree_block<NBANK, L>(r, carries, counter);
        if (++nb == a.flush_threshold) flush(L);
    }
    if (base < end) {  // partial tile: zero inputs leave every count unchanged
        uint32_t r[REGS];
#pragma unroll
        for (int v = 0; v < V; ++v) {
            const unsigned long long idx = base + (unsigned long long)v * blockDim.x + threadIdx.x;
            const uint4 x = idx < end ? ldg_stream(a.body + idx) : make_uint4(0u, 0u, 0u, 0u);
            r[4 * v + 0] = x.x;
            r[4 * v + 1] = x.y;
            r[4 * v + 2] = x.z;
            r[4 * v + 3] = x.w;
        }
        tree_block<NBANK, L>(r, carries, counter);
        if (++nb == a.flush_threshold) flush(L);
    }

    // Final flush of the lane bank (weight 2^L) fused with the carry drain.
#pragma unroll
    for (int b = 0; b < NBANK; ++b) {
        uint32_t d[16];
        drain<L>(d, carries[b]);
        const uint32_t t = bank_warp_total(counter[b], L, d);
        if (t) atomicAdd(&s_acc[b * 32 + lane], (unsigned long long)t);
    }
    __syncthreads();

    for (int c = threadIdx.x; c < 32 * NBANK; c += blockDim.x)
        if (s_acc[c]) atomicAdd(&a.acc[c], s_acc[c]);
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(a.ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;

    // Last CTA: every other CTA has fenced its channel atomics.
    __threadfence();
    const int k = a.k;
    const int wb = k >> 3;
    for (int pos = threadIdx.x; pos < k; pos += blockDim.x) {
        unsigned long long sum = 0;
        if (k == 64) {
            sum = atomicExch(&a.acc[pos], 0ull);
        } else {
            const int m = channels_per_position(k);
            for (int j = 0; j < m; ++j) sum += atomicExch(&a.acc[pos + j * k], 0ull);
        }
        sum += count_pos_words(a.head, a.head_bytes, wb, pos);
        sum += count_pos_words(a.tail, a.tail_bytes, wb, pos);
        a.out[pos] = a.accumulate ? a.out[pos] + sum : sum;
    }
    if (threadIdx.x == 0) *a.ticket = 0u;
}

template <int NBANK, int L>
__global__ void __launch_bounds__(256) segmented_kernel(const uint8_t* data,
                                                        const unsigned long long* offsets,
                                                        unsigned long long n_arrays, int k,
                                                        uint32_t flush_threshold,
                                                        unsigned long long* out) {
    constexpr int REGS = NBANK << L;
    constexpr int V = REGS / 4;
    const uint32_t lane = threadIdx.x & 31u;
    const unsigned long long warp = (blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x) >> 5;
    const unsigned long long nwarps = (gridDim.x * (unsigned long long)blockDim.x) >> 5;
    const int wb = k >> 3;

    for (unsigned long long arr = warp; arr < n_arrays; arr += nwarps) {
        const uint8_t* start = data + offsets[arr] * wb;
        const uint8_t* stop = data + offsets[arr + 1] * wb;
        const uint8_t* bstart = (const uint8_t*)(((uintptr_t)start + 15) & ~(uintptr_t)15);
        const uint8_t* bstop = (const uint8_t*)((uintptr_t)stop & ~(uintptr_t)15);
        if (bstart > bstop) bstart = bstop = stop;  // shorter than one aligned vector: all head
        const uint4* body = (const uint4*)bstart;
        const unsigned long long nvec = (unsigned long long)(bstop - bstart) >> 4;

        uint32_t carries[NBANK][L];
        uint32_t counter[NBANK][16];
#pragma unroll
        for (int b = 0; b < NBANK; ++b)
#pragma unroll
            for (int j = 0; j < L; ++j) carries[b][j] = 0;
        zero_bank<NBANK>(counter);
        uint32_t nb = 0;
        unsigned long long tot[NBANK];
#pragma unroll
        for (int b = 0; b < NBANK; ++b) tot[b] = 0;

        for (unsigned long long base = 0; base < nvec; base += 32ull * V) {
            uint32_t r[REGS];
#pragma unroll
            for (int v = 0; v < V; ++v) {
                const unsigned long long idx = base + 32ull * v + lane;
                const uint4 x = idx < nvec ? ldg_stream(body + idx) : make_uint4(0u, 0u, 0u, 0u);
                r[4 * v + 0] = x.x;
                r[4 * v + 1] = x.y;
                r[4 * v + 2] = x.z;
                r[4 * v + 3] = x.w;
            }
            tree_block<NBANK, L>(r, carries, counter);
            if (++nb == flush_threshold) {
                uint32_t d[16];
#pragma unroll
                for (int p = 0; p < 16; ++p) d[p] = 0;
#pragma unroll
                for (int b = 0; b < NBANK; ++b) tot[b] += bank_warp_total(counter[b], L, d);
                zero_bank<NBANK>(counter);
                nb = 0;
            }
        }
#pragma unroll
        for (int b = 0; b < NBANK; ++b) {
            uint32_t d[16];
            drain<L>(d, carries[b]);
            tot[b] += bank_warp_total(counter[b], L, d);
        }

        // lane c holds channel c (bank b: channel 32b + c).  Fold to positions.
        unsigned long long* row = out + arr * (unsigned long long)k;
        if (NBANK == 2) {  // k == 64
#pragma unroll
            for (int b = 0; b < NBANK; ++b) {
                const int pos = 32 * b + lane;
                row[pos] = tot[b] + count_pos_words(start, (uint32_t)(bstart - start), wb, pos) +
                           count_pos_words(bstop, (uint32_t)(stop - bstop), wb, pos);
            }
        } else {
            unsigned long long t = tot[0];
            for (int w = 16; w >= k; w >>= 1) t += __shfl_down_sync(0xFFFFFFFFu, t, w);
            if ((int)lane < k)
                row[lane] = t + count_pos_words(start, (uint32_t)(bstart - start), wb, lane) +
                            count_pos_words(bstop, (uint32_t)(stop - bstop), wb, lane);
        }
    }
}

__global__ void generate_kernel(int kind, uint64_t key, uint64_t index_base, unsigned long long n,
                                void* out) {
    constexpr uint32_t kZipf[15] = {1417819056u, 2079255034u, 2502690694u, 2811261488u,
                                    3052670681u, 3250210401u, 3416940100u, 3560893466u,
                                    3687353720u, 3799975090u, 3901386976u, 3993542513u,
                                    4077930985u, 4155713140u, 4227810676u};
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long l = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; l < n;
         l += stride) {
        const uint64_t i = index_base + l;
        switch (kind) {
            case 1:
                ((uint16_t*)out)[l] = (uint16_t)(mix64(key + ((i >> 2) + 1) * kGamma) >> (16 * (i & 3)));
                break;
            case 2: {
                const uint32_t u = (uint32_t)(mix64(key + (i + 1) * kGamma) >> 32);
                int bit = 0;
#pragma unroll
                for (int t = 0; t < 15; ++t) bit += kZipf[t] <= u;
                ((uint16_t*)out)[l] = (uint16_t)(1u << bit);
                break;
            }
            case 3: {
                const uint8_t b = (uint8_t)(mix64(key + ((i >> 3) + 1) * kGamma) >> (8 * (i & 7)));
                ((uint8_t*)out)[l] = ((i >> 12) & 1) ? b : (uint8_t)(1u << (b & 7));
                break;
            }
            case 4: {
                uint32_t w = 0;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const uint64_t h = mix64(key + (4 * i + j + 1) * kGamma);
#pragma unroll
                    for (int m = 0; m < 4; ++m)
                        w |= (uint32_t)(((h >> (16 * m)) & 0xFFFF) < 6554u) << (4 * j + m);
                }
                ((uint16_t*)out)[l] = (uint16_t)w;
                break;
            }
            case 5:
                ((uint32_t*)out)[l] = (uint32_t)(mix64(key + ((i >> 1) + 1) * kGamma) >> (32 * (i & 1)));
                break;
            case 6:
                ((uint64_t*)out)[l] = mix64(key + (i + 1) * kGamma);
                break;
        }
    }
}

__global__ void digest_kernel(const uint8_t* data, unsigned long long nbytes, unsigned long long* d) {
    const unsigned long long nw = (nbytes + 7) >> 3;
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    unsigned long long s = 0;
    for (unsigned long long j = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; j < nw;
         j += stride) {
        uint64_t w = 0;
        if (8 * j + 8 <= nbytes) {
            w = ((const uint64_t*)data)[j];
        } else {
            for (unsigned long long t = 0; 8 * j + t < nbytes; ++t) w |= (uint64_t)data[8 * j + t] << (8 * t);
        }
        s += mix64(w + j * kGamma);
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) s += __shfl_xor_sync(0xFFFFFFFFu, s, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(d, s);
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------

constexpr int kDefaultBlock = 256;
constexpr int kDefaultDepth1 = 6;  // k = 8/16/32: 64 registers = 256 B per thread per tree block
constexpr int kDefaultDepth2 = 5;  // k = 64: two banks of 32 registers

int env_int(const char* name, int dflt) {
    const char* v = std::getenv(name);
    return v && *v ? std::atoi(v) : dflt;
}

struct DeviceInfo {
    int sms = 0;
};

DeviceInfo device_info() {
    static thread_local int cached_dev = -1;
    static thread_local DeviceInfo info;
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev != cached_dev) {
        cudaDeviceGetAttribute(&info.sms, cudaDevAttrMultiProcessorCount, dev);
        cached_dev = dev;
    }
    return info;
}

template <class Kernel>
int resident_blocks(Kernel kernel, int block) {
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, block, 0) != cudaSuccess || n < 1) n = 1;
    return n;
}

using StreamKernel = void (*)(const StreamArgs);

StreamKernel pick_stream(int nbank, int depth) {
    if (nbank == 1) {
        switch (depth) {
            case 3: return stream_kernel<1, 3>;
            case 4: return stream_kernel<1, 4>;
            case 5: return stream_kernel<1, 5>;
            case 7: return stream_kernel<1, 7>;
            default: return stream_kernel<1, 6>;
        }
    }
    switch (depth) {
        case 2: return stream_kernel<2, 2>;
        case 3: return stream_kernel<2, 3>;
        case 4: return stream_kernel<2, 4>;
        case 6: return stream_kernel<2, 6>;
        default: return stream_kernel<2, 5>;
    }
}

using SegKernel = void (*)(const uint8_t*, const unsigned long long*, unsigned long long, int, uint32_t,
                           unsigned long long*);

SegKernel pick_segmented(int nbank, int depth) {
    if (nbank == 1) {
        switch (depth) {
            case 3: return segmented_kernel<1, 3>;
            case 4: return segmented_kernel<1, 4>;
            case 6: return segmented_kernel<1, 6>;
            default: return segmented_kernel<1, 5>;
        }
    }
    switch (depth) {
        case 2: return segmented_kernel<2, 2>;
        case 3: return segmented_kernel<2, 3>;
        case 5: return segmented_kernel<2, 5>;
        default: return segmented_kernel<2, 4>;
    }
}

}  // namespace

unsigned long long kernel_launches() { return g_launches.load(); }

cudaError_t launch_stream(int k, const void* data, size_t len_words, unsigned long long* d_out,
                          bool accumulate, const LaunchOptions& opt, const StreamWorkspace& ws,
                          cudaStream_t stream) {
    const int nbank = k == 64 ? 2 : 1;
    const int depth = opt.depth ? opt.depth
                                : env_int("POSPOP_TREE_DEPTH", nbank == 1 ? kDefaultDepth1 : kDefaultDepth2);
    const int block = opt.block ? opt.block : env_int("POSPOP_BLOCK", kDefaultBlock);
    StreamKernel kernel = pick_stream(nbank, depth);

    const uint8_t* p = static_cast<const uint8_t*>(data);
    const size_t nbytes = len_words * (size_t)(k / 8);
    const uint8_t* bstart = (const uint8_t*)(((uintptr_t)p + 15) & ~(uintptr_t)15);
    const uint8_t* bstop = (const uint8_t*)((uintptr_t)(p + nbytes) & ~(uintptr_t)15);
    if (bstart > bstop || nbytes == 0) bstart = bstop = p + nbytes;

    StreamArgs a;
    a.body = reinterpret_cast<const uint4*>(bstart);
    a.nvec = (unsigned long long)(bstop - bstart) >> 4;
    a.head = p;
    a.head_bytes = (uint32_t)(bstart - p);
    a.tail = bstop;
    a.tail_bytes = (uint32_t)(p + nbytes - bstop);
    a.k = k;
    a.flush_threshold = opt.flush_threshold;
    a.acc = ws.acc;
    a.ticket = ws.ticket;
    a.out = d_out;
    a.accumulate = accumulate ? 1 : 0;

    int grid = opt.grid;
    if (grid <= 0) {
        const int depth_regs = nbank << (depth < 2 ? 2 : depth);
        const unsigned long long tile = (unsigned long long)(depth_regs / 4) * block;
        const unsigned long long want = (a.nvec + tile - 1) / tile;
        const int per_sm = env_int("POSPOP_BLOCKS_PER_SM", resident_blocks(kernel, block));
        const unsigned long long cap = (unsigned long long)device_info().sms * per_sm;
        grid = (int)(want < 1 ? 1 : (want < cap ? want : cap));
    }
    kernel<<<grid, block, 0, stream>>>(a);
    ++g_launches;
    return cudaGetLastError();
}

cudaError_t launch_segmented(int k, const void* data, const unsigned long long* d_offsets, size_t n,
                             unsigned long long* d_out, const LaunchOptions& opt, cudaStream_t stream) {
    if (n == 0) return cudaSuccess;
    const int nbank = k == 64 ? 2 : 1;
    const int depth = opt.depth ? opt.depth : env_int("POSPOP_SEG_DEPTH", nbank == 1 ? 5 : 4);
    const int block = opt.block ? opt.block : env_int("POSPOP_SEG_BLOCK", kDefaultBlock);
    SegKernel kernel = pick_segmented(nbank, depth);
    int grid = opt.grid;
    if (grid <= 0) {
        const unsigned long long warps_per_block = block / 32;
        const unsigned long long want = (n + warps_per_block - 1) / warps_per_block;
        const int per_sm = env_int("POSPOP_SEG_BLOCKS_PER_SM", resident_blocks(kernel, block));
        const unsigned long long cap = (unsigned long long)device_info().sms * per_sm;
        grid = (int)(want < cap ? want : cap);
    }
    kernel<<<grid, block, 0, stream>>>(static_cast<const uint8_t*>(data), d_offsets, n, k,
                                       opt.flush_threshold, d_out);
    ++g_launches;
    return cudaGetLastError();
}

cudaError_t launch_generate(int kind, uint64_t seed, uint64_t index_base, size_t n, void* out,
                            cudaStream_t stream) {
    if (n == 0) return cudaSuccess;
    const uint64_t key = mix64(seed ^ ((uint64_t)kind * 0xD1B54A32D192ED03ull));
    const int block = 256;
    const unsigned long long want = (n + block - 1) / block;
    const unsigned long long cap = (unsigned long long)device_info().sms * 16;
    generate_kernel<<<(int)(want < cap ? want : cap), block, 0, stream>>>(kind, key, index_base, n, out);
    ++g_launches;
    return cudaGetLastError();
}

cudaError_t launch_digest(const void* data, size_t nbytes, unsigned long long* d_digest,
                          cudaStream_t stream) {
    if (nbytes == 0) return cudaSuccess;
    const int block = 256;
    const unsigned long long want = ((nbytes + 7) / 8 + block - 1) / block;
    const unsigned long long cap = (unsigned long long)device_info().sms * 16;
    digest_kernel<<<(int)(want < cap ? want : cap), block, 0, stream>>>(
        static_cast<const uint8_t*>(data), nbytes, d_digest);
    ++g_launches;
    return cudaGetLastError();
}

}  // namespace pospop_b200
