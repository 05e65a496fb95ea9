// pospop_aux.cuh -- auxiliary kernels: synthetic-input generators, the order-independent
// digest, and the device micro-op harness (test/bench infrastructure).
// Device code only; included by pospop_kernels.cu (the single CUDA translation
// unit, which instantiates the kernels and owns the host-side launchers).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "pospop_device.cuh"
#include "pospop_stream.cuh"

namespace pospop_b200 {
namespace dev {

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
            case 7:  // SAM FLAG words: the 12 defined bits uniform, bits 12-15 clear
                ((uint16_t*)out)[l] = (uint16_t)((mix64(key + ((i >> 2) + 1) * kGamma) >> (16 * (i & 3))) & 0x0FFF);
                break;
            case 8: {  // SAM FLAG words, a paired-end-like mix (oracle/pospop_oracle.c gen_range)
                constexpr uint16_t kProper[4] = {99, 147, 83, 163};
                constexpr uint16_t kPaired[8] = {65, 129, 113, 177, 97, 145, 81, 161};
                constexpr uint16_t kHalf[8] = {73, 133, 89, 121, 137, 153, 185, 69};
                const uint64_t u = mix64(key + (i + 1) * kGamma);
                const uint32_t c = (uint32_t)(u & 0xFF), sel = (uint32_t)((u >> 8) & 7);
                uint32_t f = c < 220 ? kProper[sel & 3] : c < 240 ? kPaired[sel] : c < 250 ? kHalf[sel]
                           : c < 254 ? ((sel & 1) ? 141u : 77u) : ((sel & 1) ? 16u : 0u);
                if (((u >> 16) & 0xF) < 2) f |= 0x400;     // duplicate, 1/8
                if (((u >> 20) & 0x7F) == 0) f |= 0x100;   // secondary, 1/128
                if (((u >> 27) & 0x7F) == 1) f |= 0x800;   // supplementary, 1/128
                if (((u >> 34) & 0xFFFF) == 0) f |= 0x200; // QC-fail, 2^-16
                ((uint16_t*)out)[l] = (uint16_t)f;
                break;
            }
        }
    }
}

// Device micro-op harness: runs the exact device
// primitives the stream kernel inlines -- csa, Tree<L>, extract, drain,
// bank_warp_total -- on caller-supplied 32-bit registers, so tests can pin
// them against the reference's micro-op KATs (proj/tests/test_csa.cpp).
//   op 0 csa:      in[3i..3i+2] -> out[2i] = high, out[2i+1] = low
//   op 1 tree:     carries in[0..L), blocks of 2^L inputs follow; out = tops
//                  per block, then the final carries
//   op 2 extract:  tops in[0..n) into a zeroed bank; out = 16 counters
//   op 3 drain:    carries in[0..L); out = 16 packed Horner lanes
//   op 4 total:    32 lanes x (16 counters, shift) -> lane c's warp total of channel c
template <int L>
__device__ void micro_tree(const uint32_t* in, size_t nblocks, uint32_t* out) {
    uint32_t carries[L];
    for (int j = 0; j < L; ++j) carries[j] = in[j];
    for (size_t b = 0; b < nblocks; ++b) {
        uint32_t r[1 << L];
        for (int i = 0; i < (1 << L); ++i) r[i] = in[L + b * (1 << L) + i];
        out[b] = Tree<L, 1>::run(carries, r);
    }
    for (int j = 0; j < L; ++j) out[nblocks + j] = carries[j];
}

__global__ void microop_kernel(int op, int depth, const uint32_t* in, unsigned long long n, uint32_t* out) {
    if (op == 4) {  // one full warp
        uint32_t counter[16], d[16];
        for (int p = 0; p < 16; ++p) {
            counter[p] = in[threadIdx.x * 17 + p];
            d[p] = 0;
        }
        out[threadIdx.x] = bank_warp_total(counter, (int)in[threadIdx.x * 17 + 16], d);
        return;
    }
    if (threadIdx.x != 0) return;
    switch (op) {
        case 0:
            for (unsigned long long i = 0; i < n; ++i) csa(out[2 * i], out[2 * i + 1], in[3 * i], in[3 * i + 1], in[3 * i + 2]);
            break;
        case 1: {
            const unsigned long long nb = (n - depth) >> depth;
            switch (depth) {
                case 1: micro_tree<1>(in, nb, out); break;
                case 2: micro_tree<2>(in, nb, out); break;
                case 3: micro_tree<3>(in, nb, out); break;
                case 4: micro_tree<4>(in, nb, out); break;
                case 5: micro_tree<5>(in, nb, out); break;
                case 6: micro_tree<6>(in, nb, out); break;
                default: micro_tree<7>(in, nb, out); break;
            }
            break;
        }
        case 2: {
            uint32_t counter[16];
            for (int p = 0; p < 16; ++p) counter[p] = 0;
            for (unsigned long long i = 0; i < n; ++i) extract(counter, in[i]);
            for (int p = 0; p < 16; ++p) out[p] = counter[p];
            break;
        }
        case 3: {
            uint32_t d[16];
            switch (depth) {
                case 1: drain<1>(d, in); break;
                case 2: drain<2>(d, in); break;
                case 3: drain<3>(d, in); break;
                case 4: drain<4>(d, in); break;
                case 5: drain<5>(d, in); break;
                case 6: drain<6>(d, in); break;
                default: drain<7>(d, in); break;
            }
            for (int p = 0; p < 16; ++p) out[p] = d[p];
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

// The reduce kernel: one CTA, launched right after the count on the same
// stream (programmatic dependent launch: it starts once every CTA of the
// count is running, so its spin never keeps a count CTA off an SM).
__global__ void __launch_bounds__(64) exchange_reduce_kernel(unsigned long long* own, int n, int k, int S,
                                                             unsigned long long step, unsigned long long* out) {
    pdl_allow_next();
    xchg_reduce(own, n, k, S, step, out, [] { pdl_wait_prev(); });
}

// Test harness for the protocol with fewer GPUs than ranks (B200_PROFILING:
// ranks that wait on one another must not be separate launches on one GPU):
// one cooperative launch, block r plays rank r for `steps` consecutive steps
// -- optional device sleep, credit wait, row stores + tags into every block's
// buffer, reduce of its own buffer -- with the same device functions as the
// counting and reduce kernels.  inputs: steps x n x k; totals: n x steps x k.
__global__ void __launch_bounds__(64) exchange_emulate_kernel(unsigned long long* const* bufs, int n, int k, int S,
                                                              int steps, const unsigned long long* inputs,
                                                              const unsigned* sleep_ns, unsigned long long* totals) {
    __shared__ unsigned long long vals[64];
    const int r = blockIdx.x;
    for (int step = 0; step < steps; ++step) {
        if (threadIdx.x == 0 && sleep_ns[step * n + r]) {
            const unsigned long long t0 = globaltimer();
            while (globaltimer() - t0 < sleep_ns[step * n + r]) __nanosleep(1000);
        }
        for (int p = threadIdx.x; p < k; p += blockDim.x) vals[p] = inputs[((size_t)step * n + r) * k + p];
        __syncthreads();
        xchg_wait_credit(bufs, n, r, S, (unsigned long long)step);
        __syncthreads();
        xchg_store_rows(bufs, n, r, k, S, (unsigned long long)step, vals, blockDim.x);
        xchg_reduce(bufs[r], n, k, S, (unsigned long long)step, totals + ((size_t)r * steps + step) * k, [] {});
    }
}

}  // namespace dev
}  // namespace pospop_b200
