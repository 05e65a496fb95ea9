// pospop_device.cuh -- device primitives for the sm_100a pospopcnt kernels.
//
// The reference's width-generic engine (proj/core/src/detail/csa_engine.hpp)
// works on SIMD registers of W bits split into 16-bit lanes.  On B200 the
// "lane vector" is one 32-bit register per thread: 32 independent 1-bit
// channels for the carry-save arithmetic and two 16-bit lanes for the
// counters.  A warp is 32 such registers (1024 channels) per instruction.
//
//   channel c of a 32-bit register  <->  bit c of the little-endian dword
//   k=16 : channel c counts position c mod 16   (two words per register)
//   k=8  : channel c counts position c mod 8    (four bytes per register)
//   k=32 : channel c counts position c
//   k=64 : two banks; even dwords (low halves) -> positions 0..31,
//          odd dwords (high halves) -> positions 32..63
#pragma once

#include <cstdint>

namespace pospop_b200 {

// ---------------------------------------------------------------------------
// Carry-save adder: two LOP3.LUT with the AVX-512 vpternlogd immediates.
// PTX lop3 LUT operands are a=0xF0, b=0xCC, c=0xAA, so 0xE8 is the majority
// (carry, weight 2) and 0x96 the parity (sum, weight 1): 2h + l = a + b + c.
// Reference: proj/core/src/csa_avx512.cpp:42-45, backend64.hpp:39-43.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void csa(uint32_t& h, uint32_t& l, uint32_t a, uint32_t b, uint32_t c) {
    asm("lop3.b32 %0, %1, %2, %3, 0xE8;" : "=r"(h) : "r"(a), "r"(b), "r"(c));
    asm("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(l) : "r"(a), "r"(b), "r"(c));
}

// Harley-Seal tree over 2^L registers (csa_engine.hpp:36-52): carries[j]
// holds the bit-plane of weight 2^j; returns the emitted plane of weight 2^L.
// Fully unrolled; STRIDE lets a bank pick every other register (k=64).
template <int L, int STRIDE = 1>
struct Tree {
    static __device__ __forceinline__ uint32_t run(uint32_t* carries, const uint32_t* in) {
        uint32_t h, l;
        if constexpr (L == 1) {
            csa(h, l, carries[0], in[0], in[STRIDE]);
        } else {
            const uint32_t first = Tree<L - 1, STRIDE>::run(carries, in);
            const uint32_t second = Tree<L - 1, STRIDE>::run(carries, in + (STRIDE << (L - 1)));
            csa(h, l, carries[L - 1], first, second);
        }
        carries[L - 1] = l;
        return h;
    }
};

// ---------------------------------------------------------------------------
// Lane bank: counter[p] holds two 16-bit lanes, channel p (bits 0..15) and
// channel p+16 (bits 16..31).  Each extract adds 0/1 per lane, so a lane
// stays <= the flush threshold (<= 65535).  csa_engine.hpp:67-74.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void extract(uint32_t (&counter)[16], uint32_t top) {
#pragma unroll
    for (int p = 0; p < 16; ++p) counter[p] += (top & (0x00010001u << p)) >> p;
}

// Residual-carry drain (csa_engine.hpp:86-95) in Horner form on packed lanes:
// d[p] = sum_j 2^j * bit_{p / p+16}(B_j).  Lanes stay < 2^L <= 2^8.
template <int L>
__device__ __forceinline__ void drain(uint32_t (&d)[16], const uint32_t* carries) {
#pragma unroll
    for (int p = 0; p < 16; ++p) d[p] = 0;
#pragma unroll
    for (int j = L - 1; j >= 0; --j) {
#pragma unroll
        for (int p = 0; p < 16; ++p) d[p] = (d[p] << 1) + ((carries[j] >> p) & 0x00010001u);
    }
}

// ---------------------------------------------------------------------------
// Warp transpose-reduce ("reduce-scatter"): every lane holds v[0..32); after
// 16+8+4+2+1 = 31 shuffles lane i holds sum over the warp of v[i].
// Must be called by all 32 lanes (uniform control flow).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t warp_transpose_reduce(uint32_t (&v)[32]) {
    const uint32_t lane = threadIdx.x & 31u;
#pragma unroll
    for (int half = 16; half >= 1; half >>= 1) {
        const bool upper = (lane & half) != 0;
#pragma unroll
        for (int i = 0; i < half; ++i) {
            const uint32_t send = upper ? v[i] : v[i + half];
            const uint32_t keep = upper ? v[i + half] : v[i];
            v[i] = keep + __shfl_xor_sync(0xFFFFFFFFu, send, half);
        }
    }
    return v[0];
}

// Unpacks the lane bank into 32 per-channel values scaled by 2^shift, plus an
// optional weight-1 drain bank, and reduces them across the warp.  Lane i
// returns the warp total of channel i.  Values: lane <= 65535, so
// (65535 << 8) + 255 < 2^24 and a 32-lane sum < 2^29 fits in u32.
__device__ __forceinline__ uint32_t bank_warp_total(const uint32_t (&counter)[16], int shift,
                                                    const uint32_t (&d)[16]) {
    uint32_t v[32];
#pragma unroll
    for (int p = 0; p < 16; ++p) {
        v[p] = ((counter[p] & 0xFFFFu) << shift) + (d[p] & 0xFFFFu);
        v[p + 16] = ((counter[p] >> 16) << shift) + (d[p] >> 16);
    }
    return warp_transpose_reduce(v);
}

// Byte-lane counters: counter[p] byte lane j counts channel 8j + p (p < 8);
// a lane takes at most 255 extracts between flushes.
__device__ __forceinline__ void extract_bytes(uint32_t (&counter)[16], uint32_t top) {
#pragma unroll
    for (int p = 0; p < 8; ++p)  // shifts on the FMA pipe (IMAD.HI): the FLAG kernel is ALU-bound
        counter[p] += (p ? __umulhi(top, 1u << (32 - p)) : top) & 0x01010101u;
}

__device__ __forceinline__ uint32_t bank_warp_total_bytes(const uint32_t (&counter)[16], int shift,
                                                          const uint32_t (&d)[16]) {
    uint32_t v[32];
#pragma unroll
    for (int c = 0; c < 32; ++c)
        v[c] = (((counter[c & 7] >> (8 * (c >> 3))) & 0xFFu) << shift) +
               (c < 16 ? (d[c] & 0xFFFFu) : (d[c - 16] >> 16));
    return warp_transpose_reduce(v);
}

// ---------------------------------------------------------------------------
// Debug bounds checks (libpospopcnt_b200_debug.so, built with
// -DPOSPOP_DEBUG_BOUNDS): every vector load asserts that its index lies in the
// valid range of the stream / array; a violation traps the kernel, which the
// host sees as a CUDA error.  No-ops in the product build.
// ---------------------------------------------------------------------------
#ifdef POSPOP_DEBUG_BOUNDS
#define POSPOP_CHECK(cond)          \
    do {                            \
        if (!(cond)) __trap();      \
    } while (0)
#else
#define POSPOP_CHECK(cond) \
    do {                   \
    } while (0)
#endif

// ---------------------------------------------------------------------------
// Streaming vector loads: read-only path, no L1 allocation (each byte is
// touched exactly once).  VB = 16 -> LDG.E.NA.128 (512 B per warp),
// VB = 32 -> LDG.E.NA.256 (1 KiB per warp; Blackwell's 256-bit load).
// HINT 0: default L2 policy; 1: L2 evict_first (256-bit form only);
// 2: L2 256 B prefetch hint (128-bit form only); 3: allocate in L1 (128-bit
// form only).
// ---------------------------------------------------------------------------
template <int VB, int HINT>
__device__ __forceinline__ void ldg_stream(const uint8_t* p, uint32_t (&r)[VB / 4]) {
    static_assert(VB == 16 || VB == 32, "vector width");
    if constexpr (VB == 16) {
        if constexpr (HINT == 3) {  // L1-allocating (lanes reading half sectors: the other half hits L1)
            asm("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];"
                : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "l"(p));
        } else if constexpr (HINT == 2) {
            asm("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
                : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "l"(p));
        } else {
            asm("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "l"(p));
        }
    } else {
        if constexpr (HINT == 1) {
            asm("ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                  "=r"(r[7])
                : "l"(p));
        } else {
            asm("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                  "=r"(r[7])
                : "l"(p));
        }
    }
}

// Keeps only bytes [lo, hi) of a VB-byte vector (0 <= lo <= hi <= VB).
// Zeroed bytes contribute nothing to any positional count, so masked
// vectors replace scalar head/tail loops for unaligned starts and ragged ends.
template <int VB>
__device__ __forceinline__ void mask_bytes(uint32_t (&r)[VB / 4], int lo, int hi) {
#pragma unroll
    for (int j = 0; j < VB / 4; ++j) {
        const int a = min(max(lo - 4 * j, 0), 4);
        const int b = min(max(hi - 4 * j, 0), 4);
        const uint32_t below_b = b >= 4 ? 0xFFFFFFFFu : ((1u << (8 * b)) - 1u);
        const uint32_t below_a = a >= 4 ? 0xFFFFFFFFu : ((1u << (8 * a)) - 1u);
        r[j] &= below_b & ~below_a;
    }
}

// ---------------------------------------------------------------------------
// Counter-based generator (device twin of oracle/pospop_oracle.c's
// orc_generate; tests hash both and compare).  SplitMix64 finaliser.
// ---------------------------------------------------------------------------
constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ull;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

}  // namespace pospop_b200
