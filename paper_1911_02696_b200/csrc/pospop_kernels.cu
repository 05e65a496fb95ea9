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
#include <cstdio>
#include <cstdlib>
#include <map>

#include "pospop_device.cuh"
#include "pospop_launch.h"

namespace pospop_b200 {

namespace {

std::atomic<unsigned long long> g_launches{0};

// The stream is addressed in VB-byte vectors from `base`, the largest
// 32*VB-aligned address <= data.  Vectors [v0, v1) hold the data; the first
// and last are byte-masked to [lo_byte, VB) and [0, hi_byte), so unaligned
// starts and ragged ends need no scalar code, and every warp load (32
// consecutive vectors) stays 32*VB-aligned.  Vector indices below v0 are
// never dereferenced.  Work is split over CTAs in whole groups of 32 vectors.
struct StreamArgs {
    const uint8_t* base;
    unsigned long long v0, v1;  // valid vectors
    unsigned long long f0, f1;  // fully valid (unmasked) vectors [f0, f1)
    unsigned long long g0, ng;  // first group, number of groups
    int lo_byte, hi_byte;       // valid bytes of vector v0 / vector v1-1
    int k;
    uint32_t flush_threshold;
    unsigned long long* acc;
    unsigned int* ticket;
    unsigned long long* out;
    int accumulate;
    unsigned long long* trace;  // diagnostics: per CTA {t_start, t_loop_end, t_flushed, t_done, smid} or null
    // dynamic schedule (SCHED 1): warp tiles, chunk counter, chunk sizes
    unsigned long long* next;   // global chunk counter (zero on entry, re-zeroed by the last CTA)
    unsigned long long nwt, nA, CA, CB;
    unsigned long long pool;    // SCHED 2: warp tiles in the global tail pool
    // MODE 1 (FLAG statistics)
    unsigned long long data_off;  // data start - base, bytes
    unsigned long long word_base; // global index of the first word (host-staged chunks)
    unsigned long long* bad;      // max of ~(index of an invalid FLAG word); 0 = none
};

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ unsigned smid() {
    unsigned r;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
    return r;
}

// Programmatic dependent launch (sm_90+): `pdl_allow_next` lets the next
// kernel in the stream start launching (its CTAs take SMs as ours retire);
// `pdl_wait_prev` blocks until the previous kernel in the stream has completed
// and its writes are visible.  Both are no-ops for launches without the
// programmatic-serialization attribute.
__device__ __forceinline__ void pdl_allow_next() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait_prev() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

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

// Loads one tree block for this thread: VPT vectors at first + v * stride.
// `fast`: the whole tile lies in the fully valid range (no predicates, no
// masks, immediate offsets when stride is a compile-time constant).
template <int VB, int HINT, int VPT>
__device__ __forceinline__ void load_tree_block(const StreamArgs& a, unsigned long long first, unsigned stride,
                                                bool fast, uint32_t (&r)[VPT * (VB / 4)]) {
    constexpr int RPV = VB / 4;
    if (fast) {
        const uint8_t* p = a.base + first * VB;
#pragma unroll
        for (int v = 0; v < VPT; ++v) {
            uint32_t x[RPV];
            ldg_stream<VB, HINT>(p + (unsigned long long)v * stride * VB, x);
#pragma unroll
            for (int j = 0; j < RPV; ++j) r[v * RPV + j] = x[j];
        }
    } else {
#pragma unroll
        for (int v = 0; v < VPT; ++v) {
            const unsigned long long idx = first + (unsigned long long)v * stride;
            uint32_t x[RPV];
#pragma unroll
            for (int j = 0; j < RPV; ++j) x[j] = 0;
            if (idx >= a.v0 && idx < a.v1) {
                ldg_stream<VB, HINT>(a.base + idx * VB, x);
                if (idx == a.v0 || idx + 1 == a.v1)
                    mask_bytes<VB>(x, idx == a.v0 ? a.lo_byte : 0, idx + 1 == a.v1 ? a.hi_byte : VB);
            }
#pragma unroll
            for (int j = 0; j < RPV; ++j) r[v * RPV + j] = x[j];
        }
    }
}

// Lane-bank flush (weight 2^L) into the CTA's shared channel totals; must be
// called by all 32 lanes of a warp together.
template <int NBANK, int L>
__device__ __forceinline__ void flush_bank_to_smem(uint32_t (&counter)[NBANK][16], unsigned long long* s_acc,
                                                   uint32_t lane) {
    uint32_t d[16];
#pragma unroll
    for (int p = 0; p < 16; ++p) d[p] = 0;
#pragma unroll
    for (int b = 0; b < NBANK; ++b) {
        const uint32_t tot = bank_warp_total(counter[b], L, d);
        if (tot) atomicAdd(&s_acc[b * 32 + lane], (unsigned long long)tot);
    }
    zero_bank<NBANK>(counter);
}

// CTA epilogue: final flush fused with the carry drain, CTA channel totals to
// the global accumulator, ticket; the last CTA folds channels to positions,
// writes/accumulates out[k] and leaves the scratch (acc, ticket, chunk
// counter) zeroed for the next launch.
template <int NBANK, int L, int MODE>
__device__ __forceinline__ void cta_finish(const StreamArgs& a, uint32_t (&carries)[NBANK][L],
                                           uint32_t (&counter)[NBANK][16], unsigned long long* s_acc,
                                           int* s_last, unsigned block, uint32_t lane) {
    if (a.trace && threadIdx.x == 0) a.trace[blockIdx.x * 5 + 1] = globaltimer();
    pdl_wait_prev();  // the previous launch on this stream owns acc/ticket/next until it completes
#pragma unroll
    for (int b = 0; b < NBANK; ++b) {
        uint32_t d[16];
        drain<L>(d, carries[b]);
        const uint32_t tot = bank_warp_total(counter[b], L, d);
        if (tot) atomicAdd(&s_acc[b * 32 + lane], (unsigned long long)tot);
    }
    __syncthreads();
    for (int c = threadIdx.x; c < 32 * NBANK; c += block)
        if (s_acc[c]) atomicAdd(&a.acc[c], s_acc[c]);
    __threadfence();
    __syncthreads();
    if (a.trace && threadIdx.x == 0) a.trace[blockIdx.x * 5 + 2] = globaltimer();
    if (threadIdx.x == 0) *s_last = atomicAdd(a.ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!*s_last) return;

    // Last CTA: every other CTA has fenced its channel atomics.
    __threadfence();
    if constexpr (MODE == 1) {  // two banks of k = 16: out[16 b + p] = acc[32 b + p] + acc[32 b + p + 16]
        for (int pos = threadIdx.x; pos < 32; pos += block) {
            const int b = pos >> 4, p = pos & 15;
            const unsigned long long sum =
                atomicExch(&a.acc[32 * b + p], 0ull) + atomicExch(&a.acc[32 * b + p + 16], 0ull);
            a.out[pos] = a.accumulate ? a.out[pos] + sum : sum;
        }
        if (threadIdx.x == 0) {  // ~index: the larger code is the earlier word
            const unsigned long long code = atomicExch(a.bad, 0ull);
            a.out[32] = a.accumulate && a.out[32] > code ? a.out[32] : code;
        }
    } else {
        const int k = a.k;
        for (int pos = threadIdx.x; pos < k; pos += block) {
            unsigned long long sum = 0;
            if (k == 64) {
                sum = atomicExch(&a.acc[pos], 0ull);
            } else {
                const int m = channels_per_position(k);
                for (int j = 0; j < m; ++j) sum += atomicExch(&a.acc[pos + j * k], 0ull);
            }
            a.out[pos] = a.accumulate ? a.out[pos] + sum : sum;
        }
    }
    if (threadIdx.x == 0) {
        *a.ticket = 0u;
        if (a.next) *a.next = 0ull;
    }
    if (a.trace && threadIdx.x == 0) a.trace[blockIdx.x * 5 + 3] = globaltimer();
}

// ---------------------------------------------------------------------------
// FLAG statistics (reference proj/core/src/flagstats.cpp).
// SWAR form of flag_transform (flagstats.cpp:94-125) on a register holding two
// SAM FLAG words.  Only the positions bucket_from_counts reads (1,2,3,6,7,8,
// 9,10,11,12; flagstats.cpp:39-63) are produced.  Per 16-bit lane:
//   G  = paired & !secondary & !supplementary ;  GU = G & !unmapped
//   bits 1,3 = w & GU ; bits 6,7 = w & G ; bits 2,8,9,10 = w ;
//   bit 11 = supplementary & !secondary ; bit 12 (pair_map) = GU & !mate_unmapped
// `all` is that word for every read; `fail` keeps it only for QC-fail reads.
// The QC-pass plane is never formed: pass counts = all counts - fail counts
// (exact integers, derived on the host).  The kernel is ALU-bound, so the
// shifts run on the FMA pipe (IMAD.HI / IMAD.SHL) and the G/GU selections are
// built by multiplying the lane predicate into the target bit positions
// (g * 0x00C0 + gu * 0x100A) instead of full lane masks.
// ---------------------------------------------------------------------------
template <int S>
__device__ __forceinline__ uint32_t shr_fma(uint32_t x) { return __umulhi(x, 1u << (32 - S)); }
template <int S>
__device__ __forceinline__ uint32_t shl_fma(uint32_t x) { return x * (1u << S); }

__device__ __forceinline__ void flag_transform2(uint32_t w, uint32_t& all, uint32_t& fail) {
    constexpr uint32_t L1 = 0x00010001u;
    const uint32_t g0 = w & ~shr_fma<8>(w) & ~shr_fma<11>(w);  // bit 0 / 16: paired & primary
    const uint32_t g = g0 & L1;
    const uint32_t gu = g0 & ~shr_fma<2>(w) & L1;
    const uint32_t t = g * 0x00C0u + gu * 0x100Au;              // bits 6,7 <- G ; bits 1,3,12 <- GU
    const uint32_t mf = (shr_fma<9>(w) & L1) * 0xFFFFu;           // QC-fail lane mask
    all = (w & (t | 0x07040704u)) | (t & ~shl_fma<9>(w) & 0x10001000u) | (w & ~shl_fma<3>(w) & 0x08000800u);
    fail = all & mf;
}

// Tree-block consumer.  MODE 0: positional counts of the words (NBANK banks).
// MODE 1: FLAG statistics -- transform, then bank 0 counts the transformed
// words of all reads and bank 1 those of QC-fail reads; words with reserved bits 12-15 set are
// reported through a.bad (the first such index wins, as the reference's
// check_reserved throws at the first one, flagstats.cpp:34-36).
template <int MODE, int NBANK, int L, int VB, int REGS>
__device__ __forceinline__ void consume(const StreamArgs& a, const uint32_t (&r)[REGS], unsigned long long first,
                                        unsigned stride, uint32_t (&carries)[NBANK][L],
                                        uint32_t (&counter)[NBANK][16]) {
    if constexpr (MODE == 0) {
        tree_block<NBANK, L>(r, carries, counter);
    } else {
        static_assert(NBANK == 2 && REGS == (1 << L), "FLAG mode: two banks of 2^L registers");
        constexpr int RPV = VB / 4;
        uint32_t all[REGS], fail[REGS];
        uint32_t bad = 0;
#pragma unroll
        for (int i = 0; i < REGS; ++i) {
            bad |= r[i];
            flag_transform2(r[i], all[i], fail[i]);
        }
        extract(counter[0], Tree<L, 1>::run(carries[0], all));
        extract(counter[1], Tree<L, 1>::run(carries[1], fail));
        if (bad & 0xF000F000u) {  // rare: locate this thread's first invalid word
            // Fully unrolled: a runtime index into r[] would force the whole
            // tile through local memory on the hot path.
            unsigned long long best = ~0ull;
#pragma unroll
            for (int i = 0; i < REGS; ++i)
#pragma unroll
                for (int h = 0; h < 2; ++h)
                    if ((r[i] >> (16 * h)) & 0xF000u) {
                        const unsigned long long byte =
                            (first + (unsigned long long)(i / RPV) * stride) * VB + 4 * (i % RPV) + 2 * h;
                        const unsigned long long word = ((byte - a.data_off) >> 1) + a.word_base;
                        best = word < best ? word : best;
                    }
            atomicMax(a.bad, ~best);
        }
    }
}

// SCHED 0 (static): CTA b owns a contiguous range of whole 32-vector groups and
// walks it in CTA tiles of BLOCK x VPT vectors.
// SCHED 1 (dynamic): warps pull chunks of warp tiles (32 lanes x VPT vectors,
// VPT 1 KiB-aligned warp loads) from a global counter, large chunks first
// (nA chunks of CA warp tiles) then small ones (CB) so no warp or CTA idles
// while another still holds a big share; the next chunk index is fetched one
// chunk ahead so the atomic's latency hides behind the loads.
// BLOCK > 0: compile-time block size; BLOCK == 0: runtime blockDim.x.
template <int NBANK, int L, int VB, int HINT, int BLOCK, int SCHED, int MODE, int MINB = 1>
__global__ void __launch_bounds__(BLOCK > 0 ? BLOCK : 256, MINB) stream_kernel(const StreamArgs a) {
    constexpr int REGS = MODE == 1 ? (1 << L) : (NBANK << L);  // 32-bit input registers per tree block
    constexpr int RPV = VB / 4;       // registers per vector
    constexpr int VPT = REGS / RPV;   // vectors per thread per tree block
    static_assert(VPT >= 1, "tree must consume at least one vector");
    const unsigned block = BLOCK > 0 ? (unsigned)BLOCK : blockDim.x;

    __shared__ unsigned long long s_acc[32 * NBANK];
    __shared__ int s_last;
    if (a.trace && threadIdx.x == 0) {
        a.trace[blockIdx.x * 5 + 0] = globaltimer();
        a.trace[blockIdx.x * 5 + 4] = smid();
    }
    for (int i = threadIdx.x; i < 32 * NBANK; i += block) s_acc[i] = 0;
    pdl_allow_next();
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31u;

    uint32_t carries[NBANK][L];
    uint32_t counter[NBANK][16];
#pragma unroll
    for (int b = 0; b < NBANK; ++b)
#pragma unroll
        for (int j = 0; j < L; ++j) carries[b][j] = 0;
    zero_bank<NBANK>(counter);
    uint32_t nb = 0;

    if constexpr (SCHED == 0) {
        const unsigned long long tile = (unsigned long long)VPT * block;
        const unsigned long long gb = a.g0 + a.ng * blockIdx.x / gridDim.x;
        const unsigned long long ge = a.g0 + a.ng * (blockIdx.x + 1) / gridDim.x;
        const unsigned long long E = ge * 32 < a.v1 ? ge * 32 : a.v1;
        const unsigned long long F = E < a.f1 ? E : a.f1;
        for (unsigned long long t = gb * 32; t < E; t += tile) {
            uint32_t r[REGS];
            const bool fast = t >= a.f0 && t + tile <= F;
            if (fast) load_tree_block<VB, HINT, VPT>(a, t + threadIdx.x, block, true, r);
            else {
                // Edge tile of this CTA: loads past E belong to the next CTA.
                load_tree_block<VB, HINT, VPT>(a, t + threadIdx.x, block, false, r);
#pragma unroll
                for (int v = 0; v < VPT; ++v)
                    if (t + (unsigned long long)v * block + threadIdx.x >= E)
#pragma unroll
                        for (int j = 0; j < RPV; ++j) r[v * RPV + j] = 0;
            }
            consume<MODE, NBANK, L, VB>(a, r, t + threadIdx.x, block, carries, counter);
            if (++nb == a.flush_threshold) {  // block-uniform: every thread runs the same tiles
                flush_bank_to_smem<NBANK, L>(counter, s_acc, lane);
                nb = 0;
            }
        }
    } else if constexpr (SCHED == 2) {
        // Warp tiles [0, P) are split statically into contiguous CTA ranges
        // (DRAM locality); inside a CTA, warps claim warp tiles from a shared
        // counter, so no warp idles while another still holds a share.  Warp
        // tiles [P, nwt) form a global pool handed out in chunks of CB, so
        // CTAs on faster SMs absorb the tail.
        constexpr unsigned long long WT = 32ull * VPT;
        const unsigned long long S0 = a.g0 * 32;
        const unsigned long long P = a.nwt - a.pool;
        const unsigned long long lo = P * blockIdx.x / gridDim.x;
        const unsigned long long hi = P * (blockIdx.x + 1) / gridDim.x;
        __shared__ unsigned s_claim;
        if (threadIdx.x == 0) s_claim = 0u;
        __syncthreads();
        unsigned mine = lane == 0 ? atomicAdd(&s_claim, 1u) : 0u;
        unsigned long long w = lo + __shfl_sync(0xFFFFFFFFu, mine, 0);
        mine = lane == 0 ? atomicAdd(&s_claim, 1u) : 0u;  // prefetch
        while (w < hi) {
            const unsigned long long t = S0 + w * WT;
            uint32_t r[REGS];
            load_tree_block<VB, HINT, VPT>(a, t + lane, 32u, t >= a.f0 && t + WT <= a.f1, r);
            consume<MODE, NBANK, L, VB>(a, r, t + lane, 32u, carries, counter);
            if (++nb == a.flush_threshold) {  // warp-uniform
                flush_bank_to_smem<NBANK, L>(counter, s_acc, lane);
                nb = 0;
            }
            w = lo + __shfl_sync(0xFFFFFFFFu, mine, 0);
            mine = lane == 0 ? atomicAdd(&s_claim, 1u) : 0u;
        }
        if (a.pool) {
            pdl_wait_prev();  // the pool counter is shared with the previous launch
            unsigned long long m = lane == 0 ? atomicAdd(a.next, 1ull) : 0ull;
            unsigned long long c = __shfl_sync(0xFFFFFFFFu, m, 0);
            m = lane == 0 ? atomicAdd(a.next, 1ull) : 0ull;
            for (;;) {
                const unsigned long long w0 = P + c * a.CB;
                if (w0 >= a.nwt) break;  // warp-uniform
                const unsigned long long w1 = w0 + a.CB < a.nwt ? w0 + a.CB : a.nwt;
                for (unsigned long long ww = w0; ww < w1; ++ww) {
                    const unsigned long long t = S0 + ww * WT;
                    uint32_t r[REGS];
                    load_tree_block<VB, HINT, VPT>(a, t + lane, 32u, t >= a.f0 && t + WT <= a.f1, r);
                    consume<MODE, NBANK, L, VB>(a, r, t + lane, 32u, carries, counter);
                    if (++nb == a.flush_threshold) {
                        flush_bank_to_smem<NBANK, L>(counter, s_acc, lane);
                        nb = 0;
                    }
                }
                c = __shfl_sync(0xFFFFFFFFu, m, 0);
                m = lane == 0 ? atomicAdd(a.next, 1ull) : 0ull;
            }
        }
    } else {
        constexpr unsigned long long WT = 32ull * VPT;  // vectors per warp tile
        const unsigned long long S0 = a.g0 * 32;
        pdl_wait_prev();
        unsigned long long mine = lane == 0 ? atomicAdd(a.next, 1ull) : 0ull;
        unsigned long long c = __shfl_sync(0xFFFFFFFFu, mine, 0);
        mine = lane == 0 ? atomicAdd(a.next, 1ull) : 0ull;  // prefetch: consumed one chunk later
        for (;;) {
            unsigned long long w0, w1;
            if (c < a.nA) {
                w0 = c * a.CA;
                w1 = w0 + a.CA;
            } else {
                w0 = a.nA * a.CA + (c - a.nA) * a.CB;
                w1 = w0 + a.CB < a.nwt ? w0 + a.CB : a.nwt;
            }
            if (w0 >= a.nwt) break;  // warp-uniform
            for (unsigned long long w = w0; w < w1; ++w) {
                const unsigned long long t = S0 + w * WT;
                uint32_t r[REGS];
                load_tree_block<VB, HINT, VPT>(a, t + lane, 32u, t >= a.f0 && t + WT <= a.f1, r);
                consume<MODE, NBANK, L, VB>(a, r, t + lane, 32u, carries, counter);
                if (++nb == a.flush_threshold) {  // warp-uniform
                    flush_bank_to_smem<NBANK, L>(counter, s_acc, lane);
                    nb = 0;
                }
            }
            c = __shfl_sync(0xFFFFFFFFu, mine, 0);
            mine = lane == 0 ? atomicAdd(a.next, 1ull) : 0ull;
        }
    }
    cta_finish<NBANK, L, MODE>(a, carries, counter, s_acc, &s_last, block, lane);
}

// One warp per array.  Array a spans bytes [data + off[a]*wb, data + off[a+1]*wb);
// it is read as VB-byte vectors from the VB-aligned address at or below its
// start, the first/last vector byte-masked, 32 lanes x VPT vectors per step.
// Warps pull array indices from a global counter (prefetched one array
// ahead), so arrays of any length mix balance across warps and SMs; the last
// CTA re-zeroes the counter and ticket for the next launch.
// SCHED 0: warp w takes arrays w, w + nwarps, ... (strided, no atomics).
// SCHED 1: warps pull runs of `per_grab` consecutive arrays from a global
// counter (prefetched one run ahead).
// (SCHED 2 / 3: segmented_pipe_entry below, software-pipelined; 3 = bounded
// to 2 CTAs/SM, which keeps it at <= 128 registers.)
template <int NBANK, int L, int VB, int SCHED>
__global__ void __launch_bounds__(256) segmented_kernel(const uint8_t* data,
                                                        const unsigned long long* offsets,
                                                        unsigned long long n_arrays, int k,
                                                        uint32_t flush_threshold,
                                                        unsigned long long* out,
                                                        unsigned long long* next,
                                                        unsigned int* ticket, unsigned per_grab) {
    constexpr int REGS = NBANK << L;
    constexpr int RPV = VB / 4;
    constexpr int VPT = REGS / RPV;
    constexpr unsigned long long STEP = 32ull * VPT;
    const uint32_t lane = threadIdx.x & 31u;
    const int wb = k >> 3;
    __shared__ int s_last;

    const unsigned long long warp = (blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x) >> 5;
    const unsigned long long nwarps = (gridDim.x * (unsigned long long)blockDim.x) >> 5;
    unsigned long long mine = 0, run = 0, arr = warp, stop = n_arrays;
    if (SCHED == 1) {
        mine = lane == 0 ? atomicAdd(next, 1ull) : 0ull;
        run = __shfl_sync(0xFFFFFFFFu, mine, 0);
        mine = lane == 0 ? atomicAdd(next, 1ull) : 0ull;
        arr = run * per_grab;
        stop = arr + per_grab < n_arrays ? arr + per_grab : n_arrays;
    }
    for (;;) {
        if (arr >= stop) {
            if (SCHED == 0) break;
            run = __shfl_sync(0xFFFFFFFFu, mine, 0);
            mine = lane == 0 ? atomicAdd(next, 1ull) : 0ull;
            arr = run * per_grab;
            if (arr >= n_arrays) break;
            stop = arr + per_grab < n_arrays ? arr + per_grab : n_arrays;
        }
        const uintptr_t P = (uintptr_t)(data + offsets[arr] * wb);
        const uintptr_t Q = (uintptr_t)(data + offsets[arr + 1] * wb);
        const uintptr_t B = P & ~(uintptr_t)(VB - 1);
        const unsigned long long nv = Q > P ? (Q - B + VB - 1) / VB : 0;
        const int lo = (int)(P - B);
        const int hi = nv ? (int)(Q - (B + (nv - 1) * VB)) : VB;
        const uint8_t* base = (const uint8_t*)B;
        const unsigned long long f0 = lo ? 1 : 0;                    // fully valid vectors [f0, f1)
        const unsigned long long f1 = nv - (nv && hi != VB ? 1 : 0);

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

        for (unsigned long long t = 0; t < nv; t += STEP) {
            uint32_t r[REGS];
            if (t >= f0 && t + STEP <= f1) {  // interior: unpredicated, unmasked
#pragma unroll
                for (int v = 0; v < VPT; ++v) {
                    uint32_t x[RPV];
                    ldg_stream<VB, 0>(base + (t + 32ull * v + lane) * VB, x);
#pragma unroll
                    for (int j = 0; j < RPV; ++j) r[v * RPV + j] = x[j];
                }
            } else {
#pragma unroll
                for (int v = 0; v < VPT; ++v) {
                    const unsigned long long idx = t + 32ull * v + lane;
                    uint32_t x[RPV];
#pragma unroll
                    for (int j = 0; j < RPV; ++j) x[j] = 0;
                    if (idx < nv) {
                        ldg_stream<VB, 0>(base + idx * VB, x);
                        if (idx == 0 || idx + 1 == nv) mask_bytes<VB>(x, idx == 0 ? lo : 0, idx + 1 == nv ? hi : VB);
                    }
#pragma unroll
                    for (int j = 0; j < RPV; ++j) r[v * RPV + j] = x[j];
                }
            }
            tree_block<NBANK, L>(r, carries, counter);
            if (++nb == flush_threshold) {  // warp-uniform: nv is per array
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
        if (NBANK == 2) {  // k == 64: lane c -> positions c and 32 + c
            row[lane] = tot[0];
            row[32 + lane] = tot[NBANK - 1];
        } else {
            unsigned long long t = tot[0];
            for (int w = 16; w >= k; w >>= 1) t += __shfl_down_sync(0xFFFFFFFFu, t, w);
            if ((int)lane < k) row[lane] = t;
        }
        arr += SCHED == 0 ? nwarps : 1;
    }
    if (SCHED == 0) return;
    // Every warp has drawn an index >= n_arrays; once all CTAs are past that
    // point the counter can be reset.
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
        if (s_last) {
            *next = 0ull;
            *ticket = 0u;
        }
    }
}

// Segmented, software-pipelined (SCHED 2): warp w owns arrays w, w + nwarps,
// ... and walks the concatenation of their steps (32 lanes x VPT vectors) with
// a one-step register double buffer: the loads of step s+1 -- possibly the
// first step of the warp's next array, whose offsets were fetched one array
// ahead -- are issued before step s is consumed and before an array's
// epilogue (drain + transpose-reduce + row store), so the memory pipe never
// drains at array boundaries.
struct SegView {
    const uint8_t* base;     // VB-aligned start
    unsigned long long nv;   // vectors
    unsigned long long f0, f1;
    int lo, hi;
};

template <int VB>
__device__ __forceinline__ SegView seg_view(const uint8_t* data, unsigned long long w0, unsigned long long w1, int wb) {
    SegView v;
    const uintptr_t P = (uintptr_t)(data + w0 * wb);
    const uintptr_t Q = (uintptr_t)(data + w1 * wb);
    const uintptr_t B = P & ~(uintptr_t)(VB - 1);
    v.base = (const uint8_t*)B;
    v.nv = Q > P ? (Q - B + VB - 1) / VB : 0;
    v.lo = (int)(P - B);
    v.hi = v.nv ? (int)(Q - (B + (v.nv - 1) * VB)) : VB;
    v.f0 = v.lo ? 1 : 0;
    v.f1 = v.nv - (v.nv && v.hi != VB ? 1 : 0);
    return v;
}

template <int VB, int VPT>
__device__ __forceinline__ void seg_load(const SegView& v, unsigned long long t, uint32_t lane,
                                         uint32_t (&r)[VPT * (VB / 4)]) {
    constexpr int RPV = VB / 4;
    constexpr unsigned long long STEP = 32ull * VPT;
    if (t >= v.f0 && t + STEP <= v.f1) {
#pragma unroll
        for (int q = 0; q < VPT; ++q) {
            uint32_t x[RPV];
            ldg_stream<VB, 0>(v.base + (t + 32ull * q + lane) * VB, x);
#pragma unroll
            for (int j = 0; j < RPV; ++j) r[q * RPV + j] = x[j];
        }
    } else {
#pragma unroll
        for (int q = 0; q < VPT; ++q) {
            const unsigned long long idx = t + 32ull * q + lane;
            uint32_t x[RPV];
#pragma unroll
            for (int j = 0; j < RPV; ++j) x[j] = 0;
            if (idx < v.nv) {
                ldg_stream<VB, 0>(v.base + idx * VB, x);
                if (idx == 0 || idx + 1 == v.nv) mask_bytes<VB>(x, idx == 0 ? v.lo : 0, idx + 1 == v.nv ? v.hi : VB);
            }
#pragma unroll
            for (int j = 0; j < RPV; ++j) r[q * RPV + j] = x[j];
        }
    }
}

template <int NBANK>
__device__ __forceinline__ void seg_store_row(unsigned long long* out, unsigned long long arr, int k, uint32_t lane,
                                              const unsigned long long (&tot)[NBANK]) {
    unsigned long long* row = out + arr * (unsigned long long)k;
    if (NBANK == 2) {
        row[lane] = tot[0];
        row[32 + lane] = tot[NBANK - 1];
    } else {
        unsigned long long t = tot[0];
        for (int w = 16; w >= k; w >>= 1) t += __shfl_down_sync(0xFFFFFFFFu, t, w);
        if ((int)lane < k) row[lane] = t;
    }
}

template <int NBANK, int L, int VB>
__device__ __forceinline__ void segmented_pipe_body(const uint8_t* data, const unsigned long long* offsets,
                                                    unsigned long long n_arrays, int k, uint32_t flush_threshold,
                                                    unsigned long long* out) {
    constexpr int REGS = NBANK << L;
    constexpr int RPV = VB / 4;
    constexpr int VPT = REGS / RPV;
    constexpr unsigned long long STEP = 32ull * VPT;
    const uint32_t lane = threadIdx.x & 31u;
    const unsigned long long nwarps = (gridDim.x * (unsigned long long)blockDim.x) >> 5;
    const int wb = k >> 3;

    // Current array: skip (and zero) empty arrays.
    unsigned long long arr = (blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x) >> 5;
    SegView cur;
    for (;; arr += nwarps) {
        if (arr >= n_arrays) return;
        cur = seg_view<VB>(data, offsets[arr], offsets[arr + 1], wb);
        if (cur.nv) break;
        unsigned long long z[NBANK];
#pragma unroll
        for (int b = 0; b < NBANK; ++b) z[b] = 0;
        seg_store_row<NBANK>(out, arr, k, lane, z);
    }
    // Offsets of the warp's next array, fetched one array ahead.
    unsigned long long nxt_w0 = 0, nxt_w1 = 0;
    if (arr + nwarps < n_arrays) {
        nxt_w0 = offsets[arr + nwarps];
        nxt_w1 = offsets[arr + nwarps + 1];
    }

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

    unsigned long long t = 0;
    uint32_t rc[REGS];
    seg_load<VB, VPT>(cur, t, lane, rc);
    for (;;) {
        // Where the next step is: later in this array, or the next non-empty array.
        unsigned long long t_n = t + STEP, arr_n = arr;
        SegView nxt = cur;
        bool have_next = true;
        if (t_n >= cur.nv) {
            t_n = 0;
            arr_n = arr + nwarps;
            have_next = false;
            while (arr_n < n_arrays) {
                nxt = seg_view<VB>(data, nxt_w0, nxt_w1, wb);
                if (arr_n + nwarps < n_arrays) {  // prefetch the offsets after that
                    nxt_w0 = offsets[arr_n + nwarps];
                    nxt_w1 = offsets[arr_n + nwarps + 1];
                }
                if (nxt.nv) {
                    have_next = true;
                    break;
                }
                unsigned long long z[NBANK];
#pragma unroll
                for (int b = 0; b < NBANK; ++b) z[b] = 0;
                seg_store_row<NBANK>(out, arr_n, k, lane, z);
                arr_n += nwarps;
            }
        }
        uint32_t rn[REGS];
        if (have_next) seg_load<VB, VPT>(nxt, t_n, lane, rn);

        tree_block<NBANK, L>(rc, carries, counter);
        if (++nb == flush_threshold) {
            uint32_t d[16];
#pragma unroll
            for (int p = 0; p < 16; ++p) d[p] = 0;
#pragma unroll
            for (int b = 0; b < NBANK; ++b) tot[b] += bank_warp_total(counter[b], L, d);
            zero_bank<NBANK>(counter);
            nb = 0;
        }
        if (t + STEP >= cur.nv) {  // last step of this array: epilogue while rn is in flight
#pragma unroll
            for (int b = 0; b < NBANK; ++b) {
                uint32_t d[16];
                drain<L>(d, carries[b]);
                tot[b] += bank_warp_total(counter[b], L, d);
#pragma unroll
                for (int j = 0; j < L; ++j) carries[b][j] = 0;
            }
            zero_bank<NBANK>(counter);
            nb = 0;
            seg_store_row<NBANK>(out, arr, k, lane, tot);
#pragma unroll
            for (int b = 0; b < NBANK; ++b) tot[b] = 0;
        }
        if (!have_next) break;
#pragma unroll
        for (int i = 0; i < REGS; ++i) rc[i] = rn[i];
        cur = nxt;
        arr = arr_n;
        t = t_n;
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
            case 7:  // SAM FLAG words: the 12 defined bits uniform, bits 12-15 clear
                ((uint16_t*)out)[l] = (uint16_t)((mix64(key + ((i >> 2) + 1) * kGamma) >> (16 * (i & 3))) & 0x0FFF);
                break;
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

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------

constexpr int kDefaultBlock = 256;
constexpr int kDefaultDepth1 = 7;  // k = 8/16/32: 128 registers = 512 B per thread per tree block
constexpr int kDefaultDepth2 = 6;  // k = 64: two banks of 64 registers

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
    // The occupancy query costs microseconds; cache it per (device, kernel, block).
    struct Key {
        int dev;
        const void* fn;
        int block;
        bool operator<(const Key& o) const {
            return dev != o.dev ? dev < o.dev : fn != o.fn ? fn < o.fn : block < o.block;
        }
    };
    static thread_local std::map<Key, int> cache;
    int dev = 0;
    cudaGetDevice(&dev);
    const Key key{dev, reinterpret_cast<const void*>(kernel), block};
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, block, 0) != cudaSuccess || n < 1) n = 1;
    cache[key] = n;
    return n;
}

using StreamKernel = void (*)(const StreamArgs);

struct StreamVariant {
    int nbank, depth, vb, hint, block, sched, mode;
    StreamKernel fn;
};

#define SV(NB, L, VB, H, B, S) {NB, L, VB, H, B, S, 0, stream_kernel<NB, L, VB, H, B, S, 0>}
#define SVF(L, VB, B, S) {2, L, VB, 0, B, S, 1, stream_kernel<2, L, VB, 0, B, S, 1>}
// FLAG variants that must fit 2 CTAs/SM (<= 128 registers); hint slot = 2 marks them.
#define SVF2(L, VB, B, S) {2, L, VB, 2, B, S, 1, stream_kernel<2, L, VB, 0, B, S, 1, 2>}
// Production variants first (the defaults), then tuning variants selectable
// through POSPOP_STREAM_VARIANT="depth,vb,hint,block,sched" (POSPOP_FLAG_VARIANT
// for MODE 1).
const StreamVariant kStreamVariants[] = {
    SV(1, 7, 32, 0, 256, 2), SV(2, 6, 32, 0, 256, 2),  // defaults (k <= 32 / k = 64)
    SV(1, 7, 32, 0, 0, 2), SV(2, 6, 32, 0, 0, 2),      // runtime block size (test launches)
    SV(1, 7, 32, 0, 256, 0), SV(2, 6, 32, 0, 256, 0),  // static CTA partition
    SV(1, 7, 32, 0, 0, 0), SV(2, 6, 32, 0, 0, 0),
    SV(1, 7, 32, 0, 256, 1), SV(2, 6, 32, 0, 256, 1),  // per-warp guided chunks
    SV(1, 7, 32, 0, 0, 1), SV(2, 6, 32, 0, 0, 1), SV(1, 6, 32, 0, 256, 2), SV(1, 7, 16, 0, 256, 2),
    SVF(5, 32, 512, 2), SVF(5, 32, 0, 2),               // FLAG statistics defaults (16 warps/SM)
    SVF(6, 32, 256, 2),
    SVF(5, 32, 256, 2), SVF(6, 16, 256, 2), SVF(7, 32, 256, 2),
    SVF2(5, 32, 256, 2), SVF2(5, 16, 256, 2), SVF2(4, 32, 256, 2), SVF(4, 32, 512, 2), SVF(5, 16, 512, 2),
};
#undef SV
#undef SVF
#undef SVF2

const StreamVariant* pick_stream(int nbank, int depth, int vb, int hint, int block, int sched, int mode) {
    for (const StreamVariant& v : kStreamVariants)
        if (v.nbank == nbank && v.depth == depth && v.vb == vb && v.hint == hint && v.block == block &&
            v.sched == sched && v.mode == mode)
            return &v;
    return nullptr;
}

using SegKernel = void (*)(const uint8_t*, const unsigned long long*, unsigned long long, int, uint32_t,
                           unsigned long long*, unsigned long long*, unsigned int*, unsigned);

struct SegVariant {
    int nbank, depth, vb, sched;
    SegKernel fn;
};

template <int NBANK, int L, int VB, int MINB = 1>
__global__ void __launch_bounds__(256, MINB) segmented_pipe_entry(const uint8_t* data, const unsigned long long* offsets,
                                                            unsigned long long n, int k, uint32_t thr,
                                                            unsigned long long* out, unsigned long long*,
                                                            unsigned int*, unsigned) {
    segmented_pipe_body<NBANK, L, VB>(data, offsets, n, k, thr, out);
}

#define SG(NB, L, VB, S) {NB, L, VB, S, segmented_kernel<NB, L, VB, S>}
#define SGP(NB, L, VB) {NB, L, VB, 2, segmented_pipe_entry<NB, L, VB>}
#define SGP2(NB, L, VB) {NB, L, VB, 3, segmented_pipe_entry<NB, L, VB, 2>}  // sched 3: pipelined, 2 CTAs/SM
const SegVariant kSegVariants[] = {
    SG(1, 5, 16, 0), SG(2, 5, 16, 1),  // defaults (k <= 32 / k = 64)
    SG(1, 5, 16, 1), SG(2, 5, 16, 0), SG(1, 4, 16, 0), SG(1, 4, 16, 1), SG(1, 5, 32, 0), SG(1, 5, 32, 1),
    SG(2, 4, 16, 0), SG(2, 4, 16, 1), SG(2, 4, 32, 1),
    SGP(1, 5, 16), SGP(1, 4, 16), SGP(1, 4, 32), SGP(1, 5, 32), SGP(2, 4, 16), SGP(2, 3, 32), SGP(2, 4, 32),
    SGP2(2, 4, 16), SGP2(2, 3, 32), SGP2(2, 3, 16), SGP2(1, 5, 16), SGP2(1, 5, 32),
};
#undef SGP2
#undef SG
#undef SGP

const SegVariant* pick_segmented(int nbank, int depth, int vb, int sched) {
    for (const SegVariant& v : kSegVariants)
        if (v.nbank == nbank && v.depth == depth && v.vb == vb && v.sched == sched) return &v;
    return nullptr;
}

}  // namespace

unsigned long long kernel_launches() { return g_launches.load(); }

static cudaError_t launch_stream_mode(int mode, int k, const void* data, size_t len_words,
                                      unsigned long long* d_out, bool accumulate, const LaunchOptions& opt,
                                      const StreamWorkspace& ws, cudaStream_t stream, int* grid_used) {
    const int nbank = (k == 64 || mode == 1) ? 2 : 1;
    // Tuning override: POSPOP_STREAM_VARIANT / POSPOP_FLAG_VARIANT="depth,vb,hint,block,sched".
    int depth = mode == 1 ? 5 : (nbank == 1 ? kDefaultDepth1 : kDefaultDepth2), vb = 32, hint = 0,
        block = mode == 1 ? 512 : kDefaultBlock, sched = 2;
    if (const char* v = std::getenv(mode == 1 ? "POSPOP_FLAG_VARIANT" : "POSPOP_STREAM_VARIANT"))
        std::sscanf(v, "%d,%d,%d,%d,%d", &depth, &vb, &hint, &block, &sched);
    if (opt.depth) depth = opt.depth;
    if (opt.block) block = 0;  // explicit (test) block size: the runtime-block instantiation
    const StreamVariant* var = pick_stream(nbank, depth, vb, hint, block, sched, mode);
    if (!var) var = pick_stream(nbank, depth, vb, 0, 0, sched, mode);
    if (!var) return cudaErrorInvalidConfiguration;
    const int threads = var->block ? var->block : (opt.block ? opt.block : kDefaultBlock);
    const int vpt = (mode == 1 ? (1 << var->depth) : (nbank << var->depth)) / (var->vb / 4);

    const uintptr_t P = reinterpret_cast<uintptr_t>(data);
    const size_t nbytes = len_words * (size_t)(k / 8);
    const uintptr_t VBu = (uintptr_t)var->vb;
    const uintptr_t group = 32 * VBu;
    StreamArgs a;
    a.base = reinterpret_cast<const uint8_t*>(P & ~(group - 1));
    if (nbytes == 0) {
        a.v0 = a.v1 = a.f0 = a.f1 = a.g0 = a.ng = 0;
        a.lo_byte = 0;
        a.hi_byte = (int)VBu;
    } else {
        const uintptr_t B = reinterpret_cast<uintptr_t>(a.base);
        a.v0 = (P - B) / VBu;
        a.v1 = (P + nbytes - B + VBu - 1) / VBu;
        a.lo_byte = (int)(P - (B + a.v0 * VBu));
        a.hi_byte = (int)(P + nbytes - (B + (a.v1 - 1) * VBu));
        a.f0 = a.v0 + (a.lo_byte != 0 ? 1 : 0);
        a.f1 = a.v1 - (a.hi_byte != (int)VBu ? 1 : 0);
        a.g0 = a.v0 / 32;
        a.ng = (a.v1 + 31) / 32 - a.g0;
    }
    a.k = k;
    a.flush_threshold = opt.flush_threshold;
    a.acc = ws.acc;
    a.ticket = ws.ticket;
    a.out = d_out;
    a.accumulate = accumulate ? 1 : 0;
    a.trace = opt.trace;
    a.next = ws.next;
    a.bad = ws.bad;
    a.word_base = opt.word_base;
    a.data_off = nbytes ? (unsigned long long)(P - reinterpret_cast<uintptr_t>(a.base)) : 0ull;

    int grid = opt.grid;
    if (grid <= 0) {
        const unsigned long long tile = (unsigned long long)vpt * threads;
        const unsigned long long want = (a.ng * 32 + tile - 1) / tile;
        const int per_sm = env_int("POSPOP_BLOCKS_PER_SM", resident_blocks(var->fn, threads));
        const unsigned long long cap = (unsigned long long)device_info().sms * per_sm;
        grid = (int)(want < 1 ? 1 : (want < cap ? want : cap));
    }
    // Dynamic schedule: nwt warp tiles; the last ~tail_per_warp warp tiles per
    // warp go out in small chunks of CB, everything before in chunks of CA.
    const unsigned long long wt = 32ull * vpt;
    a.nwt = a.ng ? (a.v1 - a.g0 * 32 + wt - 1) / wt : 0;
    a.CA = (unsigned long long)env_int("POSPOP_CHUNK_A", 16);
    a.CB = (unsigned long long)env_int("POSPOP_CHUNK_B", 2);
    if (a.CA < 1) a.CA = 1;
    if (a.CB < 1) a.CB = 1;
    const unsigned long long warps = (unsigned long long)grid * (threads / 32);
    unsigned long long tail = warps * (unsigned long long)env_int("POSPOP_TAIL_TILES_PER_WARP", 8);
    if (tail > a.nwt) tail = a.nwt;
    a.nA = (a.nwt - tail) / a.CA;
    // SCHED 2: the global tail pool, in warp tiles.
    a.pool = warps * (unsigned long long)env_int("POSPOP_POOL_TILES_PER_WARP", 16);
    if (a.pool > a.nwt) a.pool = a.nwt;

    if (grid_used) *grid_used = grid;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3((unsigned)threads);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = env_int("POSPOP_PDL", 1) ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, var->fn, a);
    ++g_launches;
    return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_stream(int k, const void* data, size_t len_words, unsigned long long* d_out,
                          bool accumulate, const LaunchOptions& opt, const StreamWorkspace& ws,
                          cudaStream_t stream, int* grid_used) {
    return launch_stream_mode(0, k, data, len_words, d_out, accumulate, opt, ws, stream, grid_used);
}

cudaError_t launch_flagstats(const uint16_t* flags, size_t len, unsigned long long* d_out33, bool accumulate,
                             const LaunchOptions& opt, const StreamWorkspace& ws, cudaStream_t stream) {
    return launch_stream_mode(1, 16, flags, len, d_out33, accumulate, opt, ws, stream, nullptr);
}

cudaError_t launch_segmented(int k, const void* data, const unsigned long long* d_offsets, size_t n,
                             unsigned long long* d_out, const LaunchOptions& opt, const StreamWorkspace& ws,
                             cudaStream_t stream) {
    if (n == 0) return cudaSuccess;
    const int nbank = k == 64 ? 2 : 1;
    // Tuning override: POSPOP_SEG_VARIANT="depth,vb,sched".
    // measured: pipelined with 2 CTAs/SM (k <= 32), dynamic claiming (k = 64)
    int depth = 5, vb = 16, sched = nbank == 1 ? 3 : 1;
    if (const char* v = std::getenv("POSPOP_SEG_VARIANT")) std::sscanf(v, "%d,%d,%d", &depth, &vb, &sched);
    if (opt.depth) depth = opt.depth;
    const SegVariant* var = pick_segmented(nbank, depth, vb, sched);
    if (!var) var = pick_segmented(nbank, 5, 16, nbank == 1 ? 3 : 1);
    const int block = opt.block ? opt.block : env_int("POSPOP_SEG_BLOCK", kDefaultBlock);
    int grid = opt.grid;
    if (grid <= 0) {
        const unsigned long long warps_per_block = block / 32;
        const unsigned long long want = (n + warps_per_block - 1) / warps_per_block;
        // measured (r01 sweep): 4 CTAs/SM for the strided schedule, one resident wave otherwise
        const int per_sm = env_int("POSPOP_SEG_BLOCKS_PER_SM", var->sched == 0 ? 4 : resident_blocks(var->fn, block));
        const unsigned long long cap = (unsigned long long)device_info().sms * per_sm;
        grid = (int)(want < cap ? want : cap);
    }
    const unsigned per_grab = (unsigned)env_int("POSPOP_SEG_PER_GRAB", 1);
    var->fn<<<grid, block, 0, stream>>>(static_cast<const uint8_t*>(data), d_offsets, n, k,
                                        opt.flush_threshold, d_out, ws.next, ws.ticket,
                                        per_grab < 1 ? 1u : per_grab);
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

cudaError_t launch_microop(int op, int depth, const uint32_t* d_in, size_t n, uint32_t* d_out, cudaStream_t stream) {
    microop_kernel<<<1, 32, 0, stream>>>(op, depth, d_in, n, d_out);
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
