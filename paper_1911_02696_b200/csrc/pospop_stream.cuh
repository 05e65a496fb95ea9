// pospop_stream.cuh -- the stream kernel family (k = 8/16/32/64 counts and the fused FLAG-statistics
// mode): vector addressing, tree blocks, work distribution, CTA epilogue.
// Device code only; included by pospop_kernels.cu (the single CUDA translation
// unit, which instantiates the kernels and owns the host-side launchers).
#pragma once

#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "pospop_device.cuh"
#include "pospop_exchange.h"

namespace pospop_b200 {
namespace dev {

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
    // Fused exchange (MODE 0): the last CTA also stores out[k] as row `rank`
    // of slot xstep % xslots in every rank's exchange buffer peers[j] (peer
    // memory mapped through CUDA IPC; plain stores over NVLink), j < n_peers,
    // then release-stores the row's step tag (pospop_exchange.h).
    unsigned long long* const* peers;
    int n_peers, rank;
    unsigned long long xstep;
    int xslots;
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

// System-scope accesses for the cross-GPU exchange (peer memory over NVLink).
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Producer half of the exchange, in two parts, run by the counting kernel's
// last CTA once out[k] is final.  (1) Credit: before rewriting slot step % S
// in peer j's buffer, thread j waits (bounded) until j's reducer has consumed
// the slot's previous step, step - S.  (2) The CTA stores its k counts `vals`
// (shared memory) as row `rank` in every peer's slot, fences, and each thread
// j < n release-stores the row's tag step + 1 in peer j.  A timeout sets
// error 1 in the rank's own buffer and publishes anyway (the host reports it).
__device__ __forceinline__ void xchg_wait_credit(unsigned long long* const* peers, int n, int rank, int S,
                                                 unsigned long long step) {
    if ((int)threadIdx.x < n && step >= (unsigned long long)S) {
        const unsigned long long need = step - S + 1;
        const unsigned long long t0 = globaltimer();
        while (ld_acquire_sys(peers[threadIdx.x]) < need) {
            if (globaltimer() - t0 > kXTimeoutNs) {
                peers[rank][1] = 1ull;
                break;
            }
            __nanosleep(256);
        }
    }
}

__device__ __forceinline__ void xchg_store_rows(unsigned long long* const* peers, int n, int rank, int k, int S,
                                                unsigned long long step, const unsigned long long* vals,
                                                unsigned nthreads) {
    const size_t so = xslot_off((unsigned)(step % (unsigned long long)S), n, k);
    for (int i = threadIdx.x; i < n * k; i += nthreads) {
        const int j = i / k, pos = i - j * k;
        peers[j][so + n + (size_t)rank * k + pos] = vals[pos];
    }
    __threadfence_system();
    __syncthreads();
    if ((int)threadIdx.x < n) st_release_sys(peers[threadIdx.x] + so + rank, step + 1);
}

// Consumer half: waits (bounded) for the n tags of `step` in this rank's own
// buffer, sums the n rows into out[k] (merge_counts, pospop.cpp:33-37), then
// release-stores "consumed = step + 1" so the producers may reuse the slot.
// `before_out` runs between the wait and the stores to out (the reduce kernel
// waits there for the stream's previous kernel).
template <class BeforeOut>
__device__ __forceinline__ void xchg_reduce(unsigned long long* own, int n, int k, int S, unsigned long long step,
                                            unsigned long long* out, BeforeOut before_out) {
    const size_t so = xslot_off((unsigned)(step % (unsigned long long)S), n, k);
    if ((int)threadIdx.x < n) {
        const unsigned long long t0 = globaltimer();
        while (ld_acquire_sys(own + so + threadIdx.x) != step + 1) {
            if (globaltimer() - t0 > kXTimeoutNs) {
                own[1] = 2ull;
                break;
            }
            __nanosleep(128);
        }
    }
    __syncthreads();
    before_out();
    for (int pos = threadIdx.x; pos < k; pos += blockDim.x) {
        unsigned long long sum = 0;
        for (int j = 0; j < n; ++j) sum += ld_relaxed_sys(own + so + n + (size_t)j * k + pos);
        out[pos] = sum;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        st_release_sys(own, step + 1);
    }
}

// Channel -> position fold: the channels (of 32 * NBANK) that count position
// p are p + m * k for m = 0 .. 32/k - 1 (k <= 32), or channel p (k = 64).
__device__ __forceinline__ int channels_per_position(int k) { return k >= 32 ? 1 : 32 / k; }

// Byte-frame FLAG mode with shallow trees (L <= 4): two consecutive tiles are
// joined by one more CSA level, so the byte-lane extract runs once per pair.
// (At L = 5 the two extra carry words per bank cost more in spills than the
// halved extract saves.)
template <int MODE, int L>
__host__ __device__ constexpr bool pair_tiles() { return MODE == 2 && L <= 4; }

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
            POSPOP_CHECK(first + (unsigned long long)v * stride >= a.v0 &&
                         first + (unsigned long long)v * stride < a.v1);
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
template <int NBANK, int L, int MODE = 0>
__device__ __forceinline__ void flush_bank_to_smem(uint32_t (&counter)[NBANK][16], unsigned long long* s_acc,
                                                   uint32_t lane) {
    uint32_t d[16];
#pragma unroll
    for (int p = 0; p < 16; ++p) d[p] = 0;
#pragma unroll
    for (int b = 0; b < NBANK; ++b) {
        // paired tiles extract once per pair: weight 2^(L+1)
        constexpr int W = pair_tiles<MODE, L>() ? L + 1 : L;
        const uint32_t tot = MODE == 2 ? bank_warp_total_bytes(counter[b], W, d) : bank_warp_total(counter[b], W, d);
        if (tot) atomicAdd(&s_acc[b * 32 + lane], (unsigned long long)tot);
    }
    zero_bank<NBANK>(counter);
}

// CTA epilogue: final flush fused with the carry drain, CTA channel totals to
// the global accumulator, ticket; the last CTA folds channels to positions,
// writes/accumulates out[k] and leaves the scratch (acc, ticket, chunk
// counter) zeroed for the next launch.
template <int NBANK, int L, int MODE, int CD>
__device__ __forceinline__ void cta_finish(const StreamArgs& a, uint32_t (&carries)[NBANK][CD],
                                           uint32_t (&counter)[NBANK][16], unsigned long long* s_acc,
                                           int* s_last, unsigned block, uint32_t lane) {
    if (a.trace && threadIdx.x == 0) a.trace[blockIdx.x * 5 + 1] = globaltimer();
    pdl_wait_prev();  // the previous launch on this stream owns acc/ticket/next until it completes
    if constexpr (pair_tiles<MODE, L>()) {  // fold a pending (unpaired) top into level L
#pragma unroll
        for (int b = 0; b < NBANK; ++b) {
            extract_bytes(counter[b], carries[b][L] & carries[b][L + 1]);
            carries[b][L] ^= carries[b][L + 1];
        }
    }
#pragma unroll
    for (int b = 0; b < NBANK; ++b) {
        uint32_t d[16];
        constexpr int W = pair_tiles<MODE, L>() ? L + 1 : L;  // carry levels / counter weight 2^W
        drain<W>(d, carries[b]);
        const uint32_t tot = MODE == 2 ? bank_warp_total_bytes(counter[b], W, d) : bank_warp_total(counter[b], W, d);
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
    if constexpr (MODE == 2) {
        // Byte-frame banks: stat j of bank b = sum of channels 8i + j.  Written
        // in MODE 1's layout (flag_transform positions, flagstats.cpp:39-49):
        // out[p] all reads, out[16 + p] QC-fail reads.
        for (int c = threadIdx.x; c < 96; c += block) {  // see the MODE 0 branch
            s_acc[c] = __ldcg(&a.acc[c]);
            __stcg(&a.acc[c], 0ull);
        }
        __syncthreads();
        for (int pos = threadIdx.x; pos < 32; pos += block) {
            const int f = pos >> 4, p = pos & 15;
            auto stat = [&](int b, int j) {
                return s_acc[32 * b + j] + s_acc[32 * b + 8 + j] + s_acc[32 * b + 16 + j] + s_acc[32 * b + 24 + j];
            };
            unsigned long long v = 0;
            if (p == 1 || p == 2 || p == 3 || p == 6 || p == 7) v = stat(f, p);
            else if (p >= 8 && p <= 11) v = stat(2, p - 8 + 4 * f);
            else if (p == 12) v = stat(f, 0) - stat(f, 3);  // pair_map = GU - GU & mate_unmapped
            a.out[pos] = a.accumulate ? a.out[pos] + v : v;
        }
        if (threadIdx.x == 0) {
            const unsigned long long code = atomicExch(a.bad, 0ull);
            a.out[32] = a.accumulate && a.out[32] > code ? a.out[32] : code;
        }
    } else if constexpr (MODE == 1) {  // two banks of k = 16: out[16 b + p] = acc[32 b + p] + acc[32 b + p + 16]
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
        // Channel totals: one L2 load per channel, all in parallel (the other
        // CTAs' atomics were fenced before their tickets), then re-zeroed with
        // plain stores -- the next launch on the stream touches acc only after
        // griddepcontrol.wait, i.e. after this launch completed.
        for (int c = threadIdx.x; c < 32 * NBANK; c += block) {
            s_acc[c] = __ldcg(&a.acc[c]);
            __stcg(&a.acc[c], 0ull);
        }
        __syncthreads();
        for (int pos = threadIdx.x; pos < k; pos += block) {
            unsigned long long sum = 0;
            if (k == 64) {
                sum = s_acc[pos];
            } else {
                const int m = channels_per_position(k);
                for (int j = 0; j < m; ++j) sum += s_acc[pos + j * k];
            }
            if (a.accumulate) sum += a.out[pos];
            a.out[pos] = sum;
            if (a.n_peers) s_acc[pos] = sum;
        }
        if (a.n_peers) {
            xchg_wait_credit(a.peers, a.n_peers, a.rank, a.xslots, a.xstep);
            __syncthreads();
            xchg_store_rows(a.peers, a.n_peers, a.rank, k, a.xslots, a.xstep, s_acc, block);
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

// Two Harley-Seal trees fed from one register tile through flag_transform2:
// each leaf transforms its two inputs and immediately feeds both trees, so
// the transformed planes never exist as whole arrays (fewer live registers,
// more warps per SM for this latency-bound kernel).  Same CSA sequence per
// tree as Tree<L> over the transformed arrays.
template <int L>
struct FlagDualTree {
    static __device__ __forceinline__ void run(uint32_t* ca, uint32_t* cf, const uint32_t* in, uint32_t& top_a,
                                               uint32_t& top_f) {
        uint32_t h, l;
        if constexpr (L == 1) {
            uint32_t a0, f0, a1, f1;
            flag_transform2(in[0], a0, f0);
            flag_transform2(in[1], a1, f1);
            csa(h, l, ca[0], a0, a1);
            ca[0] = l;
            top_a = h;
            csa(h, l, cf[0], f0, f1);
            cf[0] = l;
            top_f = h;
        } else {
            uint32_t a0, f0, a1, f1;
            FlagDualTree<L - 1>::run(ca, cf, in, a0, f0);
            FlagDualTree<L - 1>::run(ca, cf, in + (1 << (L - 1)), a1, f1);
            csa(h, l, ca[L - 1], a0, a1);
            ca[L - 1] = l;
            top_a = h;
            csa(h, l, cf[L - 1], f0, f1);
            cf[L - 1] = l;
            top_f = h;
        }
    }
};

// ---------------------------------------------------------------------------
// FLAG statistics, byte-frame form (MODE 2, the default).  A leaf takes two
// registers = four FLAG words and regroups them with two PRMTs into
//   Lb = the four low bytes (bits 0-7: paired .. read2)
//   Hb = the four high bytes (bits 8-15: secondary, qcfail, dup, supplementary, reserved)
// so every SWAR operation below works on four words at once (8-bit lanes)
// instead of two.  Three planes leave the leaf, each counted by its own
// Harley-Seal tree (bank 0/1/2); per byte lane:
//   AL  bit 0 GU, 1 GU&proper, 2 unmapped, 3 GU&mate_unmapped, 6 G&read1, 7 G&read2
//   FL  = AL of QC-fail reads
//   AHF bits 0-3 secondary, qcfail, dup, supplementary&!secondary; bits 4-7 the
//       same for QC-fail reads (AH << 4 under the QC-fail mask)
// with G = paired & !secondary & !supplementary and GU = G & !unmapped, so
// pair_map = GU - GU&mate_unmapped (flagstats.cpp:84).  G/GU are formed at bit 0
// of each byte and multiplied into their target bits (no carries: g, gu are
// 0/1 per byte); the QC-fail byte mask is PRMT's sign-replicate of bit 9
// moved to each byte's msb.  Bits 4,5 of AL are don't-care (never read).
// Reserved bits 12-15 sit in Hb's high nibbles, so `bad |= Hb` tracks them.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
    return d;
}

// Plane sets (P): 0 = all three planes (AL, FL, AHF -> banks 0, 1, 2);
// 1 = the QC-fail-free tile (AL, AH -> banks 0, 2: FL and the fail half of AHF
// are zero); 2 = the fail planes only (FL, AH<<4 & mf -> banks 1, 2), added
// to a tile first counted with P = 1.  AHF = AH | (AH<<4 & mf) has disjoint
// halves, so counting them in two passes gives the same positional counts.
template <int P>
struct FlagPlanes {
    static constexpr int N = P == 0 ? 3 : 2;
    static __device__ __forceinline__ int bank(int i) { return P == 0 ? i : P == 1 ? (i == 0 ? 0 : 2) : (i == 0 ? 1 : 2); }
};

template <int P>
__device__ __forceinline__ void flag_leaf(uint32_t r0, uint32_t r1, uint32_t (&o)[FlagPlanes<P>::N], uint32_t& hb) {
    constexpr uint32_t B1 = 0x01010101u;
    const uint32_t lb = prmt(r0, r1, 0x6420u);
    hb = prmt(r0, r1, 0x7531u);
    const uint32_t g = lb & ~hb & ~shr_fma<3>(hb) & B1;        // paired & !secondary & !supplementary
    const uint32_t gu = g & ~shr_fma<2>(lb);                    // ... & !unmapped
    const uint32_t t = g * 0xC0u + gu * 0x0Bu;                  // G -> bits 6,7 ; GU -> bits 0,1,3
    const uint32_t al = lb & (t | 0x04040404u);
    const uint32_t ah = hb & ~(shl_fma<3>(hb) & 0x08080808u);  // bit 3: supplementary & !secondary
    if constexpr (P == 1) {
        o[0] = al;
        o[1] = ah;
    } else {
        const uint32_t mf = prmt(shl_fma<6>(hb), 0u, 0xBA98u);  // 0xFF per QC-fail byte
        if constexpr (P == 0) {
            o[0] = al;
            o[1] = al & mf;
            o[2] = ah | (shl_fma<4>(ah) & mf);
        } else {
            o[0] = al & mf;
            o[1] = shl_fma<4>(ah) & mf;
        }
    }
}

template <int CD, int L, int P = 0>
struct FlagByteTree {  // 2^L leaves = 2^(L+1) input registers; c[b][j] = carry of weight 2^j
    static constexpr int N = FlagPlanes<P>::N;
    static __device__ __forceinline__ void run(uint32_t (&c)[3][CD], const uint32_t* in, uint32_t (&top)[N],
                                               uint32_t& bad) {
        uint32_t x[N], y[N];
        if constexpr (L == 1) {
            uint32_t hx, hy;
            flag_leaf<P>(in[0], in[1], x, hx);
            flag_leaf<P>(in[2], in[3], y, hy);
            bad = bad | hx | hy;  // one LOP3 per two leaves
        } else {
            FlagByteTree<CD, L - 1, P>::run(c, in, x, bad);
            FlagByteTree<CD, L - 1, P>::run(c, in + (2 << (L - 1)), y, bad);
        }
#pragma unroll
        for (int i = 0; i < N; ++i) {
            const int b = FlagPlanes<P>::bank(i);
            uint32_t h, l;
            csa(h, l, c[b][L - 1], x[i], y[i]);
            c[b][L - 1] = l;
            top[i] = h;
        }
    }
};

// Rare path: this thread's tile holds a FLAG word with reserved bits 12-15
// set; report the smallest such word index through a.bad (max of ~index).
// Fully unrolled: a runtime index into r[] would force the whole tile through
// local memory on the hot path.
template <int REGS, int RPV, int VB>
__device__ __forceinline__ void flag_locate_bad(const StreamArgs& a, const uint32_t (&r)[REGS], unsigned long long first,
                                             unsigned stride) {
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

// The rare reserved-bit path.  CANON: r[] holds the tile in the canonical
// register order (vector v of the lane at r[v * RPV ..]); otherwise (the ring
// kernel reads its tile from shared memory with swizzled halves) the tile is
// reloaded from global memory first.
template <bool CANON, int REGS, int RPV, int VB>
__device__ __forceinline__ void locate_bad(const StreamArgs& a, const uint32_t (&r)[REGS], unsigned long long first,
                                           unsigned stride) {
    if constexpr (CANON) {
        flag_locate_bad<REGS, RPV, VB>(a, r, first, stride);
    } else {
        uint32_t rc[REGS];
        load_tree_block<VB, 0, REGS / RPV>(a, first, stride, false, rc);
        flag_locate_bad<REGS, RPV, VB>(a, rc, first, stride);
    }
}

// Tree-block consumer.  MODE 0: positional counts of the words (NBANK banks).
// MODE 2: byte-frame FLAG statistics (three banks, see flag_leaf).
// MODE 1: FLAG statistics -- transform, then bank 0 counts the transformed
// words of all reads and bank 1 those of QC-fail reads; words with reserved bits 12-15 set are
// reported through a.bad (the first such index wins, as the reference's
// check_reserved throws at the first one, flagstats.cpp:34-36).
// CANON: see locate_bad.
template <int MODE, int NBANK, int L, int VB, bool CANON = true, int REGS, int CD>
__device__ __forceinline__ void consume(const StreamArgs& a, const uint32_t (&r)[REGS], unsigned long long first,
                                        unsigned stride, uint32_t (&carries)[NBANK][CD],
                                        uint32_t (&counter)[NBANK][16], uint32_t& phase) {
    if constexpr (MODE == 0) {
        tree_block<NBANK, L>(r, carries, counter);
    } else if constexpr (MODE == 2) {
        static_assert(NBANK == 3 && REGS == (2 << L), "byte-frame FLAG mode: three banks, 2^(L+1) registers");
        constexpr int RPV = VB / 4;
        if constexpr (!pair_tiles<MODE, L>()) {
            // `phase` predicts whether this warp's tile has QC-fail reads:
            // 0 = expect them (all three planes), 1/2 = expect none (AL and
            // AH only; if a QC-fail word shows up after all -- bit 9 = bit 1
            // of Hb -- reload the tile, an L2 hit, and add the fail planes).
            // Two consecutive tiles with QC-fail reads switch to 0, one
            // fail-free tile back to 1, so rare QC-fail reads cost one fix-up
            // each and QC-fail-heavy streams run the three-plane tree.
            // Warp-uniform throughout; exact either way.
            uint32_t bad = 0;
            if (phase) {
                uint32_t top[2];
                FlagByteTree<CD, L, 1>::run(carries, r, top, bad);
                extract_bytes(counter[0], top[0]);
                extract_bytes(counter[2], top[1]);
                if (bad & 0xF0F0F0F0u) locate_bad<CANON, REGS, RPV, VB>(a, r, first, stride);  // r[] dies here
                if (__any_sync(0xFFFFFFFFu, bad & 0x02020202u)) {
                    uint32_t r2[REGS];
                    load_tree_block<VB, 0, REGS / RPV>(a, first, stride, false, r2);
                    uint32_t bad2 = 0, top2[2];
                    FlagByteTree<CD, L, 2>::run(carries, r2, top2, bad2);
                    extract_bytes(counter[1], top2[0]);
                    extract_bytes(counter[2], top2[1]);
                    phase = phase == 1u ? 2u : 0u;
                } else {
                    phase = 1u;
                }
            } else {
                uint32_t top[3];
                FlagByteTree<CD, L>::run(carries, r, top, bad);
#pragma unroll
                for (int b = 0; b < 3; ++b) extract_bytes(counter[b], top[b]);
                if (bad & 0xF0F0F0F0u) locate_bad<CANON, REGS, RPV, VB>(a, r, first, stride);
                phase = __any_sync(0xFFFFFFFFu, bad & 0x02020202u) ? 0u : 1u;
            }
            return;
        }
        uint32_t bad = 0, top[3];
        FlagByteTree<CD, L>::run(carries, r, top, bad);
        if (phase) {  // second tile of the pair: level-L CSA, one extract per two tiles
#pragma unroll
            for (int b = 0; b < 3; ++b) {
                uint32_t h, l;
                csa(h, l, carries[b][L], carries[b][L + 1], top[b]);
                carries[b][L] = l;
                carries[b][L + 1] = 0;
                extract_bytes(counter[b], h);
            }
        } else {
#pragma unroll
            for (int b = 0; b < 3; ++b) carries[b][L + 1] = top[b];
        }
        phase ^= 1u;
        if (bad & 0xF0F0F0F0u) locate_bad<CANON, REGS, RPV, VB>(a, r, first, stride);
    } else {
        static_assert(NBANK == 2 && REGS == (1 << L), "FLAG mode: two banks of 2^L registers");
        constexpr int RPV = VB / 4;
        uint32_t bad = 0;
#pragma unroll
        for (int i = 0; i < REGS; ++i) bad |= r[i];
        uint32_t top_all, top_fail;
        FlagDualTree<L>::run(carries[0], carries[1], r, top_all, top_fail);
        extract(counter[0], top_all);
        extract(counter[1], top_fail);
        if (bad & 0xF000F000u) locate_bad<CANON, REGS, RPV, VB>(a, r, first, stride);
    }
}

// consume()'s MODE 2 branch for a tile read in place from shared memory
// (the ring kernel's direct mode): leaves load their 8 bytes as the tree
// needs them, so no register tile is live and more warps fit per SM.  The
// QC-fail fix-up pass re-reads the slot; the reserved-bit report reloads the
// tile from global memory in canonical order.
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
    constexpr int REGS = MODE == 1 ? (1 << L) : MODE == 2 ? (2 << L) : (NBANK << L);  // registers per tree block
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

    // MODE 2 keeps two extra words per bank: the level-L carry and the pending
    // top of the previous tile (tiles are paired into one depth-L+1 tree).
    constexpr int CD = pair_tiles<MODE, L>() ? L + 2 : L;
    uint32_t carries[NBANK][CD];
    uint32_t counter[NBANK][16];
    uint32_t phase = 0;
#pragma unroll
    for (int b = 0; b < NBANK; ++b)
#pragma unroll
        for (int j = 0; j < CD; ++j) carries[b][j] = 0;
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
            consume<MODE, NBANK, L, VB>(a, r, t + threadIdx.x, block, carries, counter, phase);
            if (++nb == a.flush_threshold) {  // block-uniform: every thread runs the same tiles
                flush_bank_to_smem<NBANK, L, MODE>(counter, s_acc, lane);
                nb = 0;
            }
        }
    } else if constexpr (SCHED == 4 || SCHED == 5) {
        // SCHED 2's work split with double-buffered tile registers: the next
        // warp tile is claimed and its loads issued before the current tile is
        // consumed, so each warp keeps a tile in flight while it computes
        // (for the ALU-heavy FLAG mode, whose warps would otherwise alternate
        // between waiting and computing).  SCHED 5 (MODE 2): the tile is
        // loaded in two halves and the pipeline runs at half-tile grain, so
        // the same registers as SCHED 2 keep one half-tile always in flight
        // while the depth-L tree is built from two depth-(L-1) halves.
        constexpr unsigned long long WT = 32ull * VPT;
        const unsigned long long S0 = a.g0 * 32;
        const unsigned long long P = a.nwt - a.pool;
        const unsigned long long lo = P * blockIdx.x / gridDim.x;
        const unsigned long long hi = P * (blockIdx.x + 1) / gridDim.x;
        constexpr unsigned long long kEnd = ~0ull;
        __shared__ unsigned s_claim;
        if (threadIdx.x == 0) s_claim = 0u;
        __syncthreads();
        bool local = true;
        unsigned long long pw = 0, pe = 0;  // current pool chunk [pw, pe)
        unsigned long long pm = 0;          // prefetched pool chunk index (lane 0)
        // Warp-uniform: the next warp tile of this warp, or kEnd.
        auto claim = [&]() -> unsigned long long {
            if (local) {
                const unsigned m = lane == 0 ? atomicAdd(&s_claim, 1u) : 0u;
                const unsigned long long w = lo + __shfl_sync(0xFFFFFFFFu, m, 0);
                if (w < hi) return w;
                local = false;
                if (!a.pool) return kEnd;
                pdl_wait_prev();  // the pool counter is shared with the previous launch
                pm = lane == 0 ? atomicAdd(a.next, 1ull) : 0ull;
            }
            if (pw >= pe) {
                const unsigned long long c = __shfl_sync(0xFFFFFFFFu, pm, 0);
                pm = lane == 0 ? atomicAdd(a.next, 1ull) : 0ull;
                pw = P + c * a.CB;
                if (pw >= a.nwt) {
                    pe = pw;
                    return kEnd;
                }
                pe = pw + a.CB < a.nwt ? pw + a.CB : a.nwt;
            }
            return pw++;
        };
        if constexpr (SCHED == 5) {
            static_assert(MODE == 2 && !pair_tiles<MODE, L>() && VPT % 2 == 0, "SCHED 5: byte-frame FLAG, L >= 5");
            constexpr int HR = REGS / 2, HV = VPT / 2;  // registers / vectors per half tile
            auto load_half = [&](unsigned long long w, int h, uint32_t (&r)[HR]) {
                const unsigned long long t = S0 + w * WT;
                load_tree_block<VB, HINT, HV>(a, t + lane + 32ull * HV * h, 32u, t >= a.f0 && t + WT <= a.f1, r);
            };
            auto half_tree = [&](const uint32_t (&r)[HR], unsigned long long w, int h, uint32_t (&top)[3]) {
                uint32_t bad = 0;
                FlagByteTree<CD, L - 1>::run(carries, r, top, bad);
                if (bad & 0xF0F0F0F0u)
                    flag_locate_bad<HR, RPV, VB>(a, r, S0 + w * WT + lane + 32ull * HV * h, 32u);
            };
            uint32_t ra[HR], rb[HR];
            unsigned long long w = claim();
            if (w != kEnd) load_half(w, 0, ra);
            while (w != kEnd) {
                load_half(w, 1, rb);
                uint32_t x[3], y[3];
                half_tree(ra, w, 0, x);
                const unsigned long long wn = claim();
                if (wn != kEnd) load_half(wn, 0, ra);
                half_tree(rb, w, 1, y);
#pragma unroll
                for (int b = 0; b < 3; ++b) {
                    uint32_t h, l;
                    csa(h, l, carries[b][L - 1], x[b], y[b]);
                    carries[b][L - 1] = l;
                    extract_bytes(counter[b], h);
                }
                if (++nb == a.flush_threshold) {
                    flush_bank_to_smem<NBANK, L, MODE>(counter, s_acc, lane);
                    nb = 0;
                }
                w = wn;
            }
        } else {
        auto load = [&](unsigned long long w, uint32_t (&r)[REGS]) {
            const unsigned long long t = S0 + w * WT;
            load_tree_block<VB, HINT, VPT>(a, t + lane, 32u, t >= a.f0 && t + WT <= a.f1, r);
        };
        uint32_t ra[REGS], rb[REGS];
        unsigned long long w0 = claim();
        if (w0 != kEnd) load(w0, ra);
        for (;;) {
            if (w0 == kEnd) break;
            const unsigned long long w1 = claim();
            if (w1 != kEnd) load(w1, rb);
            consume<MODE, NBANK, L, VB>(a, ra, S0 + w0 * WT + lane, 32u, carries, counter, phase);
            if (++nb == a.flush_threshold) {
                flush_bank_to_smem<NBANK, L, MODE>(counter, s_acc, lane);
                nb = 0;
            }
            if (w1 == kEnd) break;
            w0 = claim();
            if (w0 != kEnd) load(w0, ra);
            consume<MODE, NBANK, L, VB>(a, rb, S0 + w1 * WT + lane, 32u, carries, counter, phase);
            if (++nb == a.flush_threshold) {
                flush_bank_to_smem<NBANK, L, MODE>(counter, s_acc, lane);
                nb = 0;
            }
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
            consume<MODE, NBANK, L, VB>(a, r, t + lane, 32u, carries, counter, phase);
            if (++nb == a.flush_threshold) {  // warp-uniform
                flush_bank_to_smem<NBANK, L, MODE>(counter, s_acc, lane);
                nb = 0;
            }
            w = lo + __shfl_sync(0xFFFFFFFFu, mine, 0);
            mine = lane == 0 ? atomicAdd(&s_claim, 1u) : 0u;
        }
        // diagnostics: per-warp end of the CTA-range phase, then of the pool
        // phase, after the 5 per-CTA stamps (tools/trace.py)
        unsigned long long* wtrace = a.trace ? a.trace + gridDim.x * 5ull + (blockIdx.x * (block / 32) + (threadIdx.x >> 5)) * 3 : nullptr;
        if (wtrace && lane == 0) wtrace[0] = globaltimer();
        unsigned pool_tiles = 0;
        if (a.pool) {
            pdl_wait_prev();  // the pool counter is shared with the previous launch
            unsigned long long m = lane == 0 ? atomicAdd(a.next, 1ull) : 0ull;
            unsigned long long c = __shfl_sync(0xFFFFFFFFu, m, 0);
            m = lane == 0 ? atomicAdd(a.next, 1ull) : 0ull;
            for (;;) {
                const unsigned long long w0 = P + c * a.CB;
                if (w0 >= a.nwt) break;  // warp-uniform
                const unsigned long long w1 = w0 + a.CB < a.nwt ? w0 + a.CB : a.nwt;
                pool_tiles += (unsigned)(w1 - w0);
                for (unsigned long long ww = w0; ww < w1; ++ww) {
                    const unsigned long long t = S0 + ww * WT;
                    uint32_t r[REGS];
                    load_tree_block<VB, HINT, VPT>(a, t + lane, 32u, t >= a.f0 && t + WT <= a.f1, r);
                    consume<MODE, NBANK, L, VB>(a, r, t + lane, 32u, carries, counter, phase);
                    if (++nb == a.flush_threshold) {
                        flush_bank_to_smem<NBANK, L, MODE>(counter, s_acc, lane);
                        nb = 0;
                    }
                }
                c = __shfl_sync(0xFFFFFFFFu, m, 0);
                m = lane == 0 ? atomicAdd(a.next, 1ull) : 0ull;
            }
        }
        if (wtrace && lane == 0) {
            wtrace[1] = globaltimer();
            wtrace[2] = pool_tiles;
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
                consume<MODE, NBANK, L, VB>(a, r, t + lane, 32u, carries, counter, phase);
                if (++nb == a.flush_threshold) {  // warp-uniform
                    flush_bank_to_smem<NBANK, L, MODE>(counter, s_acc, lane);
                    nb = 0;
                }
            }
            c = __shfl_sync(0xFFFFFFFFu, mine, 0);
            mine = lane == 0 ? atomicAdd(a.next, 1ull) : 0ull;
        }
    }
    cta_finish<NBANK, L, MODE>(a, carries, counter, s_acc, &s_last, block, lane);
}

// ---------------------------------------------------------------------------
// Small inputs (the latency path): ONE CTA counts 16-byte
// vectors [v0, v1) (edges byte-masked like the stream kernel), four vectors
// per thread per tree block (depth 4; k = 64: two depth-3 banks), then drains,
// transpose-reduces per warp, sums channels in shared memory and writes
// out[k] directly -- no workspace, no global atomics, no ticket, so the
// launch is load latency + one reduction.
// ---------------------------------------------------------------------------
constexpr int kSmallBlock = 256;

template <int NBANK>
__global__ void __launch_bounds__(kSmallBlock, 1) small_kernel(const StreamArgs a) {
    constexpr int VPT = 4, REGS = 16, L = NBANK == 1 ? 4 : 3;
    static_assert((NBANK << L) == REGS, "one tree block = four 16-byte vectors");
    constexpr unsigned long long TILE = (unsigned long long)VPT * kSmallBlock;
    __shared__ uint32_t s_ch[32 * NBANK];
    for (int i = threadIdx.x; i < 32 * NBANK; i += kSmallBlock) s_ch[i] = 0;
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
    for (unsigned long long t = a.v0; t < a.v1; t += TILE) {
        uint32_t r[REGS];
        load_tree_block<16, 0, VPT>(a, t + threadIdx.x, kSmallBlock, t >= a.f0 && t + TILE <= a.f1, r);
        tree_block<NBANK, L>(r, carries, counter);
    }
#pragma unroll
    for (int b = 0; b < NBANK; ++b) {
        uint32_t d[16];
        drain<L>(d, carries[b]);
        const uint32_t tot = bank_warp_total(counter[b], L, d);
        if (tot) atomicAdd(&s_ch[b * 32 + lane], tot);
    }
    __syncthreads();
    pdl_wait_prev();  // out[] may belong to the previous launch on this stream
    const int k = a.k;
    for (int pos = threadIdx.x; pos < k; pos += kSmallBlock) {
        unsigned long long sum = 0;
        if (k == 64) {
            sum = s_ch[pos];
        } else {
            for (int j = 0; j < channels_per_position(k); ++j) sum += s_ch[pos + j * k];
        }
        a.out[pos] = a.accumulate ? a.out[pos] + sum : sum;
    }
}

// ---------------------------------------------------------------------------
// Medium inputs (the latency path above the single-CTA size): ONE thread-block
// cluster of gridDim.x CTAs (one per SM) counts the stream with the small
// kernel's tree; each CTA reduces to shared-memory channel totals and, after a
// cluster barrier, CTA 0 sums the other CTAs' totals through distributed
// shared memory and writes out[k] -- still no workspace, no global atomics and
// no last-CTA ticket, with gridDim.x times the single CTA's bandwidth.
// ---------------------------------------------------------------------------
template <int NBANK>
__global__ void __launch_bounds__(kSmallBlock, 1) cluster_kernel(const StreamArgs a) {
    namespace cg = cooperative_groups;
    constexpr int VPT = 4, REGS = 16, L = NBANK == 1 ? 4 : 3;
    const unsigned long long tile = (unsigned long long)VPT * kSmallBlock;
    const unsigned long long stride = tile * gridDim.x;
    __shared__ uint32_t s_ch[32 * NBANK];
    for (int i = threadIdx.x; i < 32 * NBANK; i += kSmallBlock) s_ch[i] = 0;
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
    for (unsigned long long t = a.v0 + blockIdx.x * tile; t < a.v1; t += stride) {
        uint32_t r[REGS];
        load_tree_block<16, 0, VPT>(a, t + threadIdx.x, kSmallBlock, t >= a.f0 && t + tile <= a.f1, r);
        tree_block<NBANK, L>(r, carries, counter);
    }
#pragma unroll
    for (int b = 0; b < NBANK; ++b) {
        uint32_t d[16];
        drain<L>(d, carries[b]);
        const uint32_t tot = bank_warp_total(counter[b], L, d);
        if (tot) atomicAdd(&s_ch[b * 32 + lane], tot);
    }
    cg::cluster_group cluster = cg::this_cluster();
    cluster.sync();  // every CTA's totals are in its shared memory
    if (cluster.block_rank() == 0) {
        pdl_wait_prev();  // out[] may belong to the previous launch on this stream
        for (int c = threadIdx.x; c < 32 * NBANK; c += kSmallBlock) {
            uint32_t sum = s_ch[c];
            for (unsigned r = 1; r < cluster.num_blocks(); ++r) sum += cluster.map_shared_rank(s_ch, r)[c];
            s_ch[c] = sum;
        }
        __syncthreads();
        const int k = a.k;
        for (int pos = threadIdx.x; pos < k; pos += kSmallBlock) {
            unsigned long long sum = 0;
            if (k == 64) {
                sum = s_ch[pos];
            } else {
                for (int j = 0; j < channels_per_position(k); ++j) sum += s_ch[pos + j * k];
            }
            a.out[pos] = a.accumulate ? a.out[pos] + sum : sum;
        }
    }
    cluster.sync();  // keep every CTA's shared memory alive until CTA 0 has read it
}

// ---------------------------------------------------------------------------
// TMA-staged variant (SCHED 3).  One producer warp per CTA pulls stage indices
// from the global counter and moves each 32 KiB (NC warp tiles) stage of the
// stream into a shared-memory ring with one cp.async.bulk (UBLKCP), tracked by
// a full/empty mbarrier pair per slot; NC consumer warps wait on `full`, read
// their warp tile with LDS.128 (vectors outside the valid range read as zero,
// the first/last vector byte-masked), release the slot on `empty` and run the
// same tree/flush/epilogue as the LDG kernel.  Memory latency is covered by
// the ring depth instead of by registers and warps, which matters for the
// ALU-heavy FLAG mode.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(unsigned long long* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done)
                     : "r"(smem_addr(bar)), "r"(parity)
                     : "memory");
}

__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, uint32_t bytes, unsigned long long* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_addr(dst)),
                 "l"(src), "r"(bytes), "r"(smem_addr(bar))
                 : "memory");
}

// Stage s of the ring holds NC * 32 * VPT 16-byte vectors.
template <int NBANK, int L, int MODE, int NC, int STAGES>
__global__ void __launch_bounds__(32 * (NC + 1), 1) stream_tma_kernel(const StreamArgs a) {
    constexpr int REGS = MODE == 1 ? (1 << L) : MODE == 2 ? (2 << L) : (NBANK << L);
    constexpr int VPT = REGS / 4;                                   // 16-byte vectors per lane per tree block
    constexpr unsigned long long WTV = 32ull * VPT;                 // vectors per warp tile
    constexpr unsigned long long STV = NC * WTV;                    // vectors per stage
    constexpr uint32_t STB = (uint32_t)(STV * 16);                  // bytes per stage
    extern __shared__ __align__(128) uint8_t ring[];                // STAGES x STB
    __shared__ __align__(8) unsigned long long full[STAGES], empty[STAGES];
    __shared__ unsigned long long stage_idx[STAGES];
    __shared__ unsigned long long s_acc[32 * NBANK];
    __shared__ int s_last;

    const unsigned block = blockDim.x;
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t warp = threadIdx.x >> 5;
    if (a.trace && threadIdx.x == 0) {
        a.trace[blockIdx.x * 5 + 0] = globaltimer();
        a.trace[blockIdx.x * 5 + 4] = smid();
    }
    for (int i = threadIdx.x; i < 32 * NBANK; i += block) s_acc[i] = 0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NC * 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    pdl_allow_next();
    __syncthreads();

    // MODE 2 keeps two extra words per bank: the level-L carry and the pending
    // top of the previous tile (tiles are paired into one depth-L+1 tree).
    constexpr int CD = pair_tiles<MODE, L>() ? L + 2 : L;
    uint32_t carries[NBANK][CD];
    uint32_t counter[NBANK][16];
    uint32_t phase = 0;
#pragma unroll
    for (int b = 0; b < NBANK; ++b)
#pragma unroll
        for (int j = 0; j < CD; ++j) carries[b][j] = 0;
    zero_bank<NBANK>(counter);

    const unsigned long long S0 = a.g0 * 32;
    const unsigned long long NS = a.ng ? (a.v1 - S0 + STV - 1) / STV : 0;  // stages in the stream

    if (warp == NC) {  // producer
        if (lane == 0) {
            pdl_wait_prev();  // the stage counter is shared with the previous launch
            for (unsigned it = 0;; ++it) {
                const unsigned s = it % STAGES;
                if (it >= STAGES) mbar_wait(&empty[s], ((it / STAGES) - 1) & 1u);
                const unsigned long long idx = atomicAdd(a.next, 1ull);
                stage_idx[s] = idx;
                if (idx >= NS) {  // end marker: wake the consumers without data
                    mbar_arrive(&full[s]);
                    break;
                }
                const unsigned long long t0 = S0 + idx * STV;
                const unsigned long long lo = t0 > a.v0 ? t0 : a.v0;
                const unsigned long long hi = t0 + STV < a.v1 ? t0 + STV : a.v1;
                const uint32_t bytes = (uint32_t)((hi - lo) * 16);
                POSPOP_CHECK(lo >= a.v0 && hi <= a.v1 && lo < hi);
                mbar_arrive_expect_tx(&full[s], bytes);
                tma_bulk_g2s(ring + (size_t)s * STB + (lo - t0) * 16, a.base + lo * 16, bytes, &full[s]);
            }
        }
    } else {  // consumers
        uint32_t nb = 0;
        for (unsigned it = 0;; ++it) {
            const unsigned s = it % STAGES;
            mbar_wait(&full[s], (it / STAGES) & 1u);
            const unsigned long long idx = stage_idx[s];
            if (idx >= NS) break;
            const unsigned long long t0 = S0 + idx * STV;
            const unsigned long long first = t0 + warp * WTV + lane;  // lane's first vector (global index)
            const uint8_t* tile = ring + (size_t)s * STB + (warp * WTV + lane) * 16;
            const bool fast = t0 + warp * WTV >= a.f0 && t0 + (warp + 1) * WTV <= a.f1;
            uint32_t r[REGS];
#pragma unroll
            for (int v = 0; v < VPT; ++v) {
                uint32_t x[4];
                const unsigned long long g = first + 32ull * v;
                if (fast || (g >= a.v0 && g < a.v1)) {
                    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                                 : "=r"(x[0]), "=r"(x[1]), "=r"(x[2]), "=r"(x[3])
                                 : "r"(smem_addr(tile + 512 * v)));
                    if (!fast && (g == a.v0 || g + 1 == a.v1))
                        mask_bytes<16>(x, g == a.v0 ? a.lo_byte : 0, g + 1 == a.v1 ? a.hi_byte : 16);
                } else {
                    x[0] = x[1] = x[2] = x[3] = 0;
                }
#pragma unroll
                for (int j = 0; j < 4; ++j) r[v * 4 + j] = x[j];
            }
            mbar_arrive(&empty[s]);  // this lane's reads are in registers: the slot may be refilled
            consume<MODE, NBANK, L, 16>(a, r, first, 32u, carries, counter, phase);
            if (++nb == a.flush_threshold) {  // warp-uniform
                flush_bank_to_smem<NBANK, L, MODE>(counter, s_acc, lane);
                nb = 0;
            }
        }
    }
    cta_finish<NBANK, L, MODE>(a, carries, counter, s_acc, &s_last, block, lane);
}


// ---------------------------------------------------------------------------
// Per-warp bulk-copy ring (SCHED 6).  The SCHED 2 work split (CTA ranges of
// warp tiles claimed through a shared counter, then the global tail pool),
// but each warp stages its own next S warp tiles in shared memory: lane 0
// issues one cp.async.bulk per tile into the warp's slot, tracked by the
// slot's mbarrier, so while the warp computes on tile i the loads of tiles
// i+1 .. i+S are in flight without holding registers.  No slot is shared
// between warps (the SCHED 3 ring serialised its consumers on a common
// stage).  The warp copies a ready slot into registers with LDS.128 (16-byte
// halves swapped on every other quarter-warp: conflict-free, and the
// counts do not depend on register order; k = 64's lo/hi parity is kept),
// refills the slot, then runs the same tree/extract as the LDG kernel.
// Tiles not fully inside [f0, f1) (the stream's first and last vectors) are
// loaded with the masked LDG path instead.  One CTA of NW warps per SM.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

template <int NBANK, int L, int MODE, int NW, int S>
__global__ void __launch_bounds__(32 * NW, 1) stream_ring_kernel(const StreamArgs a) {
    constexpr int VB = 32;
    constexpr int REGS = MODE == 2 ? (2 << L) : (NBANK << L);  // registers per tree block
    constexpr int RPV = VB / 4;
    constexpr int VPT = REGS / RPV;
    constexpr unsigned long long WT = 32ull * VPT;  // vectors per warp tile
    constexpr uint32_t TB = (uint32_t)(WT * VB);    // bytes per warp tile
    constexpr unsigned long long kEnd = ~0ull;
    extern __shared__ __align__(128) uint8_t ring[];  // NW x S x TB
    __shared__ __align__(8) unsigned long long bar[NW * S];
    __shared__ unsigned long long s_acc[32 * NBANK];
    __shared__ int s_last;
    __shared__ unsigned s_claim;

    constexpr unsigned block = 32 * NW;
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t warp = threadIdx.x >> 5;
    if (a.trace && threadIdx.x == 0) {
        a.trace[blockIdx.x * 5 + 0] = globaltimer();
        a.trace[blockIdx.x * 5 + 4] = smid();
    }
    for (int i = threadIdx.x; i < 32 * NBANK; i += block) s_acc[i] = 0;
    if (threadIdx.x == 0) {
        s_claim = 0u;
        for (int i = 0; i < NW * S; ++i) mbar_init(&bar[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    pdl_allow_next();
    __syncthreads();

    constexpr int CD = pair_tiles<MODE, L>() ? L + 2 : L;
    uint32_t carries[NBANK][CD];
    uint32_t counter[NBANK][16];
    uint32_t phase = 0;
#pragma unroll
    for (int b = 0; b < NBANK; ++b)
#pragma unroll
        for (int j = 0; j < CD; ++j) carries[b][j] = 0;
    zero_bank<NBANK>(counter);
    uint32_t nb = 0;

    const unsigned long long S0 = a.g0 * 32;
    const unsigned long long P = a.nwt - a.pool;
    const unsigned long long lo = P * blockIdx.x / gridDim.x;
    const unsigned long long hi = P * (blockIdx.x + 1) / gridDim.x;
    bool local = true;
    unsigned long long pw = 0, pe = 0;  // current pool chunk [pw, pe)
    unsigned long long pm = 0;          // prefetched pool chunk index (lane 0)
    // Warp-uniform: the next warp tile of this warp, or kEnd.
    auto claim = [&]() -> unsigned long long {
        if (local) {
            const unsigned m = lane == 0 ? atomicAdd(&s_claim, 1u) : 0u;
            const unsigned long long w = lo + __shfl_sync(0xFFFFFFFFu, m, 0);
            if (w < hi) return w;
            local = false;
            if (!a.pool) return kEnd;
            pdl_wait_prev();  // the pool counter is shared with the previous launch
            pm = lane == 0 ? atomicAdd(a.next, 1ull) : 0ull;
        }
        if (pw >= pe) {
            const unsigned long long c = __shfl_sync(0xFFFFFFFFu, pm, 0);
            pm = lane == 0 ? atomicAdd(a.next, 1ull) : 0ull;
            pw = P + c * a.CB;
            if (pw >= a.nwt) {
                pe = pw;
                return kEnd;
            }
            pe = pw + a.CB < a.nwt ? pw + a.CB : a.nwt;
        }
        return pw++;
    };

    uint8_t* mine = ring + (size_t)warp * S * TB;
    unsigned long long* mbar = bar + warp * S;
    unsigned long long held[S];  // warp-uniform: the tile slot s holds (kEnd: none)
    bool bulk[S];                // slot s was filled by a bulk copy (else: masked LDG at consume time)
    // Fills slot s with tile w: one bulk copy of TB bytes (fully valid tile),
    // or a bare arrive (no data: the end marker, or an edge tile loaded later).
    auto fill = [&](int s, unsigned long long w) {
        const unsigned long long t = S0 + w * WT;
        const bool full = w != kEnd && t >= a.f0 && t + WT <= a.f1;
        held[s] = w;
        bulk[s] = full;
        if (lane == 0) {
            if (full) {
                POSPOP_CHECK(t >= a.v0 && t + WT <= a.v1);
                fence_proxy_async_smem();  // this warp's earlier LDS reads of the slot precede the copy
                mbar_arrive_expect_tx(&mbar[s], TB);
                tma_bulk_g2s(mine + (size_t)s * TB, a.base + t * VB, TB, &mbar[s]);
            } else {
                mbar_arrive(&mbar[s]);
            }
        }
    };
#pragma unroll
    for (int s = 0; s < S; ++s) fill(s, claim());
    const uint32_t h = (lane >> 2) & 1u;  // 16-byte half read first
    for (uint32_t use = 0;; ++use) {
        bool done = false;
#pragma unroll
        for (int s = 0; s < S; ++s) {
            if (done) break;
            mbar_wait(&mbar[s], use & 1u);
            const unsigned long long w = held[s];
            if (w == kEnd) {
                done = true;
                break;
            }
            const unsigned long long first = S0 + w * WT + lane;
            uint32_t r[REGS];
            if (bulk[s]) {
                const uint8_t* base = mine + (size_t)s * TB + (size_t)lane * VB;
#pragma unroll
                for (int v = 0; v < VPT; ++v) {
#pragma unroll
                    for (int q = 0; q < 2; ++q) {
                        uint32_t* x = r + v * RPV + 4 * q;
                        asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                                     : "=r"(x[0]), "=r"(x[1]), "=r"(x[2]), "=r"(x[3])
                                     : "r"(smem_addr(base + (size_t)v * 32 * VB + 16 * (q ^ h)))
                                     : "memory");
                    }
                }
            } else {
                load_tree_block<VB, 0, VPT>(a, first, 32u, false, r);
            }
            __syncwarp();
            fill(s, claim());
            consume<MODE, NBANK, L, VB, false>(a, r, first, 32u, carries, counter, phase);
            if (++nb == a.flush_threshold) {  // warp-uniform
                flush_bank_to_smem<NBANK, L, MODE>(counter, s_acc, lane);
                nb = 0;
            }
        }
        if (done) break;
    }
    cta_finish<NBANK, L, MODE>(a, carries, counter, s_acc, &s_last, block, lane);
}

}  // namespace dev
}  // namespace pospop_b200
