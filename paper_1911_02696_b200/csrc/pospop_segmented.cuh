// pospop_segmented.cuh -- the segmented / batched kernels (one k-row per array): strided,
// dynamically claimed and software-pipelined schedules.
// Device code only; included by pospop_kernels.cu (the single CUDA translation
// unit, which instantiates the kernels and owns the host-side launchers).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "pospop_device.cuh"
#include "pospop_stream.cuh"

namespace pospop_b200 {
namespace dev {

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
__device__ __forceinline__ void seg_warp_loop(const uint8_t* data, const unsigned long long* offsets,
                                              unsigned long long n_arrays, int k, uint32_t flush_threshold,
                                              unsigned long long* out, unsigned long long* next, unsigned per_grab) {
    constexpr int REGS = NBANK << L;
    constexpr int RPV = VB / 4;
    constexpr int VPT = REGS / RPV;
    constexpr unsigned long long STEP = 32ull * VPT;
    const uint32_t lane = threadIdx.x & 31u;
    const int wb = k >> 3;
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
                    POSPOP_CHECK(t + 32ull * v + lane < nv);
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
}

// Every warp has drawn a claim index past the end; once all CTAs are past that
// point the claim counter can be reset for the next launch.
__device__ __forceinline__ void seg_claims_done(unsigned long long* next, unsigned int* ticket) {
    __shared__ int s_last;
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

template <int NBANK, int L, int VB, int SCHED>
__global__ void __launch_bounds__(256) segmented_kernel(const uint8_t* data,
                                                        const unsigned long long* offsets,
                                                        unsigned long long n_arrays, int k,
                                                        uint32_t flush_threshold,
                                                        unsigned long long* out,
                                                        unsigned long long* next,
                                                        unsigned int* ticket, unsigned per_grab) {
    pdl_allow_next();
    pdl_wait_prev();  // the claim counter, the ticket and the rows may belong to the previous launch
    seg_warp_loop<NBANK, L, VB, SCHED>(data, offsets, n_arrays, k, flush_threshold, out, next, per_grab);
    if (SCHED == 1) seg_claims_done(next, ticket);
}

// ---------------------------------------------------------------------------
// Bit-plane epilogue (EPI 1).  A lane's per-channel count is held as bit
// planes: the tree carries (weight 2^j, j < L) and a bit-sliced counter of the
// tree tops (weight 2^(L+i), i < M, incremented by a half-adder ripple, two
// LOP3 per level per tree block, instead of the 16-lane extract).  The warp
// sum of channel c over the 32 lanes is then, per plane P, popc of column c of
// the 32x32 bit matrix whose row r is lane r's P -- a warp bit transpose
// (5 x {SHFL, SHF funnel rotate, LOP3 bit-select}) followed by one POPC on lane
// c.  16 instructions per plane replace the 16-lane drain (Horner over L
// planes), the 32-value unpack and the 31-shuffle transpose-reduce.
// ---------------------------------------------------------------------------
struct PlaneXpose {
    uint32_t sh[5], mk[5];  // per level: rotate amount and keep-mask for this lane
    __device__ __forceinline__ explicit PlaneXpose(uint32_t lane) {
#pragma unroll
        for (int s = 0; s < 5; ++s) {
            const uint32_t j = 16u >> s;
            const uint32_t m = s == 0 ? 0x0000FFFFu : s == 1 ? 0x00FF00FFu : s == 2 ? 0x0F0F0F0Fu
                             : s == 3 ? 0x33333333u : 0x55555555u;  // columns c with (c & j) == 0
            const bool bottom = (lane & j) != 0;
            sh[s] = bottom ? 32u - j : j;
            mk[s] = bottom ? ~m : m;
        }
    }
    // Number of lanes whose plane has bit `lane` set.  All 32 lanes together.
    __device__ __forceinline__ uint32_t column_popc(uint32_t x) const {
#pragma unroll
        for (int s = 0; s < 5; ++s) {
            const uint32_t y = __shfl_xor_sync(0xFFFFFFFFu, x, 16u >> s);
            const uint32_t r = __funnelshift_l(y, y, sh[s]);
            x = (x & mk[s]) | (r & ~mk[s]);
        }
        return __popc(x);
    }
};

// tops counter: U[i] has weight 2^(L+i); adds one plane (ripple half-adders).
template <int M>
__device__ __forceinline__ void plane_count_add(uint32_t (&U)[M], uint32_t top) {
#pragma unroll
    for (int i = 0; i < M; ++i) {
        const uint32_t c = U[i] & top;
        U[i] ^= top;
        top = c;
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

template <int VB, int VPT, int HINT = 0>
__device__ __forceinline__ void seg_load(const SegView& v, unsigned long long t, uint32_t lane,
                                         uint32_t (&r)[VPT * (VB / 4)]) {
    constexpr int RPV = VB / 4;
    constexpr unsigned long long STEP = 32ull * VPT;
    if (t >= v.f0 && t + STEP <= v.f1) {
#pragma unroll
        for (int q = 0; q < VPT; ++q) {
            uint32_t x[RPV];
            POSPOP_CHECK(t + 32ull * q + lane < v.nv);
            ldg_stream<VB, HINT>(v.base + (t + 32ull * q + lane) * VB, x);
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

// seg_load for a whole CTA counting one view together: thread `tid` of
// `nthreads` loads vectors t + tid + q * nthreads (q < VPT), so each step of
// the CTA reads one contiguous window of nthreads * VPT vectors.
template <int VB, int VPT>
__device__ __forceinline__ void seg_load_cta(const SegView& v, unsigned long long t, unsigned tid, unsigned nthreads,
                                             uint32_t (&r)[VPT * (VB / 4)]) {
    constexpr int RPV = VB / 4;
    if (t >= v.f0 && t + (unsigned long long)nthreads * VPT <= v.f1) {
#pragma unroll
        for (int q = 0; q < VPT; ++q) {
            uint32_t x[RPV];
            POSPOP_CHECK(t + tid + (unsigned long long)nthreads * q < v.nv);
            ldg_stream<VB, 0>(v.base + (t + tid + (unsigned long long)nthreads * q) * VB, x);
#pragma unroll
            for (int j = 0; j < RPV; ++j) r[q * RPV + j] = x[j];
        }
    } else {
#pragma unroll
        for (int q = 0; q < VPT; ++q) {
            const unsigned long long idx = t + tid + (unsigned long long)nthreads * q;
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

// ---------------------------------------------------------------------------
// Workspace regions after the stream scratch (pospop_launch.h), addressed
// from the claim counter `next` (u64 97 of the workspace): the range mode's
// slots (u64 104 on) and the giant-array queue after them.  Zero between
// launches.
// ---------------------------------------------------------------------------
constexpr int kSegRangeSlots = 16384;  // = kSegRangeSlotsHost (pospop_launch.h); range mode: one per array
constexpr int kGiantQ = 512;           // = kGiantQHost
constexpr int kGiantEntry = 72;        // u64 per queue entry
__device__ __forceinline__ unsigned long long* seg_range_slots(unsigned long long* next) { return next + 7; }

// Giant arrays (above `giant_bytes`) met by the array-per-warp / per-lane
// schedules are not counted by one warp: the warp publishes the array in this
// queue and counts its chunks together with every warp that reaches a claim
// point (or its exit) while chunks are left; chunk partials are summed in the
// entry with u64 atomics and the warp finishing the last chunk moves them into
// the row.  The publisher keeps helping until its entry has no chunk left, so
// no array waits for a warp that already exited; a helper never waits for an
// entry that is counted but not yet marked ready -- it skips it (its publisher
// counts it; a helper spinning on that flag hung intermittently).  Entry: [0]
// array, [1] chunks, [2] chunk claim counter, [3] ready flag, [4, 68) counts,
// [68] chunks done.  [0] of the queue = entries published (beyond kGiantQ the publisher
// counts the array alone).  The last CTA resets the queue (seg_launch_done).
struct GiantQueue {
    unsigned long long* base;
    unsigned long long giant_bytes;  // 0: off
    __device__ __forceinline__ unsigned long long* entry(unsigned long long e) const {
        return base + 8 + e * kGiantEntry;
    }
    __device__ __forceinline__ unsigned long long chunk_bytes() const { return giant_bytes / 4; }
};
__device__ __forceinline__ GiantQueue seg_giant_queue(unsigned long long* next, unsigned long long giant_bytes) {
    return GiantQueue{next + 7 + (unsigned long long)kSegRangeSlots * 65, giant_bytes};
}

// Warp totals (lane c: channel c) of one vector view, depth-L tree steps.
template <int NBANK, int L, int VB>
__device__ __forceinline__ void seg_count_view(const SegView& v, uint32_t lane, const PlaneXpose& xp,
                                               unsigned long long (&tot)[NBANK]) {
    constexpr int M = 3;
    constexpr int REGS = NBANK << L;
    constexpr int VPT = REGS / (VB / 4);
    constexpr unsigned long long STEP = 32ull * VPT;
    uint32_t carries[NBANK][L], U[NBANK][M];
#pragma unroll
    for (int b = 0; b < NBANK; ++b) {
#pragma unroll
        for (int j = 0; j < L; ++j) carries[b][j] = 0;
#pragma unroll
        for (int i = 0; i < M; ++i) U[b][i] = 0;
        tot[b] = 0;
    }
    uint32_t nb = 0;
    for (unsigned long long t = 0; t < v.nv; t += STEP) {
        uint32_t r[REGS];
        seg_load<VB, VPT>(v, t, lane, r);
#pragma unroll
        for (int b = 0; b < NBANK; ++b)
            plane_count_add<M>(U[b], NBANK == 1 ? Tree<L, 1>::run(carries[b], r) : Tree<L, 2>::run(carries[b], r + b));
        if (++nb == (1u << M) - 1u) {
#pragma unroll
            for (int b = 0; b < NBANK; ++b)
#pragma unroll
                for (int i = 0; i < M; ++i) {
                    tot[b] += (unsigned long long)xp.column_popc(U[b][i]) << (L + i);
                    U[b][i] = 0;
                }
            nb = 0;
        }
    }
#pragma unroll
    for (int b = 0; b < NBANK; ++b) {
#pragma unroll
        for (int j = 0; j < L; ++j) tot[b] += (unsigned long long)xp.column_popc(carries[b][j]) << j;
#pragma unroll
        for (int i = 0; i < M; ++i) tot[b] += (unsigned long long)xp.column_popc(U[b][i]) << (L + i);
    }
}

// Publishes array `arr` of `bytes` bytes; false if the queue is full (the
// caller then counts it itself).  Warp-uniform.
__device__ __forceinline__ bool giant_publish(const GiantQueue& q, unsigned long long arr, unsigned long long bytes,
                                              uint32_t lane) {
    unsigned long long e = lane == 0 ? atomicAdd(q.base, 1ull) : 0ull;
    e = __shfl_sync(0xFFFFFFFFu, e, 0);
    if (e >= (unsigned long long)kGiantQ) return false;
    if (lane == 0) {
        unsigned long long* p = q.entry(e);
        p[0] = arr;
        p[1] = (bytes + q.chunk_bytes() - 1) / q.chunk_bytes();
        __threadfence();
        atomicExch(p + 3, 1ull);
    }
    __syncwarp();
    return true;
}

// Counts chunks of published arrays until no chunk is left to claim.
// Warp-uniform; called at a warp's exit.
template <int NBANK, int L, int VB>
__device__ __noinline__ void giant_help(const GiantQueue q, const uint8_t* data, const unsigned long long* offsets,
                                        int k, unsigned long long* out, uint32_t lane) {
    const int wb = k >> 3;
    unsigned long long cursor = 0;
    const unsigned long long cw = q.chunk_bytes() / (unsigned long long)wb;  // words per chunk
    const PlaneXpose xp(lane);
    for (;;) {
        unsigned long long cnt = __ldcg(q.base);
        if (cnt > (unsigned long long)kGiantQ) cnt = kGiantQ;
        if (cursor >= cnt) return;
        unsigned long long* p = q.entry(cursor);
        unsigned long long arr = 0, chunks = 0, c = 0;
        if (lane == 0 && atomicAdd(p + 3, 0ull) != 0ull) {  // published (else its publisher counts it)
            __threadfence();
            arr = __ldcg(p);
            chunks = __ldcg(p + 1);
            c = atomicAdd(p + 2, 1ull);
        }
        arr = __shfl_sync(0xFFFFFFFFu, arr, 0);
        chunks = __shfl_sync(0xFFFFFFFFu, chunks, 0);
        c = __shfl_sync(0xFFFFFFFFu, c, 0);
        if (c >= chunks) {  // no chunk left (or not published yet: never waited for)
            ++cursor;
            continue;
        }
        const unsigned long long w0 = offsets[arr] + c * cw, e1 = offsets[arr + 1];
        const unsigned long long w1 = w0 + cw < e1 ? w0 + cw : e1;
        unsigned long long tot[NBANK];
        seg_count_view<NBANK, L, VB>(seg_view<VB>(data, w0, w1, wb), lane, xp, tot);
        unsigned long long* acc = p + 4;
        unsigned long long v0 = tot[0];
        if (NBANK == 1)
            for (int w = 16; w >= k; w >>= 1) v0 += __shfl_down_sync(0xFFFFFFFFu, v0, w);
        if (NBANK == 2) {
            atomicAdd(acc + lane, v0);
            atomicAdd(acc + 32 + lane, tot[NBANK - 1]);
        } else if ((int)lane < k) {
            atomicAdd(acc + lane, v0);
        }
        __threadfence();
        __syncwarp();
        unsigned long long done = lane == 0 ? atomicAdd(p + 68, 1ull) : 0ull;
        done = __shfl_sync(0xFFFFFFFFu, done, 0);
        if (done + 1 == chunks) {  // the last chunk: move the counts into the row
            __threadfence();
            unsigned long long* row = out + arr * (unsigned long long)k;
            for (int ch = (int)lane; ch < k; ch += 32) row[ch] = atomicExch(acc + ch, 0ull);
            if (lane == 0) atomicExch(p + 68, 0ull);
        }
    }
}

// A warp meeting array `arr` (of `bytes` bytes): true if it was published to
// the giant queue (the caller skips it; every warp counts queued chunks when
// its own work is done -- giant_help at the warp's exit, where none of the
// schedule's registers are live -- and the publisher is among them, so every
// queued array is finished before the launch ends).
__device__ __forceinline__ bool giant_divert(const GiantQueue& q, unsigned long long arr, unsigned long long bytes,
                                             uint32_t lane) {
    if (!q.giant_bytes || bytes <= q.giant_bytes) return false;
    return giant_publish(q, arr, bytes, lane);
}

// End of a launch that may have used the claim counter and the giant queue:
// the last CTA (every warp has finished) resets both for the next launch.
__device__ __forceinline__ void seg_launch_done(unsigned long long* next, unsigned int* ticket, const GiantQueue& q) {
    __shared__ int s_last_q;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        s_last_q = atomicAdd(ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last_q) return;
    __threadfence();
    unsigned long long cnt = __ldcg(q.base);
    if (cnt > (unsigned long long)kGiantQ) cnt = kGiantQ;
    for (unsigned long long e = threadIdx.x; e < cnt; e += blockDim.x) {
        q.entry(e)[2] = 0ull;
        q.entry(e)[3] = 0ull;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        *q.base = 0ull;
        *next = 0ull;
        *ticket = 0u;
    }
}

template <int NBANK, int L, int VB, int EPI = 0, int HINT = 0>
__device__ __forceinline__ void segmented_pipe_body(const uint8_t* data, const unsigned long long* offsets,
                                                    unsigned long long n_arrays, int k, uint32_t flush_threshold,
                                                    unsigned long long* out) {
    constexpr int M = 3;  // EPI 1: bit-sliced tops counter, flushed every 2^M - 1 tree blocks
    constexpr int REGS = NBANK << L;
    constexpr int RPV = VB / 4;
    constexpr int VPT = REGS / RPV;
    constexpr unsigned long long STEP = 32ull * VPT;
    const uint32_t lane = threadIdx.x & 31u;
    const unsigned long long nwarps = (gridDim.x * (unsigned long long)blockDim.x) >> 5;
    const int wb = k >> 3;

    pdl_allow_next();
    pdl_wait_prev();  // the rows may belong to the previous launch on this stream
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
    uint32_t counter[NBANK][EPI ? 1 : 16];  // EPI 0: 16-lane counters
    uint32_t U[NBANK][M];                   // EPI 1: bit-sliced tops
#pragma unroll
    for (int b = 0; b < NBANK; ++b) {
#pragma unroll
        for (int j = 0; j < L; ++j) carries[b][j] = 0;
#pragma unroll
        for (int i = 0; i < M; ++i) U[b][i] = 0;
#pragma unroll
        for (int p = 0; p < (EPI ? 1 : 16); ++p) counter[b][p] = 0;
    }
    const PlaneXpose xp(lane);
    uint32_t nb = 0;
    unsigned long long tot[NBANK];
#pragma unroll
    for (int b = 0; b < NBANK; ++b) tot[b] = 0;

    unsigned long long t = 0;
    uint32_t rc[REGS];
    seg_load<VB, VPT, HINT>(cur, t, lane, rc);
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
        if (have_next) seg_load<VB, VPT, HINT>(nxt, t_n, lane, rn);

        if constexpr (EPI == 1) {
#pragma unroll
            for (int b = 0; b < NBANK; ++b)
                plane_count_add<M>(U[b], NBANK == 1 ? Tree<L, 1>::run(carries[b], rc)
                                                    : Tree<L, 2>::run(carries[b], rc + b));
            if (++nb == (1u << M) - 1u) {  // the tops counter is full: fold it into tot
#pragma unroll
                for (int b = 0; b < NBANK; ++b)
#pragma unroll
                    for (int i = 0; i < M; ++i) {
                        tot[b] += (unsigned long long)xp.column_popc(U[b][i]) << (L + i);
                        U[b][i] = 0;
                    }
                nb = 0;
            }
        } else {
            tree_block<NBANK, L>(rc, carries, reinterpret_cast<uint32_t(&)[NBANK][16]>(counter));
            if (++nb == flush_threshold) {
                uint32_t d[16];
#pragma unroll
                for (int p = 0; p < 16; ++p) d[p] = 0;
#pragma unroll
                for (int b = 0; b < NBANK; ++b)
                    tot[b] += bank_warp_total(reinterpret_cast<uint32_t(&)[16]>(counter[b]), L, d);
                zero_bank<NBANK>(reinterpret_cast<uint32_t(&)[NBANK][16]>(counter));
                nb = 0;
            }
        }
        if (t + STEP >= cur.nv) {  // last step of this array: epilogue while rn is in flight
            if constexpr (EPI == 1) {
#pragma unroll
                for (int b = 0; b < NBANK; ++b) {
#pragma unroll
                    for (int j = 0; j < L; ++j) {
                        tot[b] += (unsigned long long)xp.column_popc(carries[b][j]) << j;
                        carries[b][j] = 0;
                    }
#pragma unroll
                    for (int i = 0; i < M; ++i) {
                        tot[b] += (unsigned long long)xp.column_popc(U[b][i]) << (L + i);
                        U[b][i] = 0;
                    }
                }
            } else {
#pragma unroll
                for (int b = 0; b < NBANK; ++b) {
                    uint32_t d[16];
                    drain<L>(d, carries[b]);
                    tot[b] += bank_warp_total(reinterpret_cast<uint32_t(&)[16]>(counter[b]), L, d);
#pragma unroll
                    for (int j = 0; j < L; ++j) carries[b][j] = 0;
                }
                zero_bank<NBANK>(reinterpret_cast<uint32_t(&)[NBANK][16]>(counter));
            }
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

template <int NBANK, int L, int VB, int MINB = 1, int EPI = 0, int HINT = 0>
__global__ void __launch_bounds__(256, MINB) segmented_pipe_entry(const uint8_t* data, const unsigned long long* offsets,
                                                            unsigned long long n, int k, uint32_t thr,
                                                            unsigned long long* out, unsigned long long*,
                                                            unsigned int*, unsigned) {
    segmented_pipe_body<NBANK, L, VB, EPI, HINT>(data, offsets, n, k, thr, out);
}

// ---------------------------------------------------------------------------
// Multi-stage cp.async pipeline (SCHED 10): the warp-per-array walk of
// segmented_pipe_body, but the steps ahead live in a per-warp shared-memory
// ring of S slots filled with 16-byte cp.async copies (zero-filled past the
// array), so S-1 steps per warp are in flight without holding registers; the
// consumer reads its step with LDS.128.  No cross-warp synchronisation: each
// warp owns its ring (cp.async.wait_group + __syncwarp).
// ---------------------------------------------------------------------------
struct SegCursor {
    unsigned long long arr;  // n_arrays = exhausted
    unsigned long long t;    // first vector of the step
    SegView v;
};

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc, uint32_t src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_addr(smem_dst)), "l"(gsrc),
                 "r"(src_bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int NBANK>
__device__ __forceinline__ void seg_zero_row(unsigned long long* out, unsigned long long arr, int k, uint32_t lane) {
    unsigned long long z[NBANK];
#pragma unroll
    for (int b = 0; b < NBANK; ++b) z[b] = 0;
    seg_store_row<NBANK>(out, arr, k, lane, z);
}

// First non-empty array at or after `arr` (stride nwarps), zeroing the rows of
// empty arrays on the way; c.arr = n_arrays when none is left.
template <int NBANK>
__device__ __forceinline__ void seg_cursor_seek(SegCursor& c, unsigned long long arr, const uint8_t* data,
                                                const unsigned long long* offsets, unsigned long long n_arrays,
                                                unsigned long long nwarps, int k, unsigned long long* out,
                                                uint32_t lane) {
    const int wb = k >> 3;
    for (; arr < n_arrays; arr += nwarps) {
        c.v = seg_view<16>(data, offsets[arr], offsets[arr + 1], wb);
        if (c.v.nv) break;
        seg_zero_row<NBANK>(out, arr, k, lane);
    }
    c.arr = arr;
    c.t = 0;
}

template <int NBANK, int L, int S>
__device__ __forceinline__ void segmented_cpasync_body(const uint8_t* data, const unsigned long long* offsets,
                                                       unsigned long long n_arrays, int k, unsigned long long* out,
                                                       uint8_t* ring) {
    constexpr int M = 3;
    constexpr int REGS = NBANK << L;
    constexpr int VPT = REGS / 4;                     // 16-byte vectors per lane per step
    constexpr unsigned long long STEP = 32ull * VPT;  // vectors per step
    constexpr int SLOT = 32 * VPT * 16;               // bytes per ring slot
    const uint32_t lane = threadIdx.x & 31u;
    const unsigned long long nwarps = (gridDim.x * (unsigned long long)blockDim.x) >> 5;
    const unsigned long long warp = (blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x) >> 5;
    uint8_t* my = ring + (size_t)(threadIdx.x >> 5) * S * SLOT;

    SegCursor fetch;
    seg_cursor_seek<NBANK>(fetch, warp, data, offsets, n_arrays, nwarps, k, out, lane);
    SegCursor desc[S];
    auto issue = [&](int slot) {  // copy the fetch cursor's step into `slot`, then advance it
        if (fetch.arr < n_arrays) {
#pragma unroll
            for (int q = 0; q < VPT; ++q) {
                const unsigned long long idx = fetch.t + 32ull * q + lane;
                const bool in = idx < fetch.v.nv;
                POSPOP_CHECK(!in || idx < fetch.v.nv);
                cp_async16(my + slot * SLOT + (32 * q + lane) * 16, fetch.v.base + (in ? idx : 0) * 16, in ? 16u : 0u);
            }
        }
        cp_async_commit();  // one group per step, empty or not, so wait_group counts steps
        if (fetch.arr < n_arrays) {
            fetch.t += STEP;
            if (fetch.t >= fetch.v.nv)
                seg_cursor_seek<NBANK>(fetch, fetch.arr + nwarps, data, offsets, n_arrays, nwarps, k, out, lane);
        }
    };
#pragma unroll
    for (int s0 = 0; s0 < S - 1; ++s0) {
        desc[s0] = fetch;
        issue(s0);
    }

    uint32_t carries[NBANK][L];
    uint32_t U[NBANK][M];
#pragma unroll
    for (int b = 0; b < NBANK; ++b) {
#pragma unroll
        for (int j = 0; j < L; ++j) carries[b][j] = 0;
#pragma unroll
        for (int i = 0; i < M; ++i) U[b][i] = 0;
    }
    const PlaneXpose xp(lane);
    uint32_t nb = 0;
    unsigned long long tot[NBANK];
#pragma unroll
    for (int b = 0; b < NBANK; ++b) tot[b] = 0;

    for (bool more = true; more;) {
#pragma unroll
        for (int slot = 0; slot < S; ++slot) {  // unrolled: slot indices are compile-time
            constexpr int dummy = 0;
            (void)dummy;
            const int ahead = (slot + S - 1) % S;
            desc[ahead] = fetch;
            issue(ahead);
            cp_async_wait<S - 1>();  // this lane's copies of the step in `slot` have landed
            __syncwarp();            // ... and every other lane's
            const SegCursor& d = desc[slot];
            if (d.arr >= n_arrays) {
                more = false;
                break;
            }
            uint32_t r[REGS];
#pragma unroll
            for (int q = 0; q < VPT; ++q) {
                const unsigned long long idx = d.t + 32ull * q + lane;
                uint32_t x[4];
                asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                             : "=r"(x[0]), "=r"(x[1]), "=r"(x[2]), "=r"(x[3])
                             : "r"(smem_addr(my + slot * SLOT + (32 * q + lane) * 16)));
                if (idx == 0 || idx + 1 == d.v.nv) mask_bytes<16>(x, idx == 0 ? d.v.lo : 0, idx + 1 == d.v.nv ? d.v.hi : 16);
#pragma unroll
                for (int j = 0; j < 4; ++j) r[q * 4 + j] = x[j];
            }
            __syncwarp();  // the slot may be refilled once every lane has read it
#pragma unroll
            for (int b = 0; b < NBANK; ++b)
                plane_count_add<M>(U[b], NBANK == 1 ? Tree<L, 1>::run(carries[b], r) : Tree<L, 2>::run(carries[b], r + b));
            if (++nb == (1u << M) - 1u) {
#pragma unroll
                for (int b = 0; b < NBANK; ++b)
#pragma unroll
                    for (int i = 0; i < M; ++i) {
                        tot[b] += (unsigned long long)xp.column_popc(U[b][i]) << (L + i);
                        U[b][i] = 0;
                    }
                nb = 0;
            }
            if (d.t + STEP >= d.v.nv) {  // the array's last step: bit-plane epilogue and row store
#pragma unroll
                for (int b = 0; b < NBANK; ++b) {
#pragma unroll
                    for (int j = 0; j < L; ++j) {
                        tot[b] += (unsigned long long)xp.column_popc(carries[b][j]) << j;
                        carries[b][j] = 0;
                    }
#pragma unroll
                    for (int i = 0; i < M; ++i) {
                        tot[b] += (unsigned long long)xp.column_popc(U[b][i]) << (L + i);
                        U[b][i] = 0;
                    }
                }
                nb = 0;
                seg_store_row<NBANK>(out, d.arr, k, lane, tot);
#pragma unroll
                for (int b = 0; b < NBANK; ++b) tot[b] = 0;
            }
        }
    }
    cp_async_wait<0>();
}

template <int NBANK, int L, int S>
__global__ void __launch_bounds__(256, 2) segmented_cpasync_kernel(const uint8_t* data,
                                                                   const unsigned long long* offsets,
                                                                   unsigned long long n_arrays, int k, uint32_t,
                                                                   unsigned long long* out, unsigned long long*,
                                                                   unsigned int*, unsigned) {
    extern __shared__ __align__(16) uint8_t seg_ring[];
    pdl_allow_next();
    pdl_wait_prev();  // the rows may belong to the previous launch on this stream
    segmented_cpasync_body<NBANK, L, S>(data, offsets, n_arrays, k, out, seg_ring);
}

// ---------------------------------------------------------------------------
// Grouped segmented kernel (SCHED 4): G lanes per array, so one warp counts
// 32/G arrays at once and the per-array epilogue (drain + reduction + row
// store) is shared by 32/G arrays instead of paid per array by the whole
// warp.  Warps claim batches of 32/G consecutive arrays from a global counter
// (prefetched one batch ahead); a batch holding an array longer than
// `big_vectors` is counted one array at a time by all 32 lanes instead, so a
// few large arrays do not leave most lanes idle.
// ---------------------------------------------------------------------------

// Reduction over aligned groups of G lanes: each lane holds v[32] (channel c
// in v[c]); afterwards lane gl (= lane mod G) holds the group sums of channels
// [gl*32/G, (gl+1)*32/G) in v[0 .. 32/G).  Shuffle distances stay inside the
// group; all 32 lanes must call it together.
template <int G, int S = 0>
__device__ __forceinline__ void group_transpose_reduce(uint32_t (&v)[32], uint32_t lane) {
    if constexpr ((G >> (S + 1)) >= 1) {
        constexpr int D = G >> (S + 1);  // shuffle distance
        constexpr int H = 16 >> S;       // values kept: n/2
        const bool upper = (lane & D) != 0;
#pragma unroll
        for (int i = 0; i < H; ++i) {
            const uint32_t send = upper ? v[i] : v[i + H];
            const uint32_t keep = upper ? v[i + H] : v[i];
            v[i] = keep + __shfl_xor_sync(0xFFFFFFFFu, send, D);
        }
        group_transpose_reduce<G, S + 1>(v, lane);
    }
}

// tot[m] += group sum of channel gl*32/G + m of (counter << shift) + d.
template <int G>
__device__ __forceinline__ void group_bank_total(const uint32_t (&counter)[16], int shift, const uint32_t (&d)[16],
                                                 unsigned long long (&tot)[32 / G], uint32_t lane) {
    uint32_t v[32];
#pragma unroll
    for (int p = 0; p < 16; ++p) {
        v[p] = ((counter[p] & 0xFFFFu) << shift) + (d[p] & 0xFFFFu);
        v[p + 16] = ((counter[p] >> 16) << shift) + (d[p] >> 16);
    }
    group_transpose_reduce<G>(v, lane);
#pragma unroll
    for (int m = 0; m < 32 / G; ++m) tot[m] += v[m];
}

// Counts arrays a0 + lane/GX (one per group of GX lanes) and stores their rows.
template <int NBANK, int L, int VB, int GX>
__device__ __forceinline__ void seg_group_batch(const uint8_t* data, const unsigned long long* offsets,
                                                unsigned long long a0, unsigned long long n_arrays, int k,
                                                uint32_t flush_threshold, unsigned long long* out, uint32_t lane) {
    static_assert(GX >= 4 && GX <= 32 && (GX & (GX - 1)) == 0, "4..32 lanes per array");
    constexpr int REGS = NBANK << L;
    constexpr int RPV = VB / 4;
    constexpr int VPT = REGS / RPV;
    constexpr int W = 32 / GX;                                    // channels per lane after the reduction
    constexpr unsigned long long STEP = (unsigned long long)GX * VPT;  // vectors per group per tree block
    const uint32_t gl = lane % GX;
    const unsigned long long a = a0 + lane / GX;
    const int wb = k >> 3;
    SegView v;
    if (a < n_arrays) {
        v = seg_view<VB>(data, offsets[a], offsets[a + 1], wb);
    } else {
        v.base = data;
        v.nv = v.f0 = v.f1 = 0;
        v.lo = 0;
        v.hi = VB;
    }
    uint32_t carries[NBANK][L];
    uint32_t counter[NBANK][16];
#pragma unroll
    for (int b = 0; b < NBANK; ++b)
#pragma unroll
        for (int j = 0; j < L; ++j) carries[b][j] = 0;
    zero_bank<NBANK>(counter);
    unsigned long long tot[NBANK][W];
#pragma unroll
    for (int b = 0; b < NBANK; ++b)
#pragma unroll
        for (int m = 0; m < W; ++m) tot[b][m] = 0;
    uint32_t nb = 0;
    // Lockstep over the batch: groups whose array is done read zeros.
    for (unsigned long long t = 0; __any_sync(0xFFFFFFFFu, t < v.nv); t += STEP) {
        uint32_t r[REGS];
        if (t >= v.f0 && t + STEP <= v.f1) {
#pragma unroll
            for (int q = 0; q < VPT; ++q) {
                uint32_t x[RPV];
                POSPOP_CHECK(t + (unsigned long long)GX * q + gl < v.nv);
                ldg_stream<VB, 0>(v.base + (t + (unsigned long long)GX * q + gl) * VB, x);
#pragma unroll
                for (int j = 0; j < RPV; ++j) r[q * RPV + j] = x[j];
            }
        } else {
#pragma unroll
            for (int q = 0; q < VPT; ++q) {
                const unsigned long long idx = t + (unsigned long long)GX * q + gl;
                uint32_t x[RPV];
#pragma unroll
                for (int j = 0; j < RPV; ++j) x[j] = 0;
                if (idx < v.nv) {
                    ldg_stream<VB, 0>(v.base + idx * VB, x);
                    if (idx == 0 || idx + 1 == v.nv)
                        mask_bytes<VB>(x, idx == 0 ? v.lo : 0, idx + 1 == v.nv ? v.hi : VB);
                }
#pragma unroll
                for (int j = 0; j < RPV; ++j) r[q * RPV + j] = x[j];
            }
        }
        tree_block<NBANK, L>(r, carries, counter);
        if (++nb == flush_threshold) {  // warp-uniform
            uint32_t d[16];
#pragma unroll
            for (int p = 0; p < 16; ++p) d[p] = 0;
#pragma unroll
            for (int b = 0; b < NBANK; ++b) group_bank_total<GX>(counter[b], L, d, tot[b], lane);
            zero_bank<NBANK>(counter);
            nb = 0;
        }
    }
#pragma unroll
    for (int b = 0; b < NBANK; ++b) {
        uint32_t d[16];
        drain<L>(d, carries[b]);
        group_bank_total<GX>(counter[b], L, d, tot[b], lane);
    }
    // Fold channels to positions inside the group (k = 16: c, c+16; k = 8:
    // c, c+8, c+16, c+24) and store: lane gl owns channels [gl*W, gl*W + W).
    if (NBANK == 1) {
#pragma unroll
        for (int m = 0; m < W; ++m)
            for (int w = 16; w >= k; w >>= 1) tot[0][m] += __shfl_xor_sync(0xFFFFFFFFu, tot[0][m], w / W);
    }
    if (a < n_arrays && (int)(gl * W) < (NBANK == 2 ? 32 : k)) {
        unsigned long long* row = out + a * (unsigned long long)k + gl * W;
#pragma unroll
        for (int b = 0; b < NBANK; ++b)
#pragma unroll
            for (int m = 0; m < W; ++m) row[32 * b + m] = tot[b][m];
    }
}

// The claim loop of the grouped schedule (device function so the adaptive
// kernel below can run it too).  `next` must be zero on entry.
template <int NBANK, int L, int VB, int G>
__device__ __forceinline__ void seg_group_loop(const uint8_t* data, const unsigned long long* offsets,
                                               unsigned long long n_arrays, int k, uint32_t flush_threshold,
                                               unsigned long long* out, unsigned long long* next,
                                               unsigned big_vectors, unsigned long long giant_bytes = 0) {
    constexpr int NG = 32 / G;  // arrays per batch
    const uint32_t lane = threadIdx.x & 31u;
    const int wb = k >> 3;
    const GiantQueue q = seg_giant_queue(next, giant_bytes);
    unsigned long long mine = lane == 0 ? atomicAdd(next, 1ull) : 0ull;
    unsigned long long b = __shfl_sync(0xFFFFFFFFu, mine, 0);
    mine = lane == 0 ? atomicAdd(next, 1ull) : 0ull;
    for (;;) {
        const unsigned long long a0 = b * NG;
        if (a0 >= n_arrays) break;  // warp-uniform
        // Does the batch hold an array too long for G lanes?
        unsigned long long nbytes = 0;
        if (lane < (uint32_t)NG && a0 + lane < n_arrays) nbytes = (offsets[a0 + lane + 1] - offsets[a0 + lane]) * wb;
        if (!__any_sync(0xFFFFFFFFu, nbytes > (unsigned long long)big_vectors * VB)) {
            seg_group_batch<NBANK, L, VB, G>(data, offsets, a0, n_arrays, k, flush_threshold, out, lane);
        } else {
            for (int j = 0; j < NG; ++j) {
                if (a0 + j >= n_arrays) break;
                const unsigned long long bytes = __shfl_sync(0xFFFFFFFFu, nbytes, j);
                if (!giant_divert(q, a0 + j, bytes, lane))
                    seg_group_batch<NBANK, L, VB, 32>(data, offsets, a0 + j, n_arrays, k, flush_threshold, out, lane);
            }
        }
        b = __shfl_sync(0xFFFFFFFFu, mine, 0);
        mine = lane == 0 ? atomicAdd(next, 1ull) : 0ull;
    }
    if (giant_bytes) giant_help<NBANK, NBANK == 1 ? 5 : 4, 16>(q, data, offsets, k, out, lane);
}

template <int NBANK, int L, int VB, int G, int MINB>
__global__ void __launch_bounds__(256, MINB) segmented_group_kernel(const uint8_t* data,
                                                                    const unsigned long long* offsets,
                                                                    unsigned long long n_arrays, int k,
                                                                    uint32_t flush_threshold, unsigned long long* out,
                                                                    unsigned long long* next, unsigned int* ticket,
                                                                    unsigned big_vectors) {
    pdl_allow_next();
    pdl_wait_prev();  // the claim counter, the ticket and the rows may belong to the previous launch
    seg_group_loop<NBANK, L, VB, G>(data, offsets, n_arrays, k, flush_threshold, out, next, big_vectors);
    seg_claims_done(next, ticket);
}

// ---------------------------------------------------------------------------
// One lane per array (tiny arrays): each lane walks its own array's 16-byte
// vectors (masked edges), a depth-3 tree over pairs of vectors (k = 64: two
// depth-2 banks), then drains and writes its own row -- no cross-lane
// reduction at all.  Adjacent lanes take adjacent arrays, so a warp's loads
// stay within one contiguous region.  Lanes stay within 16-bit counters for
// arrays up to 2 MiB; the caller keeps arrays above `lane_cap_bytes` on the
// full-warp path.
// ---------------------------------------------------------------------------
#ifndef POSPOP_LANE_HINT
#define POSPOP_LANE_HINT 3  // L1-allocating: lanes read half sectors (64-word arrays 1626 -> 2205 GB/s)
#endif
// Counts array `a` (nothing when !valid) on this lane and hands each bank's
// 32 channel totals to sink(bank, ch).
template <int NBANK, class Sink>
__device__ __forceinline__ void seg_lane_counts(const uint8_t* data, const unsigned long long* offsets,
                                                unsigned long long a, bool valid, int k, Sink&& sink) {
    constexpr int L = NBANK == 1 ? 3 : 2;
    constexpr int REGS = NBANK << L;  // 8 registers = two 16-byte vectors
    constexpr int VPT = REGS / 4;
    const int wb = k >> 3;
    SegView v;
    if (valid) {
        v = seg_view<16>(data, offsets[a], offsets[a + 1], wb);
    } else {
        v.base = data;
        v.nv = v.f0 = v.f1 = 0;
        v.lo = 0;
        v.hi = 16;
    }
    uint32_t carries[NBANK][L];
    uint32_t counter[NBANK][16];
#pragma unroll
    for (int b = 0; b < NBANK; ++b)
#pragma unroll
        for (int j = 0; j < L; ++j) carries[b][j] = 0;
    zero_bank<NBANK>(counter);
    for (unsigned long long t = 0; t < v.nv; t += VPT) {
        uint32_t r[REGS];
#pragma unroll
        for (int q = 0; q < VPT; ++q) {
            const unsigned long long idx = t + q;
            uint32_t x[4] = {0u, 0u, 0u, 0u};
            if (idx < v.nv) {
                POSPOP_CHECK(idx < v.nv);
                ldg_stream<16, POSPOP_LANE_HINT>(v.base + idx * 16, x);
                if (idx == 0 || idx + 1 == v.nv) mask_bytes<16>(x, idx == 0 ? v.lo : 0, idx + 1 == v.nv ? v.hi : 16);
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) r[q * 4 + j] = x[j];
        }
        tree_block<NBANK, L>(r, carries, counter);
    }
#pragma unroll
    for (int b = 0; b < NBANK; ++b) {
        uint32_t d[16];
        drain<L>(d, carries[b]);
        uint32_t ch[32];
#pragma unroll
        for (int p = 0; p < 16; ++p) {
            ch[p] = ((counter[b][p] & 0xFFFFu) << L) + (d[p] & 0xFFFFu);
            ch[p + 16] = ((counter[b][p] >> 16) << L) + (d[p] >> 16);
        }
        sink(b, ch);
    }
}

// Array a's row written straight to `row` (any 8-byte-aligned address).
template <int NBANK>
__device__ __forceinline__ void seg_lane_array(const uint8_t* data, const unsigned long long* offsets,
                                               unsigned long long a, int k, unsigned long long* row) {
    seg_lane_counts<NBANK>(data, offsets, a, true, k, [&](int b, const uint32_t (&ch)[32]) {
        if (NBANK == 2 || k == 32) {
#pragma unroll
            for (int c = 0; c < 32; ++c) row[32 * b + c] = ch[c];
        } else if (k == 16) {
#pragma unroll
            for (int p = 0; p < 16; ++p) row[p] = (unsigned long long)ch[p] + ch[p + 16];
        } else {  // k == 8: channels p, p+8, p+16, p+24
#pragma unroll
            for (int p = 0; p < 8; ++p) row[p] = (unsigned long long)ch[p] + ch[p + 8] + ch[p + 16] + ch[p + 24];
        }
    });
}

// Rows staged per warp at a time in the lane mode (stride (min(k, 32) * 8 +
// 16) bytes): all 32 for the short rows of k <= 16, 16 for k = 32, 8 bank
// halves for k = 64 -- the stage's carve-out takes L1 from every mode of the
// adaptive kernel.  The launcher sizes the dynamic shared
// memory with the same rule.
__host__ __device__ __forceinline__ int seg_stage_rows(int k) { return k <= 16 ? 32 : k == 32 ? 16 : 8; }

// Copies `rows` staged rows of `half_bytes` each (stage stride `rowb`) to
// dst + r * dst_stride with coalesced 16-byte stores (two 8-byte stores when
// dst is only 8-byte aligned).  The whole warp.
__device__ __forceinline__ void seg_copy_staged(const uint8_t* wbuf, int rowb, int rows, int half_bytes, uint8_t* dst,
                                                size_t dst_stride, uint32_t lane) {
    const int cpr = half_bytes / 16;  // 16-byte chunks per row
    const bool v16 = (reinterpret_cast<uintptr_t>(dst) & 15u) == 0 && (dst_stride & 15u) == 0;
    for (int i = (int)lane; i < rows * cpr; i += 32) {
        const int r = i / cpr, c = i - r * cpr;
        const uint4 v = *reinterpret_cast<const uint4*>(wbuf + r * rowb + c * 16);
        uint8_t* p = dst + (size_t)r * dst_stride + (size_t)c * 16;
        if (v16) {
            *reinterpret_cast<uint4*>(p) = v;
        } else {
            reinterpret_cast<unsigned long long*>(p)[0] = ((unsigned long long)v.y << 32) | v.x;
            reinterpret_cast<unsigned long long*>(p)[1] = ((unsigned long long)v.w << 32) | v.z;
        }
    }
}

// Lane mode claim loop: batches of 32 consecutive arrays per warp; a batch
// holding an array above lane_cap_bytes is counted array by array by the
// whole warp instead.
// With `stage` (shared memory, k <= 32: 32 rows of k*8 + 16 bytes per warp --
// the 16-byte pad keeps each quarter-warp's row stores on distinct banks) the
// warp's 32 rows are written to shared memory first and then copied out as one
// contiguous block with coalesced 16-byte stores, instead of 32 scattered rows.
template <int NBANK, int LW, int VBW>
__device__ __forceinline__ void seg_lane_loop(const uint8_t* data, const unsigned long long* offsets,
                                              unsigned long long n_arrays, int k, uint32_t flush_threshold,
                                              unsigned long long* out, unsigned long long* next,
                                              unsigned long long lane_cap_bytes, uint8_t* stage,
                                              unsigned long long giant_bytes = 0) {
    const uint32_t lane = threadIdx.x & 31u;
    const int wb = k >> 3;
    const GiantQueue q = seg_giant_queue(next, giant_bytes);
    const int rowb = (k > 32 ? 32 : k) * 8 + 16;  // staged row stride, bytes (k = 64: half rows, one bank at a time)
    uint8_t* wbuf = stage ? stage + (threadIdx.x >> 5) * seg_stage_rows(k) * rowb : nullptr;
    unsigned long long mine = lane == 0 ? atomicAdd(next, 1ull) : 0ull;
    unsigned long long b = __shfl_sync(0xFFFFFFFFu, mine, 0);
    mine = lane == 0 ? atomicAdd(next, 1ull) : 0ull;
    for (;;) {
        const unsigned long long a0 = b * 32;
        if (a0 >= n_arrays) break;  // warp-uniform
        const unsigned long long a = a0 + lane;
        const unsigned long long nbytes = a < n_arrays ? (offsets[a + 1] - offsets[a]) * wb : 0;
        if (!__any_sync(0xFFFFFFFFu, nbytes > lane_cap_bytes)) {
            if (wbuf) {
                const unsigned long long left = n_arrays - a0;
                const int rows = left < 32 ? (int)left : 32;
                uint8_t* dst = reinterpret_cast<uint8_t*>(out + a0 * (unsigned long long)k);
                // `rp` rows at a time (k = 64: their 256-byte bank halves): a small stage keeps the L1 that
                // the other modes' in-flight loads need
                const size_t row_bytes = (size_t)k * 8;
                const int rp = seg_stage_rows(k);
                seg_lane_counts<NBANK>(data, offsets, a, a < n_arrays, k, [&](int bank, const uint32_t (&ch)[32]) {
#pragma unroll 1
                    for (int g = 0; g < 32 / rp; ++g) {
                        if ((int)lane / rp == g) {
                            unsigned long long* srow =
                                reinterpret_cast<unsigned long long*>(wbuf + ((int)lane - g * rp) * rowb);
                            if (NBANK == 2 || k == 32) {
#pragma unroll
                                for (int c = 0; c < 32; ++c) srow[c] = ch[c];
                            } else if (k == 16) {
#pragma unroll
                                for (int p = 0; p < 16; ++p) srow[p] = (unsigned long long)ch[p] + ch[p + 16];
                            } else {  // k == 8
#pragma unroll
                                for (int p = 0; p < 8; ++p)
                                    srow[p] = (unsigned long long)ch[p] + ch[p + 8] + ch[p + 16] + ch[p + 24];
                            }
                        }
                        __syncwarp();
                        const int gr = rows - rp * g;
                        if (gr > 0)
                            seg_copy_staged(wbuf, rowb, gr < rp ? gr : rp, NBANK == 2 ? 256 : (int)row_bytes,
                                            dst + (NBANK == 2 ? 256 * bank : 0) + rp * g * row_bytes, row_bytes, lane);
                        __syncwarp();
                    }
                });
            } else if (a < n_arrays) {
                seg_lane_array<NBANK>(data, offsets, a, k, out + a * (unsigned long long)k);
            }
        } else {
            for (int j = 0; j < 32; ++j) {
                if (a0 + j >= n_arrays) break;
                const unsigned long long bytes = __shfl_sync(0xFFFFFFFFu, nbytes, j);
                if (!giant_divert(q, a0 + j, bytes, lane))
                    seg_group_batch<NBANK, LW, VBW, 32>(data, offsets, a0 + j, n_arrays, k, flush_threshold, out, lane);
            }
        }
        b = __shfl_sync(0xFFFFFFFFu, mine, 0);
        mine = lane == 0 ? atomicAdd(next, 1ull) : 0ull;
    }
    if (giant_bytes) giant_help<NBANK, NBANK == 1 ? 5 : 4, 16>(q, data, offsets, k, out, lane);
}

// ---------------------------------------------------------------------------
// Warp-per-array tiles (SCHED 11): the stream kernel's shape applied to
// arrays.  A step is one full-depth tree block per lane (2^L registers, e.g.
// 16 x 32-byte loads at L = 7: 16 KiB per warp, one cfg5 u32 array), issued
// all at once and consumed once it lands; latency is hidden by the other
// warps of the SM, not by a register double buffer, so a deeper tree fits and
// no registers are copied between steps.  The warp's next array offsets are
// fetched one array ahead.  Counts are kept as bit planes (tree carries + a
// 3-plane tops counter, folded every 7 blocks) and reduced with the warp bit
// transpose (PlaneXpose), as in the pipelined kernel's EPI 1.
// ---------------------------------------------------------------------------
// Array order of one warp: `arr`, arr + stride, ... while below static_end,
// then (dyn) single arrays claimed from the global counter `next` -- the last
// rounds go to whichever warps finish first.  Claims are made one array ahead
// (the following array's bounds are prefetched with it), and only after the
// previous launch has completed (the counter is shared with it).
struct TileCursor {
    unsigned long long stride, static_end, n;
    unsigned long long* next;
    bool dyn;
    __device__ __forceinline__ bool claims(unsigned long long a) const { return dyn && a + stride >= static_end; }
    __device__ __forceinline__ unsigned long long claim(uint32_t lane) const {  // warp-uniform
        unsigned long long c = lane == 0 ? atomicAdd(next, 1ull) : 0ull;
        c = __shfl_sync(0xFFFFFFFFu, c, 0);
        return static_end + c < n ? static_end + c : n;
    }
    __device__ __forceinline__ unsigned long long following(unsigned long long a, uint32_t lane) const {
        if (a + stride < static_end) return a + stride;
        if (!dyn) return a + stride < n ? a + stride : n;
        return claim(lane);
    }
};

// EARLY: everything before the first row store -- reading the offsets and
// data and counting the first array -- overlaps the previous launch on the
// stream (programmatic dependent launch); the first row store, the first
// dynamic claim and the warp's exit wait for it, so global rows (and the
// claim counter) are only touched after the previous launch has completed.
// (Parking the rows finished before the wait in shared memory, so that the
// warp need not wait at its first store, measured slower: the carve-out it
// takes shrinks the L1 that stages the in-flight loads.)
#ifdef POSPOP_TUNING
// Diagnostics (tuning build only, tools/seg_trace.py): per warp of the tile
// mode {entry, first array counted, previous launch waited for, exit, SM id}
// in %globaltimer ns; set with pospop_tuning_seg_trace().
__device__ unsigned long long* g_seg_trace = nullptr;
#define POSPOP_SEG_STAMP(i, v)                                                                          \
    do {                                                                                                \
        if (g_seg_trace && (threadIdx.x & 31u) == 0)                                                    \
            g_seg_trace[(((unsigned long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 5 + (i)] = (v); \
    } while (0)
#else
#define POSPOP_SEG_STAMP(i, v) \
    do {                       \
    } while (0)
#endif

template <int NBANK, int L, int VB, bool EARLY = false>
__device__ __forceinline__ void seg_tile_loop(const uint8_t* data, const unsigned long long* offsets,
                                              unsigned long long n_arrays, int k, unsigned long long* out,
                                              unsigned long long arr, const TileCursor& cur,
                                              unsigned long long giant_bytes = 0) {
    constexpr int M = 3;
    constexpr int REGS = NBANK << L;
    constexpr int RPV = VB / 4;
    constexpr int VPT = REGS / RPV;
    constexpr unsigned long long STEP = 32ull * VPT;
    const uint32_t lane = threadIdx.x & 31u;
    const int wb = k >> 3;
    const PlaneXpose xp(lane);
    bool waited = !EARLY;
    POSPOP_SEG_STAMP(0, globaltimer());
    POSPOP_SEG_STAMP(4, smid());
    auto ensure_waited = [&]() {
        if (!waited) {
            POSPOP_SEG_STAMP(1, globaltimer());
            pdl_wait_prev();
            POSPOP_SEG_STAMP(2, globaltimer());
            waited = true;
        }
    };
    auto store = [&](unsigned long long a, const unsigned long long (&tot)[NBANK]) {
        ensure_waited();
        seg_store_row<NBANK>(out, a, k, lane, tot);
    };
    auto next_of = [&](unsigned long long a) {
        if (cur.claims(a)) ensure_waited();  // the claim counter belongs to the previous launch until it completes
        return cur.following(a, lane);
    };
    // giant arrays go through the queue (which belongs to the previous launch until it completes)
    const GiantQueue q = seg_giant_queue(cur.next, giant_bytes);
    auto diverted = [&](unsigned long long a, unsigned long long w0, unsigned long long w1) {
        if (!giant_bytes || (w1 - w0) * (unsigned long long)wb <= giant_bytes) return false;
        ensure_waited();
        return giant_divert(q, a, (w1 - w0) * (unsigned long long)wb, lane);
    };
    auto finish_warp = [&]() {
        ensure_waited();
        if (giant_bytes) giant_help<NBANK, NBANK == 1 ? 5 : 4, 16>(q, data, offsets, k, out, lane);
        POSPOP_SEG_STAMP(3, globaltimer());
    };
    const unsigned long long zero[NBANK] = {};
    if (arr >= cur.static_end) {  // this warp has no static array
        if (cur.dyn) {
            ensure_waited();  // the claim counter belongs to the previous launch until it completes
            arr = cur.claim(lane);
        } else {
            arr = n_arrays;
        }
    }
    // The loads of the next step -- later in this array or the first step of
    // the warp's next non-empty array -- are issued as soon as the tree has
    // consumed the registers, before the array's epilogue runs, so the warp
    // keeps its memory requests in flight across array boundaries.
    SegView v;
    for (;; arr = next_of(arr)) {  // first non-empty array
        if (arr >= n_arrays) {
            finish_warp();
            return;
        }
        const unsigned long long a_w0 = offsets[arr], a_w1 = offsets[arr + 1];
        if (diverted(arr, a_w0, a_w1)) continue;
        v = seg_view<VB>(data, a_w0, a_w1, wb);
        if (v.nv) break;
        store(arr, zero);
    }
    unsigned long long nxt = next_of(arr), w0 = 0, w1 = 0;  // the array after it, bounds prefetched
    if (nxt < n_arrays) {
        w0 = offsets[nxt];
        w1 = offsets[nxt + 1];
    }
    uint32_t carries[NBANK][L], U[NBANK][M];
    unsigned long long tot[NBANK];
#pragma unroll
    for (int b = 0; b < NBANK; ++b) {
#pragma unroll
        for (int j = 0; j < L; ++j) carries[b][j] = 0;
#pragma unroll
        for (int i = 0; i < M; ++i) U[b][i] = 0;
        tot[b] = 0;
    }
    uint32_t nb = 0;
    unsigned long long t = 0;
    uint32_t r[REGS];
    seg_load<VB, VPT>(v, t, lane, r);
    for (;;) {
#pragma unroll
        for (int b = 0; b < NBANK; ++b)
            plane_count_add<M>(U[b], NBANK == 1 ? Tree<L, 1>::run(carries[b], r) : Tree<L, 2>::run(carries[b], r + b));
        ++nb;
        t += STEP;
        const bool array_done = t >= v.nv;
        unsigned long long arr_n = arr;
        SegView vn = v;
        bool more = true;
        if (array_done) {  // the warp's next non-empty array (rows of empty ones are zeroed on the way)
            t = 0;
            more = false;
            while (nxt < n_arrays) {
                arr_n = nxt;
                const unsigned long long n_w0 = w0, n_w1 = w1;
                vn = seg_view<VB>(data, n_w0, n_w1, wb);
                nxt = next_of(arr_n);
                if (nxt < n_arrays) {
                    w0 = offsets[nxt];
                    w1 = offsets[nxt + 1];
                }
                if (diverted(arr_n, n_w0, n_w1)) continue;
                if (vn.nv) {
                    more = true;
                    break;
                }
                store(arr_n, zero);
            }
        }
        if (more) seg_load<VB, VPT>(vn, t, lane, r);  // in flight during the fold / epilogue below
        if (array_done || nb == (1u << M) - 1u) {  // warp-uniform: the step count is per array
#pragma unroll
            for (int b = 0; b < NBANK; ++b)
#pragma unroll
                for (int i = 0; i < M; ++i) {
                    tot[b] += (unsigned long long)xp.column_popc(U[b][i]) << (L + i);
                    U[b][i] = 0;
                }
            nb = 0;
        }
        if (array_done) {
#pragma unroll
            for (int b = 0; b < NBANK; ++b) {
#pragma unroll
                for (int j = 0; j < L; ++j) {
                    tot[b] += (unsigned long long)xp.column_popc(carries[b][j]) << j;
                    carries[b][j] = 0;
                }
            }
            store(arr, tot);
#pragma unroll
            for (int b = 0; b < NBANK; ++b) tot[b] = 0;
            if (!more) {
                finish_warp();
                return;
            }
            arr = arr_n;
            v = vn;
        }
    }
}

// Grid-strided tile schedule: warp w of the grid takes arrays w, w + nwarps,
// ... (the whole GPU sweeps one window of consecutive arrays); with DYN the
// last `tail_rounds` rounds are claimed dynamically from `next`.
template <int NBANK, int L, int VB, bool EARLY, bool DYN>
__device__ __forceinline__ void seg_tile_strided(const uint8_t* data, const unsigned long long* offsets,
                                                 unsigned long long n_arrays, int k, unsigned long long* out,
                                                 unsigned long long* next, unsigned tail_rounds) {
    const unsigned long long warp = (blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x) >> 5;
    const unsigned long long nwarps = (gridDim.x * (unsigned long long)blockDim.x) >> 5;
    const unsigned long long rounds = n_arrays / nwarps;
    TileCursor cur;
    cur.next = next;
    cur.dyn = DYN;
    cur.stride = nwarps;
    cur.n = n_arrays;
    cur.static_end = DYN ? (rounds > tail_rounds ? rounds - tail_rounds : 0) * nwarps : n_arrays;
    seg_tile_loop<NBANK, L, VB, EARLY>(data, offsets, n_arrays, k, out, warp, cur);
}

// ---------------------------------------------------------------------------
// Range mode (few or huge arrays): the referenced bytes [data + off[0]*wb,
// data + off[n]*wb) are split into one contiguous, 16-byte-aligned range per
// CTA (equal bytes), so an array of any size is spread over as many SMs as it
// covers.  The CTA's warps count its range together: a 32-ary warp search over
// the offsets finds the first array touching the range, then the CTA walks
// the range's arrays in order, every thread loading vectors tid, tid +
// nthreads, ... of each step (one contiguous window per CTA step, like the
// stream kernel's CTA tiles; the next step's loads -- possibly the next
// array's -- are issued before a segment's epilogue).  At the end of a segment
// the warps' counts are summed in shared memory; warp 0 stores the row of an
// array inside the range, or adds the partial counts of an array spanning
// ranges into that array's workspace slot (u64 atomics; slot = array index)
// and, if its range completes the array (a per-slot counter of the ranges it
// covers), moves the slot into the row with atomicExch, leaving the slot zero
// for the next launch.  Empty arrays are written by the CTA owning their
// position.  Starts before the previous launch completes (EARLY semantics:
// the first row store / slot update waits for it).
// ---------------------------------------------------------------------------
struct RangeSplit {
    unsigned long long base, total;  // byte positions relative to data: [base, base + total)
    unsigned long long W;            // ranges (CTAs taking part)
    // Start of range w (w <= W), 16-byte aligned in absolute address for w >= 1.
    __device__ __forceinline__ unsigned long long start(unsigned long long w) const {
        if (w >= W) return base + total;
        return base + (((total * w) / W) & ~15ull);
    }
    // The range holding position p (base <= p < base + total); empty ranges hold none.
    __device__ __forceinline__ unsigned long long owner(unsigned long long p) const {
        unsigned long long w = total ? (p - base) * W / total : 0;
        if (w >= W) w = W - 1;
        while (w > 0 && start(w) > p) --w;
        while (w + 1 < W && start(w + 1) <= p) ++w;
        return w;
    }
};

template <int NBANK, int L, int VB>
__device__ __forceinline__ void seg_range_loop(const uint8_t* data, const unsigned long long* offsets,
                                               unsigned long long n_arrays, int k, unsigned long long* out,
                                               unsigned long long* next) {
    constexpr int M = 3;
    constexpr int REGS = NBANK << L;
    constexpr int RPV = VB / 4;
    constexpr int VPT = REGS / RPV;
    constexpr int kMaxWarps = 8;  // blockDim.x <= 256
    __shared__ unsigned long long s_tot[kMaxWarps][64];
    const uint32_t lane = threadIdx.x & 31u, wic = threadIdx.x >> 5, nwc = blockDim.x >> 5;
    const unsigned long long step = (unsigned long long)blockDim.x * VPT;  // vectors per CTA step
    const unsigned long long wb = (unsigned long long)(k >> 3);
    unsigned long long* slots = seg_range_slots(next);
    const PlaneXpose xp(lane);
    bool waited = false;
    auto ensure_waited = [&]() {  // block-uniform
        if (!waited) {
            pdl_wait_prev();  // rows and slots may belong to the previous launch on this stream
            waited = true;
        }
    };
    // Byte positions are taken relative to `data` rounded down to 16 bytes
    // (`dal`): word i sits at pos(i) = sh + i * wb, so the 16-byte-aligned
    // range starts below never go negative whatever the caller's alignment.
    const unsigned long long sh = reinterpret_cast<uintptr_t>(data) & 15u;  // a multiple of wb
    const uint8_t* dal = data - sh;
    auto pos = [&](unsigned long long i) { return sh + offsets[i] * wb; };
    RangeSplit rs;
    const unsigned long long p0 = pos(0);
    rs.base = p0 & ~15ull;  // absolute 16-byte alignment
    rs.total = pos(n_arrays) - rs.base;
    // at least 4 KiB per range (so no range is empty), at most one per CTA
    rs.W = rs.total / 4096 < gridDim.x ? (rs.total / 4096 ? rs.total / 4096 : 1) : gridDim.x;
    if (blockIdx.x >= rs.W) {
        ensure_waited();
        return;
    }
    const unsigned long long r0 = rs.start(blockIdx.x), r1 = rs.start(blockIdx.x + 1);
    const bool last = blockIdx.x + 1 == rs.W;
    // First array touching [r0, r1): smallest a with end(a) > r0 or start(a) >= r0
    // (the latter catches empty arrays placed at r0).  32-ary search, every warp.
    auto touches = [&](unsigned long long i) {  // monotone in i
        return pos(i + 1) > r0 || pos(i) >= r0;
    };
    unsigned long long lo = 0, hi = n_arrays;  // the answer lies in [lo, hi]; hi = n_arrays: none
    for (;;) {
        const unsigned long long span = hi - lo;
        if (span <= 32) {  // one probe per candidate; lanes past the span stand for `hi`
            const bool pred = lane >= span || touches(lo + lane);
            const uint32_t m = __ballot_sync(0xFFFFFFFFu, pred);
            lo = m ? lo + (unsigned long long)(__ffs(m) - 1) : hi;
            break;
        }
        const unsigned long long probe = lo + span * lane / 32;  // lane 0 probes lo; all < hi <= n_arrays
        const uint32_t m = __ballot_sync(0xFFFFFFFFu, touches(probe));
        if (m & 1u) break;  // the answer is lo
        const int j = m ? __ffs(m) - 1 : 32;  // first true probe; the answer is in (probe_{j-1}, probe_j]
        const unsigned long long nlo = lo + span * (j - 1) / 32 + 1;
        if (j < 32) hi = lo + span * j / 32;
        lo = nlo;
    }
    unsigned long long a = lo;

    const unsigned long long zero[NBANK] = {};
    // The CTA finishes array `arr` (bytes [s, e)) with its warps' counts `t`.  Block-uniform.
    auto finish = [&](unsigned long long arr, unsigned long long s, unsigned long long e,
                      const unsigned long long (&t)[NBANK]) {
        ensure_waited();
        unsigned long long v0 = t[0];
        if (NBANK == 1)
            for (int w = 16; w >= k; w >>= 1) v0 += __shfl_down_sync(0xFFFFFFFFu, v0, w);
        s_tot[wic][lane] = v0;
        if (NBANK == 2) s_tot[wic][32 + lane] = t[NBANK - 1];
        __syncthreads();
        if (wic == 0) {
            unsigned long long sum0 = 0, sum1 = 0;
            for (uint32_t w = 0; w < nwc; ++w) {
                sum0 += s_tot[w][lane];
                if (NBANK == 2) sum1 += s_tot[w][32 + lane];
            }
            const bool mine = (int)lane < (NBANK == 2 ? 32 : k);
            if (s >= r0 && (e <= r1 || last)) {  // entirely in this range
                unsigned long long* row = out + arr * (unsigned long long)k;
                if (mine) row[lane] = sum0;
                if (NBANK == 2) row[32 + lane] = sum1;
            } else {
                const unsigned long long pieces = rs.owner(e - 1) - rs.owner(s) + 1;
                unsigned long long* acc = slots + arr * 65;
                if (mine) atomicAdd(acc + lane, sum0);
                if (NBANK == 2) atomicAdd(acc + 32 + lane, sum1);
                __threadfence();
                __syncwarp();
                unsigned long long done = lane == 0 ? atomicAdd(acc + 64, 1ull) : 0ull;
                done = __shfl_sync(0xFFFFFFFFu, done, 0);
                if (done + 1 == pieces) {  // this range completes the array: move the slot into the row
                    __threadfence();
                    unsigned long long* row = out + arr * (unsigned long long)k;
                    for (int c = (int)lane; c < k; c += 32) row[c] = atomicExch(acc + c, 0ull);
                    if (lane == 0) atomicExch(acc + 64, 0ull);
                }
            }
        }
        __syncthreads();  // s_tot is reused by the next segment
    };
    // Segment of array `arr` inside the range, as a vector view (nv = 0: empty).
    auto segment = [&](unsigned long long arr, unsigned long long& s, unsigned long long& e, SegView& v) {
        s = pos(arr);
        e = pos(arr + 1);
        const unsigned long long lo_b = s > r0 ? s : r0, hi_b = e < r1 || last ? e : r1;
        v = seg_view<VB>(dal, lo_b / wb, hi_b > lo_b ? hi_b / wb : lo_b / wb, (int)wb);
    };
    auto in_range = [&](unsigned long long arr) {  // array `arr` still starts in this range
        return arr < n_arrays && (last || pos(arr) < r1);
    };
    auto zero_row = [&](unsigned long long arr) {  // an empty array at a position this range owns
        ensure_waited();
        if (wic == 0) seg_store_row<NBANK>(out, arr, k, lane, zero);
    };
    unsigned long long s = 0, e = 0;
    SegView v;
    for (;; ++a) {  // first non-empty segment
        if (!in_range(a)) {
            ensure_waited();
            return;
        }
        segment(a, s, e, v);
        if (v.nv) break;
        if (s == e && s >= r0) zero_row(a);
    }
    uint32_t carries[NBANK][L], U[NBANK][M];
    unsigned long long tot[NBANK];
#pragma unroll
    for (int b = 0; b < NBANK; ++b) {
#pragma unroll
        for (int j = 0; j < L; ++j) carries[b][j] = 0;
#pragma unroll
        for (int i = 0; i < M; ++i) U[b][i] = 0;
        tot[b] = 0;
    }
    uint32_t nb = 0;
    unsigned long long t = 0;
    uint32_t r[REGS];
    seg_load_cta<VB, VPT>(v, t, threadIdx.x, blockDim.x, r);
    for (;;) {
#pragma unroll
        for (int b = 0; b < NBANK; ++b)
            plane_count_add<M>(U[b], NBANK == 1 ? Tree<L, 1>::run(carries[b], r) : Tree<L, 2>::run(carries[b], r + b));
        ++nb;
        t += step;
        const bool seg_done = t >= v.nv;
        unsigned long long a_n = a, s_n = s, e_n = e;
        SegView vn = v;
        bool more = true;
        if (seg_done) {  // next non-empty segment of this range
            t = 0;
            more = false;
            for (a_n = a + 1; in_range(a_n); ++a_n) {
                segment(a_n, s_n, e_n, vn);
                if (vn.nv) {
                    more = true;
                    break;
                }
                if (s_n == e_n) zero_row(a_n);
            }
        }
        if (more) seg_load_cta<VB, VPT>(vn, t, threadIdx.x, blockDim.x, r);  // in flight during the epilogue
        if (seg_done || nb == (1u << M) - 1u) {
#pragma unroll
            for (int b = 0; b < NBANK; ++b)
#pragma unroll
                for (int i = 0; i < M; ++i) {
                    tot[b] += (unsigned long long)xp.column_popc(U[b][i]) << (L + i);
                    U[b][i] = 0;
                }
            nb = 0;
        }
        if (seg_done) {
#pragma unroll
            for (int b = 0; b < NBANK; ++b)
#pragma unroll
                for (int j = 0; j < L; ++j) {
                    tot[b] += (unsigned long long)xp.column_popc(carries[b][j]) << j;
                    carries[b][j] = 0;
                }
            finish(a, s, e, tot);
#pragma unroll
            for (int b = 0; b < NBANK; ++b) tot[b] = 0;
            if (!more) {
                ensure_waited();
                return;
            }
            a = a_n;
            s = s_n;
            e = e_n;
            v = vn;
        }
    }
}

template <int NBANK, int L, int VB, int MINB>
__global__ void __launch_bounds__(256, MINB) segmented_range_kernel(const uint8_t* data,
                                                                    const unsigned long long* offsets,
                                                                    unsigned long long n_arrays, int k, uint32_t,
                                                                    unsigned long long* out, unsigned long long* next,
                                                                    unsigned int* ticket, unsigned) {
    pdl_allow_next();
    seg_range_loop<NBANK, L, VB>(data, offsets, n_arrays, k, out, next);  // n_arrays <= kSegRangeSlots (launcher)
    seg_claims_done(next, ticket);  // every warp has waited
}

// MODE bit 0: CTA c takes the contiguous array range [c n / G, (c + 1) n / G)
// and its warps stride over it (one DRAM region per SM, like the stream
// kernel's CTA ranges; measured slower than the strided order); otherwise
// seg_tile_strided.  Bit 1 (EARLY): reading and counting start before the
// previous launch on the stream has completed (see seg_tile_loop; the
// launcher drops programmatic dependent launch when the input may be that
// launch's output).  Bit 2 (DYN, strided only): a dynamic tail.
template <int NBANK, int L, int VB, int MINB, int MODE>
__global__ void __launch_bounds__(256, MINB) segmented_tile_kernel(const uint8_t* data,
                                                                   const unsigned long long* offsets,
                                                                   unsigned long long n_arrays, int k, uint32_t,
                                                                   unsigned long long* out, unsigned long long* next,
                                                                   unsigned int* ticket, unsigned tail_rounds) {
    constexpr bool EARLY = (MODE & 2) != 0;
    constexpr bool DYN = (MODE & 4) != 0 && (MODE & 1) == 0;
    pdl_allow_next();
    if (!EARLY) pdl_wait_prev();  // the rows may belong to the previous launch on this stream
    if constexpr (MODE & 1) {
        const unsigned long long lo = n_arrays * blockIdx.x / gridDim.x;
        const unsigned long long hi = n_arrays * (blockIdx.x + 1) / gridDim.x;
        TileCursor cur;
        cur.next = next;
        cur.dyn = false;
        cur.stride = blockDim.x >> 5;
        cur.static_end = cur.n = hi;
        seg_tile_loop<NBANK, L, VB, EARLY>(data, offsets, hi, k, out, lo + (threadIdx.x >> 5), cur);
    } else {
        seg_tile_strided<NBANK, L, VB, EARLY, DYN>(data, offsets, n_arrays, k, out, next, tail_rounds);
    }
    if constexpr (DYN) seg_claims_done(next, ticket);  // every warp has waited (seg_tile_loop exits after the wait)
}

// ---------------------------------------------------------------------------
// Adaptive segmented kernel (SCHED 8, the asynchronous entry point's default):
// every CTA reads offsets[0] and offsets[n] and picks, from the array count and
// the mean array length, the same schedule for the whole grid -- on the
// device, so device-resident offsets need no host round trip:
//   at most one array per CTA, or a mean of `range` x 32 KiB or more
//                                         -> range mode (even byte ranges per CTA)
//   mean <= lane bound                    -> one lane per array
//   mean > grouped bound, or >= the tile bound and a near multiple of the
//   tile step (NBANK x 4 KiB per warp)    -> warp-per-array tiles
//   otherwise                             -> four lanes per array
// Arrays above `giant` bytes met by the last three go through the giant queue.
// The tile and range modes start counting before the previous launch on the
// stream completed.  `thresholds`: lane bound / 64 B (bits 0-5), grouped bound
// / 256 B (6-11), tile lower bound / 256 B (12-17), range (18-23: 0 never, 63
// always, else the mean bound / 32 KiB), giant / 16 KiB (24-31, 0 = off).  (The software-pipelined warp kernel and the
// dynamic-claim warp loop remain standalone schedules, sched 1-9.)
// ---------------------------------------------------------------------------
template <int NBANK>
__global__ void __launch_bounds__(256, 2) segmented_auto_kernel(const uint8_t* data,
                                                                const unsigned long long* offsets,
                                                                unsigned long long n_arrays, int k,
                                                                uint32_t flush_threshold, unsigned long long* out,
                                                                unsigned long long* next, unsigned int* ticket,
                                                                unsigned thresholds) {
    constexpr int LW = NBANK == 1 ? 5 : 4;  // full-warp fallback tree depth
    pdl_allow_next();
    const int wb = k >> 3;
    const unsigned long long lane_max = (unsigned long long)(thresholds & 0x3Fu) * 64;  // mean bytes
    const unsigned long long group_max = (unsigned long long)((thresholds >> 6) & 0x3Fu) * 256;
    const unsigned long long tile_min = (unsigned long long)((thresholds >> 12) & 0x3Fu) * 256;
    const unsigned long long range = (thresholds >> 18) & 0x3Fu;  // 0 never, 63 always, else mean >= range x 32 KiB
    const unsigned long long giant = (unsigned long long)(thresholds >> 24) << 14;
    const GiantQueue q = seg_giant_queue(next, giant);
    const unsigned long long nwarps = (gridDim.x * (unsigned long long)blockDim.x) >> 5;
    const unsigned long long mean = n_arrays ? (offsets[n_arrays] - offsets[0]) * wb / n_arrays : 0;
    // Range mode: few arrays (at most one per CTA) or long ones (a CTA step is 32 KiB here), within the slots.
    if (range && n_arrays <= (unsigned long long)kSegRangeSlots &&
        (range == 63 || n_arrays <= gridDim.x || mean >= (range << 15))) {
        seg_range_loop<NBANK, NBANK == 1 ? 5 : 4, 16>(data, offsets, n_arrays, k, out, next);
        seg_launch_done(next, ticket, q);  // every warp has waited
        return;
    }
    // Tile mode: above the grouped bound, or from tile_min on when whole warp steps cover the mean array
    // (less than 1/8 of the last step idle; a step is NBANK x 4 KiB per warp).
    constexpr unsigned long long kStepBytes = NBANK * 4096ull;
    const unsigned long long steps = (mean + kStepBytes - 1) / kStepBytes;
    const bool whole_steps = 8 * (steps * kStepBytes - mean) < steps * kStepBytes;
    if (mean > lane_max && (mean > group_max || (mean >= tile_min && whole_steps))) {
        // depth 5 per bank over 16-byte loads: 4 KiB (k <= 32) / 8 KiB (k = 64) steps per warp (measured
        // best at two CTAs per SM: tools/seg_vs_stream.py)
        const unsigned long long warp = (blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x) >> 5;
        const unsigned long long rounds = n_arrays / nwarps;
        TileCursor cur;
        cur.next = next;
        cur.dyn = true;
        cur.stride = nwarps;
        cur.n = n_arrays;
        cur.static_end = (rounds > 4 ? rounds - 4 : 0) * nwarps;
        seg_tile_loop<NBANK, 5, 16, true>(data, offsets, n_arrays, k, out, warp, cur, giant);
        seg_launch_done(next, ticket, q);  // every warp has waited
        return;
    }
    pdl_wait_prev();  // the claim counter, the ticket and the rows may belong to the previous launch
    if (mean <= lane_max) {
        extern __shared__ __align__(16) uint8_t seg_stage[];  // launcher: 32 (half) rows per warp
        seg_lane_loop<NBANK, LW, 16>(data, offsets, n_arrays, k, flush_threshold, out, next, 16u << 10, seg_stage,
                                     giant);
    } else {
        constexpr int LG = NBANK == 1 ? 6 : 4;  // grouped-mode tree depth (measured: 6 beats 5 by ~10 % at 1 KiB)
        seg_group_loop<NBANK, LG, 16, 4>(data, offsets, n_arrays, k, flush_threshold, out, next, (256u << 10) / 16,
                                         giant);
    }
    seg_launch_done(next, ticket, q);
}

}  // namespace dev
}  // namespace pospop_b200
