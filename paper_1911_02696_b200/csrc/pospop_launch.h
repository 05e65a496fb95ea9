// pospop_launch.h -- internal host-side launchers for the sm_100a kernels.
// Plain types only; the C ABI (pospop_capi.cpp) is the only caller.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace pospop_b200 {

// Persistent device scratch for one in-flight stream launch: acc[96]
// channel totals (32 per counter bank; the FLAG kernel uses three banks) and a
// completion ticket.  Both must be zero before a
// launch; the kernel's last block leaves them zero again.
struct StreamWorkspace {
    unsigned long long* acc = nullptr;   // kAccChannels channel accumulators
    unsigned int* ticket = nullptr;      // CTA completion ticket
    unsigned long long* next = nullptr;  // dynamic-schedule chunk counter
    unsigned long long* bad = nullptr;   // FLAG mode: ~(first invalid word index), 0 = none
};

// Bytes of one workspace allocation (u64 units): acc[0, 96), ticket (u32 at
// u64 96), next (97), bad (98), then from u64 104 the segmented range mode's
// kSegRangeSlots slots (one per array) of 64 partial counts + 1 byte counter
// (dev::seg_range_slots: `next` + 7), then the segmented giant-array queue
// (8 + kGiantQ entries of kGiantEntry u64; dev::GiantQueue).  Zero between
// launches.  Stream and FLAG launches use only the first 104 u64
// (kStreamWorkspaceBytes); the segmented regions are allocated only for
// segmented launches.
constexpr int kAccChannels = 96;
constexpr int kSegRangeSlotsHost = 16384;
constexpr int kGiantQHost = 512;
constexpr int kGiantEntryHost = 72;
constexpr size_t kStreamWorkspaceBytes = 104 * sizeof(unsigned long long);  // stream / FLAG launches
constexpr size_t kWorkspaceBytes =
    (104 + (size_t)kSegRangeSlotsHost * 65 + 8 + (size_t)kGiantQHost * kGiantEntryHost) * sizeof(unsigned long long);

struct LaunchOptions {
    uint32_t flush_threshold = 65535;  // tree blocks between lane flushes, [1, 65535]
    int grid = 0;                      // 0 = persistent: SMs x resident blocks
    int block = 0;                     // 0 = default (256); multiple of 32
    int depth = 0;                     // 0 = default tree depth (k=64: per bank)
    unsigned long long* trace = nullptr;  // diagnostics: 5 u64 per CTA (see pospopcnt_trace_async)
    unsigned long long word_base = 0;     // FLAG mode: global index of the first word
    unsigned long long* const* peers = nullptr;  // fused exchange: device array of n_peers exchange buffers
    int n_peers = 0;
    int rank = 0;
    unsigned long long xstep = 0;  // fused exchange: step (slot xstep % xslots, tag xstep + 1)
    int xslots = 2;
    // Launch without programmatic dependent launch: the input may have been
    // written by a preceding launch of this library on the same stream (which
    // lets its dependents start before it finishes; our kernels read their
    // input before griddepcontrol.wait).
    bool no_pdl = false;
};

// Counts len_words k-bit words at `data` (device memory, k/8-aligned) into
// d_out[0..k).  accumulate: d_out += counts instead of d_out = counts.
// One kernel launch.
cudaError_t launch_stream(int k, const void* data, size_t len_words, unsigned long long* d_out,
                          bool accumulate, const LaunchOptions& opt, const StreamWorkspace& ws,
                          cudaStream_t stream, int* grid_used = nullptr);

// FLAG statistics (reference flagstats_pospopcnt, flagstats.cpp:127-145) in one
// pass: d_out33[0..16) = positional counts of the transformed words of all
// reads, [16..32) = of QC-fail reads (QC-pass = all - fail), [32] = ~(index of
// the first word with reserved bits 12-15 set) or 0.  One kernel launch.
cudaError_t launch_flagstats(const uint16_t* flags, size_t len, unsigned long long* d_out33, bool accumulate,
                             const LaunchOptions& opt, const StreamWorkspace& ws, cudaStream_t stream);

// Batched form: array a = words [d_offsets[a], d_offsets[a+1]) of `data`;
// row a of d_out (k entries) is overwritten.  One kernel launch.
cudaError_t launch_segmented(int k, const void* data, const unsigned long long* d_offsets,
                             size_t n_arrays, unsigned long long* d_out, const LaunchOptions& opt,
                             const StreamWorkspace& ws, cudaStream_t stream);

// Consumer half of the fused exchange (pospop_exchange.h): waits for the
// n_ranks rows of `step` in this rank's buffer `own`, sums them into
// d_total[0..k), then releases the slot.  One single-CTA launch.
cudaError_t launch_exchange_reduce(int k, unsigned long long* own, int n_ranks, unsigned long long step, int slots,
                                   unsigned long long* d_total, cudaStream_t stream);

// Protocol self-test: n_ranks co-resident blocks of one cooperative launch
// play the ranks (exchange_emulate_kernel).  bufs: device array of n_ranks
// zeroed exchange buffers; inputs steps x n x k, sleep_ns steps x n, totals
// n x steps x k (all device memory).
cudaError_t launch_exchange_emulate(unsigned long long* const* bufs, int n_ranks, int k, int slots, int steps,
                                    const unsigned long long* inputs, const unsigned* sleep_ns,
                                    unsigned long long* totals, cudaStream_t stream);

// Synthetic inputs (see oracle/pospop_oracle.h orc_generate for the kinds).
cudaError_t launch_generate(int kind, uint64_t seed, uint64_t index_base, size_t n, void* out,
                            cudaStream_t stream);

// *d_digest += order-independent digest of nbytes at an 8-byte-aligned data.
cudaError_t launch_digest(const void* data, size_t nbytes, unsigned long long* d_digest,
                          cudaStream_t stream);

// Device micro-op harness (see microop_kernel in pospop_aux.cuh).
cudaError_t launch_microop(int op, int depth, const uint32_t* d_in, size_t n, uint32_t* d_out, cudaStream_t stream);

// Number of kernels launched by this library in this process.
unsigned long long kernel_launches();

}  // namespace pospop_b200
