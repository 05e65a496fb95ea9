/*
 * pospopcnt_b200.h -- C ABI of the B200-native positional population count.
 *
 * Drop-in boundary for the reference's entry point
 *     pospop::PositionalCounts pospop::pospopcnt(pospop::Word16Span words,
 *                                                const pospop::PospopcntConfig& = {})
 *     (/root/reference/proj/core/include/pospop/pospop.hpp:34,
 *      dispatcher proj/core/src/pospop.cpp:80-111)
 * and for the paper's C signature
 *     void pospopcnt_u16_scalar_basic(uint16_t* data, uint32_t len, uint32_t* counters)
 *     (Fig. 6).
 * The reference ships no extern "C" surface; this one is derived from it as
 * "word pointer + length + k-counter output array" (BASELINE.json north_star).
 * The header-only C++ shim include/pospop_gpu.hpp restores the reference's
 * own C++ signature on top of it.  INTEGRATION.md shows the bindings.
 *
 * Conventions (mirroring the reference's behaviour):
 *  - counts[] is OVERWRITTEN, like the reference's return-by-value
 *    PositionalCounts (types.hpp:35-46); except pospopcnt_u16_c32, which
 *    ACCUMULATES like Fig. 6.
 *  - data == NULL is allowed iff len == 0 (Word16Span{} is valid, types.hpp:29-31).
 *  - data must be aligned to the word size (as a uint16_t* / uint32_t* /
 *    uint64_t* is in C++); any alignment beyond that is handled (unaligned
 *    heads and ragged tails count exactly).
 *  - data may be DEVICE memory (the fast path: counted in place in HBM) or
 *    HOST memory (pinned or pageable: streamed to the GPU in chunks with
 *    copy/compute overlap).  The classification uses cudaPointerGetAttributes.
 *  - Every call is synchronous, thread-safe and re-entrant (each call leases
 *    its own per-device streams and workspace from a bounded pool; see
 *    "resources" below), like the reference.
 *    Synchronous calls on device memory are ordered after prior work on the
 *    legacy default stream; data produced on another (non-blocking) stream
 *    must be synchronised by the caller, or counted with pospopcnt_async on
 *    the producing stream.
 *  - No exception or CUDA error crosses the ABI; failures return a status
 *    and set a thread-local message (pospop_last_error).  There is NO CPU
 *    fallback: without a usable sm_100 device every counting call returns
 *    POSPOP_EUNAVAILABLE.
 */
#ifndef POSPOPCNT_B200_H
#define POSPOPCNT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    POSPOP_OK = 0,
    POSPOP_EINVAL = 1,       /* std::invalid_argument          (pospop.cpp:63-70) */
    POSPOP_EUNAVAILABLE = 2, /* pospop::KernelUnavailableError (types.hpp:68-71)  */
    POSPOP_ECUDA = 3,        /* CUDA runtime failure (message in pospop_last_error) */
    POSPOP_ENOMEM = 4,       /* device / pinned allocation failed                  */
    POSPOP_EFLAG = 5         /* pospop::InvalidFlagWordError (flagstats.hpp:64-75)  */
} pospop_status;

/* pospop::KernelKind, same order (types.hpp:52-60).  On the GPU every kind
 * computes identical counts with the same device kernel (pospop.hpp:28-33:
 * "All kernels produce identical counts; they differ only in speed"); the
 * kind is validated and otherwise ignored. */
typedef enum {
    POSPOP_KERNEL_SCALAR = 0,
    POSPOP_KERNEL_CSA4 = 1,
    POSPOP_KERNEL_CSA8 = 2,
    POSPOP_KERNEL_CSA16 = 3,
    POSPOP_KERNEL_FOREST = 4,
    POSPOP_KERNEL_BYTEBLEND = 5,
    POSPOP_KERNEL_AUTO = 6
} pospop_kernel_kind;

/* pospop::PospopcntConfig (types.hpp:73-89), same fields and defaults. */
typedef struct {
    int32_t kernel;                  /* pospop_kernel_kind, default AUTO            */
    uint32_t register_width_bits;    /* 0 or a supported width (pospop_supported_widths) */
    uint32_t flush_threshold_blocks; /* [1, 65535], default 65535                   */
    uint64_t auto_threshold_words;   /* default 4096                                */
} pospop_config;

#define POSPOP_CONFIG_DEFAULT {POSPOP_KERNEL_AUTO, 0u, 65535u, 4096u}

/* ---- validation / capability (pospop.cpp:63-70, cpu.cpp:39-55) ---------- */

/* POSPOP_EINVAL when register_width_bits % 16 != 0, flush_threshold_blocks
 * is outside [1, 65535] or kernel is not a pospop_kernel_kind.  Needs no GPU. */
pospop_status pospop_validate(const pospop_config* config);

/* Register widths the GPU path accepts, ascending (the analogue of
 * supported_csa_widths()).  A 32-bit register is one thread's lane vector;
 * 64..512 are accepted as the reference's CPU widths and map to the same
 * kernel.  Returns the number of widths; writes at most cap. */
int pospop_supported_widths(uint32_t* out, int cap);

/* 1 when an sm_100-class device is usable (device count > 0, CC 10.x). */
int pospop_device_available(void);

/* Thread-local description of the last failure on this thread ("" if none). */
const char* pospop_last_error(void);

/* ---- single-stream counting: counts OVERWRITTEN ------------------------- */

pospop_status pospopcnt_u8(const uint8_t* data, size_t len, uint64_t counts[8]);
pospop_status pospopcnt_u16(const uint16_t* data, size_t len, uint64_t counts[16]);
pospop_status pospopcnt_u32(const uint32_t* data, size_t len, uint64_t counts[32]);
pospop_status pospopcnt_u64(const uint64_t* data, size_t len, uint64_t counts[64]);

/* The reference entry point: pospop::pospopcnt(Word16Span, PospopcntConfig).
 * config == NULL means POSPOP_CONFIG_DEFAULT.  Validation and errors as the
 * reference: EINVAL for out-of-range fields, EUNAVAILABLE for a width with
 * no GPU mapping (e.g. 16, 48, 1024) or no device. */
pospop_status pospopcnt_u16_config(const uint16_t* data, size_t len, const pospop_config* config,
                                   uint64_t counts[16]);

/* Any k in {8,16,32,64} with an explicit flush threshold (tree blocks per
 * thread between lane-counter flushes, [1,65535]). */
pospop_status pospopcnt_k(int k, const void* data, size_t len, uint32_t flush_threshold_blocks,
                          uint64_t* counts);

/* Fig. 6 signature width: uint32 counters, ACCUMULATED (counters[p] += ...),
 * as pospopcnt_u16_scalar_basic in PAPER.md:315-325.  Counters wrap modulo
 * 2^32 exactly as the paper's uint32_t counters would. */
pospop_status pospopcnt_u16_c32(const uint16_t* data, uint32_t len, uint32_t counters[16]);

/* ---- batched / segmented ------------------------------------------------- */

/* Array a is words [offsets[a], offsets[a+1]) of data (offsets: n_arrays+1
 * non-decreasing entries, in words).  Row a of counts (k entries,
 * row-major n_arrays x k) is overwritten.  data/offsets/counts may be
 * device or host memory (each classified independently). */
pospop_status pospopcnt_segmented(int k, const void* data, const uint64_t* offsets, size_t n_arrays,
                                  uint64_t* counts);

/* Typed forms (the shape SURVEY.md 8b recommends): pospopcnt_segmented with
 * k = 8 / 16 / 32 / 64; counts is n_arrays x k, row-major. */
pospop_status pospopcnt_u8_segmented(const uint8_t* data, const uint64_t* offsets, size_t n_arrays,
                                     uint64_t* counts);
pospop_status pospopcnt_u16_segmented(const uint16_t* data, const uint64_t* offsets, size_t n_arrays,
                                      uint64_t* counts);
pospop_status pospopcnt_u32_segmented(const uint32_t* data, const uint64_t* offsets, size_t n_arrays,
                                      uint64_t* counts);
pospop_status pospopcnt_u64_segmented(const uint64_t* data, const uint64_t* offsets, size_t n_arrays,
                                      uint64_t* counts);

/* ---- file / pipe ingestion (the reference CLI's input path) ------------- */

/* Counts a raw little-endian stream of k-bit words read from `fd` (a regular
 * file: parallel pread; a pipe/stdin: sequential read) through pinned double
 * buffers, overlapping host reads with H2D copies and the kernel.  As the
 * reference's read_word_stream/decode_words (proj/tools/pospopcnt.cpp:52-75):
 * a byte length that is not a multiple of k/8 is POSPOP_EINVAL ("odd byte
 * length").  *n_words (may be NULL) receives the word count. */
pospop_status pospopcnt_fd(int fd, int k, uint64_t* counts, uint64_t* n_words);

/* Same for a path; "-" reads stdin.  Unopenable path: POSPOP_EINVAL. */
pospop_status pospopcnt_file(const char* path, int k, uint64_t* counts, uint64_t* n_words);

/* ---- FLAG statistics: the reference's application of the path ----------- */

/* pospop::FlagBucket / FlagSummary (proj/core/include/pospop/flagstats.hpp:39-62),
 * same fields in the same order. */
typedef struct {
    uint64_t total, secondary, supplementary, n_pair_good, n_read1, n_read2, n_sgltn, pair_map, mapped, dup;
} pospop_flag_bucket;

typedef struct {
    pospop_flag_bucket pass; /* FQCFAIL clear */
    pospop_flag_bucket fail; /* FQCFAIL set   */
} pospop_flag_summary;

/* pospop::flagstats_pospopcnt (flagstats.hpp:100, flagstats.cpp:127-145) fused
 * into ONE pass over the FLAG words on the GPU: branchless transform, QC-pass
 * and QC-fail positional counts, bucket derivation.  Equals
 * flagstats_reference on every valid input.  A word with any of bits 12-15
 * set returns POSPOP_EFLAG with *bad_offset / *bad_word of the FIRST such
 * word (InvalidFlagWordError, flagstats.cpp:34-36); either pointer may be
 * NULL.  `flags` may be host or device memory, 2-byte aligned. */
pospop_status pospop_flagstats(const uint16_t* flags, size_t len, pospop_flag_summary* out,
                               uint64_t* bad_offset, uint16_t* bad_word);

/* ---- multi-device, one process (the cfg4 shard/reduce driver) ----------- */

/* shards[i] (lens[i] words) are counted concurrently on devices[i], then the
 * k-vectors are summed (merge_counts, pospop.cpp:33-37; the fork-join of
 * proj/tests/test_core.cpp:155-175).  A shard is either device memory that
 * lives on devices[i] (counted in place) or host memory, pinned or pageable
 * (streamed to devices[i] by a worker thread bound to that device's local
 * CPUs, through its own staging ring: N devices use N host links at once).
 * A device may appear more than once.  Use torch.distributed / NCCL for the
 * one-process-per-GPU layout (paper_1911_02696_b200.shard). */
pospop_status pospopcnt_sharded(int k, const void* const* shards, const size_t* lens,
                                const int* devices, int n_shards, uint64_t* counts);

/* Host-memory fork-join in one call: the len words at `data` are split into
 * n_devices contiguous ranges (sizes differ by at most one word), range i is
 * counted on devices[i] as a host shard of pospopcnt_sharded, and the counts
 * are summed.  Device-resident `data` is accepted when every listed device
 * is the one it lives on. */
pospop_status pospopcnt_split(int k, const void* data, size_t len, const int* devices, int n_devices,
                              uint64_t* counts);

/* Segmented fork-join over devices in one call (the batched
 * variant shards by arrays, no exchange): arrays are cut into n_devices
 * contiguous groups of about equal bytes, group i is counted on devices[i]
 * -- host data streamed over that device's own link by a worker bound to its
 * local CPUs -- and its rows land in counts[a * k ...] as with
 * pospopcnt_segmented.  data, offsets and counts in host memory; operands in
 * device memory are accepted when every listed device is the one holding
 * them (then one device counts them all). */
pospop_status pospopcnt_segmented_split(int k, const void* data, const uint64_t* offsets, size_t n,
                                        const int* devices, int n_devices, uint64_t* counts);

/* The 16-bit form (BASELINE cfg4): pospopcnt_sharded with k = 16. */
pospop_status pospopcnt_u16_sharded(const uint16_t* const* shards, const size_t* lens, const int* devices,
                                    int n_devices, uint64_t counts[16]);

/* ---- resources ----------------------------------------------------------- */

/* The library keeps no per-thread state.  A synchronous call leases a
 * per-device context (streams, result buffers, a 832-byte workspace and,
 * for host input, a 3 x 64 MiB device staging ring and 4 x 16 MiB pinned
 * host ring) from a pool of at most 8 per device and returns it when the
 * call returns; the asynchronous entry points keep one workspace per
 * (device, stream).  pospop_release_resources() frees every idle context
 * and every per-stream workspace (it synchronises the devices that own
 * per-stream workspaces; contexts leased by calls in flight are kept).  It
 * must not run concurrently with an asynchronous entry point (whose
 * workspace it may free); synchronous calls on other threads are safe.  The
 * library stays usable: later calls allocate again. */
pospop_status pospop_release_resources(void);

/* Synchronises `stream` and frees the library's workspaces for it (call
 * before destroying a stream used with the asynchronous entry points). */
pospop_status pospop_release_stream(void* stream);

/* Diagnostics: contexts alive (leased + idle) and idle on `device`, and
 * per-stream workspaces held for it.  Any pointer may be NULL. */
pospop_status pospop_resource_stats(int device, int* contexts, int* idle_contexts, int* stream_workspaces);

/* ---- asynchronous device-resident entry points (timing / integration) --- */

/* Enqueues one count of device-resident data on `stream` (a cudaStream_t,
 * used verbatim: NULL = the legacy default stream); d_counts (k u64 in device
 * memory on the current device) is overwritten, or accumulated when
 * accumulate != 0.  Returns without synchronising.  Each (device, stream)
 * pair owns one small workspace, so launches on one stream are serialised by
 * stream order and launches on different streams never share state;
 * grid/block 0 = automatic. */
pospop_status pospopcnt_async(int k, const void* d_data, size_t len, uint64_t* d_counts,
                              int accumulate, uint32_t flush_threshold_blocks, int grid, int block,
                              void* stream);

/* The 16-bit form: d_counts[16] overwritten, default flush threshold and grid. */
pospop_status pospopcnt_u16_async(const uint16_t* d_data, size_t len, uint64_t* d_counts, void* stream);

/* Diagnostics: pospopcnt_async with per-CTA %globaltimer timestamps.
 * d_trace (device, >= 5 * trace_ctas u64, trace_ctas >= 32 * SMs) receives,
 * per CTA: {start, main-loop end, CTA channels flushed, exit, SM id}, then
 * (the default multi-CTA kernel) per warp, after grid x 5 u64:
 * {end of the CTA-range phase, end of the pool phase, pool tiles counted};
 * *grid_used is the grid size.  Used by tools/trace.py to measure the
 * launch/ramp/tail/epilogue overheads of the persistent grid. */
pospop_status pospopcnt_trace_async(int k, const void* d_data, size_t len, uint64_t* d_counts,
                                    uint64_t* d_trace, size_t trace_ctas, int* grid_used, void* stream);

/* Multi-GPU, one process per GPU: count fused with a device-side all-reduce
 * over peer memory.  The k-vector sum across GPUs (reference
 * merge_counts, pospop.cpp:33-37, the sanctioned chunk-and-merge) needs no
 * separate collective: every rank owns an exchange buffer of
 * pospop_exchange_bytes(k, n_ranks, slots) bytes from pospop_ipc_alloc,
 * exports its handle (64 bytes, exchanged by the caller, e.g. over
 * torch.distributed), and maps the peers' buffers with pospop_ipc_open.
 *
 * Per step (consecutive steps 0, 1, 2, ... on one stream per rank):
 *  - pospopcnt_allgather_async counts d_data like pospopcnt_async (d_counts
 *    gets this rank's counts); its last CTA then stores them as row `rank` of
 *    slot step % slots in every rank's buffer (plain stores over NVLink) and
 *    release-stores the row's step tag.  Before rewriting a slot it waits
 *    until every peer has consumed that slot's previous step (credit).
 *    d_peers is a DEVICE array of n_ranks buffer pointers (own included).
 *  - pospop_exchange_reduce_async (same stream, own buffer) waits for the
 *    n_ranks tags of the step, writes their row sum to d_total[0..k) -- the
 *    all-reduced counts -- and returns the slot's credit.
 * Both waits are bounded (20 s); a timeout sets an error code in the own
 * buffer, which pospop_exchange_status (synchronous) reports as POSPOP_ECUDA.
 * At most 64 ranks. */
pospop_status pospop_ipc_alloc(size_t bytes, void** d_ptr, unsigned char handle[64]);  /* zeroed */
pospop_status pospop_ipc_open(const unsigned char handle[64], void** d_ptr);
pospop_status pospop_ipc_close(void* d_ptr);
pospop_status pospop_ipc_free(void* d_ptr);
size_t pospop_exchange_bytes(int k, int n_ranks, int slots);  /* 0 for invalid arguments */
pospop_status pospopcnt_allgather_async(int k, const void* d_data, size_t len, uint64_t* d_counts,
                                        uint64_t* const* d_peers, int n_ranks, int rank, uint64_t step, int slots,
                                        void* stream);
pospop_status pospop_exchange_reduce_async(int k, uint64_t* d_own, int n_ranks, uint64_t step, int slots,
                                           uint64_t* d_total, void* stream);
pospop_status pospop_exchange_status(const uint64_t* d_own, uint64_t* consumed, uint64_t* error);
/* Protocol self-test on one GPU (tests): n_ranks blocks of ONE cooperative
 * launch play the ranks for `steps` consecutive steps with the same device
 * code as the two kernels above -- optional sleep (sleep_ns, steps x n_ranks),
 * credit wait, row stores + tags into every block's buffer, reduce of its own
 * buffer.  inputs: steps x n_ranks x k host u64 (rank r's counts of step s);
 * totals: n_ranks x steps x k host u64 (what each rank's reducer summed). */
pospop_status pospop_exchange_selftest(int k, int n_ranks, int slots, int steps, const uint64_t* inputs,
                                       const uint32_t* sleep_ns, uint64_t* totals);

/* CUDA-graph replay for repeated counts of one device buffer, where launch
 * latency dominates (small inputs).  The graph is bound to (d_data, len,
 * d_counts) and reads the buffer's current contents at every replay; d_counts
 * is overwritten.  Each graph owns its workspace: different graphs may run
 * concurrently, one graph must not overlap itself.  NULL stream = legacy
 * default stream. */
typedef struct pospop_graph_s* pospop_graph;
pospop_status pospopcnt_graph_create(int k, const void* d_data, size_t len, uint64_t* d_counts,
                                     pospop_graph* out);
pospop_status pospopcnt_graph_launch(pospop_graph graph, void* stream);
void pospopcnt_graph_destroy(pospop_graph graph);

/* Segmented, device-resident, asynchronous: one launch of the adaptive kernel,
 * which picks its schedule on the device from n_arrays and the mean array
 * length (no host round trip for device offsets).  Consecutive launches on a
 * stream overlap (programmatic dependent launch): a launch starts reading and
 * counting while the previous one finishes, writes rows only after it has
 * completed, and runs fully serialised when the device allocation holding
 * d_data or d_offsets may hold one of the stream's recent outputs.  Rows are
 * overwritten; the flush threshold is accepted for API symmetry (every
 * schedule gives the same counts). */
pospop_status pospopcnt_segmented_async(int k, const void* d_data, const uint64_t* d_offsets,
                                        size_t n_arrays, uint64_t* d_counts,
                                        uint32_t flush_threshold_blocks, int grid, int block,
                                        void* stream);

/* ---- synthetic inputs and digests (device-side, for tests and bench) ---- */

/* Fills n elements at d_out with generator `kind` (1..8, oracle/pospop_oracle.h):
 * element l is global element index_base + l.  Asynchronous on `stream`. */
pospop_status pospop_generate(int kind, uint64_t seed, uint64_t index_base, size_t n, void* d_out,
                              void* stream);

/* Order-independent digest of nbytes at 8-byte-aligned device memory;
 * synchronous. */
pospop_status pospop_digest(const void* d_data, size_t nbytes, uint64_t* digest);

/* Diagnostics: runs the DEVICE primitives of the counting kernels on given
 * 32-bit registers (op 0 csa, 1 Harley-Seal tree of the given depth, 2 lane
 * extraction, 3 carry drain, 4 warp channel totals) so tests can pin them
 * against the reference's micro-op KATs (proj/tests/test_csa.cpp).  Synchronous. */
pospop_status pospop_microop(int op, int depth, const uint32_t* in, size_t n_in, uint32_t* out, size_t n_out);

/* Kernels launched by this library in this process (launch accounting). */
uint64_t pospop_kernel_launches(void);

#ifdef __cplusplus
}
#endif

#endif /* POSPOPCNT_B200_H */
