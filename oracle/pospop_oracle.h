/*
 * pospop_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference's positional-population-count algorithm
 * (/root/reference/proj/core), used exclusively as the CHECKER by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg.  Nothing in the
 * product (paper_1911_02696_b200/) links, loads or calls this library.
 *
 * Parity pinning: every function below is checked against the reference's own
 * known-answer tests (tests/test_oracle.py) and against golden vectors produced
 * by the reference library itself (oracle/_ref, tests/golden/make_golden.py).
 */
#ifndef POSPOP_ORACLE_H
#define POSPOP_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- ground truth ------------------------------------------------------ */

/* Plain double loop over words x bit positions, any k in {8,16,32,64};
 * words are little-endian k-bit integers starting at `data` (any alignment).
 * counts[0..k) are OVERWRITTEN.  Restates proj/core/src/pospop.cpp:72-78
 * (oracle_pospopcnt) and PAPER.md:315-325 (Fig. 6) for general k. */
void orc_naive(const void* data, size_t len_words, int k, uint64_t* counts);

/* ---- 64-bit carry-save-adder engine (Backend64) ------------------------ */

/* One CSA over 64 channels: 2*high + low == a + b + c per channel.
 * Restates proj/core/src/detail/backend64.hpp:39-43. */
void orc_csa(uint64_t a, uint64_t b, uint64_t c, uint64_t* high, uint64_t* low);

/* Recursive Harley-Seal tree over 2^depth inputs (depth 1..8), carries
 * updated in place, returns the emitted register of weight 2^depth.
 * Restates proj/core/src/detail/csa_engine.hpp:36-52.  *csa_calls (if not
 * NULL) is incremented once per CSA evaluation (csa_portable.cpp:29-38). */
uint64_t orc_csa_tree(int depth, uint64_t* carries, const uint64_t* in, uint64_t* csa_calls);

/* Lane-counter extraction: counter[p] += (top >> p) & 0x0001000100010001 for
 * p = 0..15, lanes shifted with srl1_epi16.  csa_engine.hpp:67-74. */
void orc_extract_top(uint64_t top, uint64_t counter[16], uint32_t* blocks_since_flush);

/* counts[p] += weight * lane_sum(counter[p]); clears the bank.
 * csa_engine.hpp:76-81, backend64.hpp:53-55. */
void orc_flush_bank(uint64_t counter[16], uint32_t* blocks_since_flush, uint64_t counts[16],
                    uint32_t weight);

/* counts[channel mod 16] += 2^j * bit(B_j).  csa_engine.hpp:86-95. */
void orc_finalize_carries(const uint64_t* carries, int depth, uint64_t counts[16]);

/* Full run_csa<Backend64, block_log2> over a u16 stream: blocks of
 * 2^block_log2 64-bit registers (4 words each), flush when the block clock
 * reaches flush_threshold, final flush, drain, scalar tail.
 * csa_engine.hpp:100-132.  Returns 0, or 1 on an out-of-range argument
 * (flush_threshold outside [1,65535], block_log2 outside [1,8]). */
int orc_run_csa64(const uint16_t* words, size_t len, int block_log2, uint32_t flush_threshold,
                  uint64_t counts[16]);

/* ---- k != 16 restated on the 16-bit API ------------------ */

/* Positional counts for k in {8,16,32,64} computed through the 16-bit CSA
 * engine: k=8 folds byte pairs (c8[p] = c16[p] + c16[p+8], odd head/tail
 * bytes counted naively), k=32/64 deinterleave into k/16 half-streams.
 * `threads` > 1 splits into contiguous chunks and merges (merge_counts,
 * pospop.cpp:33-37; fork-join as proj/tests/test_core.cpp:155-175). */
int orc_pospopcnt(const void* data, size_t len_words, int k, int threads, uint64_t* counts);

/* Batched form: array a spans words [offsets[a], offsets[a+1]); row a of
 * counts (k entries) is overwritten.  Per-array repeated calls, as
 * BASELINE.json's cfg5 CPU recipe states. */
int orc_segmented(const void* data, const uint64_t* offsets, size_t n_arrays, int k, int threads,
                  uint64_t* counts);

/* ---- FLAG statistics ---------------------------------- */

/* FlagBucket field order (proj/core/include/pospop/flagstats.hpp:39-50):
 * total, secondary, supplementary, n_pair_good, n_read1, n_read2, n_sgltn,
 * pair_map, mapped, dup.  out20[0..10) = QC-pass bucket, out20[10..20) = QC-fail. */

/* Branchy SAMtools-style reference: proj/core/src/flagstats.cpp:70-92.
 * Returns 0, or 1 with *bad_offset = index of the first word with any of
 * bits 12-15 set (InvalidFlagWordError, flagstats.cpp:34-36). */
int orc_flagstats_reference(const uint16_t* flags, size_t len, uint64_t out20[20], uint64_t* bad_offset);

/* Mask-select transform of one word: flagstats.cpp:94-125. */
void orc_flag_transform(uint16_t word, uint16_t* pass, uint16_t* fail);

/* Transform-then-count pipeline: flagstats.cpp:127-145 (two positional
 * counts, buckets read from positions 1,2,3,6,7,8,9,10,11,12). */
int orc_flagstats_pospopcnt(const uint16_t* flags, size_t len, uint64_t out20[20], uint64_t* bad_offset);

/* ---- input generators (host twins of the device generators) ------------ */

/* std::mt19937_64(seed), one word per draw from the low 16 bits:
 * proj/core/src/bench.cpp:115-120 (bench::generate_stream). */
void orc_mt_generate_stream(uint64_t seed, size_t len, uint16_t* out);

/* mt19937_64 raw draws (for replaying the reference tests' rng sequences). */
typedef struct { uint64_t mt[312]; int idx; } orc_mt64;
void orc_mt64_seed(orc_mt64* s, uint64_t seed);
uint64_t orc_mt64_next(orc_mt64* s);
void orc_mt64_draws(uint64_t seed, size_t n, uint64_t* out);

/* Counter-based synthetic inputs, identical bytes to the device generators
 * (see DESIGN.md "Synthetic inputs").  Element index i is GLOBAL
 * (index_base + local index) so shards generate in place.
 *   kind 1: uniform u16          (4 u16 per 64-bit draw)
 *   kind 2: cfg2 one-hot u16, Zipf(1.1) position
 *   kind 3: cfg3 bytes: 4 KiB runs, even runs one-hot over 8, odd uniform
 *   kind 4: cfg4 u16, every bit Bernoulli(6554/65536)
 *   kind 5: cfg5 uniform u32     (2 u32 per draw)
 *   kind 6: cfg5 uniform u64     (Bernoulli 0.5 per bit)
 *   kind 7: SAM FLAG words, uniform over the 12 defined bits (bits 12-15 clear)
 *   kind 8: SAM FLAG words, a paired-end-like mix: proper pairs 86%, other paired 8%,
 *           one end unmapped 4%, both unmapped 1.6%, single-end 0.8%; duplicate 1/8,
 *           secondary 1/128, supplementary 1/128, QC-fail 2^-16 (one 64-bit draw per word)
 * Returns 0, or 1 for an unknown kind. */
int orc_generate(int kind, uint64_t seed, uint64_t index_base, size_t n, void* out, int threads);

/* 64-bit FNV-1a style digest of a byte buffer (host/device generator check). */
uint64_t orc_digest(const void* data, size_t nbytes);

#ifdef __cplusplus
}
#endif

#endif /* POSPOP_ORACLE_H */
