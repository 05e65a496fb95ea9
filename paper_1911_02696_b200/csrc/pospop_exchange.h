// pospop_exchange.h -- layout of one rank's exchange buffer (the fused
// count + all-reduce over peer memory).  Shared by the device
// code and the host runtime.
//
// merge_counts over ranks (proj/core/src/pospop.cpp:33-37) needs every
// partial k-vector before the sum is final, so each row carries a step tag
// and each slot a credit:
//
//   u64 [0]      steps consumed by this rank's reducer (release-stored after
//                it has read slot `step % slots`: peers may then reuse it)
//   u64 [1]      error code (0 = none, 1 = credit wait timed out in a
//                producer, 2 = row wait timed out in the reducer)
//   u64 [2, 8)   spare
//   slot s       n_ranks step tags (tag j = step + 1 once rank j's row of
//                that step is in place; release-stored after the row), then
//                n_ranks rows of k counts
#pragma once

#include <cstddef>
#include <cstdint>

#ifdef __CUDACC__
#define POSPOP_HD __host__ __device__
#else
#define POSPOP_HD
#endif

namespace pospop_b200 {

constexpr int kXHeader = 8;
constexpr int kXMaxRanks = 64;
constexpr unsigned long long kXTimeoutNs = 20ull * 1000 * 1000 * 1000;  // bounded waits: 20 s

POSPOP_HD inline size_t xslot_off(unsigned slot, int n_ranks, int k) {
    return kXHeader + (size_t)slot * ((size_t)n_ranks + (size_t)n_ranks * (size_t)k);
}

POSPOP_HD inline size_t xbuffer_words(int n_ranks, int k, int slots) { return xslot_off((unsigned)slots, n_ranks, k); }

}  // namespace pospop_b200
