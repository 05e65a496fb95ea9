// pospop_gpu_flagstats.hpp -- header-only C++ shim for the reference's FLAG
// statistics entry point on top of the B200 C ABI (pospopcnt_b200.h):
//
//   pospop::FlagSummary pospop::flagstats_pospopcnt(pospop::Word16Span, const pospop::PospopcntConfig& = {})
//   (/root/reference/proj/core/include/pospop/flagstats.hpp:100, flagstats.cpp:127-145)
//
// becomes pospop_gpu::flagstats_pospopcnt with the same types and errors:
// the reference's pospop::FlagSummary result (its FlagBucket fields in the
// same order as pospop_flag_bucket), pospop::InvalidFlagWordError(offset,
// word) for the FIRST word with reserved bits 12-15 set (flagstats.cpp:34-36),
// std::invalid_argument / pospop::KernelUnavailableError as pospop_gpu.hpp.
// InvalidFlagWordError's constructor lives in the reference library, which a
// caller of pospop::flagstats_* already links.
#pragma once

#include <cstdint>
#include <type_traits>

#include "pospop/flagstats.hpp"
#include "pospop_gpu.hpp"

namespace pospop_gpu {

inline pospop::FlagBucket to_bucket(const pospop_flag_bucket& b) {
    pospop::FlagBucket r;
    r.total = b.total;
    r.secondary = b.secondary;
    r.supplementary = b.supplementary;
    r.n_pair_good = b.n_pair_good;
    r.n_read1 = b.n_read1;
    r.n_read2 = b.n_read2;
    r.n_sgltn = b.n_sgltn;
    r.pair_map = b.pair_map;
    r.mapped = b.mapped;
    r.dup = b.dup;
    return r;
}

/// Drop-in for pospop::flagstats_pospopcnt: one fused GPU pass (transform,
/// QC-pass / QC-fail positional counts, bucket derivation).  `config` is
/// validated like the reference's (the GPU runs one kernel for every kind).
/// `flags` may live in host or device memory.
inline pospop::FlagSummary flagstats_pospopcnt(pospop::Word16Span flags, const pospop::PospopcntConfig& config = {}) {
    pospop_gpu::validate(config);  // qualified: ADL would also find pospop::validate
    pospop_flag_summary s{};
    std::uint64_t bad_offset = 0;
    std::uint16_t bad_word = 0;
    const pospop_status st = pospop_flagstats(flags.data(), flags.size(), &s, &bad_offset, &bad_word);
    if (st == POSPOP_EFLAG) throw pospop::InvalidFlagWordError(static_cast<std::size_t>(bad_offset), bad_word);
    throw_on(st);
    pospop::FlagSummary out;
    out.pass = to_bucket(s.pass);
    out.fail = to_bucket(s.fail);
    return out;
}

}  // namespace pospop_gpu
