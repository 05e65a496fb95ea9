// pospop_gpu.hpp -- header-only C++ shim: the reference's own C++ entry point
// on top of the B200 C ABI (pospopcnt_b200.h).
//
//   pospop::PositionalCounts pospop::pospopcnt(pospop::Word16Span, const pospop::PospopcntConfig& = {})
//   (/root/reference/proj/core/include/pospop/pospop.hpp:34)
//
// becomes
//
//   pospop::PositionalCounts pospop_gpu::pospopcnt(pospop::Word16Span, const pospop::PospopcntConfig& = {})
//
// with the reference's types (pospop/types.hpp must be on the include path --
// the caller already has it) and the reference's exceptions:
//   std::invalid_argument          <- POSPOP_EINVAL       (pospop.cpp:63-70)
//   pospop::KernelUnavailableError <- POSPOP_EUNAVAILABLE (types.hpp:68-71)
//   std::runtime_error             <- POSPOP_ECUDA / POSPOP_ENOMEM
// A separate namespace avoids clashing with libpospop's own pospop::pospopcnt,
// so both can be linked into one binary (e.g. the reference's verify_kernels
// with a GPU KernelRunner, proj/core/include/pospop/verify.hpp:47).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>

#include "pospop/types.hpp"
#include "pospopcnt_b200.h"

namespace pospop_gpu {

inline void throw_on(pospop_status s) {
    switch (s) {
        case POSPOP_OK:
            return;
        case POSPOP_EINVAL:
            throw std::invalid_argument(pospop_last_error());
        case POSPOP_EUNAVAILABLE:
            throw pospop::KernelUnavailableError(pospop_last_error());
        default:
            throw std::runtime_error(std::string("pospopcnt_b200: ") + pospop_last_error());
    }
}

inline pospop_config to_c(const pospop::PospopcntConfig& c) {
    return pospop_config{static_cast<int32_t>(c.kernel), c.register_width_bits, c.flush_threshold_blocks,
                         static_cast<uint64_t>(c.auto_threshold_words)};
}

/// Drop-in for pospop::pospopcnt: same arguments, same result, same errors.
/// `words` may live in host memory or in device memory (cudaMalloc'd).
inline pospop::PositionalCounts pospopcnt(pospop::Word16Span words,
                                          const pospop::PospopcntConfig& config = {}) {
    pospop::PositionalCounts out;
    const pospop_config c = to_c(config);
    throw_on(pospopcnt_u16_config(words.data(), words.size(), &c, out.counts.data()));
    return out;
}

/// Drop-in for pospop::validate (pospop.cpp:63-70).
inline void validate(const pospop::PospopcntConfig& config) {
    const pospop_config c = to_c(config);
    throw_on(pospop_validate(&c));
}

/// The reference's fork-join + merge_counts (proj/tests/test_core.cpp:155-175)
/// in one call: `words` (host memory) is cut into one contiguous range per
/// entry of `devices`, each streamed over its own device's host link, and the
/// counts are merged.  A device may be listed more than once.
inline pospop::PositionalCounts pospopcnt_split(pospop::Word16Span words, const int* devices, int n_devices) {
    pospop::PositionalCounts out;
    throw_on(::pospopcnt_split(16, words.data(), words.size(), devices, n_devices, out.counts.data()));
    return out;
}

/// Frees the library's idle per-device contexts and per-stream workspaces.
inline void release_resources() { throw_on(pospop_release_resources()); }

/// A pospop::KernelRunner (verify.hpp:47) that runs the GPU path, for the
/// reference's own verify_kernels / bench harnesses.
struct GpuRunner {
    pospop::PositionalCounts operator()(pospop::Word16Span words, const pospop::PospopcntConfig& config) const {
        return pospop_gpu::pospopcnt(words, config);  // qualified: ADL would also find pospop::pospopcnt
    }
};

}  // namespace pospop_gpu
