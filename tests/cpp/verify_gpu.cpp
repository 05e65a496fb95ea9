// verify_gpu.cpp -- the reference's own verification harness driving the GPU path.
//
// Built by oracle/Makefile (target `verify`) against the UNMODIFIED reference
// headers and library (oracle/_ref/libpospop_ref.so) plus libpospopcnt_b200.so.
// It proves three things a maintainer needs before swapping the GPU in:
//   1. include/pospop_gpu.hpp compiles against pospop/types.hpp and is a
//      drop-in: pospop_gpu::pospopcnt has pospop::pospopcnt's signature;
//   2. pospop::verify_kernels (proj/core/src/verify.cpp:33-75) with a GPU
//      KernelRunner (proj/core/include/pospop/verify.hpp:47) passes: the
//      exhaustive single-word domain + every length 0..max_len, bit-exact
//      against pospop::oracle_pospopcnt;
//   3. the error conventions match (std::invalid_argument,
//      pospop::KernelUnavailableError);
//   4. the harness still catches faults with the GPU underneath (the
//      reference's own fault-injection self-test, test_verify.cpp:42-76);
//   5. the fork-join over host memory (pospop_gpu::pospopcnt_split) equals
//      the reference's single call;
//   6. pospop_gpu::flagstats_pospopcnt (include/pospop_gpu_flagstats.hpp) is
//      a drop-in for pospop::flagstats_pospopcnt, exception included.
// Exit code 0 = all passed.
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <vector>

#include "pospop/bench.hpp"
#include "pospop/flagstats.hpp"
#include "pospop/pospop.hpp"
#include "pospop/verify.hpp"
#include "pospop_gpu.hpp"
#include "pospop_gpu_flagstats.hpp"

int main(int argc, char** argv) {
    const std::size_t max_len = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 3000;
    int failures = 0;

    // (2) the reference harness with the GPU runner
    const pospop::KernelKind kinds[] = {pospop::KernelKind::Auto, pospop::KernelKind::Csa16,
                                        pospop::KernelKind::ScalarBasic};
    const pospop::VerifyReport report =
        pospop::verify_kernels(0xACCE97, max_len, kinds, pospop_gpu::GpuRunner{});
    if (report.ok()) {
        std::printf("PASS verify_kernels(GpuRunner): %zu cases (65536 single words + lengths 0..%zu) x 3 kinds\n",
                    report.cases_run, max_len);
    } else {
        std::printf("FAIL verify_kernels(GpuRunner):\n%s\n", pospop::format_failure(*report.first_failure).c_str());
        ++failures;
    }

    // (1) drop-in on a large stream, against the reference's own kernel
    const std::vector<std::uint16_t> big = pospop::bench::generate_stream({1, std::size_t{1} << 24});
    if (pospop_gpu::pospopcnt(big) == pospop::pospopcnt(big)) {
        std::printf("PASS pospop_gpu::pospopcnt == pospop::pospopcnt on 2^24 words\n");
    } else {
        std::printf("FAIL drop-in mismatch on 2^24 words\n");
        ++failures;
    }

    // (1b) the reference's fork-join over host memory (test_core.cpp:155-175),
    //      one call over several devices' links (device 0 listed 2 and 3 times
    //      on a one-GPU box), then every resource handed back
    {
        const int devs[3] = {0, 0, 0};
        const std::vector<std::uint16_t> odd(big.begin(), big.end() - 3);  // a length not divisible by 2 or 3
        const bool ok = pospop_gpu::pospopcnt_split(big, devs, 2) == pospop::pospopcnt(big) &&
                        pospop_gpu::pospopcnt_split(odd, devs, 3) == pospop::pospopcnt(odd);
        pospop_gpu::release_resources();
        const bool again = pospop_gpu::pospopcnt(big) == pospop::pospopcnt(big);  // usable after a release
        std::printf("%s pospop_gpu::pospopcnt_split (fork-join over devices) == pospop::pospopcnt; release\n",
                    ok && again ? "PASS" : "FAIL");
        failures += ok && again ? 0 : 1;
    }

    // (1c) FLAG statistics: pospop_gpu::flagstats_pospopcnt against the
    //      reference's flagstats_reference and flagstats_pospopcnt, and the
    //      first-invalid-word exception (flagstats.cpp:34-36)
    {
        std::vector<std::uint16_t> flags(big.size());
        for (std::size_t i = 0; i < flags.size(); ++i) flags[i] = big[i] & 0x0FFF;  // valid words
        const pospop::FlagSummary want = pospop::flagstats_reference(flags);
        bool ok = pospop_gpu::flagstats_pospopcnt(flags) == want && pospop::flagstats_pospopcnt(flags) == want;
        flags[777] |= 0x2000;
        flags[123456] |= 0x8000;
        try {
            pospop_gpu::flagstats_pospopcnt(flags);
            ok = false;
        } catch (const pospop::InvalidFlagWordError& e) {
            ok = ok && e.offset() == 777 && e.word() == flags[777];
        }
        std::printf("%s pospop_gpu::flagstats_pospopcnt == pospop::flagstats_reference; InvalidFlagWordError(777)\n",
                    ok ? "PASS" : "FAIL");
        failures += ok ? 0 : 1;
    }

    // (3) error conventions (proj/tests/test_core.cpp:184-201)
    pospop::PospopcntConfig bad;
    bad.flush_threshold_blocks = 0;
    try {
        pospop_gpu::pospopcnt(big, bad);
        std::printf("FAIL threshold 0 accepted\n");
        ++failures;
    } catch (const std::invalid_argument&) {
        std::printf("PASS threshold 0 -> std::invalid_argument\n");
    }
    pospop::PospopcntConfig w128;
    w128.kernel = pospop::KernelKind::Csa16;
    w128.register_width_bits = 128;
    try {
        pospop_gpu::pospopcnt(std::vector<std::uint16_t>(8), w128);
        std::printf("FAIL width 128 accepted\n");
        ++failures;
    } catch (const pospop::KernelUnavailableError&) {
        std::printf("PASS width 128 -> pospop::KernelUnavailableError\n");
    }
    // (4) the harness catches a faulty GPU runner and minimises it
    //     (restates proj/tests/test_verify.cpp:42-76 with the GPU underneath)
    {
        const pospop::KernelRunner faulty = [](pospop::Word16Span words, const pospop::PospopcntConfig& config) {
            pospop::PositionalCounts counts = pospop_gpu::pospopcnt(words, config);
            if (words.size() == 37 && counts[3] > 0) counts[3] -= 1;
            return counts;
        };
        const pospop::KernelKind csa16[] = {pospop::KernelKind::Csa16};
        const pospop::VerifyReport r = pospop::verify_kernels(123, 50, csa16, faulty);
        const bool ok = !r.ok() && r.first_failure->len == 37 && r.first_failure->seed == 123 &&
                        !r.first_failure->single_word.has_value() &&
                        r.first_failure->expected[3] == r.first_failure->actual[3] + 1 &&
                        pospop::format_failure(*r.first_failure).find("len=37") != std::string::npos;
        std::printf("%s injected fault (len 37, bit 3) caught and minimised through the GPU runner\n",
                    ok ? "PASS" : "FAIL");
        failures += ok ? 0 : 1;
        const pospop::KernelRunner faulty1 = [](pospop::Word16Span words, const pospop::PospopcntConfig& config) {
            pospop::PositionalCounts counts = pospop_gpu::pospopcnt(words, config);
            if (words.size() == 1 && words[0] == 0x00FF) counts[0] += 1;
            return counts;
        };
        const pospop::KernelKind scalar[] = {pospop::KernelKind::ScalarBasic};
        const pospop::VerifyReport r1 = pospop::verify_kernels(1, 0, scalar, faulty1);
        const bool ok1 = !r1.ok() && r1.first_failure->single_word.has_value() && *r1.first_failure->single_word == 0x00FF;
        std::printf("%s single-word fault reports 0x00FF through the GPU runner\n", ok1 ? "PASS" : "FAIL");
        failures += ok1 ? 0 : 1;
    }
    return failures;
}
