// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" face over the UNMODIFIED reference library
// (/root/reference/proj/core, compiled from its own sources by
// oracle/Makefile into oracle/_ref/libpospop_ref.so).  Used by tests/ to
// pin the C restatement (oracle/pospop_oracle.c) and the golden fixtures,
// and by bench.py's cpu_baseline / --impl reference leg to time the
// reference's own CPU path.  Never linked into the product.
//
// Error mapping follows the reference's exception types
// (proj/core/include/pospop/types.hpp:68-71, proj/core/src/pospop.cpp:63-70):
//   0 ok, 1 std::invalid_argument, 2 KernelUnavailableError, 3 other.
#include <cstdint>
#include <cstring>
#include <span>
#include <stdexcept>
#include <thread>
#include <vector>

#include "pospop/bench.hpp"
#include "pospop/csa.hpp"
#include "pospop/flagstats.hpp"
#include "pospop/kernels.hpp"
#include "pospop/pospop.hpp"
#include "pospop/verify.hpp"

using namespace pospop;

namespace {

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const KernelUnavailableError&) {
        return 2;
    } catch (const std::invalid_argument&) {
        return 1;
    } catch (...) {
        return 3;
    }
}

void put(const PositionalCounts& c, uint64_t* out) {
    for (int p = 0; p < 16; ++p) out[p] = c[p];
}

}  // namespace

extern "C" {

// pospop::pospopcnt(Word16Span, PospopcntConfig)  (pospop.hpp:34, pospop.cpp:80-111)
int ref_pospopcnt_u16(const uint16_t* data, size_t len, int kernel, uint32_t width,
                      uint32_t flush, uint64_t auto_threshold, uint64_t* out) {
    return guarded([&] {
        PospopcntConfig cfg;
        cfg.kernel = static_cast<KernelKind>(kernel);
        cfg.register_width_bits = width;
        cfg.flush_threshold_blocks = flush;
        cfg.auto_threshold_words = auto_threshold;
        put(pospopcnt(Word16Span(data, len), cfg), out);
    });
}

// pospop::validate (pospop.cpp:63-70)
int ref_validate(int kernel, uint32_t width, uint32_t flush, uint64_t auto_threshold) {
    return guarded([&] {
        PospopcntConfig cfg;
        cfg.kernel = static_cast<KernelKind>(kernel);
        cfg.register_width_bits = width;
        cfg.flush_threshold_blocks = flush;
        cfg.auto_threshold_words = auto_threshold;
        validate(cfg);
    });
}

// pospop::oracle_pospopcnt (pospop.cpp:72-78)
void ref_oracle_u16(const uint16_t* data, size_t len, uint64_t* out) {
    put(oracle_pospopcnt(Word16Span(data, len)), out);
}

// Fork-join over `threads` contiguous chunks combined with merge_counts,
// the reference's sanctioned parallel use (proj/tests/test_core.cpp:155-175,
// SPEC.md:62,91).  Auto dispatch per chunk.
int ref_pospopcnt_u16_mt(const uint16_t* data, size_t len, int threads, uint64_t* out) {
    return guarded([&] {
        if (threads < 1) threads = 1;
        const Word16Span all(data, len);
        const std::size_t chunk = len / static_cast<std::size_t>(threads);
        std::vector<PositionalCounts> partial(static_cast<std::size_t>(threads));
        {
            std::vector<std::jthread> workers;
            for (int i = 0; i < threads; ++i) {
                const std::size_t begin = static_cast<std::size_t>(i) * chunk;
                const std::size_t end = i + 1 == threads ? len : begin + chunk;
                workers.emplace_back([&partial, all, begin, end, i] {
                    partial[static_cast<std::size_t>(i)] = pospopcnt(all.subspan(begin, end - begin));
                });
            }
        }
        PositionalCounts merged;
        for (const PositionalCounts& part : partial) merged = merge_counts(merged, part);
        put(merged, out);
    });
}

// cfg5 / k != 16 on the reference's own 16-bit API, as SURVEY.md 8c restates
// it (the reference is 16-bit only): k = 16 direct; k = 32 / 64
// deinterleaved into k/16 u16 streams (half h = bits 16h..16h+15), one
// pospop::pospopcnt per stream, concatenated; k = 8 as c16[p] + c16[p+8] over
// the 2-byte-aligned body with an odd head/tail byte counted directly.
// Arrays a = words [offsets[a], offsets[a+1]) of `data`, row a of out (k u64);
// fork-join over `threads` contiguous array ranges.  Returns 0 or an error code.
int ref_segmented(int k, const void* data, const uint64_t* offsets, size_t n_arrays, int threads, uint64_t* out) {
    return guarded([&] {
        if (k != 8 && k != 16 && k != 32 && k != 64) throw std::invalid_argument("k");
        if (threads < 1) threads = 1;
        const size_t wb = static_cast<size_t>(k) / 8;
        auto one = [&](size_t a, std::vector<uint16_t>& scratch) {
            const uint8_t* p = static_cast<const uint8_t*>(data) + offsets[a] * wb;
            const size_t n = offsets[a + 1] - offsets[a];
            uint64_t* row = out + a * static_cast<size_t>(k);
            for (int i = 0; i < k; ++i) row[i] = 0;
            if (k == 16) {
                put(pospopcnt(Word16Span(reinterpret_cast<const uint16_t*>(p), n)), row);
            } else if (k == 8) {
                size_t head = reinterpret_cast<uintptr_t>(p) & 1u ? 1 : 0;
                if (head > n) head = n;
                const size_t body = (n - head) / 2;
                for (size_t i = 0; i < head; ++i)
                    for (int b = 0; b < 8; ++b) row[b] += (p[i] >> b) & 1u;
                const PositionalCounts c = pospopcnt(Word16Span(reinterpret_cast<const uint16_t*>(p + head), body));
                for (int b = 0; b < 8; ++b) row[b] += c[b] + c[b + 8];
                for (size_t i = head + 2 * body; i < n; ++i)
                    for (int b = 0; b < 8; ++b) row[b] += (p[i] >> b) & 1u;
            } else {
                const int halves = k / 16;
                scratch.resize(n);
                for (int h = 0; h < halves; ++h) {
                    for (size_t i = 0; i < n; ++i) {
                        uint16_t w;
                        std::memcpy(&w, p + i * wb + 2 * static_cast<size_t>(h), 2);
                        scratch[i] = w;
                    }
                    put(pospopcnt(Word16Span(scratch.data(), n)), row + 16 * h);
                }
            }
        };
        std::vector<std::jthread> workers;
        for (int t = 0; t < threads; ++t) {
            const size_t lo = n_arrays * static_cast<size_t>(t) / static_cast<size_t>(threads);
            const size_t hi = n_arrays * static_cast<size_t>(t + 1) / static_cast<size_t>(threads);
            workers.emplace_back([&one, lo, hi] {
                std::vector<uint16_t> scratch;
                for (size_t a = lo; a < hi; ++a) one(a, scratch);
            });
        }
    });
}

// bench::generate_stream (bench.cpp:115-120)
void ref_generate_stream(uint64_t seed, size_t len, uint16_t* out) {
    const std::vector<uint16_t> s = bench::generate_stream({seed, len});
    if (len) std::memcpy(out, s.data(), len * sizeof(uint16_t));
}

// supported_csa_widths / native_csa_width (cpu.cpp:39-55)
int ref_supported_widths(uint32_t* out, int cap) {
    const auto w = supported_csa_widths();
    int n = 0;
    for (const uint32_t x : w) {
        if (n < cap) out[n] = x;
        ++n;
    }
    return n;
}

int ref_cpu_has_avx512bw(void) { return cpu_has_avx512bw() ? 1 : 0; }

// ---- micro-ops (csa.hpp:31-87, csa_portable.cpp:50-102) ----------------
void ref_csa(uint64_t a, uint64_t b, uint64_t c, uint64_t* high, uint64_t* low) {
    const CsaOutput o = csa(a, b, c);
    *high = o.high;
    *low = o.low;
}

int ref_csa_block(int depth, uint64_t* regs4, const uint64_t* inputs, size_t n, uint64_t* top,
                  uint64_t* calls) {
    return guarded([&] {
        CarrySet carries(static_cast<std::size_t>(depth));
        for (int j = 0; j < 4; ++j) carries.regs[static_cast<std::size_t>(j)] = regs4[j];
        reset_csa_call_count();
        *top = csa_block(carries, std::span<const uint64_t>(inputs, n));
        *calls = csa_call_count();
        for (int j = 0; j < 4; ++j) regs4[j] = carries.regs[static_cast<std::size_t>(j)];
    });
}

void ref_extract_top(uint64_t top, uint64_t* counter16, uint32_t* blocks) {
    VectorCounterBank bank;
    for (int p = 0; p < 16; ++p) bank.counter[static_cast<std::size_t>(p)] = counter16[p];
    bank.blocks_since_flush = *blocks;
    extract_top(top, bank);
    for (int p = 0; p < 16; ++p) counter16[p] = bank.counter[static_cast<std::size_t>(p)];
    *blocks = bank.blocks_since_flush;
}

void ref_flush_bank(uint64_t* counter16, uint32_t* blocks, uint64_t* counts16, uint32_t weight) {
    VectorCounterBank bank;
    for (int p = 0; p < 16; ++p) bank.counter[static_cast<std::size_t>(p)] = counter16[p];
    bank.blocks_since_flush = *blocks;
    PositionalCounts c;
    for (int p = 0; p < 16; ++p) c[static_cast<std::size_t>(p)] = counts16[p];
    flush_bank(bank, c, weight);
    for (int p = 0; p < 16; ++p) counter16[p] = bank.counter[static_cast<std::size_t>(p)];
    *blocks = bank.blocks_since_flush;
    put(c, counts16);
}

void ref_finalize_carries(const uint64_t* regs4, int depth, uint64_t* counts16) {
    CarrySet carries(static_cast<std::size_t>(depth));
    for (int j = 0; j < 4; ++j) carries.regs[static_cast<std::size_t>(j)] = regs4[j];
    PositionalCounts c;
    for (int p = 0; p < 16; ++p) c[static_cast<std::size_t>(p)] = counts16[p];
    finalize_carries(carries, c);
    put(c, counts16);
}

// ---- FLAG statistics (flagstats.hpp:80-116), for the f1 "next" row -------
// out[0..20): pass bucket fields then fail bucket fields, FlagBucket order.
int ref_flagstats(const uint16_t* data, size_t len, int use_pospopcnt, uint64_t* out20,
                  uint64_t* bad_offset) {
    try {
        const Word16Span s(data, len);
        const FlagSummary f = use_pospopcnt ? flagstats_pospopcnt(s) : flagstats_reference(s);
        const FlagBucket* b[2] = {&f.pass, &f.fail};
        for (int i = 0; i < 2; ++i) {
            uint64_t* o = out20 + 10 * i;
            o[0] = b[i]->total;
            o[1] = b[i]->secondary;
            o[2] = b[i]->supplementary;
            o[3] = b[i]->n_pair_good;
            o[4] = b[i]->n_read1;
            o[5] = b[i]->n_read2;
            o[6] = b[i]->n_sgltn;
            o[7] = b[i]->pair_map;
            o[8] = b[i]->mapped;
            o[9] = b[i]->dup;
        }
        return 0;
    } catch (const InvalidFlagWordError& e) {
        *bad_offset = e.offset();
        return 1;
    } catch (...) {
        return 3;
    }
}

}  // extern "C"
