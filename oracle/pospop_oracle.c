/*
 * pospop_oracle.c -- TEST INFRASTRUCTURE ONLY (see pospop_oracle.h).
 *
 * A plain-C restatement of the reference CPU algorithm for the pospopcnt hot
 * path.  It is the checker for the CUDA product path, never the thing
 * measured or shipped.  Each function names the reference file:line it
 * restates (paths relative to /root/reference/proj).
 */
#define _GNU_SOURCE
#include "pospop_oracle.h"

#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* ground truth                                                              */
/* ------------------------------------------------------------------------ */

/* core/src/pospop.cpp:72-78: for each word, for each position p, add
 * (w >> p) & 1.  Generalised to k-bit little-endian words. */
void orc_naive(const void* data, size_t len, int k, uint64_t* counts) {
    const uint8_t* bytes = (const uint8_t*)data;
    const size_t wbytes = (size_t)k / 8;
    for (int p = 0; p < k; ++p) counts[p] = 0;
    for (size_t i = 0; i < len; ++i) {
        uint64_t w = 0;
        for (size_t b = 0; b < wbytes; ++b) w |= (uint64_t)bytes[i * wbytes + b] << (8 * b);
        for (int p = 0; p < k; ++p) counts[p] += (w >> p) & 1u;
    }
}

/* ------------------------------------------------------------------------ */
/* Backend64 CSA engine                                                      */
/* ------------------------------------------------------------------------ */

#define ONES_EPI16 0x0001000100010001ull

/* core/src/detail/backend64.hpp:39-43 (5-op full adder). */
void orc_csa(uint64_t a, uint64_t b, uint64_t c, uint64_t* high, uint64_t* low) {
    const uint64_t u = a ^ b;
    *high = (a & b) | (u & c);
    *low = u ^ c;
}

/* core/src/detail/csa_engine.hpp:36-52: tree<1> is one CSA against carries[0];
 * tree<L> = tree<L-1>(first half), tree<L-1>(second half), then one CSA of
 * the two emitted registers against carries[L-1].  2^L - 1 CSAs. */
uint64_t orc_csa_tree(int depth, uint64_t* carries, const uint64_t* in, uint64_t* calls) {
    uint64_t high, low, first, second;
    if (depth == 1) {
        orc_csa(carries[0], in[0], in[1], &high, &low);
        if (calls) ++*calls;
        carries[0] = low;
        return high;
    }
    first = orc_csa_tree(depth - 1, carries, in, calls);
    second = orc_csa_tree(depth - 1, carries, in + ((size_t)1 << (depth - 1)), calls);
    orc_csa(carries[depth - 1], first, second, &high, &low);
    if (calls) ++*calls;
    carries[depth - 1] = low;
    return high;
}

/* csa_engine.hpp:67-74 with backend64.hpp:47-49 (add) and 51 (srl1_epi16). */
void orc_extract_top(uint64_t top, uint64_t counter[16], uint32_t* blocks) {
    for (int pos = 0; pos < 16; ++pos) {
        counter[pos] += top & ONES_EPI16;
        top = (top >> 1) & 0x7FFF7FFF7FFF7FFFull;
    }
    if (blocks) ++*blocks;
}

static uint64_t lane_sum_u16(uint64_t v) { /* backend64.hpp:53-55 */
    return (v & 0xFFFF) + ((v >> 16) & 0xFFFF) + ((v >> 32) & 0xFFFF) + (v >> 48);
}

/* csa_engine.hpp:76-81. */
void orc_flush_bank(uint64_t counter[16], uint32_t* blocks, uint64_t counts[16], uint32_t weight) {
    for (int pos = 0; pos < 16; ++pos) {
        counts[pos] += (uint64_t)weight * lane_sum_u16(counter[pos]);
        counter[pos] = 0;
    }
    if (blocks) *blocks = 0;
}

/* csa_engine.hpp:86-95: bit j of B_j weighs 2^j at position (channel mod 16). */
void orc_finalize_carries(const uint64_t* carries, int depth, uint64_t counts[16]) {
    for (int j = 0; j < depth; ++j)
        for (int ch = 0; ch < 64; ++ch)
            counts[ch & 15] += ((carries[j] >> ch) & 1u) << j;
}

/* backend64.hpp:34-37: word i of a register sits at bits [16i, 16i+16). */
static uint64_t load4(const uint16_t* src) {
    return (uint64_t)src[0] | (uint64_t)src[1] << 16 | (uint64_t)src[2] << 32 |
           (uint64_t)src[3] << 48;
}

/* csa_engine.hpp:100-132 (run_csa<Backend64, N>). */
int orc_run_csa64(const uint16_t* words, size_t len, int n, uint32_t thr, uint64_t counts[16]) {
    if (n < 1 || n > 8 || thr < 1 || thr > 65535) return 1;
    const size_t regs_per_block = (size_t)1 << n;
    const size_t words_per_block = regs_per_block * 4;
    const uint32_t weight = 1u << n;
    uint64_t carries[8] = {0};
    uint64_t counter[16] = {0};
    uint64_t in[256];
    uint32_t blocks = 0;
    for (int p = 0; p < 16; ++p) counts[p] = 0;

    const size_t full_blocks = len / words_per_block;
    const uint16_t* src = words;
    for (size_t b = 0; b < full_blocks; ++b) {
        for (size_t r = 0; r < regs_per_block; ++r) in[r] = load4(src + 4 * r);
        orc_extract_top(orc_csa_tree(n, carries, in, NULL), counter, &blocks);
        if (blocks == thr) orc_flush_bank(counter, &blocks, counts, weight);
        src += words_per_block;
    }
    orc_flush_bank(counter, &blocks, counts, weight);
    orc_finalize_carries(carries, n, counts);
    for (size_t i = full_blocks * words_per_block; i < len; ++i)
        for (int p = 0; p < 16; ++p) counts[p] += (words[i] >> p) & 1u;
    return 0;
}

/* ------------------------------------------------------------------------ */
/* k restatements on the 16-bit API                                          */
/* ------------------------------------------------------------------------ */

#define DEINTERLEAVE_CHUNK 4096 /* words per half-stream chunk */

/* One contiguous chunk, k in {8,16,32,64}; counts overwritten. */
static void count_chunk(const uint8_t* data, size_t len, int k, uint64_t* counts) {
    uint64_t c16[16];
    for (int p = 0; p < k; ++p) counts[p] = 0;
    if (len == 0) return;
    if (k == 16) {
        if (((uintptr_t)data & 1) == 0) {
            orc_run_csa64((const uint16_t*)data, len, 4, 65535, counts);
        } else { /* unaligned u16 pointer: copy through an aligned buffer */
            uint16_t buf[DEINTERLEAVE_CHUNK];
            for (size_t s = 0; s < len; s += DEINTERLEAVE_CHUNK) {
                size_t m = len - s < DEINTERLEAVE_CHUNK ? len - s : DEINTERLEAVE_CHUNK;
                memcpy(buf, data + 2 * s, 2 * m);
                orc_run_csa64(buf, m, 4, 65535, c16);
                for (int p = 0; p < 16; ++p) counts[p] += c16[p];
            }
        }
        return;
    }
    if (k == 8) {
        /* PAPER.md:300 / SURVEY 8c: odd head byte naive, even-aligned body as
         * u16 with c8[p] = c16[p] + c16[p+8], odd tail byte naive. */
        size_t i = 0;
        uint64_t one[8];
        if ((uintptr_t)data & 1) {
            orc_naive(data, 1, 8, one);
            for (int p = 0; p < 8; ++p) counts[p] += one[p];
            i = 1;
        }
        const size_t pairs = (len - i) / 2;
        orc_run_csa64((const uint16_t*)(data + i), pairs, 4, 65535, c16);
        for (int p = 0; p < 8; ++p) counts[p] += c16[p] + c16[p + 8];
        i += 2 * pairs;
        if (i < len) {
            orc_naive(data + i, 1, 8, one);
            for (int p = 0; p < 8; ++p) counts[p] += one[p];
        }
        return;
    }
    /* k = 32 / 64: deinterleave 16-bit half h (bits 16h..16h+15) of every
     * word into its own stream; reinterpreting would fold p+16 onto p. */
    const int halves = k / 16;
    const size_t wb = (size_t)k / 8;
    uint16_t* buf = (uint16_t*)malloc(sizeof(uint16_t) * DEINTERLEAVE_CHUNK);
    for (int h = 0; h < halves; ++h) {
        for (size_t s = 0; s < len; s += DEINTERLEAVE_CHUNK) {
            size_t m = len - s < DEINTERLEAVE_CHUNK ? len - s : DEINTERLEAVE_CHUNK;
            for (size_t j = 0; j < m; ++j) {
                const uint8_t* w = data + (s + j) * wb + 2 * h;
                buf[j] = (uint16_t)(w[0] | (w[1] << 8));
            }
            orc_run_csa64(buf, m, 4, 65535, c16);
            for (int p = 0; p < 16; ++p) counts[16 * h + p] += c16[p];
        }
    }
    free(buf);
}

typedef struct {
    const uint8_t* data;
    size_t len;
    int k;
    uint64_t counts[64];
} chunk_job;

static void* chunk_worker(void* arg) {
    chunk_job* j = (chunk_job*)arg;
    count_chunk(j->data, j->len, j->k, j->counts);
    return NULL;
}

int orc_pospopcnt(const void* data, size_t len, int k, int threads, uint64_t* counts) {
    if (k != 8 && k != 16 && k != 32 && k != 64) return 1;
    if (threads < 1) threads = 1;
    if ((size_t)threads > len / 65536 + 1) threads = (int)(len / 65536 + 1);
    const size_t wb = (size_t)k / 8;
    if (threads == 1) {
        count_chunk((const uint8_t*)data, len, k, counts);
        return 0;
    }
    chunk_job* jobs = (chunk_job*)calloc((size_t)threads, sizeof(chunk_job));
    pthread_t* tids = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
    const size_t chunk = len / (size_t)threads;
    for (int t = 0; t < threads; ++t) {
        const size_t begin = (size_t)t * chunk;
        const size_t end = t + 1 == threads ? len : begin + chunk;
        jobs[t].data = (const uint8_t*)data + begin * wb;
        jobs[t].len = end - begin;
        jobs[t].k = k;
        pthread_create(&tids[t], NULL, chunk_worker, &jobs[t]);
    }
    for (int p = 0; p < k; ++p) counts[p] = 0;
    for (int t = 0; t < threads; ++t) {
        pthread_join(tids[t], NULL);
        for (int p = 0; p < k; ++p) counts[p] += jobs[t].counts[p]; /* merge_counts */
    }
    free(jobs);
    free(tids);
    return 0;
}

typedef struct {
    const uint8_t* data;
    const uint64_t* offsets;
    size_t a0, a1;
    int k;
    uint64_t* counts;
} seg_job;

static void* seg_worker(void* arg) {
    seg_job* j = (seg_job*)arg;
    const size_t wb = (size_t)j->k / 8;
    for (size_t a = j->a0; a < j->a1; ++a)
        count_chunk(j->data + j->offsets[a] * wb, j->offsets[a + 1] - j->offsets[a], j->k,
                    j->counts + a * (size_t)j->k);
    return NULL;
}

int orc_segmented(const void* data, const uint64_t* offsets, size_t n, int k, int threads,
                  uint64_t* counts) {
    if (k != 8 && k != 16 && k != 32 && k != 64) return 1;
    for (size_t a = 0; a < n; ++a)
        if (offsets[a + 1] < offsets[a]) return 1;
    if (threads < 1) threads = 1;
    if ((size_t)threads > n) threads = n ? (int)n : 1;
    seg_job* jobs = (seg_job*)calloc((size_t)threads, sizeof(seg_job));
    pthread_t* tids = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
    for (int t = 0; t < threads; ++t) {
        jobs[t] = (seg_job){(const uint8_t*)data, offsets, n * (size_t)t / (size_t)threads,
                            n * (size_t)(t + 1) / (size_t)threads, k, counts};
        pthread_create(&tids[t], NULL, seg_worker, &jobs[t]);
    }
    for (int t = 0; t < threads; ++t) pthread_join(tids[t], NULL);
    free(jobs);
    free(tids);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* FLAG statistics                                                           */
/* ------------------------------------------------------------------------ */

enum { FPAIRED = 0x1, FPROPER_PAIR = 0x2, FUNMAP = 0x4, FMUNMAP = 0x8, FREAD1 = 0x40, FREAD2 = 0x80,
       FSECONDARY = 0x100, FQCFAIL = 0x200, FDUP = 0x400, FSUPPLEMENTARY = 0x800, PAIRMAP = 0x1000,
       RESERVED = 0xF000 };

/* proj/core/src/flagstats.cpp:70-92 */
int orc_flagstats_reference(const uint16_t* flags, size_t len, uint64_t out[20], uint64_t* bad) {
    for (int i = 0; i < 20; ++i) out[i] = 0;
    for (size_t i = 0; i < len; ++i) {
        const uint16_t c = flags[i];
        if (c & RESERVED) {
            *bad = i;
            return 1;
        }
        uint64_t* b = (c & FQCFAIL) ? out + 10 : out;
        ++b[0];
        if (c & FSECONDARY) {
            ++b[1];
        } else if (c & FSUPPLEMENTARY) {
            ++b[2];
        } else if (c & FPAIRED) {
            if ((c & FPROPER_PAIR) && !(c & FUNMAP)) ++b[3];
            if (c & FREAD1) ++b[4];
            if (c & FREAD2) ++b[5];
            if ((c & FMUNMAP) && !(c & FUNMAP)) ++b[6];
            if (!(c & FUNMAP) && !(c & FMUNMAP)) ++b[7];
        }
        if (!(c & FUNMAP)) ++b[8];
        if (!(c & FDUP)) ++b[9];
    }
    return 0;
}

/* proj/core/src/flagstats.cpp:94-125 */
void orc_flag_transform(uint16_t word, uint16_t* pass, uint16_t* fail) {
    const uint16_t keep_secsupp = FUNMAP | FSECONDARY | FDUP | FSUPPLEMENTARY | FQCFAIL;
    const uint16_t pairing = FPROPER_PAIR | FMUNMAP | FREAD1 | FREAD2;
    const uint16_t is_secsupp = (word & (FSECONDARY | FSUPPLEMENTARY)) ? 0xFFFF : 0;
    const uint16_t is_sec = (word & FSECONDARY) ? 0xFFFF : 0;
    const uint16_t is_paired = (word & FPAIRED) ? 0xFFFF : 0;
    const uint16_t is_unmap = (word & FUNMAP) ? 0xFFFF : 0;
    const uint16_t is_munmap = (word & FMUNMAP) ? 0xFFFF : 0;
    uint16_t dat = word;
    dat &= (uint16_t)~(is_secsupp & (uint16_t)~keep_secsupp);
    dat &= (uint16_t)~(is_sec & FSUPPLEMENTARY);
    dat &= (uint16_t)~((uint16_t)~is_paired & pairing);
    dat &= (uint16_t)~(is_unmap & (FPROPER_PAIR | FMUNMAP));
    dat |= (uint16_t)(is_paired & (uint16_t)~is_secsupp & (uint16_t)~is_unmap & (uint16_t)~is_munmap & PAIRMAP);
    const uint16_t is_fail = (word & FQCFAIL) ? 0xFFFF : 0;
    *pass = (uint16_t)(dat & (uint16_t)~is_fail);
    *fail = (uint16_t)(dat & is_fail);
}

/* flagstats.cpp:50-63 (bucket_from_counts) */
static void bucket_from_counts(const uint64_t c[16], uint64_t total, uint64_t b[10]) {
    b[0] = total;
    b[1] = c[8];
    b[2] = c[11];
    b[3] = c[1];
    b[4] = c[6];
    b[5] = c[7];
    b[6] = c[3];
    b[7] = c[12];
    b[8] = total - c[2];
    b[9] = total - c[10];
}

/* proj/core/src/flagstats.cpp:127-145 */
int orc_flagstats_pospopcnt(const uint16_t* flags, size_t len, uint64_t out[20], uint64_t* bad) {
    uint64_t pc[16] = {0}, fc[16] = {0};
    for (size_t i = 0; i < len; ++i) {
        if (flags[i] & RESERVED) {
            *bad = i;
            return 1;
        }
        uint16_t p, f;
        orc_flag_transform(flags[i], &p, &f);
        for (int q = 0; q < 16; ++q) {
            pc[q] += (p >> q) & 1u;
            fc[q] += (f >> q) & 1u;
        }
    }
    const uint64_t fail_total = fc[9];
    bucket_from_counts(fc, fail_total, out + 10);
    bucket_from_counts(pc, len - fail_total, out);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* generators                                                                */
/* ------------------------------------------------------------------------ */

/* std::mt19937_64 as the C++ standard specifies it ([rand.eng.mers]):
 * w=64 n=312 m=156 r=31 a=0xB5026F5AA96619E9 u=29 d=0x5555555555555555
 * s=17 b=0x71D67FFFEDA60000 t=37 c=0xFFF7EEE000000000 l=43
 * f=6364136223846793005.  Used by proj/core/src/bench.cpp:115-120. */
void orc_mt64_seed(orc_mt64* s, uint64_t seed) {
    s->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        s->mt[i] = 6364136223846793005ull * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
    s->idx = 312;
}

uint64_t orc_mt64_next(orc_mt64* s) {
    static const uint64_t UPPER = 0xFFFFFFFF80000000ull, LOWER = 0x7FFFFFFFull;
    if (s->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            const uint64_t x = (s->mt[i] & UPPER) | (s->mt[(i + 1) % 312] & LOWER);
            uint64_t xa = x >> 1;
            if (x & 1) xa ^= 0xB5026F5AA96619E9ull;
            s->mt[i] = s->mt[(i + 156) % 312] ^ xa;
        }
        s->idx = 0;
    }
    uint64_t y = s->mt[s->idx++];
    y ^= (y >> 29) & 0x5555555555555555ull;
    y ^= (y << 17) & 0x71D67FFFEDA60000ull;
    y ^= (y << 37) & 0xFFF7EEE000000000ull;
    y ^= y >> 43;
    return y;
}

void orc_mt64_draws(uint64_t seed, size_t n, uint64_t* out) {
    orc_mt64 s;
    orc_mt64_seed(&s, seed);
    for (size_t i = 0; i < n; ++i) out[i] = orc_mt64_next(&s);
}

void orc_mt_generate_stream(uint64_t seed, size_t len, uint16_t* out) {
    orc_mt64 s;
    orc_mt64_seed(&s, seed);
    for (size_t i = 0; i < len; ++i) out[i] = (uint16_t)orc_mt64_next(&s);
}

/* Counter-based generator.  Written independently of the CUDA generator in
 * paper_1911_02696_b200/csrc; tests hash both outputs to prove they agree. */
#define GAMMA 0x9E3779B97F4A7C15ull

static uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static uint64_t gen_key(uint64_t seed, int kind) {
    return mix64(seed ^ ((uint64_t)kind * 0xD1B54A32D192ED03ull));
}

static uint64_t draw(uint64_t key, uint64_t j) { return mix64(key + (j + 1) * GAMMA); }

static const uint32_t ZIPF_THRESHOLDS[15] = {
    1417819056u, 2079255034u, 2502690694u, 2811261488u, 3052670681u,
    3250210401u, 3416940100u, 3560893466u, 3687353720u, 3799975090u,
    3901386976u, 3993542513u, 4077930985u, 4155713140u, 4227810676u};

static void gen_range(int kind, uint64_t key, uint64_t base, size_t lo, size_t hi, void* out) {
    for (size_t l = lo; l < hi; ++l) {
        const uint64_t i = base + l;
        switch (kind) {
            case 1:
                ((uint16_t*)out)[l] = (uint16_t)(draw(key, i >> 2) >> (16 * (i & 3)));
                break;
            case 2: {
                const uint32_t u = (uint32_t)(draw(key, i) >> 32);
                int bit = 0;
                for (int t = 0; t < 15; ++t) bit += ZIPF_THRESHOLDS[t] <= u;
                ((uint16_t*)out)[l] = (uint16_t)(1u << bit);
                break;
            }
            case 3: {
                const uint8_t b = (uint8_t)(draw(key, i >> 3) >> (8 * (i & 7)));
                ((uint8_t*)out)[l] = ((i >> 12) & 1) ? b : (uint8_t)(1u << (b & 7));
                break;
            }
            case 4: {
                uint16_t w = 0;
                for (int j = 0; j < 4; ++j) {
                    const uint64_t h = draw(key, 4 * i + (uint64_t)j);
                    for (int m = 0; m < 4; ++m)
                        if (((h >> (16 * m)) & 0xFFFF) < 6554u) w |= (uint16_t)(1u << (4 * j + m));
                }
                ((uint16_t*)out)[l] = w;
                break;
            }
            case 5:
                ((uint32_t*)out)[l] = (uint32_t)(draw(key, i >> 1) >> (32 * (i & 1)));
                break;
            case 6:
                ((uint64_t*)out)[l] = draw(key, i);
                break;
            case 7:
                ((uint16_t*)out)[l] = (uint16_t)((draw(key, i >> 2) >> (16 * (i & 3))) & 0x0FFF);
                break;
            case 8: { /* SAM FLAG words, a paired-end-like mix with rare QC-fail reads */
                static const uint16_t proper[4] = {99, 147, 83, 163};
                static const uint16_t paired[8] = {65, 129, 113, 177, 97, 145, 81, 161};
                static const uint16_t half[8] = {73, 133, 89, 121, 137, 153, 185, 69};
                const uint64_t u = draw(key, i);
                const unsigned c = (unsigned)(u & 0xFF), sel = (unsigned)((u >> 8) & 7);
                unsigned f;
                if (c < 220) f = proper[sel & 3];
                else if (c < 240) f = paired[sel];
                else if (c < 250) f = half[sel];
                else if (c < 254) f = (sel & 1) ? 141u : 77u;
                else f = (sel & 1) ? 16u : 0u;
                if (((u >> 16) & 0xF) < 2) f |= 0x400u;
                if (((u >> 20) & 0x7F) == 0) f |= 0x100u;
                if (((u >> 27) & 0x7F) == 1) f |= 0x800u;
                if (((u >> 34) & 0xFFFF) == 0) f |= 0x200u;
                ((uint16_t*)out)[l] = (uint16_t)f;
                break;
            }
        }
    }
}

typedef struct {
    int kind;
    uint64_t key, base;
    size_t lo, hi;
    void* out;
} gen_job;

static void* gen_worker(void* arg) {
    gen_job* j = (gen_job*)arg;
    gen_range(j->kind, j->key, j->base, j->lo, j->hi, j->out);
    return NULL;
}

int orc_generate(int kind, uint64_t seed, uint64_t base, size_t n, void* out, int threads) {
    if (kind < 1 || kind > 8) return 1;
    const uint64_t key = gen_key(seed, kind);
    if (threads < 1) threads = 1;
    if ((size_t)threads > n / 65536 + 1) threads = (int)(n / 65536 + 1);
    gen_job* jobs = (gen_job*)calloc((size_t)threads, sizeof(gen_job));
    pthread_t* tids = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
    for (int t = 0; t < threads; ++t) {
        jobs[t] = (gen_job){kind, key, base, n * (size_t)t / (size_t)threads,
                            n * (size_t)(t + 1) / (size_t)threads, out};
        pthread_create(&tids[t], NULL, gen_worker, &jobs[t]);
    }
    for (int t = 0; t < threads; ++t) pthread_join(tids[t], NULL);
    free(jobs);
    free(tids);
    return 0;
}

/* Order-independent digest: sum over little-endian u64 words w_j (last word
 * zero-padded) of mix64(w_j + j * GAMMA).  Matches the device digest. */
uint64_t orc_digest(const void* data, size_t nbytes) {
    const uint8_t* b = (const uint8_t*)data;
    uint64_t sum = 0;
    const size_t nw = (nbytes + 7) / 8;
    for (size_t j = 0; j < nw; ++j) {
        uint64_t w = 0;
        if (8 * j + 8 <= nbytes) {
            memcpy(&w, b + 8 * j, 8); /* little-endian host */
        } else {
            for (size_t t = 0; 8 * j + t < nbytes; ++t) w |= (uint64_t)b[8 * j + t] << (8 * t);
        }
        sum += mix64(w + j * GAMMA);
    }
    return sum;
}
