// pospop_kernels.cu -- the single CUDA translation unit of libpospopcnt_b200:
// instantiates the sm_100a kernels and owns their host-side launchers.
//
//   pospop_device.cuh     CSA (LOP3 0xE8/0x96), Harley-Seal tree, lane bank,
//                         drain, warp transpose-reduce, vector loads
//   pospop_stream.cuh     stream_kernel: the hot path (reference run_csa,
//                         proj/core/src/detail/csa_engine.hpp:100-132) for
//                         k = 8/16/32/64 and the fused FLAG-statistics mode
//   pospop_segmented.cuh  segmented / batched kernels (one k-row per array)
//   pospop_aux.cuh        generators, digest, micro-op harness
//
// Each launcher picks a tuned instantiation (the defaults below were chosen
// by tools/sweep.py on a B200) and launches it once; counting
// launches carry the programmatic-stream-serialization attribute so back-to-
// back counts overlap.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <utility>

#include "pospop_aux.cuh"
#include "pospop_device.cuh"
#include "pospop_launch.h"
#include "pospop_segmented.cuh"
#include "pospop_stream.cuh"
#include "pospop_variants.h"

extern char** environ;

namespace pospop_b200 {

namespace {

using namespace dev;

std::atomic<unsigned long long> g_launches{0};

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------

constexpr int kDefaultBlock = 256;
constexpr int kDefaultDepth1 = 7;  // k = 8/16/32: 128 registers = 512 B per thread per tree block
constexpr int kDefaultDepth2 = 6;  // k = 64: two banks of 64 registers

// Tuning knobs (POSPOP_*; tuning build only) are read from one snapshot of the environment
// taken at the top of each public launcher: a single pass over `environ`
// instead of a getenv() scan per knob (~0.25 us each with ~130 variables --
// several microseconds on the small-call latency path otherwise).
struct EnvSnapshot {
    static constexpr int kMax = 32;
    const char* entry[kMax];
    int n = 0;
};
#ifdef POSPOP_TUNING
thread_local EnvSnapshot t_env;

void env_refresh() {
    t_env.n = 0;
    for (char** e = environ; e && *e; ++e)
        if ((*e)[0] == 'P' && std::strncmp(*e, "POSPOP_", 7) == 0 && t_env.n < EnvSnapshot::kMax)
            t_env.entry[t_env.n++] = *e;
}

const char* env_get(const char* name) {
    const size_t len = std::strlen(name);
    for (int i = 0; i < t_env.n; ++i)
        if (std::strncmp(t_env.entry[i], name, len) == 0 && t_env.entry[i][len] == '=') return t_env.entry[i] + len + 1;
    return nullptr;
}
#else
// The release library reads no tuning knobs: the kernel, grid and flush
// threshold depend on the call's arguments only.
inline void env_refresh() {}
inline const char* env_get(const char*) { return nullptr; }
#endif

int env_int(const char* name, int dflt) {
    const char* v = env_get(name);
    return v && *v ? std::atoi(v) : dflt;
}

struct DeviceInfo {
    int sms = 0;
};

DeviceInfo device_info() {
    static thread_local int cached_dev = -1;
    static thread_local DeviceInfo info;
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev != cached_dev) {
        cudaDeviceGetAttribute(&info.sms, cudaDevAttrMultiProcessorCount, dev);
        cached_dev = dev;
    }
    return info;
}

template <class Kernel>
int resident_blocks(Kernel kernel, int block) {
    // The occupancy query costs microseconds; cache it per (device, kernel, block).
    struct Key {
        int dev;
        const void* fn;
        int block;
        bool operator<(const Key& o) const {
            return dev != o.dev ? dev < o.dev : fn != o.fn ? fn < o.fn : block < o.block;
        }
    };
    static thread_local std::map<Key, int> cache;
    int dev = 0;
    cudaGetDevice(&dev);
    const Key key{dev, reinterpret_cast<const void*>(kernel), block};
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, block, 0) != cudaSuccess || n < 1) n = 1;
    cache[key] = n;
    return n;
}

const StreamVariant* pick_stream(int nbank, int depth, int vb, int hint, int block, int sched, int mode) {
    size_t n = 0;
    const StreamVariant* v = mode == 0 ? stream_variants_counts(&n) : mode == 1 ? stream_variants_flag16(&n)
                                                                              : stream_variants_flag8(&n);
    for (size_t i = 0; i < n; ++i)
        if (v[i].nbank == nbank && v[i].depth == depth && v[i].vb == vb && v[i].hint == hint &&
            v[i].block == block && v[i].sched == sched && v[i].mode == mode)
            return &v[i];
    return nullptr;
}

const TmaVariant* pick_tma(int nbank, int depth, int mode, int nc, int stages) {
    size_t n = 0;
    const TmaVariant* v = tma_variants(&n);
    for (size_t i = 0; i < n; ++i)
        if (v[i].nbank == nbank && v[i].depth == depth && v[i].mode == mode && v[i].nc == nc && v[i].stages == stages)
            return &v[i];
    return nullptr;
}

const TmaVariant* pick_ring(int nbank, int depth, int mode, int nw, int stages) {
    size_t n = 0;
    const TmaVariant* v = ring_variants(&n);
    for (size_t i = 0; i < n; ++i)
        if (v[i].nbank == nbank && v[i].depth == depth && v[i].mode == mode && v[i].nc == nw && v[i].stages == stages)
            return &v[i];
    return nullptr;
}

const SegVariant* pick_segmented(int nbank, int depth, int vb, int sched, int group = 0) {
    size_t n = 0;
    const SegVariant* v = seg_variants(&n);
    for (size_t i = 0; i < n; ++i)
        if (v[i].nbank == nbank && v[i].depth == depth && v[i].vb == vb && v[i].sched == sched &&
            ((sched != 5 && sched != 10 && sched < 11) || v[i].group == group))
            return &v[i];
    return nullptr;
}

}  // namespace

unsigned long long kernel_launches() { return g_launches.load(); }

// Vector addressing shared by every stream launch (see StreamArgs).
static void fill_stream_args(StreamArgs& a, int k, const void* data, size_t len_words, uintptr_t vb,
                             unsigned long long* d_out, bool accumulate, const LaunchOptions& opt,
                             const StreamWorkspace& ws) {
    const uintptr_t P = reinterpret_cast<uintptr_t>(data);
    const size_t nbytes = len_words * (size_t)(k / 8);
    const uintptr_t group = 32 * vb;
    a.base = reinterpret_cast<const uint8_t*>(P & ~(group - 1));
    if (nbytes == 0) {
        a.v0 = a.v1 = a.f0 = a.f1 = a.g0 = a.ng = 0;
        a.lo_byte = 0;
        a.hi_byte = (int)vb;
    } else {
        const uintptr_t B = reinterpret_cast<uintptr_t>(a.base);
        a.v0 = (P - B) / vb;
        a.v1 = (P + nbytes - B + vb - 1) / vb;
        a.lo_byte = (int)(P - (B + a.v0 * vb));
        a.hi_byte = (int)(P + nbytes - (B + (a.v1 - 1) * vb));
        a.f0 = a.v0 + (a.lo_byte != 0 ? 1 : 0);
        a.f1 = a.v1 - (a.hi_byte != (int)vb ? 1 : 0);
        a.g0 = a.v0 / 32;
        a.ng = (a.v1 + 31) / 32 - a.g0;
    }
    a.k = k;
    a.flush_threshold = opt.flush_threshold;
    a.acc = ws.acc;
    a.ticket = ws.ticket;
    a.out = d_out;
    a.accumulate = accumulate ? 1 : 0;
    a.trace = opt.trace;
    a.next = ws.next;
    a.bad = ws.bad;
    a.word_base = opt.word_base;
    a.data_off = nbytes ? (unsigned long long)(P - reinterpret_cast<uintptr_t>(a.base)) : 0ull;
    a.nwt = a.nA = a.pool = 0;
    a.CA = a.CB = 1;
    a.peers = opt.peers;
    a.n_peers = opt.peers ? opt.n_peers : 0;
    a.rank = opt.rank;
    a.xstep = opt.xstep;
    a.xslots = opt.xslots > 0 ? opt.xslots : 1;
}

// Tree blocks between lane flushes: the caller's threshold, lowered by
// POSPOP_FLUSH_THRESHOLD (tests: exercise the flush path) and, for the
// byte-lane counters of the FLAG byte-frame kernel (MODE 2; <= 255 per lane,
// and a tile that takes the QC-fail fix-up extracts twice into bank 2), at
// most 127.
static uint32_t flush_threshold_for(int mode, const LaunchOptions& opt) {
    uint32_t thr = opt.flush_threshold;
    const int env_thr = env_int("POSPOP_FLUSH_THRESHOLD", 0);
    if (env_thr > 0 && (uint32_t)env_thr < thr) thr = (uint32_t)env_thr;
    return mode == 2 && thr > 127 ? 127 : thr;
}

static cudaError_t launch_with_pdl(StreamKernel fn, int grid, int threads, size_t smem, cudaStream_t stream,
                                   const StreamArgs& a, bool pdl) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3((unsigned)threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl && env_int("POSPOP_PDL", 1) ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, fn, a);
    ++g_launches;
    return e != cudaSuccess ? e : cudaGetLastError();
}

// TMA-staged launch (SCHED 3): one CTA per SM, a producer warp + nc consumer
// warps, `stages` x stage-bytes of dynamic shared memory.
static cudaError_t launch_stream_tma(int mode, int nbank, int depth, int k, const void* data, size_t len_words,
                                     unsigned long long* d_out, bool accumulate, const LaunchOptions& opt,
                                     const StreamWorkspace& ws, cudaStream_t stream, int* grid_used) {
    int nc = 8, stages = mode == 1 ? 6 : 6;
    if (const char* v = env_get("POSPOP_TMA")) std::sscanf(v, "%d,%d", &nc, &stages);
    const TmaVariant* var = pick_tma(nbank, depth, mode, nc, stages);
    if (!var) return cudaErrorInvalidConfiguration;
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, bool> configured;
    int dev = 0;
    cudaGetDevice(&dev);
    {
        std::lock_guard<std::mutex> lock(mu);
        auto key = std::make_pair(dev, reinterpret_cast<const void*>(var->fn));
        if (!configured[key]) {
            const cudaError_t e =
                cudaFuncSetAttribute(var->fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)var->smem);
            if (e != cudaSuccess) return e;
            configured[key] = true;
        }
    }
    StreamArgs a;
    fill_stream_args(a, k, data, len_words, 16, d_out, accumulate, opt, ws);
    a.flush_threshold = flush_threshold_for(mode, opt);
    const int grid = device_info().sms;
    if (grid_used) *grid_used = grid;
    return launch_with_pdl(var->fn, grid, 32 * (var->nc + 1), var->smem, stream, a, !opt.no_pdl);
}

static void set_schedule(StreamArgs& a, int grid, int threads, int vpt);
static cudaError_t launch_stream_ring(int mode, int nbank, int depth, int k, const void* data, size_t len_words,
                                      unsigned long long* d_out, bool accumulate, const LaunchOptions& opt,
                                      const StreamWorkspace& ws, cudaStream_t stream, int* grid_used);

static cudaError_t launch_stream_mode(int mode, int k, const void* data, size_t len_words,
                                      unsigned long long* d_out, bool accumulate, const LaunchOptions& opt,
                                      const StreamWorkspace& ws, cudaStream_t stream, int* grid_used) {
    // Tuning override: POSPOP_STREAM_VARIANT="depth,vb,hint,block,sched";
    // FLAG statistics: POSPOP_FLAG_VARIANT="depth,vb,hint,block,sched[,mode]"
    // (mode 2 byte-frame kernel, the default; mode 1 the 16-bit-lane kernel).
    // FLAG statistics default: the per-warp bulk-copy ring kernel, 16 warps
    // x 1 slot (sched 6; tools/ring_sweep.sh: uniform FLAG words 6276-6380 ->
    // 6398-6400 GB/s, the paired-end-like mix 6946 -> 7162).
    int depth = mode == 0 ? (k == 64 ? kDefaultDepth2 : kDefaultDepth1) : 5, vb = 32, hint = 0,
        block = mode == 0 ? kDefaultBlock : 512, sched = mode == 0 ? 2 : 6;
    if (mode != 0) {
        int fmode = mode;
        if (const char* v = env_get("POSPOP_FLAG_VARIANT")) {
            const int n = std::sscanf(v, "%d,%d,%d,%d,%d,%d", &depth, &vb, &hint, &block, &sched, &fmode);
            if (n < 6) fmode = 1;  // five-field strings name the 16-bit-lane kernel (r01 sweeps)
        }
        mode = fmode;
    } else if (const char* v = env_get("POSPOP_STREAM_VARIANT")) {
        std::sscanf(v, "%d,%d,%d,%d,%d", &depth, &vb, &hint, &block, &sched);
    }
    const int nbank = mode == 2 ? 3 : (k == 64 || mode == 1) ? 2 : 1;
    if (opt.depth) depth = opt.depth;
    if (sched == 3 && !opt.block && !opt.grid)
        return launch_stream_tma(mode, nbank, depth, k, data, len_words, d_out, accumulate, opt, ws, stream, grid_used);
    if (sched == 6 && !opt.block && !opt.grid)
        return launch_stream_ring(mode, nbank, depth, k, data, len_words, d_out, accumulate, opt, ws, stream, grid_used);
    if (sched == 3 || sched == 6) sched = 2;  // explicit test geometry: the LDG kernel
    if (opt.block) block = 0;  // explicit (test) block size: the runtime-block instantiation
    const StreamVariant* var = pick_stream(nbank, depth, vb, hint, block, sched, mode);
    if (!var) var = pick_stream(nbank, depth, vb, 0, 0, sched, mode);
    if (!var) return cudaErrorInvalidConfiguration;
    const int threads = var->block ? var->block : (opt.block ? opt.block : kDefaultBlock);
    const int vpt = (mode == 1 ? (1 << var->depth) : mode == 2 ? (2 << var->depth) : (nbank << var->depth)) /
                    (var->vb / 4);

    StreamArgs a;
    fill_stream_args(a, k, data, len_words, (uintptr_t)var->vb, d_out, accumulate, opt, ws);
    a.flush_threshold = flush_threshold_for(mode, opt);
    if (mode != 0) {  // the fused exchange is a count-mode feature
        a.peers = nullptr;
        a.n_peers = 0;
    }

    int grid = opt.grid;
    if (grid <= 0) {
        const unsigned long long tile = (unsigned long long)vpt * threads;
        const unsigned long long want = (a.ng * 32 + tile - 1) / tile;
        const int per_sm = env_int("POSPOP_BLOCKS_PER_SM", resident_blocks(var->fn, threads));
        const unsigned long long cap = (unsigned long long)device_info().sms * per_sm;
        grid = (int)(want < 1 ? 1 : (want < cap ? want : cap));
    }
    set_schedule(a, grid, threads, vpt);
    if (grid_used) *grid_used = grid;
    return launch_with_pdl(var->fn, grid, threads, 0, stream, a, !opt.no_pdl);
}

// Work split shared by the LDG and ring kernels: nwt warp tiles of 32 x vpt
// vectors; SCHED 1 hands them out in chunks of CA then CB; SCHED 2 / 6 split
// [0, nwt - pool) into CTA ranges and hand the pool out in chunks of CB.
static void set_schedule(StreamArgs& a, int grid, int threads, int vpt) {
    // Dynamic schedule: nwt warp tiles; the last ~tail_per_warp warp tiles per
    // warp go out in small chunks of CB, everything before in chunks of CA.
    const unsigned long long wt = 32ull * vpt;
    a.nwt = a.ng ? (a.v1 - a.g0 * 32 + wt - 1) / wt : 0;
    a.CA = (unsigned long long)env_int("POSPOP_CHUNK_A", 16);
    a.CB = (unsigned long long)env_int("POSPOP_CHUNK_B", 2);
    if (a.CA < 1) a.CA = 1;
    if (a.CB < 1) a.CB = 1;
    const unsigned long long warps = (unsigned long long)grid * (threads / 32);
    unsigned long long tail = warps * (unsigned long long)env_int("POSPOP_TAIL_TILES_PER_WARP", 8);
    if (tail > a.nwt) tail = a.nwt;
    a.nA = (a.nwt - tail) / a.CA;
    // SCHED 2: the global tail pool, in warp tiles: ~1/27 of each warp's
    // share, 1..16 tiles per warp (measured, tools/size_curve.py, 16 KiB warp
    // tiles at the default depth: 8 GiB (442 tiles per warp) wants 16 to
    // absorb the tail; at 128 MiB a 16-tile pool would be 58 % of the input
    // and costs 26 % -- pool chunks are claimed by global atomics with worse
    // DRAM locality than the CTA ranges).
    const unsigned long long share = warps ? a.nwt / warps : 0;
    unsigned long long ppw = (unsigned long long)env_int("POSPOP_POOL_TILES_PER_WARP", 0);
    if (ppw == 0) ppw = share / 27 < 1 ? 1 : (share / 27 > 16 ? 16 : share / 27);
    a.pool = warps * ppw;
    if (a.pool > a.nwt) a.pool = a.nwt;
}

// Per-warp bulk-copy ring (SCHED 6, stream_ring_kernel): one CTA of nw warps
// per SM, each warp staging its next `stages` warp tiles in shared memory.
static cudaError_t launch_stream_ring(int mode, int nbank, int depth, int k, const void* data, size_t len_words,
                                      unsigned long long* d_out, bool accumulate, const LaunchOptions& opt,
                                      const StreamWorkspace& ws, cudaStream_t stream, int* grid_used) {
    int nw = 16, stages = 1;
    if (const char* v = env_get("POSPOP_RING")) std::sscanf(v, "%d,%d", &nw, &stages);
    const TmaVariant* var = pick_ring(nbank, depth, mode, nw, stages);
    if (!var) return cudaErrorInvalidConfiguration;
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, bool> configured;
    int dev = 0;
    cudaGetDevice(&dev);
    {
        std::lock_guard<std::mutex> lock(mu);
        auto key = std::make_pair(dev, reinterpret_cast<const void*>(var->fn));
        if (!configured[key]) {
            const cudaError_t e =
                cudaFuncSetAttribute(var->fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)var->smem);
            if (e != cudaSuccess) return e;
            configured[key] = true;
        }
    }
    StreamArgs a;
    fill_stream_args(a, k, data, len_words, 32, d_out, accumulate, opt, ws);
    a.flush_threshold = flush_threshold_for(mode, opt);
    if (mode != 0) {
        a.peers = nullptr;
        a.n_peers = 0;
    }
    const int regs = mode == 2 ? (2 << var->depth) : (nbank << var->depth);
    const int vpt = regs / 8;
    const int threads = 32 * var->nc;
    const unsigned long long tile = (unsigned long long)vpt * threads;
    const unsigned long long want = (a.ng * 32 + tile - 1) / tile;
    const int cap = device_info().sms;
    const int grid = (int)(want < 1 ? 1 : (want < (unsigned long long)cap ? want : cap));
    set_schedule(a, grid, threads, vpt);
    if (grid_used) *grid_used = grid;
    return launch_with_pdl(var->fn, grid, threads, var->smem, stream, a, !opt.no_pdl);
}

// Small inputs (<= POSPOP_SMALL_BYTES, default kSmallBytes): one CTA, no
// workspace, no cross-CTA atomics or ticket -- the latency path (SURVEY 8f
// row f3; the reference's Auto switches kernels below 4096 words too,
// pospop.cpp:84-86).
// measured (tools/latency, profiles/r01_latency_c_abi.csv): one CTA up to 64 KiB,
// one 16-CTA cluster up to 3 MiB (512 KiB: 19.0 -> 13.3 us synchronous), the
// multi-CTA stream kernel above
constexpr int kSmallBytes = 64 << 10;
constexpr int kClusterBytes = 3 << 20;

static cudaError_t launch_small(int k, const void* data, size_t len_words, unsigned long long* d_out,
                                bool accumulate, const LaunchOptions& opt, const StreamWorkspace& ws,
                                cudaStream_t stream, int* grid_used) {
    StreamArgs a;
    fill_stream_args(a, k, data, len_words, 16, d_out, accumulate, opt, ws);
    if (grid_used) *grid_used = 1;
    return launch_with_pdl(k == 64 ? small_kernel<2> : small_kernel<1>, 1, kSmallBlock, 0, stream, a, !opt.no_pdl);
}

// Medium inputs: one thread-block cluster (POSPOP_CLUSTER CTAs, default 16,
// the non-portable maximum; 8 if 16 is refused).
static cudaError_t launch_cluster(int k, const void* data, size_t len_words, unsigned long long* d_out,
                                  bool accumulate, const LaunchOptions& opt, const StreamWorkspace& ws,
                                  cudaStream_t stream, int* grid_used) {
    StreamKernel fn = k == 64 ? cluster_kernel<2> : cluster_kernel<1>;
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, bool> configured;
    int dev = 0;
    cudaGetDevice(&dev);
    {
        std::lock_guard<std::mutex> lock(mu);
        auto key = std::make_pair(dev, reinterpret_cast<const void*>(fn));
        if (!configured[key]) {
            cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
            cudaGetLastError();
            configured[key] = true;
        }
    }
    StreamArgs a;
    fill_stream_args(a, k, data, len_words, 16, d_out, accumulate, opt, ws);
    int csize = env_int("POSPOP_CLUSTER", 16);
    for (;; csize = 8) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)csize);
        cfg.blockDim = dim3((unsigned)kSmallBlock);
        cfg.stream = stream;
        cudaLaunchAttribute attr[2];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = !opt.no_pdl && env_int("POSPOP_PDL", 1) ? 1 : 0;
        attr[1].id = cudaLaunchAttributeClusterDimension;
        attr[1].val.clusterDim.x = (unsigned)csize;
        attr[1].val.clusterDim.y = 1;
        attr[1].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 2;
        const cudaError_t e = cudaLaunchKernelEx(&cfg, fn, a);
        if (e == cudaSuccess) {
            ++g_launches;
            if (grid_used) *grid_used = csize;
            return cudaGetLastError();
        }
        cudaGetLastError();
        if (csize <= 8) return e;
    }
}

cudaError_t launch_stream(int k, const void* data, size_t len_words, unsigned long long* d_out,
                          bool accumulate, const LaunchOptions& opt, const StreamWorkspace& ws,
                          cudaStream_t stream, int* grid_used) {
    env_refresh();
    const size_t nbytes = len_words * (size_t)(k / 8);
    if (!opt.grid && !opt.block && !opt.trace && !opt.depth && !opt.peers && !env_get("POSPOP_STREAM_VARIANT")) {
        if (nbytes <= (size_t)env_int("POSPOP_SMALL_BYTES", kSmallBytes))
            return launch_small(k, data, len_words, d_out, accumulate, opt, ws, stream, grid_used);
        if (nbytes <= (size_t)env_int("POSPOP_CLUSTER_BYTES", kClusterBytes))
            return launch_cluster(k, data, len_words, d_out, accumulate, opt, ws, stream, grid_used);
    }
    return launch_stream_mode(0, k, data, len_words, d_out, accumulate, opt, ws, stream, grid_used);
}

cudaError_t launch_flagstats(const uint16_t* flags, size_t len, unsigned long long* d_out33, bool accumulate,
                             const LaunchOptions& opt, const StreamWorkspace& ws, cudaStream_t stream) {
    env_refresh();
    return launch_stream_mode(2, 16, flags, len, d_out33, accumulate, opt, ws, stream, nullptr);
}

// Adaptive segmented kernel (sched 8) thresholds on the mean array length
// (tools/seg_modes.py, u32: 64-word arrays lane 1523 vs G=4 1003 GB/s;
// 256-word arrays G=4 4269 vs lane 2173; 1024 words G=4 ~ pipelined).
constexpr int kSegLaneMeanBytes = 768;    // one lane per array up to here (k <= 32)
constexpr int kSegLaneMeanBytes64 = 1024; // the same for k = 64 (rows staged one bank half at a time)
constexpr int kSegGroupMeanBytes = 16128; // grouped mode up to here unless tiles fit
constexpr int kSegTileMeanBytes = 8192;  // tile mode from here when whole tile steps cover the mean
constexpr int kSegRange = 8;   // range mode from a mean of 8 x 32 KiB = 256 KiB, or with at most one array per CTA
                               // (POSPOP_SEG_RANGE: 0 = never, 63 = always)
constexpr int kSegGiantKib = 1024;       // arrays above this go through the giant queue
static_assert(dev::kSegRangeSlots == kSegRangeSlotsHost && dev::kGiantQ == kGiantQHost &&
                  dev::kGiantEntry == kGiantEntryHost && kAccChannels + 1 + 7 == 104,
              "segmented workspace regions: pospop_launch.h and pospop_segmented.cuh disagree");

cudaError_t launch_segmented(int k, const void* data, const unsigned long long* d_offsets, size_t n,
                             unsigned long long* d_out, const LaunchOptions& opt, const StreamWorkspace& ws,
                             cudaStream_t stream) {
    if (n == 0) return cudaSuccess;
    env_refresh();
    const int nbank = k == 64 ? 2 : 1;
    // Tuning override: POSPOP_SEG_VARIANT="depth,vb,sched[,lanes per array]".
    // Default: the adaptive kernel (sched 8), which picks one lane per array,
    // 4 lanes per array or the pipelined warp-per-array kernel with the
    // bit-plane epilogue from the mean array length on the device
    // (tools/seg_modes.py).
    int depth = nbank == 1 ? 5 : 4, vb = 16, sched = 8, group = 0;  // (depth/vb name the sched-8 entry)
    if (const char* v = env_get("POSPOP_SEG_VARIANT")) std::sscanf(v, "%d,%d,%d,%d", &depth, &vb, &sched, &group);
    if (opt.depth) depth = opt.depth;
    const SegVariant* var = pick_segmented(nbank, depth, vb, sched, group);
    if (var && var->sched == 16 && n > (size_t)kSegRangeSlotsHost) var = nullptr;  // range kernel: a slot per array
    if (!var) var = pick_segmented(nbank, nbank == 1 ? 5 : 4, 16, 8);
    if (var->sched == 8 && !opt.grid && !opt.block && !env_get("POSPOP_SEG_VARIANT") && n <= (size_t)kSegRangeSlotsHost) {
        // With at most one array per SM the adaptive kernel would pick its range mode whatever the
        // lengths; that choice is made here instead, for the standalone range kernel at one CTA per SM
        // with depth-7 / 32-byte steps (twice the bytes in flight of the adaptive kernel's launch).
        const int range = env_int("POSPOP_SEG_RANGE", kSegRange);
        if (range != 0 && n <= (size_t)device_info().sms) {
            const SegVariant* r = pick_segmented(nbank, nbank == 1 ? 7 : 6, 32, 16, 1);
            if (r) var = r;
        }
    }
    const int block = opt.block ? opt.block : env_int("POSPOP_SEG_BLOCK", kDefaultBlock);
    int grid = opt.grid;
    if (grid <= 0) {
        const unsigned long long warps_per_block = block / 32;
        const unsigned long long per_warp = var->sched == 5 ? 32 / var->group : 1;  // arrays per warp batch
        const unsigned long long want = (n + warps_per_block * per_warp - 1) / (warps_per_block * per_warp);
        // measured (r01 sweep): 4 CTAs/SM for the strided schedule, one resident wave otherwise
        const int per_sm = env_int("POSPOP_SEG_BLOCKS_PER_SM", var->sched == 0 ? 4 : resident_blocks(var->fn, block));
        const unsigned long long cap = (unsigned long long)device_info().sms * per_sm;
        // the adaptive kernel's range mode and the range kernel spread few arrays over every warp
        grid = (int)(want < cap && var->sched != 8 && var->sched != 16 ? want : cap);
    }
    // Last argument: SCHED 1 arrays per grab; SCHED 5 the vector count above
    // which a batch is counted one array at a time by the whole warp.
    unsigned extra = (unsigned)env_int("POSPOP_SEG_PER_GRAB", 1);
    if (extra < 1) extra = 1;
    if (var->sched == 5) extra = (unsigned)((size_t)env_int("POSPOP_SEG_BIG_KIB", 256) * 1024 / var->vb);
    if (var->sched >= 11) extra = (unsigned)env_int("POSPOP_SEG_TAIL_ROUNDS", 4);  // tile kernels: dynamic tail
    if (var->sched == 8) {  // mode bounds: lane mean (64 B units), grouped / tile mean (256 B units), range-mode
                            // mean (32 KiB units; 0 off, 63 always) (6 bits each), giant-array bound (16 KiB, 8 bits)
        auto units = [](int v, unsigned unit, unsigned cap) {
            return (unsigned)(v < 0 ? 0 : ((unsigned)v / unit > cap ? cap : (unsigned)v / unit));
        };
        extra = units(env_int("POSPOP_SEG_LANE_MEAN_BYTES", nbank == 1 ? kSegLaneMeanBytes : kSegLaneMeanBytes64), 64,
                      0x3F) |
                (units(env_int("POSPOP_SEG_GROUP_MEAN_BYTES", kSegGroupMeanBytes), 256, 0x3F) << 6) |
                (units(env_int("POSPOP_SEG_TILE_MEAN_BYTES", kSegTileMeanBytes), 256, 0x3F) << 12) |
                (units(env_int("POSPOP_SEG_RANGE", kSegRange), 1, 0x3F) << 18) |
                (units(env_int("POSPOP_SEG_GIANT_KIB", kSegGiantKib), 16, 0xFF) << 24);
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3((unsigned)block);
    cfg.stream = stream;
    if (var->sched == 10 || (var->sched == 8 && !env_int("POSPOP_SEG_NO_STAGE", 0))) {
        // sched 8: the lane mode stages dev::seg_stage_rows(k) rows per warp at a time (k*8 + 16 bytes
        // each; k = 64: 256-byte bank halves); sched 10: each warp's ring of `group` steps of 32 x VPT
        // 16-byte vectors
        cfg.dynamicSmemBytes = var->sched == 10
                                   ? (size_t)(block / 32) * var->group * 32 * ((size_t)(nbank << var->depth) / 4) * 16
                                   : (size_t)(block / 32) * dev::seg_stage_rows(k) * ((size_t)(k > 32 ? 32 : k) * 8 + 16);
        static std::mutex mu;
        static std::map<std::pair<int, const void*>, size_t> configured;
        int dev = 0;
        cudaGetDevice(&dev);
        std::lock_guard<std::mutex> lock(mu);
        size_t& have = configured[std::make_pair(dev, reinterpret_cast<const void*>(var->fn))];
        if (have < cfg.dynamicSmemBytes) {
            const cudaError_t e = cudaFuncSetAttribute(var->fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                       (int)cfg.dynamicSmemBytes);
            if (e != cudaSuccess) return e;
            have = cfg.dynamicSmemBytes;
        }
    }
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = !opt.no_pdl && env_int("POSPOP_PDL", 1) ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, var->fn, static_cast<const uint8_t*>(data), d_offsets,
                                             (unsigned long long)n, k, opt.flush_threshold, d_out, ws.next,
                                             ws.ticket, extra);
    ++g_launches;
    return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_exchange_reduce(int k, unsigned long long* own, int n_ranks, unsigned long long step, int slots,
                                   unsigned long long* d_total, cudaStream_t stream) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(1);
    cfg.blockDim = dim3(64);
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, exchange_reduce_kernel, own, n_ranks, k, slots, step, d_total);
    ++g_launches;
    return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_exchange_emulate(unsigned long long* const* bufs, int n_ranks, int k, int slots, int steps,
                                    const unsigned long long* inputs, const unsigned* sleep_ns,
                                    unsigned long long* totals, cudaStream_t stream) {
    void* args[] = {(void*)&bufs, &n_ranks, &k, &slots, &steps, (void*)&inputs, (void*)&sleep_ns, &totals};
    const cudaError_t e = cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(exchange_emulate_kernel),
                                                      dim3((unsigned)n_ranks), dim3(64), args, 0, stream);
    ++g_launches;
    return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_generate(int kind, uint64_t seed, uint64_t index_base, size_t n, void* out,
                            cudaStream_t stream) {
    if (n == 0) return cudaSuccess;
    const uint64_t key = mix64(seed ^ ((uint64_t)kind * 0xD1B54A32D192ED03ull));
    const int block = 256;
    const unsigned long long want = (n + block - 1) / block;
    const unsigned long long cap = (unsigned long long)device_info().sms * 16;
    generate_kernel<<<(int)(want < cap ? want : cap), block, 0, stream>>>(kind, key, index_base, n, out);
    ++g_launches;
    return cudaGetLastError();
}

cudaError_t launch_microop(int op, int depth, const uint32_t* d_in, size_t n, uint32_t* d_out, cudaStream_t stream) {
    microop_kernel<<<1, 32, 0, stream>>>(op, depth, d_in, n, d_out);
    ++g_launches;
    return cudaGetLastError();
}

cudaError_t launch_digest(const void* data, size_t nbytes, unsigned long long* d_digest,
                          cudaStream_t stream) {
    if (nbytes == 0) return cudaSuccess;
    const int block = 256;
    const unsigned long long want = ((nbytes + 7) / 8 + block - 1) / block;
    const unsigned long long cap = (unsigned long long)device_info().sms * 16;
    digest_kernel<<<(int)(want < cap ? want : cap), block, 0, stream>>>(
        static_cast<const uint8_t*>(data), nbytes, d_digest);
    ++g_launches;
    return cudaGetLastError();
}

}  // namespace pospop_b200
