// pospop_capi.cpp -- extern "C" boundary and host runtime (include/pospopcnt_b200.h).
//
// Mirrors the reference dispatcher pospop::pospopcnt (proj/core/src/pospop.cpp:80-111):
// validate -> resolve kernel kind / width (errors as the reference) -> count.
// Counting always runs on the GPU: device-resident input is counted in place;
// host input is streamed through pinned-size device staging buffers with
// H2D copies on a copy stream overlapping the kernel on the compute stream.
// There is no CPU fallback path.
#include <cuda_runtime.h>

#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cctype>
#include <cerrno>
#include <pthread.h>
#include <sched.h>
#include <condition_variable>
#include <deque>
#include <cstdarg>
#include <functional>
#include <thread>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <set>
#include <string>
#include <utility>
#include <vector>

#include "../../include/pospopcnt_b200.h"
#include "pospop_exchange.h"
#include "pospop_launch.h"

using namespace pospop_b200;

namespace {

thread_local std::string t_err;

pospop_status fail(pospop_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    std::vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    t_err = buf;
    return s;
}

pospop_status cuda_fail(cudaError_t e, const char* what) {
    const pospop_status s = (e == cudaErrorMemoryAllocation) ? POSPOP_ENOMEM
                            : (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver ||
                               e == cudaErrorNoKernelImageForDevice)
                                ? POSPOP_EUNAVAILABLE
                                : POSPOP_ECUDA;
    cudaGetLastError();  // clear sticky-free errors
    return fail(s, "%s: %s (%s)", what, cudaGetErrorString(e), cudaGetErrorName(e));
}

#define CU(call)                                           \
    do {                                                   \
        const cudaError_t e_ = (call);                     \
        if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
    } while (0)

bool valid_k(int k) { return k == 8 || k == 16 || k == 32 || k == 64; }

// ---------------------------------------------------------------------------
// Device discovery: sm_100 class only (the fatbin carries sm_100a SASS).
// ---------------------------------------------------------------------------
pospop_status check_device(int dev) {
    static thread_local int checked = -1;  // last device that passed (cheap fast path per call)
    if (dev == checked) return POSPOP_OK;
    int major = 0;
    const cudaError_t e = cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceGetAttribute");
    if (major != 10)
        return fail(POSPOP_EUNAVAILABLE,
                    "kernel unavailable: device %d is compute capability %d.x, sm_100 required", dev,
                    major);
    checked = dev;
    return POSPOP_OK;
}

pospop_status current_device(int* dev) {
    int n = 0;
    const cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) {
        cudaGetLastError();
        return fail(POSPOP_EUNAVAILABLE, "kernel unavailable: no CUDA device (%s); no CPU fallback",
                    e == cudaSuccess ? "device count 0" : cudaGetErrorString(e));
    }
    CU(cudaGetDevice(dev));
    return check_device(*dev);
}

pospop_status cuda_set_device(int dev) {
    CU(cudaSetDevice(dev));
    return POSPOP_OK;
}

// Parses a sysfs CPU list ("0-15,32-47") into `set`; false if empty.
bool parse_cpulist(const char* text, cpu_set_t* set) {
    CPU_ZERO(set);
    bool any = false;
    const char* p = text;
    while (*p) {
        char* end = nullptr;
        const long lo = std::strtol(p, &end, 10);
        if (end == p) break;
        long hi = lo;
        p = end;
        if (*p == '-') {
            hi = std::strtol(p + 1, &end, 10);
            p = end;
        }
        for (long c = lo; c <= hi && c < CPU_SETSIZE; ++c) {
            CPU_SET((int)c, set);
            any = true;
        }
        if (*p == ',') ++p;
        else break;
    }
    return any;
}

// The CPUs local to device `dev` (sysfs local_cpulist of its PCI function).
bool device_cpus(int dev, cpu_set_t* set) {
    char bus[32] = {};
    if (cudaDeviceGetPCIBusId(bus, sizeof bus, dev) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    for (char* q = bus; *q; ++q) *q = (char)std::tolower((unsigned char)*q);
    const std::string path = std::string("/sys/bus/pci/devices/") + bus + "/local_cpulist";
    FILE* f = std::fopen(path.c_str(), "r");
    if (!f) return false;
    char buf[1024] = {};
    const bool ok = std::fgets(buf, sizeof buf, f) != nullptr;
    std::fclose(f);
    return ok && parse_cpulist(buf, set);
}

// Binds the calling thread to the CPUs local to device `dev` (host-shard
// workers: their memcpy / DMA source stays on the device's NUMA node).
bool bind_to_device_cpus(int dev) {
    cpu_set_t set;
    return device_cpus(dev, &set) && pthread_setaffinity_np(pthread_self(), sizeof set, &set) == 0;
}

// Runs the calling thread on device `dev`'s local CPUs for the lifetime of
// the scope (pinned host buffers allocated inside are first touched there,
// so they land on the device's NUMA node), then restores its affinity.
struct NumaScope {
    cpu_set_t saved;
    bool restore = false;
    explicit NumaScope(int dev) {
        cpu_set_t set;
        if (pthread_getaffinity_np(pthread_self(), sizeof saved, &saved) == 0 && device_cpus(dev, &set))
            restore = pthread_setaffinity_np(pthread_self(), sizeof set, &set) == 0;
    }
    ~NumaScope() {
        if (restore) pthread_setaffinity_np(pthread_self(), sizeof saved, &saved);
    }
};

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

// ---------------------------------------------------------------------------
// Per-call device context: compute + copy streams, result buffers, the
// stream workspace, and (lazily) the host-staging ring.  Contexts are leased
// from a per-device pool for the duration of one call (CtxScope), so
// resources are bounded per device -- at most kMaxCtxPerDevice contexts for
// the calls in flight (plus one per host shard of a pospopcnt_sharded call
// in flight) -- whatever the number of calling threads, and nothing is tied
// to a thread.
// pospop_release_resources() frees the idle ones.  (The reference keeps all
// per-call state on the stack, proj/core/src/detail/csa_engine.hpp:107-110;
// device allocation per call would synchronise the device, so the pool is the
// closest B200 equivalent.)
// ---------------------------------------------------------------------------
constexpr int kRing = 3;
constexpr size_t kBounceBytes = 1 << 20;  // pageable host inputs up to this size: pinned bounce copy, zero-copy kernel
constexpr size_t kZeroCopyBytes = 2 << 20;  // pinned host inputs up to this size: read in place by the kernel
constexpr int kHostRing = 4;              // pinned host slots for pageable / file input
constexpr size_t kHostChunk = 16 << 20;   // bytes per pinned host slot
constexpr int kMaxCtxPerDevice = 8;       // concurrent calls per device beyond this wait for a context

// Persistent host worker threads for the CPU side of host-input pipelines
// (parallel memcpy from pageable memory, parallel pread from files) into the
// pinned host ring; one process-wide pool, one job at a time.
class HostPool {
  public:
    static HostPool& get() {
        static HostPool pool;
        return pool;
    }
    int size() const { return (int)workers_.size() + 1; }
    // Runs fn(0 .. tasks-1) on the pool and the calling thread; returns when all are done.
    void run(int tasks, const std::function<void(int)>& fn) {
        std::lock_guard<std::mutex> job(job_mu_);
        {
            std::lock_guard<std::mutex> lk(mu_);
            fn_ = &fn;
            tasks_ = tasks;
            next_ = 0;
            done_ = 0;
            ++gen_;
        }
        cv_.notify_all();
        work();
        std::unique_lock<std::mutex> lk(mu_);
        done_cv_.wait(lk, [&] { return done_ == tasks_; });
        fn_ = nullptr;
    }

  private:
    HostPool() {
        const char* env = std::getenv("POSPOP_HOST_THREADS");
        int n = env && *env ? std::atoi(env) : (int)std::thread::hardware_concurrency();
        if (n > 32) n = 32;
        for (int i = 1; i < n; ++i) workers_.emplace_back([this] { loop(); });
    }
    ~HostPool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : workers_) t.join();
    }
    void work() {
        for (;;) {
            int t;
            const std::function<void(int)>* fn;
            {
                std::lock_guard<std::mutex> lk(mu_);
                if (!fn_ || next_ >= tasks_) return;
                t = next_++;
                fn = fn_;
            }
            (*fn)(t);
            std::lock_guard<std::mutex> lk(mu_);
            if (++done_ == tasks_) done_cv_.notify_all();
        }
    }
    void loop() {
        unsigned long long seen = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
                if (stop_) return;
                seen = gen_;
            }
            work();
        }
    }
    std::vector<std::thread> workers_;
    std::mutex job_mu_, mu_;
    std::condition_variable cv_, done_cv_;
    const std::function<void(int)>* fn_ = nullptr;
    int tasks_ = 0, next_ = 0, done_ = 0;
    unsigned long long gen_ = 0;
    bool stop_ = false;
};

// Parallel memcpy of `n` bytes in 1 MiB pieces on the host pool.
void parallel_copy(void* dst, const void* src, size_t n) {
    constexpr size_t kPiece = 1 << 20;
    const int tasks = (int)((n + kPiece - 1) / kPiece);
    HostPool::get().run(tasks, [&](int t) {
        const size_t lo = (size_t)t * kPiece;
        const size_t len = n - lo < kPiece ? n - lo : kPiece;
        std::memcpy(static_cast<uint8_t*>(dst) + lo, static_cast<const uint8_t*>(src) + lo, len);
    });
}

struct Ctx {
    int dev = -1;
    cudaStream_t stream = nullptr;
    cudaStream_t copy = nullptr;
    unsigned long long* d_out = nullptr;  // 64 u64
    unsigned long long* h_out = nullptr;  // 64 u64, pinned
    // Synchronous calls let the kernel's last CTA write the result straight
    // into mapped pinned memory: no D2H copy on the small-call latency path.
    unsigned long long* m_out = nullptr;      // 64 u64, pinned + mapped (host view)
    unsigned long long* m_out_dev = nullptr;  // its device view
    StreamWorkspace ws;      // stream / FLAG launches (kStreamWorkspaceBytes)
    StreamWorkspace seg_ws;  // segmented launches (kWorkspaceBytes, on first segmented use)
    void* stage[kRing] = {nullptr, nullptr, nullptr};
    void* bounce = nullptr;  // pinned host buffer for small host inputs (kBounceBytes)
    size_t stage_bytes = 0;
    cudaEvent_t ev_copied[kRing] = {};
    cudaEvent_t ev_done[kRing] = {};
    // grow-only device scratch for the synchronous segmented call (data, offsets, rows)
    void* scratch[3] = {};
    size_t scratch_cap[3] = {};
    // segmented calls on host data: rows come back on their own stream, per
    // chunk, through a grow-only pinned staging buffer when the caller's rows
    // are pageable; one event pair per chunk (grow-only pool)
    cudaStream_t d2h = nullptr;
    void* rows_pinned = nullptr;
    size_t rows_pinned_cap = 0;
    std::vector<cudaEvent_t> seg_ev;
    // pospopcnt_sharded: per shard on this device a stream, a workspace and a
    // mapped pinned result (kept for reuse; no allocation per call)
    struct ShardSlot {
        cudaStream_t stream = nullptr;
        StreamWorkspace ws;
        unsigned long long* m_out = nullptr;
        unsigned long long* m_out_dev = nullptr;
    };
    std::deque<ShardSlot> shard_slots;  // deque: push_back keeps references to earlier slots valid
    // pinned host ring for pageable / file input (lazily allocated)
    uint8_t* host_ring[kHostRing] = {};
    cudaEvent_t ev_h2d[kHostRing] = {};  // the H2D that last read host_ring[i] is done
    bool host_used[kHostRing] = {};
};

pospop_status alloc_workspace(StreamWorkspace* ws, bool segmented = false) {
    const size_t bytes = segmented ? kWorkspaceBytes : kStreamWorkspaceBytes;
    CU(cudaMalloc(&ws->acc, bytes));
    ws->ticket = reinterpret_cast<unsigned int*>(ws->acc + kAccChannels);
    ws->next = ws->acc + kAccChannels + 1;
    ws->bad = ws->acc + kAccChannels + 2;
    CU(cudaMemset(ws->acc, 0, bytes));
    return POSPOP_OK;
}

void free_workspace(StreamWorkspace* ws) {
    if (ws->acc) cudaFree(ws->acc);
    *ws = StreamWorkspace{};
}

// Frees everything a context owns (its device must be current).  Pending work
// on its streams is waited for first (a call that failed part-way may have
// left some).
void destroy_ctx(Ctx* c) {
    for (cudaStream_t st : {c->stream, c->copy, c->d2h})
        if (st) cudaStreamSynchronize(st);
    for (auto& slot : c->shard_slots) {
        if (slot.stream) {
            cudaStreamSynchronize(slot.stream);
            cudaStreamDestroy(slot.stream);
        }
        free_workspace(&slot.ws);
        if (slot.m_out) cudaFreeHost(slot.m_out);
    }
    free_workspace(&c->ws);
    free_workspace(&c->seg_ws);
    for (int i = 0; i < kRing; ++i) {
        if (c->stage[i]) cudaFree(c->stage[i]);
        if (c->ev_copied[i]) cudaEventDestroy(c->ev_copied[i]);
        if (c->ev_done[i]) cudaEventDestroy(c->ev_done[i]);
    }
    for (int i = 0; i < kHostRing; ++i) {
        if (c->host_ring[i]) cudaFreeHost(c->host_ring[i]);
        if (c->ev_h2d[i]) cudaEventDestroy(c->ev_h2d[i]);
    }
    for (void* p : c->scratch)
        if (p) cudaFree(p);
    for (cudaEvent_t e : c->seg_ev) cudaEventDestroy(e);
    if (c->rows_pinned) cudaFreeHost(c->rows_pinned);
    if (c->bounce) cudaFreeHost(c->bounce);
    if (c->d_out) cudaFree(c->d_out);
    if (c->h_out) cudaFreeHost(c->h_out);
    if (c->m_out) cudaFreeHost(c->m_out);
    for (cudaStream_t st : {c->stream, c->copy, c->d2h})
        if (st) cudaStreamDestroy(st);
    cudaGetLastError();
    delete c;
}

pospop_status create_ctx(int dev, Ctx** out) {
    Ctx* c = new Ctx;
    c->dev = dev;
    struct Undo {  // frees the partial context if a step below fails
        Ctx*& c;
        ~Undo() {
            if (c) destroy_ctx(c);
        }
    } undo{c};
    // Blocking streams: synchronous entry points are ordered after prior work
    // on the legacy default stream (where callers typically produced the data).
    CU(cudaStreamCreateWithFlags(&c->stream, cudaStreamDefault));
    CU(cudaStreamCreateWithFlags(&c->copy, cudaStreamDefault));
    CU(cudaMalloc(&c->d_out, 64 * sizeof(unsigned long long)));
    CU(cudaMallocHost(&c->h_out, 64 * sizeof(unsigned long long)));
    CU(cudaHostAlloc(&c->m_out, 64 * sizeof(unsigned long long), cudaHostAllocMapped));
    CU(cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->m_out_dev), c->m_out, 0));
    pospop_status s = alloc_workspace(&c->ws);
    if (s) return s;
    *out = c;
    c = nullptr;  // keep it
    return POSPOP_OK;
}

struct CtxPool {
    std::mutex mu;
    std::condition_variable cv;
    std::map<int, std::vector<Ctx*>> idle;
    std::map<int, int> live;  // leased + idle, per device
    static CtxPool& get() {
        static CtxPool* pool = new CtxPool;  // never destroyed: no CUDA calls during process exit
        return *pool;
    }
};

// The contexts one call holds, returned to the pool when the call returns.
// A call that needs several devices acquires them in ascending device order
// (pospopcnt_sharded), so bounded pools cannot deadlock.
class CtxScope {
  public:
    CtxScope() = default;
    CtxScope(const CtxScope&) = delete;
    CtxScope& operator=(const CtxScope&) = delete;
    ~CtxScope() {
        if (held_.empty()) return;
        CtxPool& pool = CtxPool::get();
        std::vector<std::pair<int, Ctx*>> surplus;  // above the bound (unbounded worker leases): freed
        {
            std::lock_guard<std::mutex> lk(pool.mu);
            for (auto& h : held_) {
                if (pool.live[h.first] > kMaxCtxPerDevice) {
                    --pool.live[h.first];
                    surplus.push_back(h);
                } else {
                    pool.idle[h.first].push_back(h.second);
                }
            }
        }
        pool.cv.notify_all();
        for (auto& h : surplus) {
            DeviceGuard g(h.first);
            destroy_ctx(h.second);
        }
    }
    // bounded = false: never wait for the per-device bound (the host-shard
    // workers of a call whose caller already holds contexts: waiting there
    // could deadlock against other callers doing the same).
    pospop_status get(int dev, Ctx** out, bool bounded = true) {
        for (auto& h : held_)
            if (h.first == dev) {
                *out = h.second;
                return POSPOP_OK;
            }
        pospop_status s = check_device(dev);
        if (s) return s;
        CtxPool& pool = CtxPool::get();
        Ctx* c = nullptr;
        {
            std::unique_lock<std::mutex> lk(pool.mu);
            if (bounded)
                pool.cv.wait(lk, [&] { return !pool.idle[dev].empty() || pool.live[dev] < kMaxCtxPerDevice; });
            if (!pool.idle[dev].empty()) {
                c = pool.idle[dev].back();
                pool.idle[dev].pop_back();
            } else {
                ++pool.live[dev];
            }
        }
        if (!c) {
            DeviceGuard g(dev);
            if ((s = create_ctx(dev, &c))) {
                {
                    std::lock_guard<std::mutex> lk(pool.mu);
                    --pool.live[dev];
                }
                pool.cv.notify_all();
                return s;
            }
        }
        held_.emplace_back(dev, c);
        *out = c;
        return POSPOP_OK;
    }

  private:
    std::vector<std::pair<int, Ctx*>> held_;
};

pospop_status ensure_seg_ws(Ctx* c) {
    if (c->seg_ws.acc) return POSPOP_OK;
    return alloc_workspace(&c->seg_ws, true);
}

pospop_status ensure_stage(Ctx* c) {
    if (c->stage[0]) return POSPOP_OK;
    const char* env = std::getenv("POSPOP_STAGE_MB");
    size_t mb = env && *env ? std::strtoull(env, nullptr, 10) : 64;
    if (mb < 1) mb = 1;
    c->stage_bytes = mb << 20;
    for (int i = 0; i < kRing; ++i) {
        CU(cudaMalloc(&c->stage[i], c->stage_bytes));
        CU(cudaEventCreateWithFlags(&c->ev_copied[i], cudaEventDisableTiming));
        CU(cudaEventCreateWithFlags(&c->ev_done[i], cudaEventDisableTiming));
    }
    return POSPOP_OK;
}

pospop_status ensure_host_ring(Ctx* c) {
    if (c->host_ring[0]) return POSPOP_OK;
    NumaScope numa(c->dev);
    for (int i = 0; i < kHostRing; ++i) {
        CU(cudaMallocHost(&c->host_ring[i], kHostChunk));
        CU(cudaEventCreateWithFlags(&c->ev_h2d[i], cudaEventDisableTiming));
    }
    return POSPOP_OK;
}

// Host input through the pinned ring: `produce(slot_ptr, offset, bytes)`
// fills a pinned slot (parallel memcpy or pread, on the host pool) while the
// previous slots' H2D copies (copy stream) and kernels (compute stream) run.
// `launch(dev_ptr, offset, bytes, chunk_index)` enqueues the counting kernel.
template <class Produce, class Launch>
pospop_status host_ring_pipeline(Ctx* c, size_t total_bytes, size_t align, Produce produce, Launch launch) {
    pospop_status s;
    if ((s = ensure_stage(c))) return s;
    if ((s = ensure_host_ring(c))) return s;
    const size_t chunk = kHostChunk < c->stage_bytes ? kHostChunk : c->stage_bytes;  // multiple of `align`
    (void)align;
    size_t i = 0;
    for (size_t off = 0; off < total_bytes; off += chunk, ++i) {
        const size_t n = total_bytes - off < chunk ? total_bytes - off : chunk;
        const int hs = (int)(i % kHostRing), ds = (int)(i % kRing);
        if (c->host_used[hs]) CU(cudaEventSynchronize(c->ev_h2d[hs]));
        if ((s = produce(c->host_ring[hs], off, n))) return s;
        if (i >= (size_t)kRing) CU(cudaStreamWaitEvent(c->copy, c->ev_done[ds], 0));
        CU(cudaMemcpyAsync(c->stage[ds], c->host_ring[hs], n, cudaMemcpyHostToDevice, c->copy));
        CU(cudaEventRecord(c->ev_h2d[hs], c->copy));
        c->host_used[hs] = true;
        CU(cudaEventRecord(c->ev_copied[ds], c->copy));
        CU(cudaStreamWaitEvent(c->stream, c->ev_copied[ds], 0));
        if ((s = launch(c->stage[ds], off, n, i))) return s;
        CU(cudaEventRecord(c->ev_done[ds], c->stream));
    }
    return POSPOP_OK;
}

// Grow-only device scratch buffer `i` of the context (no cudaMalloc/cudaFree
// per call: cudaFree synchronises the device).
pospop_status ctx_scratch(Ctx* c, int i, size_t bytes, void** out) {
    if (c->scratch_cap[i] < bytes) {
        if (c->scratch[i]) {
            CU(cudaStreamSynchronize(c->stream));
            CU(cudaFree(c->scratch[i]));
            c->scratch[i] = nullptr;
            c->scratch_cap[i] = 0;
        }
        CU(cudaMalloc(&c->scratch[i], bytes));
        c->scratch_cap[i] = bytes;
    }
    *out = c->scratch[i];
    return POSPOP_OK;
}

pospop_status ensure_seg_pipeline(Ctx* c, size_t events, size_t pinned_row_bytes) {
    if (!c->d2h) CU(cudaStreamCreateWithFlags(&c->d2h, cudaStreamNonBlocking));
    while (c->seg_ev.size() < events) {
        cudaEvent_t e;
        CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        c->seg_ev.push_back(e);
    }
    if (c->rows_pinned_cap < pinned_row_bytes) {
        if (c->rows_pinned) {
            CU(cudaStreamSynchronize(c->d2h));
            CU(cudaFreeHost(c->rows_pinned));
            c->rows_pinned = nullptr;
            c->rows_pinned_cap = 0;
        }
        CU(cudaMallocHost(&c->rows_pinned, pinned_row_bytes));
        c->rows_pinned_cap = pinned_row_bytes;
    }
    return POSPOP_OK;
}

// Host -> device copy of a contiguous range on the compute stream; pageable
// sources go through the pinned host ring with parallel memcpy.
pospop_status h2d_on_stream(Ctx* c, void* dst, const void* src, size_t bytes, bool pinned) {
    if (pinned || bytes <= kBounceBytes) {
        CU(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c->stream));
        return POSPOP_OK;
    }
    pospop_status s;
    if ((s = ensure_host_ring(c))) return s;
    size_t i = 0;
    for (size_t off = 0; off < bytes; off += kHostChunk, ++i) {
        const size_t n = bytes - off < kHostChunk ? bytes - off : kHostChunk;
        const int hs = (int)(i % kHostRing);
        if (c->host_used[hs]) CU(cudaEventSynchronize(c->ev_h2d[hs]));
        parallel_copy(c->host_ring[hs], static_cast<const uint8_t*>(src) + off, n);
        CU(cudaMemcpyAsync(static_cast<uint8_t*>(dst) + off, c->host_ring[hs], n, cudaMemcpyHostToDevice, c->stream));
        CU(cudaEventRecord(c->ev_h2d[hs], c->stream));
        c->host_used[hs] = true;
    }
    return POSPOP_OK;
}

// Workspaces for the async entry point, one per (device, stream), plus the
// output ranges of the stream's recent launches: a launch whose input overlaps
// one of them is enqueued without programmatic dependent launch (our kernels
// let dependents start early and read their own input before waiting).
struct StreamState {
    StreamWorkspace ws;      // stream / exchange launches
    StreamWorkspace seg_ws;  // segmented launches (on first use)
    static constexpr int kHist = 8;
    uintptr_t out_lo[kHist] = {}, out_hi[kHist] = {};
    int next = 0;
};
std::mutex g_ws_mu;
std::map<std::pair<int, cudaStream_t>, StreamState> g_ws;

pospop_status stream_workspace(int dev, cudaStream_t s, StreamWorkspace* out, const void* in = nullptr,
                               size_t in_bytes = 0, const void* dst = nullptr, size_t dst_bytes = 0,
                               bool* no_pdl = nullptr, const void* in2 = nullptr, size_t in2_bytes = 0,
                               bool segmented = false) {
    std::lock_guard<std::mutex> lock(g_ws_mu);
    auto key = std::make_pair(dev, s);
    auto it = g_ws.find(key);
    if (it == g_ws.end()) {
        StreamState st;
        const pospop_status e = alloc_workspace(&st.ws);
        if (e) return e;
        it = g_ws.emplace(key, st).first;
    }
    StreamState& st = it->second;
    if (segmented && !st.seg_ws.acc) {
        const pospop_status e = alloc_workspace(&st.seg_ws, true);
        if (e) return e;
    }
    if (no_pdl) {
        const uintptr_t lo = reinterpret_cast<uintptr_t>(in), hi = lo + in_bytes;
        *no_pdl = false;
        const uintptr_t lo2 = reinterpret_cast<uintptr_t>(in2), hi2 = lo2 + in2_bytes;
        for (int i = 0; i < StreamState::kHist; ++i) {
            if (in_bytes && st.out_hi[i] > lo && st.out_lo[i] < hi) *no_pdl = true;
            if (in2_bytes && st.out_hi[i] > lo2 && st.out_lo[i] < hi2) *no_pdl = true;
        }
        if (dst) {
            st.out_lo[st.next] = reinterpret_cast<uintptr_t>(dst);
            st.out_hi[st.next] = reinterpret_cast<uintptr_t>(dst) + dst_bytes;
            st.next = (st.next + 1) % StreamState::kHist;
        }
    }
    *out = segmented ? st.seg_ws : st.ws;
    return POSPOP_OK;
}

// The device allocation holding `p` (cuMemGetAddressRange through the runtime's
// driver entry point): the bound on what a kernel indexing from `p` with
// device-resident offsets can read.  False if it cannot be determined.
bool alloc_range(const void* p, const void** base, size_t* bytes) {
    using Fn = int (*)(unsigned long long*, size_t*, unsigned long long);
    static Fn fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            f = nullptr;
        return reinterpret_cast<Fn>(f);
    }();
    unsigned long long b = 0;
    size_t n = 0;
    if (!fn || !p || fn(&b, &n, reinterpret_cast<unsigned long long>(p)) != 0) return false;
    *base = reinterpret_cast<const void*>(b);
    *bytes = n;
    return true;
}

// ---------------------------------------------------------------------------
// Pointer classification.
// ---------------------------------------------------------------------------
enum class Where { Device, Host };

// mapped: for pinned host memory, its device-accessible address (UVA), or
// NULL when the allocation is not mapped.
Where classify(const void* p, int* dev, bool* pinned = nullptr, const void** mapped = nullptr) {
    cudaPointerAttributes a;
    std::memset(&a, 0, sizeof a);
    if (pinned) *pinned = false;
    if (mapped) *mapped = nullptr;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return Where::Host;
    }
    if (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) {
        *dev = a.device;
        return Where::Device;
    }
    if (pinned) *pinned = a.type == cudaMemoryTypeHost;
    if (mapped && a.type == cudaMemoryTypeHost) *mapped = a.devicePointer;
    return Where::Host;
}

// ---------------------------------------------------------------------------
// The counting core: k in {8,16,32,64}, result in out[0..k).
// ---------------------------------------------------------------------------
pospop_status count_on_ctx(Ctx* c, int k, const void* data, size_t len, bool on_device, bool pinned, uint32_t flush,
                           uint64_t* out);

pospop_status count_any(int k, const void* data, size_t len, uint32_t flush, uint64_t* out) {
    if (!valid_k(k)) return fail(POSPOP_EINVAL, "k must be 8, 16, 32 or 64, got %d", k);
    if (!out) return fail(POSPOP_EINVAL, "counts must not be NULL");
    if (flush < 1 || flush > 65535)
        return fail(POSPOP_EINVAL, "flush_threshold_blocks must be in [1, 65535], got %u", flush);
    if (!data && len) return fail(POSPOP_EINVAL, "data is NULL but len is %zu", len);
    const size_t wb = (size_t)k / 8;
    if ((uintptr_t)data % wb)
        return fail(POSPOP_EINVAL, "data %p is not aligned to the %d-bit word size", data, k);
    int dev = 0;
    pospop_status s = current_device(&dev);
    if (s) return s;
    if (len == 0) {
        for (int p = 0; p < k; ++p) out[p] = 0;
        return POSPOP_OK;
    }
    bool pinned = false;
    const Where where = classify(data, &dev, &pinned);
    DeviceGuard g(dev);
    CtxScope scope;
    Ctx* c = nullptr;
    if ((s = scope.get(dev, &c))) return s;
    return count_on_ctx(c, k, data, len, where == Where::Device, pinned, flush, out);
}

// Counts len (> 0) k-bit words at data on context c's device (current):
// device memory in place, host memory through the staging pipelines.
pospop_status count_on_ctx(Ctx* c, int k, const void* data, size_t len, bool on_device, bool pinned, uint32_t flush,
                           uint64_t* out) {
    pospop_status s;
    const size_t wb = (size_t)k / 8;
    LaunchOptions opt;
    opt.flush_threshold = flush;
    if (on_device) {
        CU(launch_stream(k, data, len, c->m_out_dev, false, opt, c->ws, c->stream));
    } else if (len * wb <= (pinned ? kZeroCopyBytes : kBounceBytes)) {
        // Small host input (the latency path): the kernel
        // reads the caller's pinned memory -- or a pinned bounce copy of
        // pageable memory -- in place over the host link (zero-copy through
        // UVA): no DMA, no device staging, one launch on one stream, the
        // result written by the last CTA into mapped memory.  Above
        // kZeroCopyBytes the copy engine's larger transfers win
        // (tools/zero_copy_probe.py).
        const void* src = data;
        const void* dsrc = nullptr;
        int hd = c->dev;
        if (!pinned) {
            if (!c->bounce) CU(cudaMallocHost(&c->bounce, kBounceBytes));
            std::memcpy(c->bounce, data, len * wb);
            src = c->bounce;
        }
        classify(src, &hd, nullptr, &dsrc);
        if (dsrc) {
            CU(launch_stream(k, dsrc, len, c->m_out_dev, false, opt, c->ws, c->stream));
        } else {  // pinned but not mapped: one DMA into the staging buffer
            if ((s = ensure_stage(c))) return s;
            CU(cudaMemcpyAsync(c->stage[0], src, len * wb, cudaMemcpyHostToDevice, c->stream));
            CU(launch_stream(k, c->stage[0], len, c->m_out_dev, false, opt, c->ws, c->stream));
        }
    } else if (!pinned) {
        // Pageable host input: parallel memcpy into the pinned host ring
        // overlapping the H2D of the previous slot and the kernel before it.
        const uint8_t* src = static_cast<const uint8_t*>(data);
        s = host_ring_pipeline(
            c, len * wb, wb,
            [&](uint8_t* dst, size_t off, size_t n) {
                parallel_copy(dst, src + off, n);
                return POSPOP_OK;
            },
            [&](const void* d, size_t, size_t n, size_t i) -> pospop_status {
                CU(launch_stream(k, d, n / wb, c->m_out_dev, i > 0, opt, c->ws, c->stream));
                return POSPOP_OK;
            });
        if (s) return s;
    } else {
        // Pinned host input: chunked H2D straight from the caller's buffer on
        // the copy stream, counting on the compute stream, kRing staging
        // buffers recycled behind ev_done.
        if ((s = ensure_stage(c))) return s;
        const size_t chunk_words = c->stage_bytes / wb;
        const uint8_t* src = static_cast<const uint8_t*>(data);
        size_t i = 0;
        for (size_t off = 0; off < len; off += chunk_words, ++i) {
            const size_t n = len - off < chunk_words ? len - off : chunk_words;
            const int slot = (int)(i % kRing);
            if (i >= (size_t)kRing) CU(cudaStreamWaitEvent(c->copy, c->ev_done[slot], 0));
            CU(cudaMemcpyAsync(c->stage[slot], src + off * wb, n * wb, cudaMemcpyHostToDevice, c->copy));
            CU(cudaEventRecord(c->ev_copied[slot], c->copy));
            CU(cudaStreamWaitEvent(c->stream, c->ev_copied[slot], 0));
            CU(launch_stream(k, c->stage[slot], n, c->m_out_dev, i > 0, opt, c->ws, c->stream));
            CU(cudaEventRecord(c->ev_done[slot], c->stream));
        }
    }
    CU(cudaStreamSynchronize(c->stream));  // the last CTA wrote c->m_out (mapped)
    for (int p = 0; p < k; ++p) out[p] = c->m_out[p];
    return POSPOP_OK;
}

// Segmented call on host data above kSegPipeMin bytes.  The arrays are cut
// at array boundaries into units of at most kSegChunk bytes; an array longer
// than that is a unit of its own, sent in kSegChunk pieces.  Unit i goes
// through device staging slot i % kRing (the count path's 3 x 64 MiB ring, so
// device memory stays bounded whatever the input size): its H2D on the copy
// stream (pageable data through the pinned host ring), its launch on the
// compute stream -- the segmented kernel over the unit's arrays, or for a
// piece of a long array the stream kernel accumulating into that array's row
// -- and the D2H of its rows on a third stream (pageable rows through a
// grow-only pinned row buffer, copied out as each D2H completes) all overlap
// the neighbouring units, so the call runs at the H2D link rate.  Each unit is
// staged at the same 32-byte phase as in host memory, with slack on both sides
// for the kernels' masked edge vectors.
constexpr size_t kSegPipeMin = 8u << 20;
constexpr size_t kSegChunk = 32u << 20;  // <= stage_bytes - 128

struct SegUnit {
    size_t a0, a1;   // arrays [a0, a1); a long array: a1 = a0 + 1
    size_t lo, hi;   // bytes relative to the first referenced byte
    bool piece;      // a piece of a long array (stream kernel, accumulating)
    bool first_piece, last_piece;
};

pospop_status segmented_host_pipeline(Ctx* c, int k, const void* data, const uint64_t* offsets, bool o_dev,
                                      const uint64_t* hoff, size_t n, uint64_t* counts, bool c_dev) {
    pospop_status s;
    if ((s = ensure_seg_ws(c))) return s;
    const size_t wb = (size_t)k / 8, row_bytes = (size_t)k * sizeof(uint64_t);
    const uint8_t* src = static_cast<const uint8_t*>(data) + hoff[0] * wb;
    bool d_pinned = false, c_pinned = false;
    int hdev = c->dev;
    classify(data, &hdev, &d_pinned);
    if (!c_dev) classify(counts, &hdev, &c_pinned);
    const bool stage_rows = !c_dev && !c_pinned;
    if ((s = ensure_stage(c))) return s;
    const size_t piece_bytes = kSegChunk < c->stage_bytes - 128 ? kSegChunk : (c->stage_bytes - 128) & ~(size_t)63;

    // units (rows of a unit go back once its last launch is done)
    std::vector<SegUnit> units;
    const size_t chunk_words = piece_bytes / wb;
    for (size_t a0 = 0; a0 < n;) {
        const size_t lo = (hoff[a0] - hoff[0]) * wb;
        if ((hoff[a0 + 1] - hoff[a0]) * wb > piece_bytes) {  // a long array, in pieces
            const size_t hi = (hoff[a0 + 1] - hoff[0]) * wb;
            for (size_t p = lo; p < hi; p += piece_bytes)
                units.push_back({a0, a0 + 1, p, hi - p < piece_bytes ? hi : p + piece_bytes, true, p == lo,
                                 p + piece_bytes >= hi});
            ++a0;
            continue;
        }
        const uint64_t* e = std::upper_bound(hoff + a0 + 1, hoff + n + 1, hoff[a0] + chunk_words);
        size_t a1 = (size_t)(e - hoff) - 1;
        if (a1 <= a0) a1 = a0 + 1;
        units.push_back({a0, a1, lo, (hoff[a1] - hoff[0]) * wb, false, true, true});
        a0 = a1;
    }
    const size_t nu = units.size();

    void *obuf = nullptr, *rbuf = nullptr;
    if (!o_dev && (s = ctx_scratch(c, 1, (n + 1) * sizeof(uint64_t), &obuf))) return s;
    if (!c_dev && (s = ctx_scratch(c, 2, n * row_bytes, &rbuf))) return s;
    if ((s = ensure_seg_pipeline(c, nu + 1, stage_rows ? n * row_bytes : 0))) return s;
    if (!d_pinned && (s = ensure_host_ring(c))) return s;
    const unsigned long long* doff = reinterpret_cast<const unsigned long long*>(o_dev ? offsets : obuf);
    unsigned long long* dout = reinterpret_cast<unsigned long long*>(c_dev ? counts : rbuf);
    uint8_t* rows_dst = stage_rows ? static_cast<uint8_t*>(c->rows_pinned) : reinterpret_cast<uint8_t*>(counts);

    // the copy/d2h streams start after the caller's prior legacy-stream work (through c->stream)
    CU(cudaEventRecord(c->seg_ev[nu], c->stream));
    CU(cudaStreamWaitEvent(c->copy, c->seg_ev[nu], 0));
    CU(cudaStreamWaitEvent(c->d2h, c->seg_ev[nu], 0));
    if (!o_dev)
        CU(cudaMemcpyAsync(obuf, offsets, (n + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice, c->copy));

    size_t drained = 0;  // units whose staged rows are in `counts` (or that have no rows of their own)
    auto drain = [&](bool wait, size_t issued) -> pospop_status {  // units [0, issued) have been enqueued
        for (; drained < issued; ++drained) {
            const SegUnit& u = units[drained];
            if (!u.last_piece) continue;
            cudaEvent_t done = c->seg_ev[drained];
            if (wait) {
                CU(cudaEventSynchronize(done));
            } else {
                const cudaError_t q = cudaEventQuery(done);
                if (q == cudaErrorNotReady) return POSPOP_OK;
                CU(q);
            }
            parallel_copy(reinterpret_cast<uint8_t*>(counts) + u.a0 * row_bytes, rows_dst + u.a0 * row_bytes,
                          (u.a1 - u.a0) * row_bytes);
        }
        return POSPOP_OK;
    };

    size_t piece = 0;  // host-ring slot counter (pageable data)
    for (size_t i = 0; i < nu; ++i) {
        const SegUnit& u = units[i];
        const int slot = (int)(i % kRing);
        const size_t pad = reinterpret_cast<uintptr_t>(src + u.lo) & 31u;
        uint8_t* dst = static_cast<uint8_t*>(c->stage[slot]) + 64 + pad;  // 64 B of slack before the unit
        if (i >= (size_t)kRing) CU(cudaStreamWaitEvent(c->copy, c->ev_done[slot], 0));
        if (d_pinned) {
            CU(cudaMemcpyAsync(dst, src + u.lo, u.hi - u.lo, cudaMemcpyHostToDevice, c->copy));
        } else {
            for (size_t off = u.lo; off < u.hi; off += kHostChunk, ++piece) {
                const size_t m = u.hi - off < kHostChunk ? u.hi - off : kHostChunk;
                const int hs = (int)(piece % kHostRing);
                if (c->host_used[hs]) CU(cudaEventSynchronize(c->ev_h2d[hs]));
                parallel_copy(c->host_ring[hs], src + off, m);
                CU(cudaMemcpyAsync(dst + (off - u.lo), c->host_ring[hs], m, cudaMemcpyHostToDevice, c->copy));
                CU(cudaEventRecord(c->ev_h2d[hs], c->copy));
                c->host_used[hs] = true;
            }
        }
        CU(cudaEventRecord(c->ev_copied[slot], c->copy));
        CU(cudaStreamWaitEvent(c->stream, c->ev_copied[slot], 0));
        LaunchOptions opt;
        if (u.piece) {
            CU(launch_stream(k, dst, (u.hi - u.lo) / wb, dout + u.a0 * k, !u.first_piece, opt, c->ws, c->stream));
        } else {
            // device pointer whose word hoff[a0] is at dst
            const uint8_t* ddata = dst - u.lo - hoff[0] * wb;
            CU(launch_segmented(k, ddata, doff + u.a0, u.a1 - u.a0, dout + u.a0 * k, opt, c->seg_ws, c->stream));
        }
        CU(cudaEventRecord(c->ev_done[slot], c->stream));
        if (!c_dev && u.last_piece) {
            CU(cudaStreamWaitEvent(c->d2h, c->ev_done[slot], 0));
            CU(cudaMemcpyAsync(rows_dst + u.a0 * row_bytes, dout + u.a0 * k, (u.a1 - u.a0) * row_bytes,
                               cudaMemcpyDeviceToHost, c->d2h));
            CU(cudaEventRecord(c->seg_ev[i], c->d2h));
            if (stage_rows && (s = drain(false, i + 1))) return s;
        }
    }
    if (stage_rows && (s = drain(true, nu))) return s;
    // the next call may reuse the staging slots and scratch: c->stream follows the d2h stream
    CU(cudaEventRecord(c->seg_ev[nu], c->d2h));
    CU(cudaStreamWaitEvent(c->stream, c->seg_ev[nu], 0));
    CU(cudaStreamSynchronize(c->stream));
    return POSPOP_OK;
}

// flagstats.cpp:50-63 (bucket_from_counts): positions of the transformed word.
void bucket_from_counts(const uint64_t* c, uint64_t total, pospop_flag_bucket* b) {
    b->total = total;
    b->secondary = c[8];
    b->supplementary = c[11];
    b->n_pair_good = c[1];
    b->n_read1 = c[6];
    b->n_read2 = c[7];
    b->n_sgltn = c[3];
    b->pair_map = c[12];
    b->mapped = total - c[2];
    b->dup = total - c[10];
}

const uint32_t kWidths[] = {64, 256, 512};

bool width_supported(uint32_t w) {
    for (uint32_t x : kWidths)
        if (x == w) return true;
    return false;
}

}  // namespace

extern "C" {

const char* pospop_last_error(void) { return t_err.c_str(); }

int pospop_supported_widths(uint32_t* out, int cap) {
    const int n = (int)(sizeof kWidths / sizeof kWidths[0]);
    for (int i = 0; i < n && i < cap; ++i) out[i] = kWidths[i];
    return n;
}

int pospop_device_available(void) {
    int dev = 0;
    return current_device(&dev) == POSPOP_OK ? 1 : 0;
}

uint64_t pospop_kernel_launches(void) { return kernel_launches(); }

pospop_status pospop_validate(const pospop_config* c) {
    if (!c) return POSPOP_OK;
    if (c->register_width_bits % 16 != 0)
        return fail(POSPOP_EINVAL, "register_width_bits must be a multiple of 16, got %u",
                    c->register_width_bits);
    if (c->flush_threshold_blocks < 1 || c->flush_threshold_blocks > 65535)
        return fail(POSPOP_EINVAL, "flush_threshold_blocks must be in [1, 65535], got %u",
                    c->flush_threshold_blocks);
    if (c->kernel < POSPOP_KERNEL_SCALAR || c->kernel > POSPOP_KERNEL_AUTO)
        return fail(POSPOP_EINVAL, "unknown kernel");
    return POSPOP_OK;
}

pospop_status pospopcnt_u8(const uint8_t* d, size_t n, uint64_t c[8]) { return count_any(8, d, n, 65535, c); }
pospop_status pospopcnt_u16(const uint16_t* d, size_t n, uint64_t c[16]) { return count_any(16, d, n, 65535, c); }
pospop_status pospopcnt_u32(const uint32_t* d, size_t n, uint64_t c[32]) { return count_any(32, d, n, 65535, c); }
pospop_status pospopcnt_u64(const uint64_t* d, size_t n, uint64_t c[64]) { return count_any(64, d, n, 65535, c); }

pospop_status pospopcnt_k(int k, const void* data, size_t len, uint32_t flush, uint64_t* counts) {
    return count_any(k, data, len, flush, counts);
}

// pospop::pospopcnt (pospop.cpp:80-111): validate, resolve Auto, then the
// per-kind width rules (forest 92-93, byteblend byteblend.cpp:60-80, CSA
// csa_portable.cpp:40-46), then count.
pospop_status pospopcnt_u16_config(const uint16_t* data, size_t len, const pospop_config* config,
                                   uint64_t counts[16]) {
    const pospop_config dflt = POSPOP_CONFIG_DEFAULT;
    const pospop_config* c = config ? config : &dflt;
    pospop_status s = pospop_validate(c);
    if (s) return s;
    int kind = c->kernel;
    if (kind == POSPOP_KERNEL_AUTO)
        kind = len < c->auto_threshold_words ? POSPOP_KERNEL_BYTEBLEND : POSPOP_KERNEL_CSA16;
    const uint32_t w = c->register_width_bits;
    switch (kind) {
        case POSPOP_KERNEL_SCALAR:
            break;
        case POSPOP_KERNEL_FOREST:
            if (w > 64) return fail(POSPOP_EUNAVAILABLE, "kernel unavailable: forest supports 64-bit registers only");
            break;
        case POSPOP_KERNEL_BYTEBLEND:
            if (c->kernel != POSPOP_KERNEL_AUTO && w != 0 && w != 64 && w != 256)
                return fail(POSPOP_EUNAVAILABLE,
                            "kernel unavailable: byteblend supports 64- or 256-bit registers, got %u", w);
            break;
        default:  // CSA kinds
            if (w != 0 && !width_supported(w))
                return fail(POSPOP_EUNAVAILABLE, "kernel unavailable: no CSA backend for %u-bit registers", w);
            break;
    }
    return count_any(16, data, len, c->flush_threshold_blocks, counts);
}

pospop_status pospopcnt_u16_c32(const uint16_t* data, uint32_t len, uint32_t counters[16]) {
    if (!counters) return fail(POSPOP_EINVAL, "counters must not be NULL");
    uint64_t c[16];
    const pospop_status s = count_any(16, data, len, 65535, c);
    if (s) return s;
    for (int p = 0; p < 16; ++p) counters[p] += (uint32_t)c[p];
    return POSPOP_OK;
}

pospop_status segmented_on_ctx(Ctx* c, int k, const void* data, bool d_dev, const uint64_t* offsets, bool o_dev,
                               size_t n, uint64_t* counts, bool c_dev);

pospop_status pospopcnt_segmented(int k, const void* data, const uint64_t* offsets, size_t n,
                                  uint64_t* counts) {
    if (!valid_k(k)) return fail(POSPOP_EINVAL, "k must be 8, 16, 32 or 64, got %d", k);
    if (n == 0) return POSPOP_OK;
    if (!offsets || !counts) return fail(POSPOP_EINVAL, "offsets/counts must not be NULL");
    const size_t wb = (size_t)k / 8;
    if ((uintptr_t)data % wb) return fail(POSPOP_EINVAL, "data is not aligned to the %d-bit word size", k);
    int dev = 0;
    pospop_status s = current_device(&dev);
    if (s) return s;
    int ddev = dev, odev = dev, cdev = dev;
    const bool d_dev = data && classify(data, &ddev) == Where::Device;
    const bool o_dev = classify(offsets, &odev) == Where::Device;
    const bool c_dev = classify(counts, &cdev) == Where::Device;
    if (d_dev) dev = ddev;
    DeviceGuard g(dev);
    CtxScope scope;
    Ctx* c = nullptr;
    if ((s = scope.get(dev, &c))) return s;
    return segmented_on_ctx(c, k, data, d_dev, offsets, o_dev, n, counts, c_dev);
}

// The segmented call on context c's device (current): data in device memory
// on that device (d_dev) or host memory; offsets / counts in device memory
// (o_dev / c_dev) or host memory.
pospop_status segmented_on_ctx(Ctx* c, int k, const void* data, bool d_dev, const uint64_t* offsets, bool o_dev,
                               size_t n, uint64_t* counts, bool c_dev) {
    pospop_status s;
    const size_t wb = (size_t)k / 8;
    const int dev = c->dev;
    // Host offsets are needed on the host for validation and sizing anyway.
    std::vector<uint64_t> h_off;
    const uint64_t* hoff = offsets;
    if (o_dev) {
        h_off.resize(n + 1);
        CU(cudaMemcpy(h_off.data(), offsets, (n + 1) * sizeof(uint64_t), cudaMemcpyDeviceToHost));
        hoff = h_off.data();
    }
    for (size_t a = 0; a < n; ++a)
        if (hoff[a + 1] < hoff[a]) return fail(POSPOP_EINVAL, "offsets must be non-decreasing (array %zu)", a);
    if (!data && hoff[n] != hoff[0]) return fail(POSPOP_EINVAL, "data is NULL but arrays are non-empty");

    if (!d_dev && (hoff[n] - hoff[0]) * wb > kSegPipeMin)
        return segmented_host_pipeline(c, k, data, offsets, o_dev, hoff, n, counts, c_dev);

    const void* ddata = data;
    if (!d_dev && hoff[n] > hoff[0]) {  // stage the referenced range [offsets[0], offsets[n]) words
        bool pinned = false;
        int hdev = dev;
        classify(data, &hdev, &pinned);
        const size_t lo = hoff[0] * wb, bytes = (hoff[n] - hoff[0]) * wb;
        // keep the start's alignment within 32 bytes so vector loads see the same offsets
        const size_t pad = reinterpret_cast<uintptr_t>(static_cast<const uint8_t*>(data) + lo) & 31u;
        void* buf = nullptr;
        if ((s = ctx_scratch(c, 0, bytes + pad + 64, &buf))) return s;  // +64: whole last vector
        if ((s = h2d_on_stream(c, static_cast<uint8_t*>(buf) + pad, static_cast<const uint8_t*>(data) + lo, bytes,
                               pinned)))
            return s;
        // device pointer whose word offsets[0] is at buf + pad
        ddata = static_cast<const uint8_t*>(buf) + pad - lo;
    }
    const unsigned long long* doff = reinterpret_cast<const unsigned long long*>(offsets);
    if (!o_dev) {
        void* buf = nullptr;
        if ((s = ctx_scratch(c, 1, (n + 1) * sizeof(uint64_t), &buf))) return s;
        CU(cudaMemcpyAsync(buf, offsets, (n + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice, c->stream));
        doff = static_cast<const unsigned long long*>(buf);
    }
    unsigned long long* dout = reinterpret_cast<unsigned long long*>(counts);
    if (!c_dev) {
        void* buf = nullptr;
        if ((s = ctx_scratch(c, 2, n * (size_t)k * sizeof(uint64_t), &buf))) return s;
        dout = static_cast<unsigned long long*>(buf);
    }
    LaunchOptions opt;
    if ((s = ensure_seg_ws(c))) return s;
    CU(launch_segmented(k, ddata ? ddata : (const void*)doff, doff, n, dout, opt, c->seg_ws, c->stream));
    if (!c_dev)
        CU(cudaMemcpyAsync(counts, dout, n * (size_t)k * sizeof(uint64_t), cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    return POSPOP_OK;
}

pospop_status pospopcnt_u8_segmented(const uint8_t* data, const uint64_t* offsets, size_t n, uint64_t* counts) {
    return pospopcnt_segmented(8, data, offsets, n, counts);
}
pospop_status pospopcnt_u16_segmented(const uint16_t* data, const uint64_t* offsets, size_t n, uint64_t* counts) {
    return pospopcnt_segmented(16, data, offsets, n, counts);
}
pospop_status pospopcnt_u32_segmented(const uint32_t* data, const uint64_t* offsets, size_t n, uint64_t* counts) {
    return pospopcnt_segmented(32, data, offsets, n, counts);
}
pospop_status pospopcnt_u64_segmented(const uint64_t* data, const uint64_t* offsets, size_t n, uint64_t* counts) {
    return pospopcnt_segmented(64, data, offsets, n, counts);
}

pospop_status pospopcnt_segmented_split(int k, const void* data, const uint64_t* offsets, size_t n,
                                        const int* devices, int n_devices, uint64_t* counts) {
    if (!valid_k(k)) return fail(POSPOP_EINVAL, "k must be 8, 16, 32 or 64, got %d", k);
    if (n_devices < 1 || !devices) return fail(POSPOP_EINVAL, "need >= 1 device");
    if (n == 0) return POSPOP_OK;
    if (!offsets || !counts) return fail(POSPOP_EINVAL, "offsets/counts must not be NULL");
    const size_t wb = (size_t)k / 8;
    if ((uintptr_t)data % wb) return fail(POSPOP_EINVAL, "data is not aligned to the %d-bit word size", k);
    int dev0 = 0;
    pospop_status s = current_device(&dev0);
    if (s) return s;
    int n_dev = 0;
    CU(cudaGetDeviceCount(&n_dev));
    for (int i = 0; i < n_devices; ++i) {
        if (devices[i] < 0 || devices[i] >= n_dev)
            return fail(POSPOP_EINVAL, "no device %d (%d visible)", devices[i], n_dev);
        if ((s = check_device(devices[i]))) return s;
    }
    int ddev = dev0, odev = dev0, cdev = dev0;
    const bool d_dev = data && classify(data, &ddev) == Where::Device;
    const bool o_dev = classify(offsets, &odev) == Where::Device;
    const bool c_dev = classify(counts, &cdev) == Where::Device;
    if (d_dev || o_dev || c_dev) {  // device-resident operands: one device holds them all
        const int home = d_dev ? ddev : o_dev ? odev : cdev;
        for (int i = 0; i < n_devices; ++i)
            if (devices[i] != home)
                return fail(POSPOP_EINVAL, "device-resident operands live on device %d; listed device %d", home,
                            devices[i]);
        return pospopcnt_segmented(k, data, offsets, n, counts);
    }
    for (size_t a = 0; a < n; ++a)
        if (offsets[a + 1] < offsets[a]) return fail(POSPOP_EINVAL, "offsets must be non-decreasing (array %zu)", a);
    // Contiguous groups of arrays with about equal bytes (each at least one
    // array when there are enough), one per listed device.
    std::vector<size_t> cut((size_t)n_devices + 1, n);
    cut[0] = 0;
    const uint64_t w0 = offsets[0], wn = offsets[n];
    for (int i = 1; i < n_devices; ++i) {
        const uint64_t target = w0 + (wn - w0) * (uint64_t)i / (uint64_t)n_devices;
        size_t a = (size_t)(std::lower_bound(offsets, offsets + n + 1, target) - offsets);
        a = std::max(a, cut[(size_t)i - 1]);
        cut[(size_t)i] = std::min(a, n);
    }
    std::vector<pospop_status> st((size_t)n_devices, POSPOP_OK);
    std::vector<std::string> err((size_t)n_devices);
    std::vector<std::thread> workers;
    for (int i = 0; i < n_devices; ++i) {
        const size_t a0 = cut[(size_t)i], a1 = cut[(size_t)i + 1];
        if (a1 <= a0) continue;
        auto work = [&, i, a0, a1](bool own_thread) {
            const int d = devices[i];
            pospop_status ws = cuda_set_device(d);
            if (!ws) {
                if (own_thread) bind_to_device_cpus(d);
                CtxScope wscope;
                Ctx* c = nullptr;
                if (!(ws = wscope.get(d, &c, false)))
                    ws = segmented_on_ctx(c, k, data, false, offsets + a0, false, a1 - a0, counts + a0 * (size_t)k,
                                          false);
            }
            st[(size_t)i] = ws;
            if (ws) err[(size_t)i] = t_err;
        };
        try {
            workers.emplace_back(work, true);
        } catch (const std::exception&) {
            work(false);
            cudaSetDevice(dev0);
        }
    }
    for (auto& t : workers) t.join();
    for (int i = 0; i < n_devices; ++i)
        if (st[(size_t)i]) return fail(st[(size_t)i], "device group %d: %s", i, err[(size_t)i].c_str());
    return POSPOP_OK;
}

pospop_status pospop_flagstats(const uint16_t* flags, size_t len, pospop_flag_summary* out, uint64_t* bad_offset,
                               uint16_t* bad_word) {
    if (!out) return fail(POSPOP_EINVAL, "out must not be NULL");
    if (!flags && len) return fail(POSPOP_EINVAL, "flags is NULL but len is %zu", len);
    if ((uintptr_t)flags % 2) return fail(POSPOP_EINVAL, "flags is not 2-byte aligned");
    int dev = 0;
    pospop_status s = current_device(&dev);
    if (s) return s;
    std::memset(out, 0, sizeof *out);
    if (len == 0) return POSPOP_OK;
    bool pinned = false;
    const Where where = classify(flags, &dev, &pinned);
    DeviceGuard g(dev);
    CtxScope scope;
    Ctx* c = nullptr;
    if ((s = scope.get(dev, &c))) return s;
    LaunchOptions opt;
    const void* mapped = nullptr;  // small host input read in place (zero-copy), as in count_on_ctx
    if (where == Where::Host && len * 2 <= (pinned ? kZeroCopyBytes : kBounceBytes)) {
        const void* src = flags;
        if (!pinned) {
            if (!c->bounce) CU(cudaMallocHost(&c->bounce, kBounceBytes));
            std::memcpy(c->bounce, flags, len * 2);
            src = c->bounce;
        }
        int hd = dev;
        classify(src, &hd, nullptr, &mapped);
    }
    if (where == Where::Device || mapped) {
        CU(launch_flagstats(mapped ? static_cast<const uint16_t*>(mapped) : flags, len, c->m_out_dev, false, opt,
                            c->ws, c->stream));
    } else if (!pinned) {  // pageable: parallel copies into the pinned host ring
        const uint8_t* src = reinterpret_cast<const uint8_t*>(flags);
        s = host_ring_pipeline(
            c, len * 2, 2,
            [&](uint8_t* dst, size_t off, size_t n) {
                parallel_copy(dst, src + off, n);
                return POSPOP_OK;
            },
            [&](const void* d, size_t off, size_t n, size_t i) -> pospop_status {
                LaunchOptions o = opt;
                o.word_base = off / 2;
                CU(launch_flagstats(static_cast<const uint16_t*>(d), n / 2, c->m_out_dev, i > 0, o, c->ws,
                                    c->stream));
                return POSPOP_OK;
            });
        if (s) return s;
    } else {
        if ((s = ensure_stage(c))) return s;
        const size_t chunk_words = c->stage_bytes / 2;
        size_t i = 0;
        for (size_t off = 0; off < len; off += chunk_words, ++i) {
            const size_t n = len - off < chunk_words ? len - off : chunk_words;
            const int slot = (int)(i % kRing);
            if (i >= (size_t)kRing) CU(cudaStreamWaitEvent(c->copy, c->ev_done[slot], 0));
            CU(cudaMemcpyAsync(c->stage[slot], flags + off, n * 2, cudaMemcpyHostToDevice, c->copy));
            CU(cudaEventRecord(c->ev_copied[slot], c->copy));
            CU(cudaStreamWaitEvent(c->stream, c->ev_copied[slot], 0));
            opt.word_base = off;
            CU(launch_flagstats(static_cast<const uint16_t*>(c->stage[slot]), n, c->m_out_dev, i > 0, opt,
                                c->ws, c->stream));
            CU(cudaEventRecord(c->ev_done[slot], c->stream));
        }
    }
    CU(cudaStreamSynchronize(c->stream));  // the last CTA wrote c->m_out (mapped)
    if (c->m_out[32]) {
        const uint64_t idx = ~c->m_out[32];
        uint16_t word = 0;
        if (where == Where::Device)
            CU(cudaMemcpy(&word, flags + idx, 2, cudaMemcpyDeviceToHost));
        else
            word = flags[idx];
        if (bad_offset) *bad_offset = idx;
        if (bad_word) *bad_word = word;
        return fail(POSPOP_EFLAG, "invalid FLAG word 0x%x at offset %llu (bits 12-15 must be clear)", word,
                    (unsigned long long)idx);
    }
    // Kernel output: [0,16) counts over all reads, [16,32) over QC-fail reads;
    // QC-pass = all - fail (flagstats.cpp:137-143 counts the two streams).
    const uint64_t* ac = reinterpret_cast<const uint64_t*>(c->m_out);
    const uint64_t* fc = ac + 16;
    uint64_t pc[16];
    for (int p = 0; p < 16; ++p) pc[p] = ac[p] - fc[p];
    const uint64_t fail_total = fc[9];
    bucket_from_counts(fc, fail_total, &out->fail);
    bucket_from_counts(pc, len - fail_total, &out->pass);
    return POSPOP_OK;
}

// ---------------------------------------------------------------------------
// File / pipe ingestion (reference read_word_stream +
// decode_words, proj/tools/pospopcnt.cpp:52-75).
// ---------------------------------------------------------------------------
namespace {

// Fills buf with up to `want` bytes from fd at `offset` (regular file:
// parallel pread stripes) or sequentially (pipe).  Returns bytes read, or -1.
ssize_t fill_buffer(int fd, bool seekable, uint8_t* buf, size_t want, uint64_t offset) {
    if (!seekable) {
        size_t got = 0;
        while (got < want) {
            const ssize_t r = ::read(fd, buf + got, want - got);
            if (r < 0) {
                if (errno == EINTR) continue;
                return -1;
            }
            if (r == 0) break;
            got += (size_t)r;
        }
        return (ssize_t)got;
    }
    // Regular file: parallel pread of 1 MiB pieces on the host pool.
    constexpr size_t kPiece = 1 << 20;
    const int tasks = (int)((want + kPiece - 1) / kPiece);
    std::vector<ssize_t> got((size_t)tasks, 0);
    HostPool::get().run(tasks, [&](int t) {
        const size_t lo = (size_t)t * kPiece;
        const size_t hi = lo + kPiece < want ? lo + kPiece : want;
        size_t done = 0;
        while (lo + done < hi) {
            const ssize_t r = ::pread(fd, buf + lo + done, hi - lo - done, (off_t)(offset + lo + done));
            if (r < 0) {
                if (errno == EINTR) continue;
                got[(size_t)t] = -1;
                return;
            }
            if (r == 0) break;
            done += (size_t)r;
        }
        got[(size_t)t] = (ssize_t)done;
    });
    size_t total = 0;
    for (int t = 0; t < tasks; ++t) {
        if (got[(size_t)t] < 0) return -1;
        total += (size_t)got[(size_t)t];
        if ((size_t)got[(size_t)t] < (t + 1 == tasks ? want - (size_t)t * kPiece : kPiece)) break;  // EOF in piece t
    }
    return (ssize_t)total;
}

}  // namespace

pospop_status pospopcnt_fd(int fd, int k, uint64_t* counts, uint64_t* n_words) {
    if (!valid_k(k)) return fail(POSPOP_EINVAL, "k must be 8, 16, 32 or 64, got %d", k);
    if (!counts) return fail(POSPOP_EINVAL, "counts must not be NULL");
    if (fd < 0) return fail(POSPOP_EINVAL, "bad file descriptor %d", fd);
    int dev = 0;
    pospop_status s = current_device(&dev);
    if (s) return s;
    CtxScope scope;
    Ctx* c = nullptr;
    if ((s = scope.get(dev, &c))) return s;
    if ((s = ensure_stage(c))) return s;
    struct stat st;
    const bool seekable = fstat(fd, &st) == 0 && S_ISREG(st.st_mode);
    const size_t wb = (size_t)k / 8;
    if ((s = ensure_host_ring(c))) return s;
    const size_t chunk = kHostChunk < c->stage_bytes ? kHostChunk : c->stage_bytes;  // a multiple of 8
    uint64_t total = 0;
    LaunchOptions opt;
    for (size_t i = 0;; ++i) {
        const int hs = (int)(i % kHostRing), slot = (int)(i % kRing);
        if (c->host_used[hs]) CU(cudaEventSynchronize(c->ev_h2d[hs]));  // the H2D that last read it is done
        uint8_t* buf = c->host_ring[hs];
        const ssize_t got = fill_buffer(fd, seekable, buf, chunk, total);
        if (got < 0) return fail(POSPOP_EINVAL, "read failed: %s", std::strerror(errno));
        if (got == 0) break;
        total += (uint64_t)got;
        if ((size_t)got % wb != 0) {
            // only the final chunk may be short; a ragged word means a bad length
            uint8_t probe;
            const ssize_t more = seekable ? ::pread(fd, &probe, 1, (off_t)total) : ::read(fd, &probe, 1);
            return fail(POSPOP_EINVAL, "input: %s byte length (%llu%s bytes); expected raw little-endian %d-bit words",
                        wb == 2 ? "odd" : "ragged", (unsigned long long)total, more > 0 ? "+" : "", k);
        }
        if (i >= (size_t)kRing) CU(cudaStreamWaitEvent(c->copy, c->ev_done[slot], 0));
        CU(cudaMemcpyAsync(c->stage[slot], buf, (size_t)got, cudaMemcpyHostToDevice, c->copy));
        CU(cudaEventRecord(c->ev_h2d[hs], c->copy));
        c->host_used[hs] = true;
        CU(cudaEventRecord(c->ev_copied[slot], c->copy));
        CU(cudaStreamWaitEvent(c->stream, c->ev_copied[slot], 0));
        CU(launch_stream(k, c->stage[slot], (size_t)got / wb, c->d_out, i > 0, opt, c->ws, c->stream));
        CU(cudaEventRecord(c->ev_done[slot], c->stream));
        if ((size_t)got < chunk) break;
    }
    if (total == 0) {
        for (int p = 0; p < k; ++p) counts[p] = 0;
    } else {
        CU(cudaMemcpyAsync(c->h_out, c->d_out, (size_t)k * sizeof(uint64_t), cudaMemcpyDeviceToHost, c->stream));
        CU(cudaStreamSynchronize(c->stream));
        for (int p = 0; p < k; ++p) counts[p] = c->h_out[p];
    }
    if (n_words) *n_words = total / wb;
    return POSPOP_OK;
}

pospop_status pospopcnt_file(const char* path, int k, uint64_t* counts, uint64_t* n_words) {
    if (!path) return fail(POSPOP_EINVAL, "path must not be NULL");
    const bool is_stdin = path[0] == '-' && path[1] == 0;
    const int fd = is_stdin ? 0 : ::open(path, O_RDONLY);
    if (fd < 0) return fail(POSPOP_EINVAL, "cannot open input file: %s", path);
    const pospop_status s = pospopcnt_fd(fd, k, counts, n_words);
    if (!is_stdin) ::close(fd);
    return s;
}

pospop_status pospopcnt_sharded(int k, const void* const* shards, const size_t* lens, const int* devices,
                                int n_shards, uint64_t* counts) {
    if (!valid_k(k)) return fail(POSPOP_EINVAL, "k must be 8, 16, 32 or 64, got %d", k);
    if (n_shards < 0 || (n_shards > 0 && (!shards || !lens || !devices)) || !counts)
        return fail(POSPOP_EINVAL, "invalid shard description");
    int dev0 = 0;
    pospop_status s = current_device(&dev0);
    if (s) return s;
    int n_dev = 0;
    CU(cudaGetDeviceCount(&n_dev));
    const size_t wb = (size_t)k / 8;
    std::vector<char> on_device((size_t)n_shards, 0), pinned((size_t)n_shards, 0);
    std::set<int> device_set;  // devices of the device-resident shards
    for (int i = 0; i < n_shards; ++i) {  // validate everything before launching anything
        if (devices[i] < 0 || devices[i] >= n_dev)
            return fail(POSPOP_EINVAL, "shard %d: no device %d (%d visible)", i, devices[i], n_dev);
        if (!shards[i] && lens[i]) return fail(POSPOP_EINVAL, "shard %d is NULL with len %zu", i, lens[i]);
        if ((uintptr_t)shards[i] % wb) return fail(POSPOP_EINVAL, "shard %d is misaligned", i);
        if ((s = check_device(devices[i]))) return s;
        if (!lens[i]) continue;
        int pd = devices[i];
        bool pin = false;
        if (classify(shards[i], &pd, &pin) == Where::Device) {
            if (pd != devices[i]) return fail(POSPOP_EINVAL, "shard %d lives on device %d, not %d", i, pd, devices[i]);
            on_device[(size_t)i] = 1;
            device_set.insert(devices[i]);
        }
        pinned[(size_t)i] = pin;
    }
    // Device shards: one context per device, acquired in ascending device
    // order.  Launch every shard before any synchronisation (launch skew,
    // SURVEY 8e).  Shard i is the j-th device shard of its device: it uses
    // that context's slot j (own stream and workspace, so shards on one device
    // may overlap), and its kernel writes the k counts straight into the
    // slot's mapped buffer.
    CtxScope scope;
    std::map<int, Ctx*> ctx;
    for (int d : device_set) {
        DeviceGuard g(d);
        if ((s = scope.get(d, &ctx[d]))) return s;
    }
    std::vector<Ctx::ShardSlot*> used((size_t)n_shards, nullptr);
    std::map<int, size_t> per_dev;
    LaunchOptions opt;
    for (int i = 0; i < n_shards; ++i) {
        if (!on_device[(size_t)i]) continue;
        const int d = devices[i];
        DeviceGuard g(d);
        Ctx* c = ctx[d];
        const size_t j = per_dev[d]++;
        if (c->shard_slots.size() <= j) {
            c->shard_slots.emplace_back();
            Ctx::ShardSlot& slot = c->shard_slots.back();
            CU(cudaStreamCreateWithFlags(&slot.stream, cudaStreamDefault));
            if ((s = alloc_workspace(&slot.ws))) return s;
            CU(cudaHostAlloc(&slot.m_out, 64 * sizeof(unsigned long long), cudaHostAllocMapped));
            CU(cudaHostGetDevicePointer(reinterpret_cast<void**>(&slot.m_out_dev), slot.m_out, 0));
        }
        Ctx::ShardSlot* slot = &c->shard_slots[j];
        used[(size_t)i] = slot;
        CU(launch_stream(k, shards[i], lens[i], slot->m_out_dev, false, opt, slot->ws, slot->stream));
    }
    // Host shards: one worker thread each, running on the CPUs local to its
    // device, streams its range through its own context's staging ring over
    // that device's host link -- N devices' links in parallel.
    std::vector<std::vector<uint64_t>> host_out;
    std::vector<pospop_status> host_st;
    std::vector<std::string> host_err;
    std::vector<std::thread> workers;
    host_out.resize((size_t)n_shards);
    host_st.assign((size_t)n_shards, POSPOP_OK);
    host_err.resize((size_t)n_shards);
    for (int i = 0; i < n_shards; ++i) {
        if (on_device[(size_t)i] || !lens[i]) continue;
        host_out[(size_t)i].assign((size_t)k, 0);
        auto work = [&, i](bool own_thread) {
            const int d = devices[i];
            pospop_status ws = cuda_set_device(d);
            if (!ws) {
                if (own_thread) bind_to_device_cpus(d);
                CtxScope wscope;
                Ctx* c = nullptr;
                if (!(ws = wscope.get(d, &c, false)))
                    ws = count_on_ctx(c, k, shards[i], lens[i], false, pinned[(size_t)i] != 0, 65535,
                                      host_out[(size_t)i].data());
            }
            host_st[(size_t)i] = ws;
            if (ws) host_err[(size_t)i] = t_err;
        };
        try {
            workers.emplace_back(work, true);
        } catch (const std::exception&) {  // no thread available: count this shard on the calling thread
            work(false);
            cudaSetDevice(dev0);
        }
    }
    for (auto& t : workers) t.join();
    for (int p = 0; p < k; ++p) counts[p] = 0;
    pospop_status first = POSPOP_OK;
    int first_i = -1;
    for (int i = 0; i < n_shards; ++i) {  // merge_counts over shards
        if (on_device[(size_t)i]) {
            DeviceGuard g(devices[i]);
            CU(cudaStreamSynchronize(used[(size_t)i]->stream));
            for (int p = 0; p < k; ++p) counts[p] += used[(size_t)i]->m_out[p];
        } else if (lens[i]) {
            if (host_st[(size_t)i] && !first) {
                first = host_st[(size_t)i];
                first_i = i;
            }
            for (int p = 0; p < k; ++p) counts[p] += host_out[(size_t)i][(size_t)p];
        }
    }
    if (first) return fail(first, "shard %d: %s", first_i, host_err[(size_t)first_i].c_str());
    return POSPOP_OK;
}

pospop_status pospopcnt_split(int k, const void* data, size_t len, const int* devices, int n_devices,
                              uint64_t* counts) {
    if (!valid_k(k)) return fail(POSPOP_EINVAL, "k must be 8, 16, 32 or 64, got %d", k);
    if (n_devices < 1 || !devices || !counts) return fail(POSPOP_EINVAL, "need >= 1 device and a counts array");
    if (!data && len) return fail(POSPOP_EINVAL, "data is NULL but len is %zu", len);
    const size_t wb = (size_t)k / 8;
    std::vector<const void*> ptrs((size_t)n_devices);
    std::vector<size_t> lens((size_t)n_devices);
    for (int i = 0; i < n_devices; ++i) {  // contiguous word ranges, sizes differing by at most one word
        const size_t lo = len / n_devices * i + ((size_t)i < len % n_devices ? i : len % n_devices);
        const size_t n = len / n_devices + ((size_t)i < len % n_devices ? 1 : 0);
        ptrs[(size_t)i] = static_cast<const uint8_t*>(data) + lo * wb;
        lens[(size_t)i] = n;
    }
    return pospopcnt_sharded(k, ptrs.data(), lens.data(), devices, n_devices, counts);
}

pospop_status pospop_release_resources(void) {
    std::vector<std::pair<int, Ctx*>> dead;
    {
        CtxPool& pool = CtxPool::get();
        std::lock_guard<std::mutex> lk(pool.mu);
        for (auto& kv : pool.idle) {
            for (Ctx* c : kv.second) dead.emplace_back(kv.first, c);
            pool.live[kv.first] -= (int)kv.second.size();
            kv.second.clear();
        }
    }
    for (auto& dc : dead) {
        DeviceGuard g(dc.first);
        destroy_ctx(dc.second);
    }
    std::lock_guard<std::mutex> lock(g_ws_mu);
    std::set<int> synced;
    for (auto& kv : g_ws) {
        const int dev = kv.first.first;
        DeviceGuard g(dev);
        if (synced.insert(dev).second) cudaDeviceSynchronize();
        free_workspace(&kv.second.ws);
        free_workspace(&kv.second.seg_ws);
    }
    g_ws.clear();
    cudaGetLastError();
    return POSPOP_OK;
}

pospop_status pospop_release_stream(void* stream) {
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    std::lock_guard<std::mutex> lock(g_ws_mu);
    for (auto it = g_ws.begin(); it != g_ws.end();) {
        if (it->first.second != st) {
            ++it;
            continue;
        }
        DeviceGuard g(it->first.first);
        CU(cudaStreamSynchronize(st));
        free_workspace(&it->second.ws);
        free_workspace(&it->second.seg_ws);
        it = g_ws.erase(it);
    }
    return POSPOP_OK;
}

pospop_status pospop_resource_stats(int device, int* contexts, int* idle_contexts, int* stream_workspaces) {
    {
        CtxPool& pool = CtxPool::get();
        std::lock_guard<std::mutex> lk(pool.mu);
        if (contexts) *contexts = pool.live.count(device) ? pool.live[device] : 0;
        if (idle_contexts) *idle_contexts = pool.idle.count(device) ? (int)pool.idle[device].size() : 0;
    }
    std::lock_guard<std::mutex> lock(g_ws_mu);
    int n = 0;
    for (auto& kv : g_ws) n += kv.first.first == device;
    if (stream_workspaces) *stream_workspaces = n;
    return POSPOP_OK;
}

pospop_status pospopcnt_u16_sharded(const uint16_t* const* shards, const size_t* lens, const int* devices,
                                    int n_devices, uint64_t counts[16]) {
    return pospopcnt_sharded(16, reinterpret_cast<const void* const*>(shards), lens, devices, n_devices, counts);
}

pospop_status pospopcnt_u16_async(const uint16_t* d_data, size_t len, uint64_t* d_counts, void* stream) {
    return pospopcnt_async(16, d_data, len, d_counts, 0, 65535, 0, 0, stream);
}

pospop_status pospopcnt_async(int k, const void* d_data, size_t len, uint64_t* d_counts, int accumulate,
                              uint32_t flush, int grid, int block, void* stream) {
    if (!valid_k(k)) return fail(POSPOP_EINVAL, "k must be 8, 16, 32 or 64, got %d", k);
    if (flush < 1 || flush > 65535)
        return fail(POSPOP_EINVAL, "flush_threshold_blocks must be in [1, 65535], got %u", flush);
    if (!d_counts || (!d_data && len)) return fail(POSPOP_EINVAL, "NULL pointer");
    if ((uintptr_t)d_data % ((size_t)k / 8)) return fail(POSPOP_EINVAL, "data is misaligned");
    if (block < 0 || block % 32 || block > 256) return fail(POSPOP_EINVAL, "block must be a multiple of 32 in [32, 256]");
    if (grid < 0) return fail(POSPOP_EINVAL, "grid must be >= 0");
    int dev = 0;
    pospop_status s = current_device(&dev);
    if (s) return s;
    // The stream is used verbatim: NULL is the legacy default stream.
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    StreamWorkspace ws;
    LaunchOptions opt;
    if ((s = stream_workspace(dev, st, &ws, d_data, len * ((size_t)k / 8), d_counts, (size_t)k * 8, &opt.no_pdl)))
        return s;
    opt.flush_threshold = flush;
    opt.grid = grid;
    opt.block = block;
    CU(launch_stream(k, len ? d_data : (const void*)d_counts, len,
                     reinterpret_cast<unsigned long long*>(d_counts), accumulate != 0, opt, ws, st));
    return POSPOP_OK;
}

pospop_status pospop_ipc_alloc(size_t bytes, void** d_ptr, unsigned char handle[64]) {
    if (!d_ptr || !handle || !bytes) return fail(POSPOP_EINVAL, "NULL pointer or zero size");
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
    int dev = 0;
    pospop_status s = current_device(&dev);
    if (s) return s;
    CU(cudaMalloc(d_ptr, bytes));
    CU(cudaMemset(*d_ptr, 0, bytes));
    cudaIpcMemHandle_t h;
    CU(cudaIpcGetMemHandle(&h, *d_ptr));
    std::memcpy(handle, &h, 64);
    return POSPOP_OK;
}

pospop_status pospop_ipc_open(const unsigned char handle[64], void** d_ptr) {
    if (!d_ptr || !handle) return fail(POSPOP_EINVAL, "NULL pointer");
    int dev = 0;
    pospop_status s = current_device(&dev);
    if (s) return s;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, 64);
    CU(cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess));
    return POSPOP_OK;
}

pospop_status pospop_ipc_close(void* d_ptr) {
    CU(cudaIpcCloseMemHandle(d_ptr));
    return POSPOP_OK;
}

pospop_status pospop_ipc_free(void* d_ptr) {
    CU(cudaFree(d_ptr));
    return POSPOP_OK;
}

size_t pospop_exchange_bytes(int k, int n_ranks, int slots) {
    if (!valid_k(k) || n_ranks < 1 || n_ranks > kXMaxRanks || slots < 1) return 0;
    return xbuffer_words(n_ranks, k, slots) * sizeof(uint64_t);
}

pospop_status pospopcnt_allgather_async(int k, const void* d_data, size_t len, uint64_t* d_counts,
                                        uint64_t* const* d_peers, int n_ranks, int rank, uint64_t step, int slots,
                                        void* stream) {
    if (!valid_k(k)) return fail(POSPOP_EINVAL, "k must be 8, 16, 32 or 64, got %d", k);
    if (!d_counts || !d_peers || (!d_data && len)) return fail(POSPOP_EINVAL, "NULL pointer");
    if (n_ranks < 1 || n_ranks > kXMaxRanks || rank < 0 || rank >= n_ranks)
        return fail(POSPOP_EINVAL, "rank %d of %d (at most %d ranks)", rank, n_ranks, kXMaxRanks);
    if (slots < 1) return fail(POSPOP_EINVAL, "slots must be >= 1, got %d", slots);
    if ((uintptr_t)d_data % ((size_t)k / 8)) return fail(POSPOP_EINVAL, "data is misaligned");
    int dev = 0;
    pospop_status s = current_device(&dev);
    if (s) return s;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    StreamWorkspace ws;
    LaunchOptions opt;
    if ((s = stream_workspace(dev, st, &ws, d_data, len * ((size_t)k / 8), d_counts, (size_t)k * 8, &opt.no_pdl)))
        return s;
    opt.peers = reinterpret_cast<unsigned long long* const*>(d_peers);
    opt.n_peers = n_ranks;
    opt.rank = rank;
    opt.xstep = step;
    opt.xslots = slots;
    CU(launch_stream(k, len ? d_data : (const void*)d_counts, len, reinterpret_cast<unsigned long long*>(d_counts),
                     false, opt, ws, st));
    return POSPOP_OK;
}

pospop_status pospop_exchange_reduce_async(int k, uint64_t* d_own, int n_ranks, uint64_t step, int slots,
                                           uint64_t* d_total, void* stream) {
    if (!valid_k(k)) return fail(POSPOP_EINVAL, "k must be 8, 16, 32 or 64, got %d", k);
    if (!d_own || !d_total) return fail(POSPOP_EINVAL, "NULL pointer");
    if (n_ranks < 1 || n_ranks > kXMaxRanks) return fail(POSPOP_EINVAL, "n_ranks %d (at most %d)", n_ranks, kXMaxRanks);
    if (slots < 1) return fail(POSPOP_EINVAL, "slots must be >= 1, got %d", slots);
    int dev = 0;
    pospop_status s = current_device(&dev);
    if (s) return s;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    StreamWorkspace ws;
    bool no_pdl = false;  // records d_total as a recent output of this stream (PDL hazard tracking)
    if ((s = stream_workspace(dev, st, &ws, nullptr, 0, d_total, (size_t)k * 8, &no_pdl))) return s;
    CU(launch_exchange_reduce(k, reinterpret_cast<unsigned long long*>(d_own), n_ranks, step, slots,
                              reinterpret_cast<unsigned long long*>(d_total), st));
    return POSPOP_OK;
}

pospop_status pospop_exchange_status(const uint64_t* d_own, uint64_t* consumed, uint64_t* error) {
    if (!d_own) return fail(POSPOP_EINVAL, "NULL pointer");
    uint64_t h[2] = {0, 0};
    CU(cudaMemcpy(h, d_own, sizeof h, cudaMemcpyDeviceToHost));
    if (consumed) *consumed = h[0];
    if (error) *error = h[1];
    if (h[1]) return fail(POSPOP_ECUDA, "exchange: %s timed out (error %llu)",
                          h[1] == 1 ? "a producer's credit wait" : "the reducer's row wait", (unsigned long long)h[1]);
    return POSPOP_OK;
}

pospop_status pospop_exchange_selftest(int k, int n_ranks, int slots, int steps, const uint64_t* inputs,
                                       const uint32_t* sleep_ns, uint64_t* totals) {
    if (!valid_k(k)) return fail(POSPOP_EINVAL, "k must be 8, 16, 32 or 64, got %d", k);
    if (n_ranks < 1 || n_ranks > kXMaxRanks || slots < 1 || steps < 0 || !inputs || !sleep_ns || !totals)
        return fail(POSPOP_EINVAL, "bad exchange self-test request");
    int dev = 0;
    pospop_status s = current_device(&dev);
    if (s) return s;
    const size_t words = xbuffer_words(n_ranks, k, slots);
    const size_t in_n = (size_t)steps * n_ranks * k, sl_n = (size_t)steps * n_ranks;
    // one allocation: n buffers, the pointer table, inputs, sleeps, totals
    const size_t bytes = (n_ranks * words + n_ranks + 2 * in_n) * 8 + sl_n * 4 + 64;
    unsigned long long* base = nullptr;
    CU(cudaMalloc(&base, bytes));
    struct Free {
        void* p;
        ~Free() { cudaFree(p); }
    } guard{base};
    CU(cudaMemset(base, 0, bytes));
    std::vector<unsigned long long*> table((size_t)n_ranks);
    for (int r = 0; r < n_ranks; ++r) table[(size_t)r] = base + (size_t)r * words;
    unsigned long long* d_table = base + (size_t)n_ranks * words;
    unsigned long long* d_in = d_table + n_ranks;
    unsigned long long* d_tot = d_in + in_n;
    unsigned* d_sleep = reinterpret_cast<unsigned*>(d_tot + in_n);
    CU(cudaMemcpy(d_table, table.data(), (size_t)n_ranks * 8, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(d_in, inputs, in_n * 8, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(d_sleep, sleep_ns, sl_n * 4, cudaMemcpyHostToDevice));
    CU(launch_exchange_emulate(reinterpret_cast<unsigned long long* const*>(d_table), n_ranks, k, slots, steps, d_in, d_sleep, d_tot, nullptr));
    CU(cudaDeviceSynchronize());
    CU(cudaMemcpy(totals, d_tot, in_n * 8, cudaMemcpyDeviceToHost));
    for (int r = 0; r < n_ranks; ++r) {
        uint64_t h[2];
        CU(cudaMemcpy(h, table[(size_t)r], sizeof h, cudaMemcpyDeviceToHost));
        if (h[1] || h[0] != (uint64_t)steps)
            return fail(POSPOP_ECUDA, "exchange self-test: rank %d consumed %llu of %d steps, error %llu", r,
                        (unsigned long long)h[0], steps, (unsigned long long)h[1]);
    }
    return POSPOP_OK;
}

pospop_status pospopcnt_trace_async(int k, const void* d_data, size_t len, uint64_t* d_counts,
                                    uint64_t* d_trace, size_t trace_ctas, int* grid_used, void* stream) {
    if (!valid_k(k)) return fail(POSPOP_EINVAL, "k must be 8, 16, 32 or 64, got %d", k);
    if (!d_counts || !d_trace || !grid_used || (!d_data && len)) return fail(POSPOP_EINVAL, "NULL pointer");
    if ((uintptr_t)d_data % ((size_t)k / 8)) return fail(POSPOP_EINVAL, "data is misaligned");
    int dev = 0;
    pospop_status s = current_device(&dev);
    if (s) return s;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    StreamWorkspace ws;
    if ((s = stream_workspace(dev, st, &ws))) return s;
    LaunchOptions opt;
    opt.trace = reinterpret_cast<unsigned long long*>(d_trace);
    // The grid is decided inside the launcher; refuse to launch if the trace
    // buffer could be too small for the largest persistent grid.
    int sms = 0;
    CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    // 5 stamps per CTA + 3 per warp (SCHED 2): at most 8 + 3 x 32 u64 per CTA of a persistent grid
    if (trace_ctas < (size_t)sms * 32) return fail(POSPOP_EINVAL, "trace buffer needs >= %d CTAs", sms * 32);
    CU(launch_stream(k, len ? d_data : (const void*)d_counts, len, reinterpret_cast<unsigned long long*>(d_counts),
                     false, opt, ws, st, grid_used));
    return POSPOP_OK;
}

// ---------------------------------------------------------------------------
// CUDA-graph replay of one count (calls where launch
// latency dominates).  The graph holds one kernel node bound to the data
// pointer, length and output; it reads the buffer's CURRENT contents at every
// replay.  Each graph owns its workspace, so different graphs may run
// concurrently; one graph must not be replayed concurrently with itself.
// ---------------------------------------------------------------------------
}  // extern "C"

struct pospop_graph_s {
    int dev = -1;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    StreamWorkspace ws;
};

extern "C" {

pospop_status pospopcnt_graph_create(int k, const void* d_data, size_t len, uint64_t* d_counts,
                                     pospop_graph* out) {
    if (!valid_k(k)) return fail(POSPOP_EINVAL, "k must be 8, 16, 32 or 64, got %d", k);
    if (!out || !d_counts || (!d_data && len)) return fail(POSPOP_EINVAL, "NULL pointer");
    if ((uintptr_t)d_data % ((size_t)k / 8)) return fail(POSPOP_EINVAL, "data is misaligned");
    *out = nullptr;
    int dev = 0;
    pospop_status s = current_device(&dev);
    if (s) return s;
    if (len && classify(d_data, &dev) != Where::Device) return fail(POSPOP_EINVAL, "graph data must be device memory");
    DeviceGuard g(dev);
    auto* gr = new pospop_graph_s;
    gr->dev = dev;
    if ((s = alloc_workspace(&gr->ws))) {
        delete gr;
        return s;
    }
    cudaStream_t cap = nullptr;
    CU(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
    CU(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
    LaunchOptions opt;
    const cudaError_t le = launch_stream(k, len ? d_data : (const void*)d_counts, len,
                                         reinterpret_cast<unsigned long long*>(d_counts), false, opt, gr->ws, cap);
    const cudaError_t ce = cudaStreamEndCapture(cap, &gr->graph);
    cudaStreamDestroy(cap);
    if (le != cudaSuccess || ce != cudaSuccess) {
        cudaFree(gr->ws.acc);
        delete gr;
        return cuda_fail(le != cudaSuccess ? le : ce, "graph capture");
    }
    const cudaError_t ie = cudaGraphInstantiate(&gr->exec, gr->graph, 0);
    if (ie != cudaSuccess) {
        cudaGraphDestroy(gr->graph);
        cudaFree(gr->ws.acc);
        delete gr;
        return cuda_fail(ie, "cudaGraphInstantiate");
    }
    *out = gr;
    return POSPOP_OK;
}

pospop_status pospopcnt_graph_launch(pospop_graph gr, void* stream) {
    if (!gr) return fail(POSPOP_EINVAL, "NULL graph");
    DeviceGuard g(gr->dev);
    CU(cudaGraphLaunch(gr->exec, static_cast<cudaStream_t>(stream)));
    return POSPOP_OK;
}

void pospopcnt_graph_destroy(pospop_graph gr) {
    if (!gr) return;
    DeviceGuard g(gr->dev);
    cudaGraphExecDestroy(gr->exec);
    cudaGraphDestroy(gr->graph);
    cudaFree(gr->ws.acc);
    delete gr;
}

pospop_status pospopcnt_segmented_async(int k, const void* d_data, const uint64_t* d_offsets, size_t n,
                                        uint64_t* d_counts, uint32_t flush, int grid, int block,
                                        void* stream) {
    if (!valid_k(k)) return fail(POSPOP_EINVAL, "k must be 8, 16, 32 or 64, got %d", k);
    if (flush < 1 || flush > 65535)
        return fail(POSPOP_EINVAL, "flush_threshold_blocks must be in [1, 65535], got %u", flush);
    if (n && (!d_offsets || !d_counts)) return fail(POSPOP_EINVAL, "NULL pointer");
    if ((uintptr_t)d_data % ((size_t)k / 8)) return fail(POSPOP_EINVAL, "data is misaligned");
    if (block < 0 || block % 32 || block > 256) return fail(POSPOP_EINVAL, "block must be a multiple of 32 in [32, 256]");
    int dev = 0;
    pospop_status s = current_device(&dev);
    if (s) return s;
    cudaStream_t st = static_cast<cudaStream_t>(stream);  // NULL = legacy default stream
    StreamWorkspace ws;
    LaunchOptions opt;
    // The default kernel reads (offsets and data) before waiting for the
    // previous launch on the stream, so programmatic dependent launch is
    // dropped when either allocation may hold a recent launch's output.
    const void *dbase = nullptr, *obase = nullptr;
    size_t dbytes = 0, obytes = 0;
    const bool known = (!d_data || alloc_range(d_data, &dbase, &dbytes)) && (!n || alloc_range(d_offsets, &obase, &obytes));
    if ((s = stream_workspace(dev, st, &ws, dbase, dbytes, d_counts, n * (size_t)k * 8, &opt.no_pdl, obase, obytes,
                              true)))
        return s;
    if (!known) opt.no_pdl = true;
    opt.flush_threshold = flush;
    opt.grid = grid;
    opt.block = block;
    CU(launch_segmented(k, d_data, reinterpret_cast<const unsigned long long*>(d_offsets), n,
                        reinterpret_cast<unsigned long long*>(d_counts), opt, ws, st));
    return POSPOP_OK;
}

pospop_status pospop_generate(int kind, uint64_t seed, uint64_t base, size_t n, void* d_out, void* stream) {
    if (kind < 1 || kind > 8) return fail(POSPOP_EINVAL, "unknown generator kind %d", kind);
    if (!d_out && n) return fail(POSPOP_EINVAL, "NULL output");
    int dev = 0;
    pospop_status s = current_device(&dev);
    if (s) return s;
    CU(launch_generate(kind, seed, base, n, d_out, static_cast<cudaStream_t>(stream)));
    return POSPOP_OK;
}

pospop_status pospop_microop(int op, int depth, const uint32_t* in, size_t n_in, uint32_t* out, size_t n_out) {
    if (op < 0 || op > 4 || depth < 1 || depth > 7 || !in || !out) return fail(POSPOP_EINVAL, "bad micro-op request");
    if (op == 1 && (n_in < (size_t)depth || (n_in - depth) % ((size_t)1 << depth)))
        return fail(POSPOP_EINVAL, "tree input must be depth carries + whole blocks of 2^depth registers");
    if (op == 4 && n_in != 32 * 17) return fail(POSPOP_EINVAL, "total needs 32 lanes x (16 counters + shift)");
    int dev = 0;
    pospop_status s = current_device(&dev);
    if (s) return s;
    CtxScope scope;
    Ctx* c = nullptr;
    if ((s = scope.get(dev, &c))) return s;
    uint32_t *d_in = nullptr, *d_out = nullptr;
    CU(cudaMalloc(&d_in, n_in * 4 + 4));
    CU(cudaMalloc(&d_out, n_out * 4 + 4));
    CU(cudaMemcpyAsync(d_in, in, n_in * 4, cudaMemcpyHostToDevice, c->stream));
    CU(cudaMemsetAsync(d_out, 0, n_out * 4, c->stream));
    CU(launch_microop(op, depth, d_in, n_in, d_out, c->stream));
    CU(cudaMemcpyAsync(out, d_out, n_out * 4, cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    cudaFree(d_in);
    cudaFree(d_out);
    return POSPOP_OK;
}

pospop_status pospop_digest(const void* d_data, size_t nbytes, uint64_t* digest) {
    if (!digest || (!d_data && nbytes)) return fail(POSPOP_EINVAL, "NULL pointer");
    if ((uintptr_t)d_data % 8) return fail(POSPOP_EINVAL, "digest input must be 8-byte aligned");
    int dev = 0;
    pospop_status s = current_device(&dev);
    if (s) return s;
    classify(d_data, &dev);
    DeviceGuard g(dev);
    CtxScope scope;
    Ctx* c = nullptr;
    if ((s = scope.get(dev, &c))) return s;
    CU(cudaMemsetAsync(c->d_out, 0, sizeof(unsigned long long), c->stream));
    CU(launch_digest(d_data, nbytes, c->d_out, c->stream));
    CU(cudaMemcpyAsync(c->h_out, c->d_out, sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    *digest = c->h_out[0];
    return POSPOP_OK;
}

}  // extern "C"
