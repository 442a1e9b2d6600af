// runtime.cpp — device context, lazy init/teardown, error boundary, counters
// and the resident-upload helpers of the B200 harness library.

#include "runtime.hpp"

#include "lilac_b200.h"

#include <algorithm>
#include <climits>
#include <map>
#include <memory>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <atomic>
#include <sched.h>

namespace b200 {

bool g_profile = [] {
    const char* e = std::getenv("LILAC_B200_PROFILE");
    return e && std::strcmp(e, "1") == 0;
}();

namespace {
std::int64_t g_phase_ns[kPhCount] = {};
std::int64_t g_phase_n[kPhCount] = {};
}  // namespace

void host_phase_add(int ph, std::int64_t ns) {
    g_phase_ns[ph] += ns;
    g_phase_n[ph] += 1;
}

namespace {
thread_local std::string t_err;
thread_local std::string t_err_code;
int g_error_mode = -1;
std::vector<RegionEntry> g_regions;
std::vector<HarnessStats*> g_hstats;
}  // namespace

const char* current_error() { return t_err.c_str(); }

void set_error(const char* code, const std::string& msg) {
    t_err_code = code;
    t_err = msg;
}

void clear_error() {
    t_err.clear();
    t_err_code.clear();
}

int error_mode() {
    if (g_error_mode < 0) {
        const char* e = std::getenv("LILAC_B200_ERRORS");
        g_error_mode = (e && std::strcmp(e, "return") == 0) ? B200_ERRORS_RETURN : B200_ERRORS_ABORT;
    }
    return g_error_mode;
}

void throw_cuda(cudaError_t e, const char* what, const char* file, int line) {
    throw Error(Errc::DeviceError, std::string(cudaGetErrorName(e)) + " (" + cudaGetErrorString(e) +
                                       ") in " + what + " at " + file + ":" + std::to_string(line));
}

// ---- DevBuf + caching pool --------------------------------------------------------
//
// Marshal objects destruct/construct their device arrays whenever a host
// region's identity changes (reference marshal.hpp:192-199) — e.g. the dot
// harness sees (r,r), (p,q), (x,z) in turn. cudaMalloc/cudaFree on that path
// would serialise the device, so freed blocks go to a size-class free list
// and are reused; everything is returned to CUDA at shutdown.

namespace {
struct PoolBlock {
    void* ptr;
    std::size_t cap;
    int device;
};
std::vector<PoolBlock> g_pool;
std::size_t g_pool_bytes = 0;
constexpr std::size_t kPoolLimit = std::size_t(8) << 30;  // cached bytes kept at most

std::size_t size_class(std::size_t n) {
    if (n <= (std::size_t(1) << 20)) {  // powers of two up to 1 MiB
        std::size_t c = 4096;
        while (c < n) c <<= 1;
        return c;
    }
    const std::size_t g = std::size_t(2) << 20;  // 2 MiB granules above
    return (n + g - 1) / g * g;
}
}  // namespace

void DevBuf::ensure(std::size_t n, bool zero_tail) {
    if (ptr && cap >= n + kPadBytes) {
        bytes = n;
        return;
    }
    release();
    ensure_init();
    int dev = 0;
    B200_CUDA(cudaGetDevice(&dev));
    const std::size_t want = size_class(n + kPadBytes);
    for (std::size_t i = 0; i < g_pool.size(); ++i) {
        if (g_pool[i].device == dev && g_pool[i].cap == want) {
            ptr = g_pool[i].ptr;
            g_pool_bytes -= want;
            g_pool.erase(g_pool.begin() + static_cast<std::ptrdiff_t>(i));
            break;
        }
    }
    if (!ptr) {
        host_phase_add(kPhMalloc, 0);
        cudaError_t e = cudaMalloc(&ptr, want);
        if (e == cudaErrorMemoryAllocation && !g_pool.empty()) {
            (void)cudaGetLastError();
            pool_trim();
            e = cudaMalloc(&ptr, want);
        }
        if (e != cudaSuccess) {
            ptr = nullptr;
            throw_cuda(e, "cudaMalloc", __FILE__, __LINE__);
        }
    }
    // zero the tail so masked over-reads of index arrays stay in range
    if (zero_tail) B200_CUDA(cudaMemsetAsync(static_cast<char*>(ptr) + n, 0, want - n, rt().stream));
    cap = want;
    bytes = n;
    device = dev;
}

void DevBuf::release() {
    if (ptr) {
        if (rt().inited && g_pool_bytes + cap <= kPoolLimit) {
            g_pool.push_back({ptr, cap, device});
            g_pool_bytes += cap;
        } else {
            cudaFree(ptr);  // teardown path: errors ignored
        }
    }
    ptr = nullptr;
    bytes = cap = 0;
}

bool keep_plain_csr() {
    static const bool keep = [] {
        const char* e = std::getenv("LILAC_B200_KEEP_CSR");
        return e && std::strcmp(e, "1") == 0;
    }();
    return keep;
}

void device_quiesce() {
    if (rt().inited) (void)cudaDeviceSynchronize();
}

void pool_trim() {
    for (const PoolBlock& b : g_pool) cudaFree(b.ptr);
    g_pool.clear();
    g_pool_bytes = 0;
}

// ---- runtime ------------------------------------------------------------------

namespace {
thread_local Runtime* tl_rt = nullptr;  // a DeviceScope's runtime
Runtime& primary_rt() {
    static Runtime r;
    return r;
}
std::map<int, std::unique_ptr<Runtime>>& secondary_rts() {
    static auto* m = new std::map<int, std::unique_ptr<Runtime>>;  // outlives atexit teardown
    return *m;
}
}  // namespace

Runtime& rt() { return tl_rt ? *tl_rt : primary_rt(); }

int harness_ngpus() {
    static const int k = [] {
        const char* e = std::getenv("LILAC_B200_NGPUS");
        // at most 64 shards: multi_dot's per-shard result slots live in the
        // runtime's 4 KB scalar block (d_result() + g)
        return e && *e ? std::min(64, std::max(1, std::atoi(e))) : 1;
    }();
    return k;
}

int shard_device(int g) {
    ensure_init();
    int count = 1;
    B200_CUDA(cudaGetDeviceCount(&count));
    return (primary_rt().device + g) % std::max(count, 1);
}

Runtime& device_runtime(int device) {
    ensure_init();
    Runtime& p = primary_rt();
    if (device == p.device) return p;
    auto& m = secondary_rts();
    auto it = m.find(device);
    if (it != m.end()) return *it->second;
    auto r = std::make_unique<Runtime>();
    Runtime* prev = tl_rt;
    int prev_dev = 0;
    B200_CUDA(cudaGetDevice(&prev_dev));
    B200_CUDA(cudaSetDevice(device));
    r->device = device;
    B200_CUDA(cudaStreamCreateWithFlags(&r->stream, cudaStreamNonBlocking));
    B200_CUDA(cudaEventCreate(&r->ev_k0));
    B200_CUDA(cudaEventCreate(&r->ev_k1));
    {
        void* h = nullptr;
        B200_CUDA(cudaHostAlloc(&h, 128, cudaHostAllocMapped | cudaHostAllocPortable));
        std::memset(h, 0, 128);
        r->h_slot_val = static_cast<double*>(h);
        r->h_slot_flag = reinterpret_cast<unsigned*>(static_cast<char*>(h) + 64);
        void* d = nullptr;
        B200_CUDA(cudaHostGetDevicePointer(&d, h, 0));
        r->dslot.value = static_cast<double*>(d);
        r->dslot.flag = reinterpret_cast<unsigned*>(static_cast<char*>(d) + 64);
    }
    r->inited = true;
    tl_rt = r.get();  // the scratch below is allocated on `device`
    r->partials.ensure(sizeof(double) * kMaxParts * 4);
    r->scalars.ensure(4096);
    r->flags.ensure(64);
    B200_CUDA(cudaMemsetAsync(r->scalars.ptr, 0, 4096, r->stream));
    B200_CUDA(cudaStreamSynchronize(r->stream));
    tl_rt = prev;
    B200_CUDA(cudaSetDevice(prev_dev));
    Runtime& out = *r;
    m.emplace(device, std::move(r));
    return out;
}

DeviceScope::DeviceScope(int device) : prev(tl_rt) {
    Runtime& r = device_runtime(device);
    const Runtime& p = primary_rt();
    // the primary's settings
    r.kernel = p.kernel;
    r.strategy = p.strategy;
    r.exact_blas = p.exact_blas;
    r.stage_bytes = p.stage_bytes;
    B200_CUDA(cudaGetDevice(&prev_dev));
    B200_CUDA(cudaSetDevice(r.device));
    tl_rt = &r;
}

DeviceScope::~DeviceScope() {
    tl_rt = prev;
    (void)cudaSetDevice(prev_dev);
}

static void at_exit_teardown() { shutdown(); }

void ensure_init() {
    Runtime& r = rt();
    if (r.inited) return;
    int dev = r.device;
    if (dev < 0) {
        const char* e = std::getenv("LILAC_B200_DEVICE");
        if (e && *e)
            dev = std::atoi(e);
        else
            B200_CUDA(cudaGetDevice(&dev));
    }
    int count = 0;
    B200_CUDA(cudaGetDeviceCount(&count));
    if (dev < 0 || dev >= count)
        throw Error(Errc::DeviceError, "device " + std::to_string(dev) + " not present (" +
                                           std::to_string(count) + " visible)");
    B200_CUDA(cudaSetDevice(dev));
    cudaDeviceProp prop;
    B200_CUDA(cudaGetDeviceProperties(&prop, dev));
    if (prop.major != 10)
        throw Error(Errc::DeviceError, std::string("built for sm_100a, found ") + prop.name + " (sm_" +
                                           std::to_string(prop.major) + std::to_string(prop.minor) + ")");
    r.device = dev;
    B200_CUDA(cudaStreamCreateWithFlags(&r.stream, cudaStreamNonBlocking));
    B200_CUDA(cudaEventCreate(&r.ev_k0));
    B200_CUDA(cudaEventCreate(&r.ev_k1));
    {
        void* h = nullptr;
        B200_CUDA(cudaHostAlloc(&h, 128, cudaHostAllocMapped));
        std::memset(h, 0, 128);
        r.h_slot_val = static_cast<double*>(h);
        r.h_slot_flag = reinterpret_cast<unsigned*>(static_cast<char*>(h) + 64);
        void* d = nullptr;
        B200_CUDA(cudaHostGetDevicePointer(&d, h, 0));
        r.dslot.value = static_cast<double*>(d);
        r.dslot.flag = reinterpret_cast<unsigned*>(static_cast<char*>(d) + 64);
    }
    r.inited = true;  // DevBuf::ensure below re-enters ensure_init
    r.partials.ensure(sizeof(double) * kMaxParts * 4);
    r.scalars.ensure(4096);
    r.flags.ensure(64);
    B200_CUDA(cudaMemsetAsync(r.scalars.ptr, 0, 4096, r.stream));
    B200_CUDA(cudaStreamSynchronize(r.stream));
    const char* k = std::getenv("LILAC_B200_KERNEL");
    if (k && *k) r.kernel = parse_csr_kernel(k);
    r.strategy = lilac::marshal::default_strategy(Strategy::Hybrid);
    const char* wb = std::getenv("LILAC_B200_WRITEBACK");
    if (wb && std::strcmp(wb, "lazy") == 0) r.lazy_writeback = true;
    // page guards see CPU stores only: tell the marshaling layer which host
    // memory DMA or device stores can reach (pinned / registered / managed)
    lilac::marshal::set_dma_probe([](const void* p) {
        cudaPointerAttributes a;
        if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
            (void)cudaGetLastError();
            return false;
        }
        return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeManaged;
    });
    const char* pin = std::getenv("LILAC_B200_PINNED");
    lilac::marshal::set_dma_always_dirty(pin && std::strcmp(pin, "always") == 0);
    // registered after the CUDA runtime initialised, so it runs before the
    // runtime's own teardown (mirrors harnessgen.cpp:98-113)
    std::atexit(at_exit_teardown);
}

double wait_host_slot(unsigned seq) {
    Runtime& r = rt();
    volatile unsigned* flag = r.h_slot_flag;
    for (unsigned long spin = 1;; ++spin) {
        if (*flag == seq) break;
        if ((spin & 1023) == 0) {
            const cudaError_t e = cudaStreamQuery(r.stream);
            if (e == cudaSuccess) {
                if (*flag == seq) break;
                throw Error(Errc::DeviceError, "result slot not posted by a completed kernel");
            }
            if (e != cudaErrorNotReady) throw_cuda(e, "cudaStreamQuery", __FILE__, __LINE__);
            if (spin > (1ul << 20)) sched_yield();  // a long queue: stop burning the core
        }
        __builtin_ia32_pause();
    }
    std::atomic_thread_fence(std::memory_order_acquire);
    return *reinterpret_cast<volatile double*>(r.h_slot_val);
}

void shutdown() {
    Runtime& r = primary_rt();
    lilac::marshal::release_all();
    mirrors_clear();
    if (!r.inited) return;
    for (auto& kv : secondary_rts()) {
        Runtime& q = *kv.second;
        (void)cudaSetDevice(q.device);
        for (DevBuf* b : {&q.partials, &q.scalars, &q.flags, &q.stage}) b->release();
        if (q.h_slot_val) cudaFreeHost(q.h_slot_val);
        if (q.ev_k0) cudaEventDestroy(q.ev_k0);
        if (q.ev_k1) cudaEventDestroy(q.ev_k1);
        if (q.stream) cudaStreamDestroy(q.stream);
    }
    secondary_rts().clear();
    (void)cudaSetDevice(r.device);
    r.partials.release();
    r.scalars.release();
    r.flags.release();
    r.stage.release();
    if (r.h_slot_val) cudaFreeHost(r.h_slot_val);
    r.h_slot_val = nullptr;
    r.h_slot_flag = nullptr;
    r.dslot = HostSlot{};
    if (r.ev_k0) cudaEventDestroy(r.ev_k0);
    if (r.ev_k1) cudaEventDestroy(r.ev_k1);
    pool_trim();
    if (r.stream) cudaStreamDestroy(r.stream);
    r.ev_k0 = r.ev_k1 = nullptr;
    r.stream = nullptr;
    r.inited = false;
}

void register_region(MarshalObjectBase* obj, const std::int64_t* h2d, const std::int64_t* d2h,
                     const std::int64_t* d2d) {
    for (auto& e : g_regions)
        if (e.obj == obj) return;
    g_regions.push_back({obj, h2d, d2h, d2d});
}

const std::vector<RegionEntry>& all_regions() { return g_regions; }

HarnessStats& harness_stats(const char* name) {
    for (HarnessStats* h : g_hstats)
        if (h->name == name) return *h;
    auto* h = new HarnessStats;
    h->name = name;
    g_hstats.push_back(h);
    return *h;
}

std::vector<HarnessStats*> all_harness_stats() { return g_hstats; }

// ---- transfers -------------------------------------------------------------------

void upload(DevArray& d, const void* host, std::size_t bytes) {
    if (bytes > 0) {
        PhaseTimer pt(kPhMirrorFetch);
        if (mirror_fetch(d, host, bytes)) {
            d.d2d += static_cast<std::int64_t>(bytes);
            return;
        }
    }
    d.lent.reset();
    d.view = nullptr;
    d.buf.ensure(bytes);
    if (bytes == 0) return;
    PhaseTimer pt(kPhH2D);
    host_in(host, bytes);
    B200_CUDA(cudaMemcpyAsync(d.buf.ptr, host, bytes, cudaMemcpyHostToDevice, rt().stream));
    d.h2d += static_cast<std::int64_t>(bytes);
}

void download(void* host, DevArray& d, std::size_t bytes, DevArray& counter) {
    if (bytes == 0) return;
    if (rt().lazy_writeback) {
        PhaseTimer pt(kPhPublish);
        std::size_t eager = 0;  // the partial edge pages of an unaligned output, written now
        if (mirror_publish_lazy(host, bytes, d.buf, &eager)) {
            counter.lazy += static_cast<std::int64_t>(bytes - eager);
            counter.d2h += static_cast<std::int64_t>(eager);
            return;
        }
    }
    {
        PhaseTimer pt(kPhD2H);
        lilac::marshal::supersede_range(host, bytes);  // lazy bytes under the destination
        d2h_copy(host, d.buf.ptr, bytes, rt().stream);
    }
    PhaseTimer pt(kPhPublish);
    // publish only after the bytes landed (pinned D2H is asynchronous: the
    // mirror's edge snapshot must see the written data)
    mirror_publish(host, bytes, d.buf);
    counter.d2h += static_cast<std::int64_t>(bytes);
}

// ---- device mirrors ------------------------------------------------------------------

namespace {

struct Mirror {
    lilac::marshal::TrackedRegion reg;
    std::shared_ptr<const DevBuf> buf;  // immutable once published; borrowed by inputs
    lilac::marshal::DeferredRange lazy;  // active while the host bytes are still on the device
};

std::map<std::uintptr_t, std::unique_ptr<Mirror>> g_mirrors;  // keyed by host base
std::size_t g_mirror_total = 0;
constexpr std::size_t kMirrorMin = std::size_t(8) << 10;  // smaller arrays: not worth a guard
constexpr std::size_t kMirrorLimit = std::size_t(4) << 30;  // device bytes kept as mirrors

bool mirrors_enabled() {
    static int on = -1;
    if (on < 0) {
        const char* e = std::getenv("LILAC_B200_MIRRORS");
        on = (e && std::strcmp(e, "0") == 0) ? 0 : 1;
    }
    return on == 1;
}

// Take src's device allocation (no copy) as an immutable shared buffer; src
// gets a fresh allocation of the same size from the pool.
std::shared_ptr<const DevBuf> steal(DevBuf& src, std::size_t bytes) {
    PhaseTimer pt(kPhSteal);
    auto* b = new DevBuf(src);
    src = DevBuf{};
    src.ensure(bytes, false);  // an f64 output: its padding is never indexed
    return std::shared_ptr<const DevBuf>(b, [](const DevBuf* p) {
        const_cast<DevBuf*>(p)->release();
        delete p;
    });
}

std::int64_t g_lazy_deferred = 0, g_lazy_filled = 0;

// Materialise a lazy write-back: the mirror holds the bytes. Runs in the
// fault handler or before a DMA read; a failure here loses data: abort.
void mirror_fill(lilac::marshal::DeferredRange* d) {
    auto* m = static_cast<Mirror*>(d->ctx);
    const std::size_t bytes = d->content_hi - d->content_lo;
    // the lazy bytes start content_lo - base into the mirror (an unaligned
    // output defers only its whole interior pages)
    const std::size_t off = d->content_lo - reinterpret_cast<std::uintptr_t>(m->reg.ref.base);
    Runtime& r = rt();
    cudaError_t e = cudaMemcpyAsync(reinterpret_cast<void*>(d->content_lo), m->buf->as<const char>() + off, bytes,
                                    cudaMemcpyDeviceToHost, r.stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(r.stream);
    if (e != cudaSuccess) {
        std::fprintf(stderr, "lilac-b200: lazy write-back of %zu bytes failed: %s\n", bytes, cudaGetErrorString(e));
        std::abort();
    }
    g_lazy_filled += static_cast<std::int64_t>(bytes);
}

// fill: materialise first if the host bytes are still lazy (false when the
// caller is about to overwrite all of them)
void drop_mirror(std::map<std::uintptr_t, std::unique_ptr<Mirror>>::iterator it, bool fill = true) {
    lilac::marshal::retire_deferred(it->second->lazy, fill);
    lilac::marshal::drop_guard(it->second->reg);
    g_mirror_total -= it->second->buf->cap;
    g_mirrors.erase(it);
}

// drop every mirror overlapping [h, h+bytes); lazy ones are filled unless the
// range covers them (their bytes are superseded)
void drop_overlapping(std::uintptr_t h, std::size_t bytes) {
    for (auto it = g_mirrors.begin(); it != g_mirrors.end();) {
        const std::uintptr_t lo = it->first, hi = lo + it->second->reg.ref.bytes;
        if (lo < h + bytes && h < hi) {
            auto nx = std::next(it);
            drop_mirror(it, !(h <= lo && hi <= h + bytes));
            it = nx;
        } else {
            ++it;
        }
    }
}

}  // namespace

bool mirror_fetch(DevArray& d, const void* host, std::size_t bytes) {
    if (g_mirrors.empty()) return false;
    const auto h = reinterpret_cast<std::uintptr_t>(host);
    auto it = g_mirrors.upper_bound(h);
    if (it == g_mirrors.begin()) return false;
    --it;
    Mirror& m = *it->second;
    if (h + bytes > it->first + m.reg.ref.bytes) return false;  // not contained
    {
        PhaseTimer pt(kPhMirrorPoll);
        if (lilac::marshal::poll_dirty(m.reg)) {  // the host wrote it since the write-back
            drop_mirror(it);
            return false;
        }
    }
    // zero-copy: borrow the mirror's buffer (the device buffer d owned, if
    // any, is kept for a later host upload)
    d.lent = m.buf;
    d.view = m.buf->as<const char>() + (h - it->first);
    return true;
}

void mirror_publish(const void* host, std::size_t bytes, DevBuf& src) {
    if (!mirrors_enabled() || bytes < kMirrorMin) return;
    const auto h = reinterpret_cast<std::uintptr_t>(host);
    drop_overlapping(h, bytes);  // stale now
    if (g_mirror_total + bytes > kMirrorLimit) mirrors_clear();
    auto m = std::make_unique<Mirror>();
    m->reg.ref = {host, bytes, nullptr};
    m->reg.strategy = lilac::marshal::Strategy::Hybrid;
    try {
        PhaseTimer pt(kPhPublishGuard);
        lilac::marshal::mark_clean(m->reg);  // guard: a host write invalidates the mirror
    } catch (const Error&) {
        return;  // pages that cannot be protected get no mirror
    }
    m->buf = steal(src, bytes);
    g_mirror_total += m->buf->cap;
    g_mirrors.emplace(h, std::move(m));
}

bool mirror_publish_lazy(const void* host, std::size_t bytes, DevBuf& src, std::size_t* eager) {
    const auto h = reinterpret_cast<std::uintptr_t>(host);
    const std::size_t pg = lilac::marshal::page_size();
    if (eager) *eager = 0;
    if (!mirrors_enabled() || bytes < kMirrorMin) return false;
    const bool aligned = h % pg == 0;
    auto same = g_mirrors.find(h);
    if (same != g_mirrors.end() && same->second->reg.ref.bytes == bytes && same->second->lazy.active &&
        lilac::marshal::reclean_covered(same->second->reg)) {
        // steady state (rewritten before the host looked): swap in the new
        // device bytes; pages stay PROT_NONE, no system call
        Mirror& m = *same->second;
        g_mirror_total -= m.buf->cap;
        m.buf = steal(src, bytes);
        g_mirror_total += m.buf->cap;
        g_lazy_deferred += static_cast<std::int64_t>(bytes);
        return true;
    }
    drop_overlapping(h, bytes);
    if (g_mirror_total + bytes > kMirrorLimit) mirrors_clear();
    // The pages the bytes touch are deferred (PROT_NONE) and only our bytes are
    // ever filled, so an unrelated neighbour on an edge page (malloc header,
    // free space) reads correctly after a one-time fault. An edge page shared
    // with another array in use (adjacent heap allocations) is written at once
    // instead: making it lazy would fill this output on every access to the
    // neighbour. Aligned: PageProtect; unaligned: Hybrid, which guards a lazy
    // edge page whole and snapshots an eager one.
    std::uintptr_t lo = h / pg * pg, hi = (h + bytes + pg - 1) / pg * pg;
    std::uintptr_t clo = h, chi = h + bytes;
    std::size_t edges = 0;
    if (!aligned || (h + bytes) % pg) {
        const std::uintptr_t last = (h + bytes - 1) / pg * pg;
        const bool head = h % pg && lilac::marshal::page_shared(lo, h, h + bytes);
        const bool tail = (h + bytes) % pg && lilac::marshal::page_shared(last, h, h + bytes) &&
                          (last != lo || !head);
        if (head) {
            lo += pg;
            clo = lo;
        }
        if (tail) {
            hi = last;
            chi = last;
        }
        if (hi <= lo || chi <= clo) return false;  // nothing left to defer
        if (head || tail) {
            Runtime& r = rt();
            lilac::marshal::supersede_range(host, bytes);
            if (head)
                B200_CUDA(cudaMemcpyAsync(const_cast<void*>(host), src.ptr, clo - h, cudaMemcpyDeviceToHost, r.stream));
            if (tail)
                B200_CUDA(cudaMemcpyAsync(reinterpret_cast<void*>(chi), src.as<char>() + (chi - h), h + bytes - chi,
                                          cudaMemcpyDeviceToHost, r.stream));
            B200_CUDA(cudaStreamSynchronize(r.stream));
            edges = (clo - h) + (h + bytes - chi);
        }
    }
    auto m = std::make_unique<Mirror>();
    m->reg.ref = {host, bytes, nullptr};
    m->reg.strategy = aligned ? lilac::marshal::Strategy::PageProtect : lilac::marshal::Strategy::Hybrid;
    m->lazy.lo = lo;
    m->lazy.hi = hi;
    m->lazy.content_lo = clo;
    m->lazy.content_hi = chi;
    m->lazy.fill = mirror_fill;
    m->lazy.ctx = m.get();
    m->buf = steal(src, bytes);  // before defer_range: a fill needs the bytes
    try {
        PhaseTimer pt(kPhPublishGuard);
        // deferred first: the guard then sees the lazy edge pages and guards
        // them whole instead of snapshotting (reading) their stale bytes
        lilac::marshal::defer_range(m->lazy);
        lilac::marshal::mark_clean(m->reg);
    } catch (const Error&) {
        lilac::marshal::retire_deferred(m->lazy, false);
        lilac::marshal::drop_guard(m->reg);
        // give the bytes back to the caller for an eager write-back
        src.release();
        src = *m->buf;
        const_cast<DevBuf&>(*m->buf) = DevBuf{};
        return false;
    }
    g_lazy_deferred += static_cast<std::int64_t>(chi - clo);
    g_mirror_total += m->buf->cap;
    g_mirrors.emplace(h, std::move(m));
    if (eager) *eager = edges;
    return true;
}

void lazy_bytes(std::int64_t* deferred, std::int64_t* filled) {
    if (deferred) *deferred = g_lazy_deferred;
    if (filled) *filled = g_lazy_filled;
}

void mirrors_forget(const void* host, std::size_t bytes) {
    const auto h = reinterpret_cast<std::uintptr_t>(host);
    for (auto it = g_mirrors.begin(); it != g_mirrors.end();) {
        const std::uintptr_t lo = it->first, hi = lo + it->second->reg.ref.bytes;
        auto nx = std::next(it);
        if (lo < h + bytes && h < hi) drop_mirror(it, false);
        it = nx;
    }
}

void mirrors_drop_all() {
    while (!g_mirrors.empty()) drop_mirror(g_mirrors.begin(), false);
}

void mirrors_clear() {
    while (!g_mirrors.empty()) drop_mirror(g_mirrors.begin());
}

std::int64_t mirror_bytes() { return static_cast<std::int64_t>(g_mirror_total); }

void upload_row_ptr(DevBuf& buf, const std::int64_t* row_ptr, std::int64_t rows, std::int64_t nnz,
                    std::int64_t* max_row, bool* monotone) {
    Runtime& r = rt();
    const std::size_t bytes = sizeof(std::int64_t) * static_cast<std::size_t>(rows + 1);
    buf.ensure(bytes);
    host_in(row_ptr, bytes);
    B200_CUDA(cudaMemcpyAsync(buf.ptr, row_ptr, bytes, cudaMemcpyHostToDevice, r.stream));
    B200_CUDA(cudaMemsetAsync(r.flags.ptr, 0, 16, r.stream));
    launch_check_row_ptr(buf.as<std::int64_t>(), rows, nnz, r.d_umax(), r.d_bad(), r.stream);
    unsigned long long mx = 0;
    int bad = 0;
    B200_CUDA(cudaMemcpyAsync(&mx, r.d_umax(), 8, cudaMemcpyDeviceToHost, r.stream));
    B200_CUDA(cudaMemcpyAsync(&bad, r.d_bad(), 4, cudaMemcpyDeviceToHost, r.stream));
    B200_CUDA(cudaStreamSynchronize(r.stream));
    if (bad & 1)
        throw Error(Errc::OutOfBounds, "row_ptr addresses nonzeros outside [0, nnz=" + std::to_string(nnz) + ")");
    *max_row = static_cast<std::int64_t>(mx);
    *monotone = (bad & 2) == 0;
}

std::int64_t upload_col_ind(DevBuf& buf, const std::int64_t* col_ind, std::int64_t nnz, bool* col32) {
    Runtime& r = rt();
    const std::size_t n = static_cast<std::size_t>(std::max<std::int64_t>(nnz, 0));
    buf.ensure(n * sizeof(std::int32_t));
    host_in(col_ind, n * sizeof(std::int64_t));
    B200_CUDA(cudaMemsetAsync(r.flags.ptr, 0, 16, r.stream));
    // narrow chunk by chunk through a bounded staging buffer
    const std::size_t chunk = std::max<std::size_t>(1, r.stage_bytes / sizeof(std::int64_t));
    if (n > 0) r.stage.ensure(std::min(n, chunk) * sizeof(std::int64_t));
    for (std::size_t off = 0; off < n; off += chunk) {
        const std::size_t m = std::min(chunk, n - off);
        B200_CUDA(cudaMemcpyAsync(r.stage.ptr, col_ind + off, m * sizeof(std::int64_t), cudaMemcpyHostToDevice,
                                  r.stream));
        launch_scan_cols(r.stage.as<std::int64_t>(), static_cast<std::int64_t>(m), buf.as<std::int32_t>() + off,
                         r.d_umax(), r.d_bad(), r.stream);
    }
    unsigned long long cols = 0;
    int bad = 0;
    B200_CUDA(cudaMemcpyAsync(&cols, r.d_umax(), 8, cudaMemcpyDeviceToHost, r.stream));
    B200_CUDA(cudaMemcpyAsync(&bad, r.d_bad(), 4, cudaMemcpyDeviceToHost, r.stream));
    B200_CUDA(cudaStreamSynchronize(r.stream));
    if (bad) throw Error(Errc::OutOfBounds, "negative column index in col_ind");
    if (cols > static_cast<unsigned long long>(INT32_MAX)) {
        // too wide for int32: keep the ABI width
        buf.ensure(n * sizeof(std::int64_t));
        if (n) B200_CUDA(cudaMemcpyAsync(buf.ptr, col_ind, n * sizeof(std::int64_t), cudaMemcpyHostToDevice, r.stream));
        B200_CUDA(cudaStreamSynchronize(r.stream));
        *col32 = false;
    } else {
        *col32 = true;
    }
    return static_cast<std::int64_t>(cols);
}

}  // namespace b200

// ---- C ABI: runtime control and counters -------------------------------------------

using namespace b200;

extern "C" {

int b200_init(int device) {
    return boundary("b200_init", [&] {
        if (rt().inited && rt().device != device && device >= 0)
            throw Error(Errc::DataError, "already initialised on device " + std::to_string(rt().device));
        if (device >= 0) rt().device = device;
        ensure_init();
    });
}

void b200_shutdown(void) {
    boundary("b200_shutdown", [] { shutdown(); });
}

void b200_set_error_mode(int mode) { g_error_mode = mode == B200_ERRORS_RETURN ? 1 : 0; }

const char* b200_last_error(void) { return t_err.c_str(); }
const char* b200_last_error_code(void) { return t_err_code.c_str(); }

int b200_set_kernel(const char* name) {
    return boundary("b200_set_kernel", [&] {
        CsrKernel k = parse_csr_kernel(name ? name : "");
        rt().kernel = k;  // layouts are (re)decided at the next upload
    });
}

int b200_set_strategy(const char* name) {
    return boundary("b200_set_strategy", [&] { rt().strategy = lilac::marshal::parse_strategy(name ? name : ""); });
}

void b200_set_exact_blas(int on) { rt().exact_blas = on != 0; }

void b200_set_profiling(int on) { g_profile = on != 0; }

int b200_set_writeback(const char* mode) {
    return boundary("b200_set_writeback", [&] {
        const std::string m = mode ? mode : "";
        if (m == "lazy")
            rt().lazy_writeback = true;
        else if (m == "eager")
            rt().lazy_writeback = false;
        else
            throw Error(Errc::DataError, "unknown write-back mode '" + m + "' (expected eager or lazy)");
    });
}

int b200_host_sync(const void* host, size_t bytes) {
    return boundary("b200_host_sync", [&] {
        if (host)
            lilac::marshal::materialize_range(host, bytes);
        else
            lilac::marshal::materialize_all();
    });
}

int b200_host_will_write(void* host, size_t bytes) {
    return boundary("b200_host_will_write", [&] {
        if (!host || bytes == 0) return;
        // a writer that does not fault (a system call, another library's DMA):
        // lazy bytes there become real first (a partial write keeps the rest),
        // guards over the range are lifted and their regions marked changed,
        // device mirrors of it are dropped
        lilac::marshal::materialize_range(host, bytes);
        lilac::marshal::note_host_write(host, bytes);
        mirrors_forget(host, bytes);
    });
}

int b200_host_forget(const void* host, size_t bytes) {
    return boundary("b200_host_forget", [&] {
        if (!host) {
            lilac::marshal::release_all();
            mirrors_drop_all();
            return;
        }
        mirrors_forget(host, bytes);
        lilac::marshal::forget_range(host, bytes);
    });
}

int b200_lazy_counters(int64_t* ranges, int64_t* fault_fills, int64_t* explicit_fills, int64_t* cancelled,
                       int64_t* bytes_deferred, int64_t* bytes_filled) {
    long a = 0, b = 0, c = 0, d = 0;
    lilac::marshal::deferred_counters(&a, &b, &c, &d);
    if (ranges) *ranges = a;
    if (fault_fills) *fault_fills = b;
    if (explicit_fills) *explicit_fills = c;
    if (cancelled) *cancelled = d;
    lazy_bytes(bytes_deferred, bytes_filled);
    return 0;
}

const char* b200_version(void) { return "lilac-b200 0.1 sm_100a"; }

int b200_region_stats_get(b200_region_stats* out, int cap) {
    const auto& regs = all_regions();
    int n = 0;
    for (const RegionEntry& e : regs) {
        if (n < cap && out) {
            b200_region_stats& s = out[n];
            std::memset(&s, 0, sizeof s);
            std::strncpy(s.region, e.obj->name().c_str(), sizeof(s.region) - 1);
            s.n_construct = e.obj->counters().n_construct;
            s.n_update = e.obj->counters().n_update;
            s.n_destruct = e.obj->counters().n_destruct;
            s.bytes_h2d = e.h2d ? *e.h2d : 0;
            s.bytes_d2h = e.d2h ? *e.d2h : 0;
            s.bytes_d2d = e.d2d ? *e.d2d : 0;
            s.strategy = static_cast<int32_t>(e.obj->strategy());
            s.fell_back = e.obj->fell_back();
            s.streaming = e.obj->streaming();
            s.constructed = e.obj->constructed();
        }
        ++n;
    }
    return n;
}

int b200_harness_stats_get(b200_harness_stats* out, int cap) {
    auto hs = all_harness_stats();
    int n = 0;
    for (HarnessStats* h : hs) {
        if (n < cap && out) {
            b200_harness_stats& s = out[n];
            std::memset(&s, 0, sizeof s);
            std::strncpy(s.harness, h->name.c_str(), sizeof(s.harness) - 1);
            s.calls = h->calls;
            s.t_total_ms = h->t_total_ms;
            s.t_poll_ms = h->t_poll_ms;
            s.t_kernel_ms = h->t_kernel_ms;
            s.t_writeback_ms = h->t_writeback_ms;
            s.bytes_h2d = h->bytes_h2d;
            s.bytes_d2h = h->bytes_d2h;
            s.bytes_d2d = h->bytes_d2d;
        }
        ++n;
    }
    return n;
}

int b200_host_profile(int64_t* ns, int64_t* counts, int cap) {
    for (int i = 0; i < kPhCount && i < cap; ++i) {
        ns[i] = g_phase_ns[i];
        counts[i] = g_phase_n[i];
    }
    return kPhCount;
}

int b200_marshal_counters(int64_t* faults, int64_t* mprotects, int64_t* hash_bytes, int64_t* mirror_bytes) {
    long f = 0, m = 0, h = 0;
    lilac::marshal::debug_counters(&f, &m, &h);
    if (faults) *faults = f;
    if (mprotects) *mprotects = m;
    if (hash_bytes) *hash_bytes = h;
    if (mirror_bytes) *mirror_bytes = b200::mirror_bytes();
    return 0;
}

int64_t b200_dma_visible_regions(void) { return lilac::marshal::dma_visible_regions(); }

void b200_stats_reset(void) {
    for (HarnessStats* h : all_harness_stats()) {
        std::string name = h->name;
        *h = HarnessStats{};
        h->name = name;
    }
}

}  // extern "C"

namespace b200 {

bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("LILAC_B200_PDL");
        return !(e && std::strcmp(e, "0") == 0);
    }();
    return on;
}

}  // namespace b200
