// marshal.cpp — change detection, registry and page guards for the B200
// marshaling runtime (include/lilac/marshal.hpp).
//
// Contract followed: reference include/lilac/marshal.hpp:108-240 (state
// machine) and src/marshal.cpp:123-243 (strategies, fault plumbing, registry).
// The guard table is per page range; a page stays write-protected while at
// least one clean region covers it (the reference unprotects unconditionally
// in drop_guard, which can leave a clean neighbour unguarded).

#include "lilac/marshal.hpp"

#include <algorithm>
#include <atomic>
#include <cerrno>
#include <cstdlib>
#include <cstring>
#include <cstdio>
#include <mutex>
#include <vector>

#include <signal.h>
#include <sys/mman.h>
#include <fcntl.h>
#include <unistd.h>
#include <sys/syscall.h>

namespace lilac::marshal {
inline namespace b200 {

const char* errc_name(Errc c) {
    switch (c) {
    case Errc::OutOfBounds: return "OutOfBounds";
    case Errc::HookFailure: return "HookFailure";
    case Errc::ProtectionUnsupported: return "ProtectionUnsupported";
    case Errc::DataError: return "DataError";
    case Errc::DeviceError: return "DeviceError";
    }
    return "?";
}

Error::Error(Errc code, const std::string& message)
    : std::runtime_error(std::string(errc_name(code)) + ": " + message), code_(code) {}

namespace {

struct Guard {
    std::uintptr_t lo, hi;
    TrackedRegion* region;
};

// Mutated in normal context under g_mu; the fault handler only reads it
// (single-threaded acquire contract).
std::vector<Guard> g_guards;
std::vector<TrackedRegion*> g_tracked;  // every region with a live snapshot
std::vector<DeferredRange*> g_deferred;  // lazy ranges (active or awaiting unlink)
std::mutex g_mu;
std::size_t g_page = 0;
volatile long g_stat_faults = 0, g_stat_mprotect = 0, g_stat_hash_bytes = 0;
volatile long g_def_n = 0, g_def_fault_fills = 0, g_def_explicit_fills = 0, g_def_cancelled = 0;
struct sigaction g_prev;
bool g_prev_valid = false;
bool (*g_dma_probe)(const void*) = nullptr;  // set_dma_probe
bool g_dma_always = false;
long g_dma_regions = 0;

// mprotect(RW) over [lo, hi). A stale range over memory the caller freed may
// contain unmapped holes (a trimmed heap); mprotect then fails as a whole at
// the first hole and leaves the pages after it protected with no guard left to
// claim their faults — so fall back to page by page. Returns whether any page
// is mapped. Async-signal-safe.
bool open_pages(std::uintptr_t lo, std::uintptr_t hi) {
    if (hi <= lo) return true;
    if (mprotect(reinterpret_cast<void*>(lo), hi - lo, PROT_READ | PROT_WRITE) == 0) return true;
    bool any = false;
    for (std::uintptr_t p = lo; p < hi; p += g_page)
        any |= mprotect(reinterpret_cast<void*>(p), g_page, PROT_READ | PROT_WRITE) == 0;
    return any;
}

// Close the parts of [lo, hi) covered by an active lazy range (PROT_NONE).
void apply_deferred(std::uintptr_t lo, std::uintptr_t hi) {
    for (std::size_t i = 0; i < g_deferred.size(); ++i) {
        const DeferredRange* d = g_deferred[i];
        if (!d->active) continue;
        const std::uintptr_t a = lo > d->lo ? lo : d->lo, b = hi < d->hi ? hi : d->hi;
        if (a < b) mprotect(reinterpret_cast<void*>(a), b - a, PROT_NONE);
    }
}

// Recompute the protection of [lo, hi): PROT_NONE under an active lazy range,
// else PROT_READ under a clean guard, else read-write. Lock-free (the fault
// handler calls it); callers in normal context hold g_mu.
void reapply(std::uintptr_t lo, std::uintptr_t hi) {
    if (hi <= lo) return;
    g_stat_mprotect = g_stat_mprotect + 1;
    open_pages(lo, hi);
    for (const Guard& g : g_guards) {
        if (g.region->dirty) continue;
        const std::uintptr_t a = lo > g.lo ? lo : g.lo, b = hi < g.hi ? hi : g.hi;
        if (a < b) mprotect(reinterpret_cast<void*>(a), b - a, PROT_READ);
    }
    apply_deferred(lo, hi);
}

// Materialise one lazy range: open its pages, let the owner write the bytes,
// then restore the guards' protections over them.
const bool g_trace = std::getenv("LILAC_MARSHAL_TRACE") != nullptr;

void trace(const char* what, std::uintptr_t a, std::uintptr_t b) {
    if (!g_trace) return;
    char buf[128];
    const int n = std::snprintf(buf, sizeof buf, "[marshal] %s %#lx..%#lx\n", what, (unsigned long)a, (unsigned long)b);
    if (n > 0) (void)!write(2, buf, static_cast<std::size_t>(n));
}

// Can the process read the byte at a? (A write(2) of it into a pipe fails
// with EFAULT instead of faulting.) Normal context only.
bool page_readable(std::uintptr_t a) {
    static int fds[2] = {-1, -1};
    if (fds[0] < 0 && pipe2(fds, O_NONBLOCK | O_CLOEXEC) != 0) return false;
    if (write(fds[1], reinterpret_cast<const void*>(a), 1) != 1) return false;
    char c;
    (void)!read(fds[0], &c, 1);
    return true;
}

void fill_one(DeferredRange& d, bool from_fault) {
    trace(from_fault ? "fill(fault)" : "fill", d.lo, d.hi);
    d.active = false;
    // A range is ours only while its pages are still PROT_NONE: memory freed
    // and mapped again (readable) must not receive the old bytes.
    if (!from_fault && (page_readable(d.lo) || page_readable(d.hi - 1))) {
        trace("stale (remapped)", d.lo, d.hi);
        return;
    }
    if (mprotect(reinterpret_cast<void*>(d.lo), d.hi - d.lo, PROT_READ | PROT_WRITE) != 0) {
        trace("stale (unmapped)", d.lo, d.hi);
        return;  // the memory is gone: nothing to fill
    }
    if (d.fill) d.fill(&d);
    trace("filled", d.lo, d.hi);
    if (from_fault)
        g_def_fault_fills = g_def_fault_fills + 1;
    else
        g_def_explicit_fills = g_def_explicit_fills + 1;
    reapply(d.lo, d.hi);
}

bool page_deferred(std::uintptr_t page) {
    for (const DeferredRange* d : g_deferred)
        if (d->active && d->lo <= page && page < d->hi) return true;
    return false;
}

// Faults from several threads (a host loop plus worker threads reading
// caller arrays) are handled one at a time: the guard walk and a lazy fill are
// not re-entrant. The owner's tid makes a nested fault on the same thread (a
// fill that itself touches a protected page) proceed instead of deadlocking.
// A thread that waited may find its page already filled; it then takes the
// guard path, which can only over-report a write (dirty), never miss one.
std::atomic<long> g_fault_owner{0};

struct FaultLock {
    bool held = false;
    FaultLock() {
        const long me = static_cast<long>(syscall(SYS_gettid));
        if (g_fault_owner.load(std::memory_order_acquire) == me) return;  // nested
        long expect = 0;
        while (!g_fault_owner.compare_exchange_weak(expect, me, std::memory_order_acq_rel)) {
            expect = 0;
            __builtin_ia32_pause();
        }
        held = true;
    }
    void release() {
        if (held) g_fault_owner.store(0, std::memory_order_release);
        held = false;
    }
    ~FaultLock() { release(); }
};

void on_fault(int sig, siginfo_t* si, void* uctx) {
    FaultLock lock;
    const auto addr = reinterpret_cast<std::uintptr_t>(si->si_addr);
    trace("fault", addr, static_cast<std::uintptr_t>(si->si_code));
    const std::uintptr_t page = addr & ~(static_cast<std::uintptr_t>(g_page) - 1);
    // only protection faults on mapped pages can be ours (an access to
    // unmapped memory inside a stale range must crash, not loop)
    if (si->si_code != SEGV_ACCERR) goto not_ours;
    {
    // a touch of lazy bytes: materialise them; a write re-faults on the
    // restored guard and is recorded below
    bool filled = false;
    for (std::size_t i = 0; i < g_deferred.size(); ++i) {
        DeferredRange* d = g_deferred[i];
        if (d->active && page < d->hi && page + g_page > d->lo) {
            fill_one(*d, true);
            filled = true;
        }
    }
    if (filled) return;
    bool hit = false;
    for (const Guard& g : g_guards) {
        if (page < g.hi && page + g_page > g.lo) {
            g.region->dirty = true;
            hit = true;
        }
    }
    if (hit) {
        g_stat_faults = g_stat_faults + 1;
        // A region is dirty after its first trapped write: open its whole
        // guard range now (one fault per region per clean cycle instead of one
        // per page), then re-close pages still covered by a clean region.
        for (const Guard& g : g_guards)
            if (page < g.hi && page + g_page > g.lo) open_pages(g.lo, g.hi);
        // the faulting page itself must end writable, or re-executing loops
        if (mprotect(reinterpret_cast<void*>(page), g_page, PROT_READ | PROT_WRITE) != 0) goto not_ours;
        for (const Guard& g : g_guards) {
            if (g.region->dirty) continue;
            for (const Guard& h : g_guards) {
                if (!h.region->dirty || !(page < h.hi && page + g_page > h.lo)) continue;
                const std::uintptr_t a = g.lo > h.lo ? g.lo : h.lo, b = g.hi < h.hi ? g.hi : h.hi;
                if (a < b) mprotect(reinterpret_cast<void*>(a), b - a, PROT_READ);
            }
        }
        for (const Guard& g : g_guards)
            if (page < g.hi && page + g_page > g.lo) apply_deferred(g.lo, g.hi);
        return;
    }
    }
not_ours:
    trace("not ours", addr, static_cast<std::uintptr_t>(g_guards.size()));
    lock.release();  // the previous handler may not return here
    // Not ours: hand the fault to whoever had SIGSEGV before us.
    if (g_prev_valid) {
        if (g_prev.sa_flags & SA_SIGINFO) {
            if (g_prev.sa_sigaction) {
                g_prev.sa_sigaction(sig, si, uctx);
                return;
            }
        } else if (g_prev.sa_handler != SIG_DFL && g_prev.sa_handler != SIG_IGN) {
            g_prev.sa_handler(sig);
            return;
        }
    }
    signal(SIGSEGV, SIG_DFL);  // re-executing the access now terminates normally
}

void ensure_handler() {
    struct sigaction cur;
    if (sigaction(SIGSEGV, nullptr, &cur) == 0 && (cur.sa_flags & SA_SIGINFO) &&
        cur.sa_sigaction == on_fault)
        return;
    struct sigaction sa;
    std::memset(&sa, 0, sizeof sa);
    sa.sa_sigaction = on_fault;
    sa.sa_flags = SA_SIGINFO | SA_ONSTACK;
    sigemptyset(&sa.sa_mask);
    struct sigaction prev;
    if (sigaction(SIGSEGV, &sa, &prev) != 0)
        throw Error(Errc::ProtectionUnsupported,
                    std::string("cannot install SIGSEGV handler: ") + std::strerror(errno));
    g_prev = prev;
    g_prev_valid = true;
}

std::uintptr_t floor_page(std::uintptr_t a) { return a & ~(static_cast<std::uintptr_t>(page_size()) - 1); }
std::uintptr_t ceil_page(std::uintptr_t a) { return floor_page(a + page_size() - 1); }

void protect(std::uintptr_t lo, std::uintptr_t hi) {
    g_stat_mprotect = g_stat_mprotect + 1;
    if (hi > lo && mprotect(reinterpret_cast<void*>(lo), hi - lo, PROT_READ) != 0) {
        const int err = errno;
        open_pages(lo, hi);  // undo a partial protection: no guard will own it
        throw Error(Errc::ProtectionUnsupported, std::string("mprotect failed: ") + std::strerror(err));
    }
}

// Unprotect [lo,hi), then re-protect the parts still covered by a clean
// guarded region other than `except`. Caller holds g_mu.
void release_pages(std::uintptr_t lo, std::uintptr_t hi, const TrackedRegion* except) {
    if (hi <= lo) return;
    g_stat_mprotect = g_stat_mprotect + 1;
    open_pages(lo, hi);
    for (const Guard& g : g_guards) {
        if (g.region == except || g.region->dirty) continue;
        std::uintptr_t a = std::max(lo, g.lo), b = std::min(hi, g.hi);
        if (a < b) mprotect(reinterpret_cast<void*>(a), b - a, PROT_READ);
    }
    apply_deferred(lo, hi);
}

void add_guard(TrackedRegion& r, std::uintptr_t lo, std::uintptr_t hi) {
    ensure_handler();
    protect(lo, hi);
    apply_deferred(lo, hi);
    if (!r.guarded) {
        g_guards.push_back({lo, hi, &r});
        r.guarded = true;
        r.guard_lo = lo;
        r.guard_hi = hi;
    }
}

void track(TrackedRegion& r) {
    if (std::find(g_tracked.begin(), g_tracked.end(), &r) == g_tracked.end()) g_tracked.push_back(&r);
}

std::uint64_t version_of(const TrackedRegion& r) {
    if (!r.ref.version)
        throw Error(Errc::DataError, "exact-version strategy needs a version word behind the region");
    return *r.ref.version;
}

// Hybrid edge hashes: the partial pages at each end that cannot be protected.
void edge_spans(const TrackedRegion& r, std::uintptr_t& in_lo, std::uintptr_t& in_hi) {
    const auto base = reinterpret_cast<std::uintptr_t>(r.ref.base);
    const std::uintptr_t end = base + r.ref.bytes;
    in_lo = ceil_page(base);
    in_hi = floor_page(end);
    if (in_hi <= in_lo) in_lo = in_hi = end;  // no whole page inside: hash everything
}

// Hybrid edge snapshot: head bytes then tail bytes.
std::size_t head_len(const TrackedRegion& r) {
    const auto base = reinterpret_cast<std::uintptr_t>(r.ref.base);
    return r.hash_head_end > base ? r.hash_head_end - base : 0;
}

std::size_t tail_len(const TrackedRegion& r) {
    const auto end = reinterpret_cast<std::uintptr_t>(r.ref.base) + r.ref.bytes;
    return r.hash_tail_begin < end ? end - r.hash_tail_begin : 0;
}

void snapshot_edges(TrackedRegion& r) {
    const std::size_t h = head_len(r), t = tail_len(r);
    r.edges.resize(h + t);
    if (h) std::memcpy(r.edges.data(), r.ref.base, h);
    if (t) std::memcpy(r.edges.data() + h, reinterpret_cast<const void*>(r.hash_tail_begin), t);
    g_stat_hash_bytes = g_stat_hash_bytes + static_cast<long>(h + t);
}

bool edges_changed(const TrackedRegion& r) {
    const std::size_t h = head_len(r), t = tail_len(r);
    g_stat_hash_bytes = g_stat_hash_bytes + static_cast<long>(h + t);
    if (r.edges.size() != h + t) return true;
    if (h && std::memcmp(r.edges.data(), r.ref.base, h) != 0) return true;
    return t && std::memcmp(r.edges.data() + h, reinterpret_cast<const void*>(r.hash_tail_begin), t) != 0;
}

// Is [lo, hi) inside one active lazy range?
// The two snapshot strategies keep one 64-bit stamp per clean cycle: the
// FNV-1a hash of the bytes (Checksum) or the interpreter buffer's write
// version (ExactVersion); `snapshot_of` is what poll_dirty compares against.
std::uint64_t snapshot_stamp(const TrackedRegion& r) {
    return r.strategy == Strategy::Checksum ? fnv1a(r.ref.base, r.ref.bytes) : version_of(r);
}

std::uint64_t& snapshot_of(TrackedRegion& r) {
    return r.strategy == Strategy::Checksum ? r.last_checksum : r.last_version;
}

// Naive / Checksum / ExactVersion: record the stamp (Naive: never clean).
// False for the page-guard strategies.
bool snapshot_clean(TrackedRegion& r) {
    switch (r.strategy) {
    case Strategy::Naive:
        r.dirty = true;
        return true;
    case Strategy::Checksum:
    case Strategy::ExactVersion:
        snapshot_of(r) = snapshot_stamp(r);
        r.dirty = false;
        return true;
    default:
        return false;
    }
}

bool covered_by_deferred(std::uintptr_t lo, std::uintptr_t hi) {
    for (const DeferredRange* d : g_deferred)
        if (d->active && d->lo <= lo && hi <= d->hi) return true;
    return false;
}

}  // namespace

namespace {
// The strategy names of the LILAC_MARSHAL_STRATEGY setting, one table for
// both directions.
struct StrategyName {
    Strategy s;
    const char* name;
};
constexpr StrategyName kStrategyNames[] = {{Strategy::PageProtect, "pageprotect"},
                                           {Strategy::Checksum, "checksum"},
                                           {Strategy::ExactVersion, "exact"},
                                           {Strategy::Naive, "naive"},
                                           {Strategy::Hybrid, "hybrid"}};
}  // namespace

const char* strategy_name(Strategy s) {
    for (const StrategyName& e : kStrategyNames)
        if (e.s == s) return e.name;
    return "?";
}

Strategy parse_strategy(const std::string& n) {
    std::string known;
    for (const StrategyName& e : kStrategyNames) {
        if (n == e.name) return e.s;
        known += known.empty() ? e.name : std::string(", ") + e.name;
    }
    throw Error(Errc::DataError, "marshal strategy '" + n + "' is not one of: " + known);
}

Strategy default_strategy(Strategy fallback) {
    const char* env = std::getenv("LILAC_MARSHAL_STRATEGY");
    return (env && *env) ? parse_strategy(env) : fallback;
}

std::uint64_t fnv1a(const void* data, std::size_t size) {
    const auto* p = static_cast<const unsigned char*>(data);
    std::uint64_t h = 0xcbf29ce484222325ULL;
    for (std::size_t i = 0; i < size; ++i) h = (h ^ p[i]) * 0x100000001b3ULL;
    return h;
}

std::size_t page_size() {
    if (g_page == 0) g_page = static_cast<std::size_t>(sysconf(_SC_PAGESIZE));
    return g_page;
}

void mark_clean(TrackedRegion& r) {
    if ((r.strategy == Strategy::PageProtect || r.strategy == Strategy::Hybrid) && g_dma_probe && r.ref.bytes) {
        const bool v = g_dma_probe(r.ref.base);
        if (v && !r.dma_visible) g_dma_regions = g_dma_regions + 1;
        r.dma_visible = v;
    }
    if (snapshot_clean(r)) return;  // the snapshot strategies (no page guard)
    switch (r.strategy) {
    case Strategy::PageProtect: {
        if (r.ref.bytes == 0) {
            r.dirty = false;
            return;
        }
        const auto base = reinterpret_cast<std::uintptr_t>(r.ref.base);
        if (base % page_size() != 0)
            throw Error(Errc::ProtectionUnsupported, "page protection needs a page-aligned region base");
        std::lock_guard<std::mutex> lk(g_mu);
        track(r);
        r.dirty = false;  // clear first: a racing fault must win
        add_guard(r, base, ceil_page(base + r.ref.bytes));
        return;
    }
    case Strategy::Hybrid: {
        if (r.ref.bytes == 0) {
            r.dirty = false;
            return;
        }
        std::uintptr_t in_lo, in_hi;
        edge_spans(r, in_lo, in_hi);
        const auto base = reinterpret_cast<std::uintptr_t>(r.ref.base);
        const std::uintptr_t end = base + r.ref.bytes;
        std::lock_guard<std::mutex> lk(g_mu);
        track(r);
        r.dirty = false;
        // edge pages that are lazy are guarded whole: hashing them would
        // materialise them (a foreign write on them only costs a refresh)
        std::uintptr_t g_lo = in_lo, g_hi = in_hi;
        r.hash_head_end = in_lo;
        r.hash_tail_begin = in_hi;
        if (!g_deferred.empty()) {
            if (in_hi <= in_lo) {  // no whole page inside: all or nothing
                bool all = true;
                for (std::uintptr_t pg = floor_page(base); pg < end && all; pg += page_size()) all = page_deferred(pg);
                if (all) {
                    g_lo = floor_page(base);
                    g_hi = ceil_page(end);
                    r.hash_head_end = base;
                    r.hash_tail_begin = end;
                }
            } else {
                if (base < in_lo && page_deferred(floor_page(base))) {
                    g_lo = floor_page(base);
                    r.hash_head_end = base;
                }
                if (in_hi < end && page_deferred(in_hi)) {
                    g_hi = ceil_page(end);
                    r.hash_tail_begin = end;
                }
            }
        }
        if (g_hi > g_lo) add_guard(r, g_lo, g_hi);
        snapshot_edges(r);
        return;
    }
    }
}

bool page_shared(std::uintptr_t page, std::uintptr_t self_lo, std::uintptr_t self_hi) {
    const std::uintptr_t pe = page + page_size();
    // the parts of the page outside our bytes
    const std::uintptr_t a0 = page, a1 = std::min(pe, std::max(page, self_lo));
    const std::uintptr_t b0 = std::max(page, std::min(pe, self_hi)), b1 = pe;
    auto hits = [&](std::uintptr_t lo, std::uintptr_t hi) {
        return (a0 < a1 && lo < a1 && a0 < hi) || (b0 < b1 && lo < b1 && b0 < hi);
    };
    std::lock_guard<std::mutex> lk(g_mu);
    for (const TrackedRegion* r : g_tracked) {
        const auto lo = reinterpret_cast<std::uintptr_t>(r->ref.base);
        if (r->ref.bytes && hits(lo, lo + r->ref.bytes)) return true;
    }
    for (const DeferredRange* d : g_deferred)
        if (d->active && hits(d->content_lo, d->content_hi)) return true;
    return false;
}

void set_dma_probe(bool (*probe)(const void*)) { g_dma_probe = probe; }
void set_dma_always_dirty(bool on) { g_dma_always = on; }
long dma_visible_regions() { return g_dma_regions; }

bool poll_dirty(TrackedRegion& r) {
    if (r.dma_visible && g_dma_always &&
        (r.strategy == Strategy::PageProtect || r.strategy == Strategy::Hybrid))
        return true;  // a DMA / device write would not fault: do not trust the guard
    // a fault already recorded a write, or nothing to compare
    if (r.dirty || r.ref.bytes == 0) return r.dirty || r.strategy == Strategy::Naive;
    if (r.strategy == Strategy::Naive) return r.dirty = true;
    if (r.strategy == Strategy::PageProtect) return false;  // clean until a store faults
    if (r.strategy == Strategy::Hybrid) return r.dirty = edges_changed(r);
    return r.dirty = snapshot_stamp(r) != snapshot_of(r);  // Checksum / ExactVersion
}

void drop_guard(TrackedRegion& r) {
    std::lock_guard<std::mutex> lk(g_mu);
    g_tracked.erase(std::remove(g_tracked.begin(), g_tracked.end(), &r), g_tracked.end());
    if (!r.guarded) return;
    g_guards.erase(std::remove_if(g_guards.begin(), g_guards.end(),
                                  [&](const Guard& g) { return g.region == &r; }),
                   g_guards.end());
    release_pages(r.guard_lo, r.guard_hi, &r);
    r.guarded = false;
    r.guard_lo = r.guard_hi = 0;
}

void debug_counters(long* faults, long* mprotects, long* hash_bytes) {
    *faults = g_stat_faults;
    *mprotects = g_stat_mprotect;
    *hash_bytes = g_stat_hash_bytes;
}

void note_host_write(const void* base, std::size_t bytes) {
    if (bytes == 0) return;
    const auto lo = reinterpret_cast<std::uintptr_t>(base);
    const std::uintptr_t hi = lo + bytes;
    std::lock_guard<std::mutex> lk(g_mu);
    for (TrackedRegion* r : g_tracked) {
        const auto rlo = reinterpret_cast<std::uintptr_t>(r->ref.base);
        if (rlo < hi && lo < rlo + r->ref.bytes) r->dirty = true;
    }
    // open the pages for the incoming write (DMA never faults; a CPU copy
    // would); lazy pages stay closed
    const std::uintptr_t plo = floor_page(lo), phi = ceil_page(hi);
    bool guarded = false;
    for (const Guard& g : g_guards) {
        if (g.lo < phi && plo < g.hi) {
            g.region->dirty = true;
            guarded = true;
        }
    }
    if (guarded && !covered_by_deferred(plo, phi)) {
        g_stat_mprotect = g_stat_mprotect + 1;
        open_pages(plo, phi);
        apply_deferred(plo, phi);
    }
}

void supersede_range(const void* base, std::size_t bytes) {
    if (g_deferred.empty() || bytes == 0) return;
    const auto lo = reinterpret_cast<std::uintptr_t>(base);
    const std::uintptr_t hi = lo + bytes;
    std::lock_guard<std::mutex> lk(g_mu);
    for (DeferredRange* d : g_deferred) {
        if (!d->active || !(d->lo < hi && lo < d->hi)) continue;
        if (lo <= d->content_lo && d->content_hi <= hi) {
            d->active = false;
            g_def_cancelled = g_def_cancelled + 1;
            reapply(d->lo, d->hi);
        } else {
            fill_one(*d, false);
        }
    }
}

bool reclean_covered(TrackedRegion& r) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!r.guarded || !covered_by_deferred(r.guard_lo, r.guard_hi)) return false;
    if (r.strategy == Strategy::Hybrid) {
        if (head_len(r) || tail_len(r)) return false;  // has hashed edges: full mark_clean
    } else if (r.strategy != Strategy::PageProtect) {
        return false;
    }
    track(r);
    r.dirty = false;
    return true;
}

// ---- lazy ranges -------------------------------------------------------------------

void defer_range(DeferredRange& d) {
    if (d.hi <= d.lo) return;
    std::lock_guard<std::mutex> lk(g_mu);
    ensure_handler();
    if (!d.linked) {
        g_deferred.push_back(&d);
        d.linked = true;
    }
    g_stat_mprotect = g_stat_mprotect + 1;
    if (mprotect(reinterpret_cast<void*>(d.lo), d.hi - d.lo, PROT_NONE) != 0) {
        reapply(d.lo, d.hi);
        throw Error(Errc::ProtectionUnsupported, std::string("mprotect failed: ") + std::strerror(errno));
    }
    d.active = true;
    g_def_n = g_def_n + 1;
}

void materialize_range(const void* base, std::size_t bytes) {
    if (g_deferred.empty() || bytes == 0) return;
    const auto lo = reinterpret_cast<std::uintptr_t>(base);
    const std::uintptr_t hi = lo + bytes;
    std::lock_guard<std::mutex> lk(g_mu);
    for (DeferredRange* d : g_deferred)
        if (d->active && d->lo < hi && lo < d->hi) fill_one(*d, false);
}

void materialize_all() {
    std::lock_guard<std::mutex> lk(g_mu);
    for (DeferredRange* d : g_deferred)
        if (d->active) fill_one(*d, false);
}

void retire_deferred(DeferredRange& d, bool fill) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (d.active) {
        if (fill) {
            fill_one(d, false);
        } else {
            d.active = false;
            reapply(d.lo, d.hi);
        }
    }
    if (d.linked) {
        g_deferred.erase(std::remove(g_deferred.begin(), g_deferred.end(), &d), g_deferred.end());
        d.linked = false;
    }
}

bool any_deferred() {
    for (const DeferredRange* d : g_deferred)
        if (d->active) return true;
    return false;
}

void deferred_counters(long* deferred, long* fault_fills, long* explicit_fills, long* cancelled) {
    if (deferred) *deferred = g_def_n;
    if (fault_fills) *fault_fills = g_def_fault_fills;
    if (explicit_fills) *explicit_fills = g_def_explicit_fills;
    if (cancelled) *cancelled = g_def_cancelled;
}

// ---- MarshalObjectBase --------------------------------------------------------

namespace {
// Every constructed marshal object, in construction order (release_all tears
// them down in that order, like the reference's registry).
class ObjectRegistry {
public:
    void add(MarshalObjectBase* o) {
        std::lock_guard<std::mutex> lk(mu_);
        if (std::find(live_.begin(), live_.end(), o) == live_.end()) live_.push_back(o);
    }
    void remove(MarshalObjectBase* o) {
        std::lock_guard<std::mutex> lk(mu_);
        live_.erase(std::remove(live_.begin(), live_.end(), o), live_.end());
    }
    // take (and unregister) every object, or those `pick` selects
    template <typename P>
    std::vector<MarshalObjectBase*> take(P pick) {
        std::lock_guard<std::mutex> lk(mu_);
        std::vector<MarshalObjectBase*> out, keep;
        for (MarshalObjectBase* o : live_) (pick(o) ? out : keep).push_back(o);
        live_.swap(keep);
        return out;
    }

private:
    std::vector<MarshalObjectBase*> live_;
    std::mutex mu_;
};

ObjectRegistry& registry() {
    static ObjectRegistry* r = new ObjectRegistry;  // usable from atexit handlers
    return *r;
}
}  // namespace

MarshalObjectBase::MarshalObjectBase(std::string name, Strategy s)
    : name_(std::move(name)), strategy_(s) {
    if (name_.empty()) name_ = "region@" + std::to_string(reinterpret_cast<std::uintptr_t>(this));
}

MarshalObjectBase::~MarshalObjectBase() = default;

void MarshalObjectBase::set_strategy(Strategy s) {
    if (constructed_) throw Error(Errc::DataError, "cannot change the strategy of a constructed object");
    strategy_ = s;
    fell_back_ = false;
}

void MarshalObjectBase::enroll() { registry().add(this); }

void MarshalObjectBase::unenroll() { registry().remove(this); }

// Snapshot the region as clean. A region the page guard cannot cover (a
// misaligned base under PageProtect, a refused mprotect) is demoted to the
// byte hash for the rest of its life — the reference's ProtectionUnsupported
// rule — and reported through fell_back().
void MarshalObjectBase::clean_with_fallback() {
    if (streaming_) return;
    bool demote = false;
    try {
        mark_clean(region_);
    } catch (const Error& e) {
        if (e.code() != Errc::ProtectionUnsupported) throw;
        demote = true;
    }
    if (!demote) return;
    fell_back_ = true;
    strategy_ = region_.strategy = Strategy::Checksum;
    mark_clean(region_);
}

bool MarshalObjectBase::region_dirty() { return streaming_ || poll_dirty(region_); }

void MarshalObjectBase::note_update_for_streaming(bool was_dirty) {
    if (!adaptive_ || streaming_) return;
    if (!was_dirty) {
        dirty_streak_ = 0;
        return;
    }
    if (++dirty_streak_ >= kStreamAfter && region_.strategy != Strategy::Naive &&
        region_.strategy != Strategy::ExactVersion) {
        // Rewritten on every call: guarding it costs a fault per page per call
        // for no saved transfer. Stop guarding; update unconditionally.
        streaming_ = true;
        drop_guard(region_);
    }
}

void MarshalObjectBase::hook_failed(const char* which, const std::exception& e) const {
    throw Error(Errc::HookFailure, "region '" + name_ + "': the " + which + " hook threw: " + e.what());
}

Diagnostics release_all() {
    Diagnostics d;
    for (MarshalObjectBase* o : registry().take([](MarshalObjectBase*) { return true; })) o->force_release(d);
    return d;
}

Diagnostics forget_range(const void* base, std::size_t bytes) {
    Diagnostics d;
    if (bytes == 0) return d;
    const auto lo = reinterpret_cast<std::uintptr_t>(base);
    const std::uintptr_t hi = lo + bytes;
    const auto hit = registry().take([&](MarshalObjectBase* o) {
        const auto rlo = reinterpret_cast<std::uintptr_t>(o->region_.ref.base);
        return o->constructed_ && rlo < hi && lo < rlo + o->region_.ref.bytes;
    });
    for (MarshalObjectBase* o : hit) o->force_release(d);
    std::lock_guard<std::mutex> lk(g_mu);
    for (DeferredRange* r : g_deferred) {
        if (r->active && r->content_lo < hi && lo < r->content_hi) {
            r->active = false;
            g_def_cancelled = g_def_cancelled + 1;
            reapply(r->lo, r->hi);
        }
    }
    return d;
}

// ---- PageBuffer -----------------------------------------------------------------

// Whole anonymous pages (at least one), so PageProtect can guard the buffer.
PageBuffer::PageBuffer(std::size_t bytes)
    : p_(nullptr), bytes_(bytes), mapped_((bytes + page_size() - 1) / page_size() * page_size()) {
    if (mapped_ == 0) mapped_ = page_size();
    void* p = mmap(nullptr, mapped_, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    if (p == MAP_FAILED)
        throw Error(Errc::DataError, "PageBuffer of " + std::to_string(bytes) + " bytes: " + std::strerror(errno));
    p_ = p;
}

PageBuffer::~PageBuffer() {
    if (p_) munmap(p_, mapped_);
}

}  // namespace b200
}  // namespace lilac::marshal
