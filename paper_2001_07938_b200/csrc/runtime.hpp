#pragma once
// runtime.hpp — process-wide device context, error boundary and counters of
// the B200 harness library (host side).

#include "b200.hpp"

#include <chrono>
#include <cstdio>
#include <functional>
#include <memory>
#include <string>
#include <vector>

namespace b200 {

using lilac::marshal::MarshalObject;
using lilac::marshal::MarshalObjectBase;
using lilac::marshal::Strategy;

// Out type of the input/output transfer classes (B200Read / B200Write): a
// device allocation plus the bytes this binding has moved.
struct DevArray {
    DevBuf buf;
    // An input served from a device mirror borrows the mirror's (immutable)
    // buffer instead of copying it; the reference keeps it alive.
    std::shared_ptr<const DevBuf> lent;
    const char* view = nullptr;
    std::int64_t h2d = 0;
    std::int64_t d2h = 0;
    std::int64_t d2d = 0;  // bytes served from a device mirror instead of the host
    std::int64_t lazy = 0;  // write-back bytes left on the device (lazy mode)

    // the device bytes of an input binding
    template <typename T>
    const T* data() const { return lent ? reinterpret_cast<const T*>(view) : buf.as<const T>(); }
    void release() {
        lent.reset();
        view = nullptr;
        buf.release();
    }
};

struct HarnessStats {
    std::string name;
    std::int64_t calls = 0;
    double t_total_ms = 0, t_poll_ms = 0, t_kernel_ms = 0, t_writeback_ms = 0;
    std::int64_t bytes_h2d = 0, bytes_d2h = 0, bytes_d2d = 0;
};

struct Runtime {
    bool inited = false;
    int device = -1;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev_k0 = nullptr, ev_k1 = nullptr;
    // scratch: partials for deterministic reductions, ticket, flags
    DevBuf partials, scalars, flags;
    CsrKernel kernel = CsrKernel::Auto;
    Strategy strategy = Strategy::Hybrid;
    bool exact_blas = false;
    bool lazy_writeback = false;  // LILAC_B200_WRITEBACK=lazy / b200_set_writeback
    std::size_t stage_bytes = std::size_t(256) << 20;  // chunk for narrowing uploads
    DevBuf stage;
    // pinned, device-mapped scalar result slot (dot results; HostSlot)
    double* h_slot_val = nullptr;
    unsigned* h_slot_flag = nullptr;
    HostSlot dslot;  // device pointers of the same
    unsigned slot_seq = 0;

    HostSlot next_slot() {
        HostSlot s = dslot;
        s.seq = ++slot_seq;
        return s;
    }

    unsigned int* d_ticket() const { return scalars.as<unsigned int>(); }
    double* d_result() const { return reinterpret_cast<double*>(scalars.as<char>() + 64); }
    unsigned long long* d_umax() const { return reinterpret_cast<unsigned long long*>(flags.as<char>()); }
    int* d_bad() const { return reinterpret_cast<int*>(flags.as<char>() + 8); }
};

Runtime& rt();
// Multi-device harness path (LILAC_B200_NGPUS = k >= 2): every device but
// the primary gets its own runtime (stream, scratch, result slot) carrying the
// primary's settings. While a DeviceScope is alive, this thread's rt() is the
// scope device's runtime and that device is current, so every upload / build /
// launch helper works on it unchanged.
Runtime& device_runtime(int device);
struct DeviceScope {
    Runtime* prev;
    int prev_dev = 0;
    explicit DeviceScope(int device);
    ~DeviceScope();
    DeviceScope(const DeviceScope&) = delete;
    DeviceScope& operator=(const DeviceScope&) = delete;
};
// LILAC_B200_NGPUS (>= 1; read once) and the device of shard g (g mod visible)
int harness_ngpus();
int shard_device(int g);
void ensure_init();  // lazy first-call init + atexit teardown
// Spin until the kernel that was given HostSlot seq `seq` posted its value
// (checking the stream for errors now and then); returns the value.
double wait_host_slot(unsigned seq);
void shutdown();

// Region stats registry (harness objects + their transfer counters).
void register_region(MarshalObjectBase* obj, const std::int64_t* h2d, const std::int64_t* d2h,
                     const std::int64_t* d2d);
HarnessStats& harness_stats(const char* name);
std::vector<HarnessStats*> all_harness_stats();
struct RegionEntry {
    MarshalObjectBase* obj;
    const std::int64_t* h2d;
    const std::int64_t* d2h;
    const std::int64_t* d2d;
};
const std::vector<RegionEntry>& all_regions();

// ---- error boundary -----------------------------------------------------------

void set_error(const char* code, const std::string& msg);
const char* current_error();
void clear_error();
int error_mode();

// Runs f; on exception records it and aborts (default) or returns -1.
template <typename F>
int boundary(const char* fn, F&& f) {
    try {
        clear_error();
        f();
        return 0;
    } catch (const Error& e) {
        set_error(lilac::marshal::errc_name(e.code()), std::string(fn) + ": " + e.what());
    } catch (const std::exception& e) {
        set_error("HookFailure", std::string(fn) + ": " + e.what());
    }
    if (error_mode() == 0) {
        std::fprintf(stderr, "lilac-b200: %s\n", current_error());
        std::fflush(stderr);
        std::abort();
    }
    return -1;
}

// ---- transfer helpers (stream-ordered, synchronous w.r.t. the host) --------------

// Before any DMA read of caller memory: lazy bytes there must be real first
// (DMA does not fault on PROT_NONE pages).
inline void host_in(const void* p, std::size_t bytes) { lilac::marshal::materialize_range(p, bytes); }

// upload: H2D, or D2D from a valid device mirror of the same host bytes.
void upload(DevArray& d, const void* host, std::size_t bytes);
// download: D2H write-back; then publishes a device mirror of the host region
// (the mirror takes d's buffer; d gets a fresh one from the pool).
// Lazy mode (regions >= 8 KiB): no D2H — the mirror is published with every
// page the region touches PROT_NONE, and its bytes land on the first touch of
// any of those pages (a neighbour on an unaligned region's edge page included).
void download(void* host, DevArray& d, std::size_t bytes, DevArray& counter);
// D2H of `bytes` into host memory on stream s, returning once the bytes landed;
// pageable destinations go through pinned chunks with parallel host copies
// (copy_engine.cpp).
void d2h_copy(void* host, const void* dev, std::size_t bytes, cudaStream_t s);

// Device mirrors (the coherence layer of SURVEY §8(f)1): after a write-back the
// device holds the exact bytes of the host region; the region is guarded like
// a Hybrid marshal region, and while no host write touched it any later upload
// of (a sub-range of) it is served device-to-device. LILAC_B200_MIRRORS=0 off.
bool mirror_fetch(DevArray& d, const void* host, std::size_t bytes);
void mirror_publish(const void* host, std::size_t bytes, DevBuf& src);
// *eager: bytes written back at once (0: all deferred)
bool mirror_publish_lazy(const void* host, std::size_t bytes, DevBuf& src, std::size_t* eager = nullptr);
void lazy_bytes(std::int64_t* deferred, std::int64_t* filled);
void mirrors_clear();                                    // lazy bytes filled first
void mirrors_forget(const void* host, std::size_t bytes);  // the caller frees it: no fill
void mirrors_drop_all();
std::int64_t mirror_bytes();

// Resident CSR / JDS uploads shared by the harnesses and the device API.
struct CsrUpload {
    DevBuf row_ptr, col, val;
    CsrDev dev;
    std::int64_t bytes_moved = 0;
};
// Upload + validate row_ptr for `rows` (nnz = row_ptr[rows]).
void upload_row_ptr(DevBuf& buf, const std::int64_t* row_ptr, std::int64_t rows, std::int64_t nnz,
                    std::int64_t* max_row, bool* monotone);
// Upload col_ind[0..nnz) narrowing to int32 when possible; returns cols.
std::int64_t upload_col_ind(DevBuf& buf, const std::int64_t* col_ind, std::int64_t nnz, bool* col32);

using Clock = std::chrono::steady_clock;

// Host-side phase accumulators (ns), read by b200_host_profile().
enum HostPhase { kPhMirrorFetch, kPhMirrorPoll, kPhD2D, kPhH2D, kPhD2H, kPhPublish, kPhPublishGuard,
                 kPhAcquire, kPhLaunch, kPhPick, kPhAcquireOut, kPhSteal, kPhMalloc, kPhCount };
// Phase timers and per-call kernel events cost clock reads and CUDA API calls
// on every harness call: off unless LILAC_B200_PROFILE=1 / b200_set_profiling.
extern bool g_profile;
void host_phase_add(int ph, std::int64_t ns);
struct PhaseTimer {
    int ph;
    Clock::time_point t0;
    explicit PhaseTimer(int p) : ph(g_profile ? p : -1) {
        if (ph >= 0) t0 = Clock::now();
    }
    void stop() {
        if (ph < 0) return;
        host_phase_add(ph, std::chrono::duration_cast<std::chrono::nanoseconds>(Clock::now() - t0).count());
        ph = -1;
    }
    ~PhaseTimer() { stop(); }
};
inline double ms_since(Clock::time_point t0) {
    return std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
}

}  // namespace b200
