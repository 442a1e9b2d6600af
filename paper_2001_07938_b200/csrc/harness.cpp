// harness.cpp — the extern "C" harness entry points of the B200 backend.
//
// Each entry point has exactly the shape the reference's harness generator
// emits (src/harnessgen.cpp:42-133; golden fixtures/gen/cusparse_spmv.gen.cpp):
// a static state record with one marshal object per binding, lazy first-run
// setup with atexit teardown, acquires in binding order, the library call,
// then write_back of every OUTPUT binding. The marshal classes are the B200
// counterparts of the fixture's CudaRead/CudaWrite/LastEntry/ReadableMax
// (fixtures/lilac/cusparse.lilac:6-43), with the fixture's two integer-width
// bugs fixed: LastEntry reads int64 (cusparse.lilac:34 reads int) and the
// device col_ind is narrowed explicitly instead of reinterpreting int64 bytes
// as int (cusparse.lilac:56-57).

#include "lilac_b200.h"
#include "runtime.hpp"
#include "tcsr.hpp"

#include <cstring>
#include <vector>

using namespace b200;

namespace {

// ---- marshal classes -------------------------------------------------------------

// LastEntry (input): out = in[n-1] of an int64 array.
void LastEntry_update(const void* in, std::size_t size, std::int64_t& out) {
    const auto* p = static_cast<const std::int64_t*>(in);
    out = size >= sizeof(std::int64_t) ? p[size / sizeof(std::int64_t) - 1] : 0;
}

// ReadableMax (input): out = 1 + max(in) of an int64 array, 0 when empty
// (the SPEC's empty-max convention, SPEC.md cached_invariant).
void ReadableMax_update(const void* in, std::size_t size, std::int64_t& out) {
    const auto* p = static_cast<const std::int64_t*>(in);
    std::int64_t m = -1;
    for (std::size_t i = 0; i < size / sizeof(std::int64_t); ++i) m = p[i] > m ? p[i] : m;
    out = m + 1;
}

// B200Read (input): resident device copy, refreshed on change.
void B200Read_update(const void* in, std::size_t size, DevArray& out) { upload(out, in, size); }
void B200Read_destruct(const void*, std::size_t, DevArray& out) { out.release(); }

// B200Write (output): device destination, write_back = device->host copy.
void B200Write_construct(const void*, std::size_t size, DevArray& out) { out.buf.ensure(size); }
void B200Write_update(const void* in, std::size_t size, DevArray& out) {
    download(const_cast<void*>(in), out, size, out);
}
void B200Write_destruct(const void*, std::size_t, DevArray& out) { out.buf.release(); }

// B200RowPtr (input): row_ptr[0..rows] resident + validated against nnz.
struct RowPtrDev {
    DevBuf buf;
    std::int64_t max_row = 0;
    bool monotone = true;
    std::int64_t h2d = 0, d2h = 0, d2d = 0;
};

// B200ColInd (input): col_ind[0..nnz) resident, narrowed to int32 when every
// index fits, with cols = 1 + max (ReadableMax) computed in the same pass.
struct ColDev {
    DevBuf buf;
    bool col32 = true;
    std::int64_t cols = 0;
    std::int64_t h2d = 0, d2h = 0, d2d = 0;
};

void ColInd_update(const void* in, std::size_t size, ColDev& out) {
    const std::int64_t nnz = static_cast<std::int64_t>(size / sizeof(std::int64_t));
    out.cols = upload_col_ind(out.buf, static_cast<const std::int64_t*>(in), nnz, &out.col32);
    out.h2d += static_cast<std::int64_t>(size);
}
void ColInd_destruct(const void*, std::size_t, ColDev& out) { out.buf.release(); }

// B200Perm (input, JDS): perm resident + its inverse (a cached invariant) when
// perm is a bijection of [0, rows).
struct PermDev {
    DevBuf perm, inv;
    bool bijective = true;
    std::int64_t h2d = 0, d2h = 0, d2d = 0;
};

void Perm_update(const void* in, std::size_t size, PermDev& out) {
    Runtime& r = rt();
    const std::int64_t rows = static_cast<std::int64_t>(size / sizeof(std::int64_t));
    out.perm.ensure(size);
    out.inv.ensure(size);
    host_in(in, size);
    if (size) B200_CUDA(cudaMemcpyAsync(out.perm.ptr, in, size, cudaMemcpyHostToDevice, r.stream));
    B200_CUDA(cudaMemsetAsync(r.flags.ptr, 0, 16, r.stream));
    launch_invert_perm(out.perm.as<std::int64_t>(), rows, out.inv.as<std::int64_t>(), r.d_bad(), r.stream);
    int bad = 0;
    B200_CUDA(cudaMemcpyAsync(&bad, r.d_bad(), 4, cudaMemcpyDeviceToHost, r.stream));
    B200_CUDA(cudaStreamSynchronize(r.stream));
    if (bad & 1) throw Error(Errc::OutOfBounds, "perm entry outside [0, rows)");
    out.bijective = (bad & 2) == 0;
    out.h2d += static_cast<std::int64_t>(size);
}
void Perm_destruct(const void*, std::size_t, PermDev& out) {
    out.perm.release();
    out.inv.release();
}

template <typename Out>
void enroll_stats(MarshalObject<Out>& m, const char* name) {
    m.set_name(name);
    m.set_strategy(rt().strategy);
    m.set_adaptive(true);
    register_region(&m, &m.out().h2d, &m.out().d2h, &m.out().d2d);
}

template <>
void enroll_stats<std::int64_t>(MarshalObject<std::int64_t>& m, const char* name) {
    m.set_name(name);
    m.set_strategy(rt().strategy);
    m.set_adaptive(true);
    register_region(&m, nullptr, nullptr, nullptr);
}

struct Timer {
    HarnessStats& st;
    Clock::time_point t0 = Clock::now(), t_mark = t0;
    explicit Timer(HarnessStats& s) : st(s) {}
    void acquired() {
        st.t_poll_ms += ms_since(t_mark);
        t_mark = Clock::now();
    }
    void written_back() { st.t_writeback_ms += ms_since(t_mark); }
    ~Timer() {
        st.t_total_ms += ms_since(t0);
        st.calls++;
    }
};

// Brackets the compute launch with events on the harness stream. No sync
// here: the write-back's stream sync completes the events, and
// collect_kernel_time reads them afterwards (one host sync per call).
template <typename F>
void timed_launch(HarnessStats& st, F&& launch) {
    PhaseTimer pt(kPhLaunch);
    Runtime& r = rt();
    if (!g_profile) {
        launch();
        return;
    }
    B200_CUDA(cudaEventRecord(r.ev_k0, r.stream));
    launch();
    B200_CUDA(cudaEventRecord(r.ev_k1, r.stream));
    (void)st;
}

void collect_kernel_time(HarnessStats& st) {
    if (!g_profile) return;
    Runtime& r = rt();
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, r.ev_k0, r.ev_k1) == cudaSuccess)
        st.t_kernel_ms += ms;
    else
        (void)cudaGetLastError();  // not complete (empty write-back): clear the non-sticky status
}

// ---- persistent state: b200_spmv_csr ------------------------------------------------

struct spmv_csr_state {
    MarshalObject<std::int64_t> m_nnz;
    MarshalObject<RowPtrDev> m_row_ptr;
    MarshalObject<ColDev> m_col_ind;
    MarshalObject<DevArray> m_val;
    MarshalObject<DevArray> m_x;
    MarshalObject<DevArray> m_output;
    TcsrOwner tiled;                // derived layouts, rebuilt when the matrix changes
    MergeOwner merge;
    SplitOwner split;
    LrcOwner lrc;
    std::int64_t tiled_stamp = -1;  // sum of matrix update/construct counters it was built at
    CsrKernel tiled_policy = CsrKernel::Auto;
    bool plain_dropped = false;     // col / val device copies freed: a derived layout serves the matrix
    bool first_run_done = false;
};

std::int64_t matrix_stamp(const spmv_csr_state& st) {
    std::int64_t s = 0;
    for (const MarshalObjectBase* m :
         {static_cast<const MarshalObjectBase*>(&st.m_row_ptr), static_cast<const MarshalObjectBase*>(&st.m_col_ind),
          static_cast<const MarshalObjectBase*>(&st.m_val)})
        s += m->counters().n_update + m->counters().n_construct;
    return s;
}

spmv_csr_state& csr_state() {
    static spmv_csr_state* st = new spmv_csr_state;  // outlives atexit teardown
    if (!st->first_run_done) {
        st->first_run_done = true;
        ensure_init();  // BeforeFirstExecution; registers the release_all atexit
        enroll_stats(st->m_nnz, "b200_spmv_csr.nnz");
        enroll_stats(st->m_row_ptr, "b200_spmv_csr.row_ptr");
        enroll_stats(st->m_col_ind, "b200_spmv_csr.col_ind");
        enroll_stats(st->m_val, "b200_spmv_csr.val");
        enroll_stats(st->m_x, "b200_spmv_csr.x");
        enroll_stats(st->m_output, "b200_spmv_csr.output");
    }
    return *st;
}

void add_bytes(HarnessStats& hs, std::int64_t h2d0, std::int64_t h2d1, std::int64_t d2h0, std::int64_t d2h1) {
    hs.bytes_h2d += h2d1 - h2d0;
    hs.bytes_d2h += d2h1 - d2h0;
}

// bytes served from device mirrors during one call (all DevArray inputs)
struct D2dMeter {
    HarnessStats& hs;
    std::vector<const std::int64_t*> ctrs;
    std::int64_t start = 0;
    D2dMeter(HarnessStats& h, std::initializer_list<const std::int64_t*> c) : hs(h), ctrs(c) {
        for (auto* p : ctrs) start += *p;
    }
    ~D2dMeter() {
        std::int64_t now = 0;
        for (auto* p : ctrs) now += *p;
        hs.bytes_d2d += now - start;
    }
};

// ---- persistent state: b200_spmv_jds -------------------------------------------------

struct spmv_jds_state {
    MarshalObject<std::int64_t> m_max_nz;   // ReadableMax of nzcnt[0..rows) - 1
    MarshalObject<std::int64_t> m_nnz;      // LastEntry of jd_ptr[0..max_nz+1)
    MarshalObject<DevArray> m_nzcnt;
    MarshalObject<PermDev> m_perm;
    MarshalObject<DevArray> m_jd_ptr;
    MarshalObject<ColDev> m_col_ind;
    MarshalObject<DevArray> m_val;
    MarshalObject<DevArray> m_x;
    MarshalObject<DevArray> m_output;
    JdsSeg seg;  // k_jds_seg zones of the marshaled nzcnt
    bool validated = false;
    bool first_run_done = false;
};

spmv_jds_state& jds_state() {
    static spmv_jds_state* st = new spmv_jds_state;
    if (!st->first_run_done) {
        st->first_run_done = true;
        ensure_init();
        enroll_stats(st->m_max_nz, "b200_spmv_jds.max_nz");
        enroll_stats(st->m_nnz, "b200_spmv_jds.nnz");
        enroll_stats(st->m_nzcnt, "b200_spmv_jds.nzcnt");
        enroll_stats(st->m_perm, "b200_spmv_jds.perm");
        enroll_stats(st->m_jd_ptr, "b200_spmv_jds.jd_ptr");
        enroll_stats(st->m_col_ind, "b200_spmv_jds.col_ind");
        enroll_stats(st->m_val, "b200_spmv_jds.val");
        enroll_stats(st->m_x, "b200_spmv_jds.x");
        enroll_stats(st->m_output, "b200_spmv_jds.output");
    }
    return *st;
}

// ---- persistent state: BLAS-1 companions ------------------------------------------------

// A binding served by K marshal objects chosen by region identity (LRU). The
// reference keeps one object per binding, so a harness called on alternating
// arrays (CG: dot(r,r), dot(p,q), dot(x,z)) destructs and reconstructs on
// every call (marshal.hpp:192-199) — re-guarding pages, re-allocating, and
// dropping the streaming state each time. Each cached object still follows
// the reference state machine for its own region.
template <typename Out, int K>
struct BindingCache {
    MarshalObject<Out> objs[K];
    std::uint64_t used[K] = {};
    std::uint64_t clock = 0;

    void enroll(const std::string& name) {
        static std::vector<std::string> keep;  // names outlive the objects' registration
        for (int i = 0; i < K; ++i) {
            keep.push_back(name + "[" + std::to_string(i) + "]");
            enroll_stats(objs[i], keep.back().c_str());
        }
    }
    MarshalObject<Out>& pick(const void* base, std::size_t bytes) {
        int victim = -1;
        for (int i = 0; i < K; ++i) {
            const auto& r = objs[i].region().ref;
            if (objs[i].constructed() && r.base == base && r.bytes == bytes) {
                used[i] = ++clock;
                return objs[i];
            }
        }
        for (int i = 0; i < K; ++i)
            if (!objs[i].constructed()) {
                victim = i;
                break;
            }
        if (victim < 0) {
            victim = 0;
            for (int i = 1; i < K; ++i)
                if (used[i] < used[victim]) victim = i;
        }
        used[victim] = ++clock;
        return objs[victim];
    }
    std::int64_t sum(std::int64_t Out::*field) {
        std::int64_t t = 0;
        for (auto& o : objs) t += o.out().*field;
        return t;
    }
};

constexpr int kBindingCache = 4;

struct dot_state {
    BindingCache<DevArray, kBindingCache> m_a, m_b;
    MarshalObject<DevArray> m_result;
    bool first_run_done = false;
};

struct gemm_state {
    MarshalObject<DevArray> m_c, m_a, m_b;
    bool first_run_done = false;
};

gemm_state& gemm_st() {
    static gemm_state* st = new gemm_state;
    if (!st->first_run_done) {
        st->first_run_done = true;
        ensure_init();
        enroll_stats(st->m_c, "b200_gemm.c");
        enroll_stats(st->m_a, "b200_gemm.a");
        enroll_stats(st->m_b, "b200_gemm.b");
    }
    return *st;
}

struct vec2_state {  // axpy / xpay: y in, x in, y out
    BindingCache<DevArray, kBindingCache> m_y_in, m_x, m_y_out;
    bool first_run_done = false;
};

dot_state& dot_st() {
    static dot_state* st = new dot_state;
    if (!st->first_run_done) {
        st->first_run_done = true;
        ensure_init();
        st->m_a.enroll("b200_dot.a");
        st->m_b.enroll("b200_dot.b");
        enroll_stats(st->m_result, "b200_dot.result");
    }
    return *st;
}

vec2_state& vec2_st(const char* which) {
    static vec2_state* axpy = new vec2_state;
    static vec2_state* xpay = new vec2_state;
    const bool is_axpy = std::strcmp(which, "b200_axpy") == 0;
    vec2_state* st = is_axpy ? axpy : xpay;
    if (!st->first_run_done) {
        st->first_run_done = true;
        ensure_init();
        const std::string w = which;
        st->m_y_in.enroll(w + ".y");
        st->m_x.enroll(w + ".x");
        st->m_y_out.enroll(w + ".y_out");
    }
    return *st;
}

std::int64_t sum_h2d(std::initializer_list<std::int64_t> v) {
    std::int64_t s = 0;
    for (auto x : v) s += x;
    return s;
}

}  // namespace

// =================================================================================
// Entry points
// =================================================================================

namespace b200 {
// multi_harness.cpp: the same entry points over LILAC_B200_NGPUS devices
void multi_spmv_csr(std::int64_t rows, double* output, const std::int64_t* row_ptr, const double* val,
                    const double* x, const std::int64_t* col_ind);
void multi_dot(double* result, std::int64_t n, const double* a, const double* b);
void multi_vec2(const char* name, std::int64_t n, double* y, double s, const double* x, bool axpy);
}  // namespace b200

extern "C" void b200_spmv_csr(std::int64_t rows, double* output, const std::int64_t* row_ptr, const double* val,
                              const double* x, const std::int64_t* col_ind) {
    boundary("b200_spmv_csr", [&] {
        if (harness_ngpus() > 1) {
            multi_spmv_csr(rows, output, row_ptr, val, x, col_ind);
            return;
        }
        spmv_csr_state& state = csr_state();
        HarnessStats& hs = harness_stats("b200_spmv_csr");
        Timer tm(hs);
        if (rows < 0) throw Error(Errc::DataError, "rows < 0");
        const std::int64_t h0 = sum_h2d({state.m_row_ptr.out().h2d, state.m_col_ind.out().h2d, state.m_val.out().h2d,
                                         state.m_x.out().h2d});
        D2dMeter dm(hs, {&state.m_x.out().d2d, &state.m_val.out().d2d});
        const std::int64_t d0 = state.m_output.out().d2h;

        // Marshaling, in binding order (cusparse.lilac:52-61)
        const std::int64_t nnz = state.m_nnz.acquire(row_ptr, (rows + 1) * sizeof(*row_ptr), nullptr,
                                                     LastEntry_update, nullptr);
        if (nnz < 0) throw Error(Errc::OutOfBounds, "row_ptr[rows] < 0");
        RowPtrDev& rp = state.m_row_ptr.acquire(
            row_ptr, (rows + 1) * sizeof(*row_ptr), nullptr,
            [rows, nnz](const void* in, std::size_t size, RowPtrDev& out) {
                upload_row_ptr(out.buf, static_cast<const std::int64_t*>(in), rows, nnz, &out.max_row, &out.monotone);
                out.h2d += static_cast<std::int64_t>(size);
            },
            [](const void*, std::size_t, RowPtrDev& out) { out.buf.release(); });
        ColDev& ci = state.m_col_ind.acquire(col_ind, nnz * sizeof(*col_ind), nullptr, ColInd_update, ColInd_destruct);
        DevArray& dval = state.m_val.acquire(val, nnz * sizeof(*val), nullptr, B200Read_update, B200Read_destruct);
        DevArray& dx = state.m_x.acquire(x, ci.cols * sizeof(*x), nullptr, B200Read_update, B200Read_destruct);
        DevArray& dout = state.m_output.acquire_out(output, rows * sizeof(*output), B200Write_construct,
                                                    B200Write_update, B200Write_destruct);
        tm.acquired();

        // body: the sm_100a SpMV
        CsrDev A;
        A.rows = rows;
        A.nnz = nnz;
        A.cols = ci.cols;
        A.max_row = rp.max_row;
        A.row_ptr = rp.buf.as<std::int64_t>();
        A.col = ci.buf.ptr;
        A.col32 = ci.col32;
        A.val = dval.data<double>();
        A.monotone = rp.monotone;
        // derived tiled layout: rebuilt only when row_ptr/col_ind/val were re-marshaled
        std::int64_t stamp = matrix_stamp(state);
        const bool rebuild = stamp != state.tiled_stamp || rt().kernel != state.tiled_policy;
        // (the flag alone is not enough: a new matrix identity re-constructs the
        // bindings, which brings the plain arrays back)
        state.plain_dropped = state.plain_dropped && (!ci.buf.ptr || (!dval.lent && !dval.buf.ptr));
        if (rebuild && state.plain_dropped) {
            // the plain col / val were freed behind the old layout: a rebuild (or
            // another kernel) needs them again — re-marshal both in full
            state.m_col_ind.release();
            state.m_val.release();
            state.plain_dropped = false;
            state.m_col_ind.acquire(col_ind, nnz * sizeof(*col_ind), nullptr, ColInd_update, ColInd_destruct);
            state.m_val.acquire(val, nnz * sizeof(*val), nullptr, B200Read_update, B200Read_destruct);
            A.col = ci.buf.ptr;
            A.col32 = ci.col32;
            A.val = dval.data<double>();
            stamp = matrix_stamp(state);
        }
        if (rebuild) {
            state.tiled.refresh(rows, row_ptr, col_ind, val, ci.cols, rp.monotone, rp.max_row, rt().kernel);
            if (!state.tiled.valid)
                state.lrc.refresh(A, row_ptr, col_ind, rt().kernel);
            else
                state.lrc.release();
            if (!state.tiled.valid && !state.lrc.valid) {
                state.split.refresh(A, row_ptr, rt().kernel);
                state.merge.refresh(A, row_ptr, rt().kernel);
            } else {
                state.split.release();
                state.merge.release();
            }
            state.tiled_stamp = stamp;
            state.tiled_policy = rt().kernel;
            // only the derived layout is read from now on: free the plain copies
            // (the marshal objects stay constructed, so change detection goes on)
            if ((state.tiled.valid || state.lrc.valid) && !keep_plain_csr() && !dval.lent) {
                ci.buf.release();
                dval.buf.release();
                state.plain_dropped = true;
            }
        }
        if (state.plain_dropped) {
            A.col = nullptr;
            A.val = nullptr;
        }
        if (state.tiled.valid) A.tiled = &state.tiled.dev;
        if (state.lrc.valid) A.lrc = &state.lrc.dev;
        if (state.merge.valid) A.merge = &state.merge.dev;
        if (state.split.valid) A.split = &state.split.dev;
        tm.acquired();
        timed_launch(hs, [&] { launch_spmv_csr(A, dx.data<double>(), dout.buf.as<double>(), rt().kernel, rt().stream); });
        tm.acquired();

        state.m_output.write_back();
        collect_kernel_time(hs);
        tm.written_back();
        add_bytes(hs, h0,
                  sum_h2d({state.m_row_ptr.out().h2d, state.m_col_ind.out().h2d, state.m_val.out().h2d,
                           state.m_x.out().h2d}),
                  d0, state.m_output.out().d2h);
    });
}

extern "C" void b200_spmv_jds(std::int64_t rows, double* output, const std::int64_t* nzcnt, const std::int64_t* perm,
                              const double* val, const std::int64_t* jd_ptr, const double* x,
                              const std::int64_t* col_ind) {
    boundary("b200_spmv_jds", [&] {
        spmv_jds_state& state = jds_state();
        HarnessStats& hs = harness_stats("b200_spmv_jds");
        Timer tm(hs);
        if (rows < 0) throw Error(Errc::DataError, "rows < 0");
        auto h2d_now = [&] {
            return sum_h2d({state.m_nzcnt.out().h2d, state.m_perm.out().h2d, state.m_jd_ptr.out().h2d,
                            state.m_col_ind.out().h2d, state.m_val.out().h2d, state.m_x.out().h2d});
        };
        const std::int64_t h0 = h2d_now();
        const std::int64_t d0 = state.m_output.out().d2h;
        D2dMeter dm(hs, {&state.m_x.out().d2d, &state.m_val.out().d2d});

        const std::int64_t max_nz =
            state.m_max_nz.acquire(nzcnt, rows * sizeof(*nzcnt), nullptr, ReadableMax_update, nullptr) - 1;
        const std::int64_t njd = max_nz >= 0 ? max_nz + 1 : 0;
        const std::int64_t nnz =
            njd > 0 ? state.m_nnz.acquire(jd_ptr, njd * sizeof(*jd_ptr), nullptr, LastEntry_update, nullptr) : 0;
        if (nnz < 0) throw Error(Errc::OutOfBounds, "jd_ptr[max_nz] < 0");
        DevArray& dnz = state.m_nzcnt.acquire(nzcnt, rows * sizeof(*nzcnt), nullptr,
                                              [&](const void* in, std::size_t size, DevArray& out) {
                                                  upload(out, in, size);
                                                  host_in(in, size);  // read on the host below (lazy ranges filled here)
                                                  state.seg = jds_segments(static_cast<const std::int64_t*>(in),
                                                                           rows);
                                                  state.validated = false;
                                              },
                                              B200Read_destruct);
        PermDev& dperm = state.m_perm.acquire(perm, rows * sizeof(*perm), nullptr, Perm_update, Perm_destruct);
        DevArray& djd = state.m_jd_ptr.acquire(jd_ptr, njd * sizeof(*jd_ptr), nullptr,
                                               [&](const void* in, std::size_t size, DevArray& out) {
                                                   upload(out, in, size);
                                                   state.validated = false;
                                               },
                                               B200Read_destruct);
        DevArray& dval = state.m_val.acquire(val, nnz * sizeof(*val), nullptr, B200Read_update, B200Read_destruct);
        ColDev& ci = state.m_col_ind.acquire(col_ind, nnz * sizeof(*col_ind), nullptr, ColInd_update, ColInd_destruct);
        DevArray& dx = state.m_x.acquire(x, ci.cols * sizeof(*x), nullptr, B200Read_update, B200Read_destruct);
        DevArray& dout = state.m_output.acquire_out(output, rows * sizeof(*output), B200Write_construct,
                                                    B200Write_update, B200Write_destruct);
        if (!state.validated) {
            // offsets jd_ptr[k] + p must stay inside [0, nnz) (what_interp.cpp:67-68)
            Runtime& r = rt();
            B200_CUDA(cudaMemsetAsync(r.flags.ptr, 0, 16, r.stream));
            launch_check_jds(dnz.data<std::int64_t>(), djd.data<std::int64_t>(), rows, njd, nnz, r.d_bad(),
                             r.stream);
            int bad = 0;
            B200_CUDA(cudaMemcpyAsync(&bad, r.d_bad(), 4, cudaMemcpyDeviceToHost, r.stream));
            B200_CUDA(cudaStreamSynchronize(r.stream));
            if (bad) throw Error(Errc::OutOfBounds, "jd_ptr[k] + perm[i] outside [0, nnz)");
            state.validated = true;
        }
        tm.acquired();

        JdsDev A;
        A.rows = rows;
        A.nnz = nnz;
        A.cols = ci.cols;
        A.njd = njd;
        A.nzcnt = dnz.data<std::int64_t>();
        A.perm = dperm.perm.as<std::int64_t>();
        A.inv_perm = dperm.bijective ? dperm.inv.as<std::int64_t>() : nullptr;
        A.jd_ptr = djd.data<std::int64_t>();
        A.col = ci.buf.ptr;
        A.col32 = ci.col32;
        A.val = dval.data<double>();
        A.seg = state.seg;
        timed_launch(hs, [&] { launch_spmv_jds(A, dx.data<double>(), dout.buf.as<double>(), rt().stream); });
        tm.acquired();

        state.m_output.write_back();
        collect_kernel_time(hs);
        tm.written_back();
        add_bytes(hs, h0, h2d_now(), d0, state.m_output.out().d2h);
    });
}

extern "C" void b200_dot(double* result, std::int64_t length, const double* a, const double* b) {
    boundary("b200_dot", [&] {
        if (harness_ngpus() > 1) {
            multi_dot(result, length, a, b);
            return;
        }
        dot_state& state = dot_st();
        HarnessStats& hs = harness_stats("b200_dot");
        Timer tm(hs);
        if (length < 0) throw Error(Errc::DataError, "length < 0");
        const std::size_t bytes = length * sizeof(double);
        auto& oa = state.m_a.pick(a, bytes);
        auto& ob = state.m_b.pick(b, bytes);
        const std::int64_t h0 = state.m_a.sum(&DevArray::h2d) + state.m_b.sum(&DevArray::h2d),
                           d0 = state.m_result.out().d2h,
                           dd0 = state.m_a.sum(&DevArray::d2d) + state.m_b.sum(&DevArray::d2d);
        DevArray& da = oa.acquire(a, bytes, nullptr, B200Read_update, B200Read_destruct);
        // dot(r, r): one binding serves both operands
        DevArray& db = (b == a) ? da : ob.acquire(b, bytes, nullptr, B200Read_update, B200Read_destruct);
        // the kernel also posts the result to the pinned mapped slot; the
        // write-back (B200Write's update) waits on it instead of D2H + sync
        const HostSlot slot = rt().next_slot();
        DevArray& dres = state.m_result.acquire_out(
            result, sizeof(*result), B200Write_construct,
            [seq = slot.seq](const void* in, std::size_t size, DevArray& out) {
                const double v = wait_host_slot(seq);
                std::memcpy(const_cast<void*>(in), &v, size < sizeof v ? size : sizeof v);
                out.d2h += static_cast<std::int64_t>(sizeof v);
            },
            B200Write_destruct);
        tm.acquired();
        timed_launch(hs, [&] {
            Runtime& r = rt();
            if (r.exact_blas)
                launch_dot_exact(da.data<double>(), db.data<double>(), length, dres.buf.as<double>(), r.stream,
                                 slot);
            else
                launch_dot(da.data<double>(), db.data<double>(), length, dres.buf.as<double>(),
                           r.partials.as<double>(), r.d_ticket(), r.stream, slot);
        });
        tm.acquired();
        state.m_result.write_back();
        collect_kernel_time(hs);
        tm.written_back();
        add_bytes(hs, h0, state.m_a.sum(&DevArray::h2d) + state.m_b.sum(&DevArray::h2d), d0,
                  state.m_result.out().d2h);
        hs.bytes_d2d += state.m_a.sum(&DevArray::d2d) + state.m_b.sum(&DevArray::d2d) - dd0;
    });
}

namespace {

void vec2_call(const char* name, std::int64_t n, double* y, double s, const double* x, bool axpy) {
    if (harness_ngpus() > 1) {
        multi_vec2(name, n, y, s, x, axpy);
        return;
    }
    vec2_state& state = vec2_st(name);
    HarnessStats& hs = harness_stats(name);
    Timer tm(hs);
    if (n < 0) throw Error(Errc::DataError, "n < 0");
    const std::size_t bytes = n * sizeof(double);
    PhaseTimer pt_pick(kPhPick);
    auto& oy = state.m_y_in.pick(y, bytes);
    auto& ox = state.m_x.pick(x, bytes);
    auto& oo = state.m_y_out.pick(y, bytes);
    const std::int64_t h0 = state.m_y_in.sum(&DevArray::h2d) + state.m_x.sum(&DevArray::h2d),
                       d0 = state.m_y_out.sum(&DevArray::d2h),
                       dd0 = state.m_y_in.sum(&DevArray::d2d) + state.m_x.sum(&DevArray::d2d);
    pt_pick.stop();
    PhaseTimer pt_acq(kPhAcquire);
    DevArray& dy = oy.acquire(y, bytes, nullptr, B200Read_update, B200Read_destruct);
    DevArray& dx = ox.acquire(x, bytes, nullptr, B200Read_update, B200Read_destruct);
    pt_acq.stop();
    PhaseTimer pt_out(kPhAcquireOut);
    DevArray& dout = oo.acquire_out(y, bytes, B200Write_construct, B200Write_update, B200Write_destruct);
    pt_out.stop();
    tm.acquired();
    timed_launch(hs, [&] {
        Runtime& r = rt();
        if (axpy)
            launch_axpy_to(n, dout.buf.as<double>(), dy.data<double>(), s, dx.data<double>(), r.stream);
        else
            launch_xpay_to(n, dout.buf.as<double>(), dy.data<double>(), s, dx.data<double>(), r.stream);
    });
    tm.acquired();
    oo.write_back();
    collect_kernel_time(hs);
    tm.written_back();
    add_bytes(hs, h0, state.m_y_in.sum(&DevArray::h2d) + state.m_x.sum(&DevArray::h2d), d0,
              state.m_y_out.sum(&DevArray::d2h));
    hs.bytes_d2d += state.m_y_in.sum(&DevArray::d2d) + state.m_x.sum(&DevArray::d2d) - dd0;
}

}  // namespace

extern "C" void b200_gemm(std::int64_t n, std::int64_t m, double* c, std::int64_t p, const double* a,
                          const double* b) {
    boundary("b200_gemm", [&] {
        gemm_state& state = gemm_st();
        HarnessStats& hs = harness_stats("b200_gemm");
        Timer tm(hs);
        if (n < 0 || m < 0 || p < 0) throw Error(Errc::DataError, "negative gemm extent");
        const std::int64_t h0 = state.m_a.out().h2d + state.m_b.out().h2d, d0 = state.m_c.out().d2h;
        D2dMeter dm(hs, {&state.m_a.out().d2d, &state.m_b.out().d2d});
        // binding order of infer_interface: c (output), a, b (kernels.lilac:14-19)
        DevArray& dc = state.m_c.acquire_out(c, n * m * sizeof(double), B200Write_construct, B200Write_update,
                                             B200Write_destruct);
        DevArray& da = state.m_a.acquire(a, n * p * sizeof(double), nullptr, B200Read_update, B200Read_destruct);
        DevArray& db = state.m_b.acquire(b, p * m * sizeof(double), nullptr, B200Read_update, B200Read_destruct);
        tm.acquired();
        timed_launch(hs, [&] {
            launch_gemm(n, m, p, da.data<double>(), db.data<double>(), dc.buf.as<double>(), rt().exact_blas,
                        rt().stream);
        });
        tm.acquired();
        state.m_c.write_back();
        collect_kernel_time(hs);
        tm.written_back();
        add_bytes(hs, h0, state.m_a.out().h2d + state.m_b.out().h2d, d0, state.m_c.out().d2h);
    });
}

extern "C" void b200_axpy(std::int64_t n, double* y, double alpha, const double* x) {
    boundary("b200_axpy", [&] { vec2_call("b200_axpy", n, y, alpha, x, true); });
}

extern "C" void b200_xpay(std::int64_t n, double* y, double beta, const double* x) {
    boundary("b200_xpay", [&] { vec2_call("b200_xpay", n, y, beta, x, false); });
}
