// multi_harness.cpp — the harness entry points over several B200s of one
// process (LILAC_B200_NGPUS = k >= 2), behind the unchanged C ABI: a program
// rewritten by LiLAC and linked against liblilac_b200.so (PAPER.md:233-238,
// harnessgen.cpp:86-131) uses k GPUs without a source change.
//
//  * b200_spmv_csr: the matrix is marshaled once into k nnz-balanced row
//    blocks (b200_partition_rows), each resident on its own device with its
//    own derived layout (tiled / lane-range) and the plain CSR freed behind it;
//    per call x goes to every device, each computes its rows, and each writes
//    its slice of `output` straight back. Change detection of row_ptr / col_ind
//    / val is the marshaling layer's (one MarshalObject per binding, as the
//    single-device path): a change re-shards the whole matrix.
//  * b200_dot / b200_axpy / b200_xpay: element ranges per device; the dot's
//    per-device partials are summed on the host in device order
//    (deterministic).
// Vectors move every call (the reference's eager semantics: no device mirrors
// or lazy write-back in this mode). Shard g lives on device (primary + g) mod
// visible: with fewer GPUs than k the shards share devices, which is how the
// path is exercised on one B200 (every shard on device 0, one stream).

#include "lilac_b200.h"
#include "runtime.hpp"
#include "tcsr.hpp"

#include <memory>
#include <vector>

namespace b200 {

namespace {

struct MShard {
    int device = 0;
    std::int64_t r0 = 0, rows = 0, nnz = 0, cols = 0;
    DevBuf rp, col, val, x, y;
    CsrDev A;
    TcsrOwner tiled;
    LrcOwner lrc;
    SplitOwner split;
    void release() {
        for (DevBuf* b : {&rp, &col, &val, &x, &y}) b->release();
        tiled.release();
        lrc.release();
        split.release();
    }
};

void count_update(const void*, std::size_t, std::int64_t& out) { ++out; }

struct MultiCsr {
    MarshalObject<std::int64_t> m_nnz, m_rp, m_col, m_val;  // change detection of the matrix bindings
    std::vector<std::unique_ptr<MShard>> shards;
    std::int64_t stamp = -1, cols = 0;
    bool first_run_done = false;

    std::int64_t matrix_stamp() const {
        std::int64_t s = 0;
        for (const MarshalObjectBase* m : {static_cast<const MarshalObjectBase*>(&m_rp),
                                           static_cast<const MarshalObjectBase*>(&m_col),
                                           static_cast<const MarshalObjectBase*>(&m_val)})
            s += m->counters().n_update + m->counters().n_construct;
        return s;
    }
};

MultiCsr& multi_csr() {
    static MultiCsr* st = new MultiCsr;
    if (!st->first_run_done) {
        st->first_run_done = true;
        ensure_init();
        const char* names[] = {"b200_spmv_csr[multi].nnz", "b200_spmv_csr[multi].row_ptr",
                               "b200_spmv_csr[multi].col_ind", "b200_spmv_csr[multi].val"};
        MarshalObject<std::int64_t>* objs[] = {&st->m_nnz, &st->m_rp, &st->m_col, &st->m_val};
        for (int i = 0; i < 4; ++i) {
            objs[i]->set_name(names[i]);
            objs[i]->set_strategy(rt().strategy);
            objs[i]->set_adaptive(true);
            register_region(objs[i], nullptr, nullptr, nullptr);
        }
    }
    return *st;
}

void last_entry(const void* in, std::size_t size, std::int64_t& out) {
    const auto* p = static_cast<const std::int64_t*>(in);
    out = size >= sizeof(std::int64_t) ? p[size / sizeof(std::int64_t) - 1] : 0;
}

// (Re)build every shard from the caller's arrays.
void shard_matrix(MultiCsr& st, std::int64_t rows, const std::int64_t* row_ptr, const std::int64_t* col_ind,
                  const double* val) {
    const int k = harness_ngpus();
    for (auto& s : st.shards) {
        DeviceScope ds(s->device);
        s->release();
    }
    st.shards.clear();
    host_in(row_ptr, sizeof(std::int64_t) * static_cast<std::size_t>(rows + 1));
    std::vector<std::int64_t> bounds(static_cast<std::size_t>(k) + 1);
    b200_partition_rows(rows, row_ptr, k, bounds.data());
    st.cols = 0;
    std::vector<std::vector<std::int64_t>> lrps(static_cast<std::size_t>(k));
    for (int g = 0; g < k; ++g) {
        auto s = std::make_unique<MShard>();
        s->device = shard_device(g);
        DeviceScope ds(s->device);
        s->r0 = bounds[g];
        s->rows = bounds[g + 1] - bounds[g];
        const std::int64_t base = row_ptr[s->r0];
        std::vector<std::int64_t>& lrp = lrps[g];
        lrp.resize(static_cast<std::size_t>(s->rows + 1));
        for (std::int64_t i = 0; i <= s->rows; ++i) lrp[i] = row_ptr[s->r0 + i] - base;
        s->nnz = lrp[s->rows];
        std::int64_t max_row = 0;
        bool monotone = true, col32 = true;
        upload_row_ptr(s->rp, lrp.data(), s->rows, s->nnz, &max_row, &monotone);
        s->cols = upload_col_ind(s->col, col_ind + base, s->nnz, &col32);
        s->val.ensure(sizeof(double) * static_cast<std::size_t>(std::max<std::int64_t>(s->nnz, 1)));
        host_in(val + base, sizeof(double) * static_cast<std::size_t>(s->nnz));
        if (s->nnz)
            B200_CUDA(cudaMemcpyAsync(s->val.ptr, val + base, sizeof(double) * static_cast<std::size_t>(s->nnz),
                                      cudaMemcpyHostToDevice, rt().stream));
        B200_CUDA(cudaStreamSynchronize(rt().stream));
        CsrDev& A = s->A;
        A.rows = s->rows;
        A.nnz = s->nnz;
        A.max_row = max_row;
        A.row_ptr = s->rp.as<std::int64_t>();
        A.col = s->col.ptr;
        A.col32 = col32;
        A.val = s->val.as<double>();
        A.monotone = monotone;
        st.cols = std::max(st.cols, s->cols);
        st.shards.push_back(std::move(s));
    }
    // the derived layouts see the full x extent (every shard reads all of x)
    for (int g = 0; g < k; ++g) {
        MShard& s = *st.shards[g];
        DeviceScope ds(s.device);
        const std::int64_t base = row_ptr[s.r0];
        CsrDev& A = s.A;
        A.cols = st.cols;
        if (s.tiled.refresh(s.rows, lrps[g].data(), col_ind + base, val + base, st.cols, A.monotone, A.max_row,
                            rt().kernel)) {
            A.tiled = &s.tiled.dev;
        } else if (s.lrc.refresh(A, lrps[g].data(), col_ind + base, rt().kernel)) {
            A.lrc = &s.lrc.dev;
        } else if (s.split.refresh(A, lrps[g].data(), rt().kernel)) {
            A.split = &s.split.dev;
        }
        if ((A.tiled || A.lrc) && !keep_plain_csr()) {
            s.col.release();
            s.val.release();
            A.col = nullptr;
            A.val = nullptr;
        }
        s.x.ensure(sizeof(double) * static_cast<std::size_t>(std::max<std::int64_t>(st.cols, 1)), false);
        s.y.ensure(sizeof(double) * static_cast<std::size_t>(std::max<std::int64_t>(s.rows, 1)), false);
    }
}

// A DMA write into caller memory: lazy bytes under it are superseded, device
// mirrors of it are stale, guards see a write.
void dma_write_target(void* host, std::size_t bytes) {
    lilac::marshal::supersede_range(host, bytes);
    mirrors_forget(host, bytes);
    lilac::marshal::note_host_write(host, bytes);
}

// per-device vector buffers of the BLAS-1 companions
struct VecBufs {
    DevBuf a, b;
};
std::vector<VecBufs>& vec_bufs() {
    static auto* v = new std::vector<VecBufs>;
    if (v->size() < static_cast<std::size_t>(harness_ngpus())) v->resize(static_cast<std::size_t>(harness_ngpus()));
    return *v;
}

}  // namespace

void multi_spmv_csr(std::int64_t rows, double* output, const std::int64_t* row_ptr, const double* val, const double* x,
                    const std::int64_t* col_ind) {
    MultiCsr& st = multi_csr();
    HarnessStats& hs = harness_stats("b200_spmv_csr");
    const auto t0 = Clock::now();
    if (rows < 0) throw Error(Errc::DataError, "rows < 0");
    const std::int64_t nnz = st.m_nnz.acquire(row_ptr, (rows + 1) * sizeof(*row_ptr), nullptr, last_entry, nullptr);
    if (nnz < 0) throw Error(Errc::OutOfBounds, "row_ptr[rows] < 0");
    st.m_rp.acquire(row_ptr, (rows + 1) * sizeof(*row_ptr), nullptr, count_update, nullptr);
    st.m_col.acquire(col_ind, nnz * sizeof(*col_ind), nullptr, count_update, nullptr);
    st.m_val.acquire(val, nnz * sizeof(*val), nullptr, count_update, nullptr);
    const std::int64_t stamp = st.matrix_stamp();
    if (stamp != st.stamp) {
        shard_matrix(st, rows, row_ptr, col_ind, val);
        st.stamp = stamp;
        hs.bytes_h2d += 8 * (rows + 1) + 16 * nnz;
    }
    const std::size_t xb = sizeof(double) * static_cast<std::size_t>(st.cols);
    host_in(x, xb);
    dma_write_target(output, sizeof(double) * static_cast<std::size_t>(rows));
    for (auto& sp : st.shards) {
        MShard& s = *sp;
        DeviceScope ds(s.device);
        if (xb) B200_CUDA(cudaMemcpyAsync(s.x.ptr, x, xb, cudaMemcpyHostToDevice, rt().stream));
        if (s.rows) {
            launch_spmv_csr(s.A, s.x.as<double>(), s.y.as<double>(), rt().kernel, rt().stream);
            B200_CUDA(cudaMemcpyAsync(output + s.r0, s.y.ptr, sizeof(double) * static_cast<std::size_t>(s.rows),
                                      cudaMemcpyDeviceToHost, rt().stream));
        }
    }
    for (auto& sp : st.shards) {
        DeviceScope ds(sp->device);
        B200_CUDA(cudaStreamSynchronize(rt().stream));
    }
    hs.calls++;
    hs.bytes_h2d += static_cast<std::int64_t>(xb * st.shards.size());
    hs.bytes_d2h += 8 * rows;
    hs.t_total_ms += ms_since(t0);
}

void multi_dot(double* result, std::int64_t n, const double* a, const double* b) {
    HarnessStats& hs = harness_stats("b200_dot");
    const auto t0 = Clock::now();
    if (n < 0) throw Error(Errc::DataError, "length < 0");
    const int k = harness_ngpus();
    host_in(a, sizeof(double) * static_cast<std::size_t>(n));
    host_in(b, sizeof(double) * static_cast<std::size_t>(n));
    std::vector<double> part(static_cast<std::size_t>(k), 0.0);
    auto& vb = vec_bufs();
    for (int g = 0; g < k; ++g) {
        const std::int64_t lo = n * g / k, hi = n * (g + 1) / k, m = hi - lo;
        DeviceScope ds(shard_device(g));
        Runtime& r = rt();
        VecBufs& v = vb[g];
        v.a.ensure(sizeof(double) * static_cast<std::size_t>(std::max<std::int64_t>(m, 1)), false);
        v.b.ensure(sizeof(double) * static_cast<std::size_t>(std::max<std::int64_t>(m, 1)), false);
        if (m) {
            B200_CUDA(cudaMemcpyAsync(v.a.ptr, a + lo, sizeof(double) * m, cudaMemcpyHostToDevice, r.stream));
            B200_CUDA(cudaMemcpyAsync(v.b.ptr, b + lo, sizeof(double) * m, cudaMemcpyHostToDevice, r.stream));
        }
        // each device's partial lands in its own result slot; summed below in device order
        double* dres = r.d_result() + g;
        if (r.exact_blas)
            launch_dot_exact(v.a.as<double>(), v.b.as<double>(), m, dres, r.stream);
        else
            launch_dot(v.a.as<double>(), v.b.as<double>(), m, dres, r.partials.as<double>(), r.d_ticket(), r.stream);
        B200_CUDA(cudaMemcpyAsync(&part[g], dres, sizeof(double), cudaMemcpyDeviceToHost, r.stream));
        hs.bytes_h2d += 16 * m;
        hs.bytes_d2h += 8;
    }
    for (int g = 0; g < k; ++g) {
        DeviceScope ds(shard_device(g));
        B200_CUDA(cudaStreamSynchronize(rt().stream));
    }
    double s = 0.0;
    for (int g = 0; g < k; ++g) s += part[g];
    *result = s;
    hs.calls++;
    hs.t_total_ms += ms_since(t0);
}

void multi_vec2(const char* name, std::int64_t n, double* y, double s, const double* x, bool axpy) {
    HarnessStats& hs = harness_stats(name);
    const auto t0 = Clock::now();
    if (n < 0) throw Error(Errc::DataError, "n < 0");
    const int k = harness_ngpus();
    host_in(x, sizeof(double) * static_cast<std::size_t>(n));
    host_in(y, sizeof(double) * static_cast<std::size_t>(n));
    dma_write_target(y, sizeof(double) * static_cast<std::size_t>(n));
    auto& vb = vec_bufs();
    for (int g = 0; g < k; ++g) {
        const std::int64_t lo = n * g / k, hi = n * (g + 1) / k, m = hi - lo;
        if (!m) continue;
        DeviceScope ds(shard_device(g));
        Runtime& r = rt();
        VecBufs& v = vb[g];
        v.a.ensure(sizeof(double) * static_cast<std::size_t>(m), false);
        v.b.ensure(sizeof(double) * static_cast<std::size_t>(m), false);
        B200_CUDA(cudaMemcpyAsync(v.a.ptr, y + lo, sizeof(double) * m, cudaMemcpyHostToDevice, r.stream));
        B200_CUDA(cudaMemcpyAsync(v.b.ptr, x + lo, sizeof(double) * m, cudaMemcpyHostToDevice, r.stream));
        if (axpy)
            launch_axpy_to(m, v.a.as<double>(), v.a.as<double>(), s, v.b.as<double>(), r.stream);
        else
            launch_xpay_to(m, v.a.as<double>(), v.a.as<double>(), s, v.b.as<double>(), r.stream);
        B200_CUDA(cudaMemcpyAsync(y + lo, v.a.ptr, sizeof(double) * m, cudaMemcpyDeviceToHost, r.stream));
        hs.bytes_h2d += 16 * m;
        hs.bytes_d2h += 8 * m;
    }
    for (int g = 0; g < k; ++g) {
        DeviceScope ds(shard_device(g));
        B200_CUDA(cudaStreamSynchronize(rt().stream));
    }
    hs.calls++;
    hs.t_total_ms += ms_since(t0);
}

}  // namespace b200
