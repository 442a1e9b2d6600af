// dist_driver.cpp — row-sharded NPB CG over 1..N B200s.
//
// Rows are split into contiguous nnz-balanced ranges (b200_partition_rows).
// Each shard keeps its row block resident (with global column indices), a
// full-length replica of p (and z) that its SpMV reads, and its own slices of
// x, z, r, q. Per CG step there is one real exchange: the p slices are
// all-gathered (variable sizes: grouped NCCL broadcasts), plus the scalar
// partials of the two dot products, gathered in rank order and summed in the
// same order on every shard (deterministic across ranks and runs).
//
//   spmv+dot(partial) -> gather d -> alpha -> z,r update + r.r(partial) ->
//   gather rho -> beta -> p update (own slice) -> all-gather p
//
// NcclExchange drives one shard per process (torchrun, one GPU each);
// LocalExchange drives k shards on one GPU with device copies, which runs the
// identical sharded algorithm for tests on a single B200.

#include "exchange.hpp"

#include <cstdlib>
#include <cstring>
#include "lilac_b200.h"
#include "runtime.hpp"
#include "tcsr.hpp"

#include <algorithm>
#include <cstddef>
#include <memory>
#include <vector>

using namespace b200;

namespace {

struct Shard {
    std::int64_t row0 = 0, rows = 0, nnz = 0;
    std::int64_t cmin = 0, cmax = 0;  // column footprint [cmin, cmax): the p / z entries its SpMV reads
    DevBuf row_ptr, col, val;
    CsrDev A;
    TcsrOwner tiled;
    MergeOwner merge;
    SplitOwner split;
    LrcOwner lrc;
    DevBuf x, q, r, p_full, z_full, partials, scalars, gathered;
    CgVectors v{};

    void release() {
        for (DevBuf* b : {&row_ptr, &col, &val, &x, &q, &r, &p_full, &z_full, &partials, &scalars, &gathered})
            b->release();
        tiled.release();
        merge.release();
        split.release();
        lrc.release();
    }
};

}  // namespace

struct b200_dist_cg {
    std::unique_ptr<Exchange> ex;
    std::vector<std::unique_ptr<Shard>> shards;
    std::vector<std::int64_t> bounds;  // world + 1
    int world = 1;
    int rank = 0;
    int transport = 0;  // 0 local device copies, 1 NCCL, 2 peer memory
    std::int64_t n = 0;
    cudaStream_t stream = nullptr;
    int steps_exchanges = 0;
    std::unique_ptr<PeerExchange> pending;  // exported, not attached yet
    // one outer iteration captured as a CUDA graph (kernels, exchange copies
    // and NCCL collectives alike), keyed by (stream, cgitmax, shift)
    cudaGraphExec_t graph = nullptr;
    cudaStream_t graph_stream = nullptr;
    int graph_cgitmax = -1;
    double graph_shift = 0.0;
    // the CG steps of every local shard in one persistent kernel
    // (k_cg_tiled_dist) once the peer-memory exchange is bound
    DevBuf fused_slots, fused_bars;
    std::size_t fused_smem = 0;
    bool fused_ready = false;
    bool fused_on = true;    // b200_dist_cg_set_fused
    bool fused_last = false;  // the last outer iteration ran k_cg_tiled_dist
};

namespace {

void init_shard_vectors(Shard& s, std::int64_t n, int nranks);

// A derived layout serves the shard: free its plain col / val (keep_plain_csr).
void drop_plain(Shard& s) {
    if (!(s.A.tiled || s.A.lrc) || keep_plain_csr()) return;
    s.col.release();
    s.val.release();
    s.A.col = nullptr;
    s.A.val = nullptr;
}

// Upload one row block [row0, row0+rows) given its host arrays (row_ptr with
// rows+1 entries, absolute offsets into col_ind/val as passed).
void load_shard(Shard& s, std::int64_t n, std::int64_t row0, std::int64_t rows, const std::int64_t* rp,
                const std::int64_t* ci, const double* val, int nranks) {
    s.row0 = row0;
    s.rows = rows;
    std::vector<std::int64_t> lrp(static_cast<std::size_t>(rows + 1));
    for (std::int64_t i = 0; i <= rows; ++i) lrp[i] = rp[i] - rp[0];
    const std::int64_t base = rp[0];
    s.nnz = lrp[rows];
    bool monotone = true, col32 = true;
    std::int64_t max_row = 0;
    upload_row_ptr(s.row_ptr, lrp.data(), rows, s.nnz, &max_row, &monotone);
    const std::int64_t cols = upload_col_ind(s.col, ci + base, s.nnz, &col32);
    if (cols > n) throw Error(Errc::OutOfBounds, "column index >= n in a shard");
    std::int64_t cmin = cols;
    for (std::int64_t j = 0; j < s.nnz; ++j) cmin = std::min(cmin, ci[base + j]);
    s.cmin = s.nnz ? cmin : 0;
    s.cmax = cols;
    s.val.ensure(s.nnz * 8);
    host_in(val + base, s.nnz * 8);
    if (s.nnz) B200_CUDA(cudaMemcpyAsync(s.val.ptr, val + base, s.nnz * 8, cudaMemcpyHostToDevice, rt().stream));
    B200_CUDA(cudaStreamSynchronize(rt().stream));
    CsrDev& A = s.A;
    A.rows = rows;
    A.nnz = s.nnz;
    A.cols = n;  // the SpMV reads the full replica
    A.max_row = max_row;
    A.row_ptr = s.row_ptr.as<std::int64_t>();
    A.col = s.col.ptr;
    A.col32 = col32;
    A.val = s.val.as<double>();
    A.monotone = monotone;
    if (s.tiled.refresh(rows, lrp.data(), ci + base, val + base, n, monotone, max_row, rt().kernel)) {
        s.tiled.dev.cols = n;
        A.tiled = &s.tiled.dev;
    } else {
        if (s.lrc.refresh(A, lrp.data(), ci + base, rt().kernel)) {
            A.lrc = &s.lrc.dev;
        } else {
            if (s.split.refresh(A, lrp.data(), rt().kernel)) A.split = &s.split.dev;
            if (s.merge.refresh(A, lrp.data(), rt().kernel)) A.merge = &s.merge.dev;
        }
    }
    drop_plain(s);
    init_shard_vectors(s, n, nranks);
}

// Per-shard CG state: owned x/q/r, full-length p/z replicas, partials and
// scalars (sharded mode), CgVectors views.
void init_shard_vectors(Shard& s, std::int64_t n, int nranks) {
    const std::int64_t rows = s.rows, row0 = s.row0;
    const std::size_t own = sizeof(double) * static_cast<std::size_t>(std::max<std::int64_t>(rows, 1));
    for (DevBuf* b : {&s.x, &s.q, &s.r}) b->ensure(own);
    s.p_full.ensure(sizeof(double) * n);
    s.z_full.ensure(sizeof(double) * n);
    s.partials.ensure(sizeof(double) * kMaxParts * 4);
    s.scalars.ensure(sizeof(CgScalars));
    s.gathered.ensure(sizeof(double) * 2 * std::max(nranks, 1));
    B200_CUDA(cudaMemsetAsync(s.scalars.ptr, 0, sizeof(CgScalars), rt().stream));
    B200_CUDA(cudaMemsetAsync(s.p_full.ptr, 0, sizeof(double) * n, rt().stream));
    B200_CUDA(cudaMemsetAsync(s.z_full.ptr, 0, sizeof(double) * n, rt().stream));
    // sharded mode flag (> 1): reductions stop at the shard partial even when
    // world == 1, since the exchange + fin_* path is always taken here
    const int nr = std::max(nranks, 2);
    B200_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(s.scalars.ptr) + offsetof(CgScalars, nranks), &nr, sizeof nr,
                              cudaMemcpyHostToDevice, rt().stream));
    CgVectors& v = s.v;
    v.n = rows;
    v.x = s.x.as<double>();
    v.q = s.q.as<double>();
    v.r = s.r.as<double>();
    v.p_full = s.p_full.as<double>();
    v.z_full = s.z_full.as<double>();
    v.p = v.p_full + row0;
    v.z = v.z_full + row0;
    v.row0 = row0;
    v.partials = s.partials.as<double>();
    v.sc = s.scalars.as<CgScalars>();
    cg_launch_reset_x(v, rt().stream);
    B200_CUDA(cudaStreamSynchronize(rt().stream));
}

// Rows [row0, row0+rows) of the 27-point stencil generated in this GPU's HBM
// (no host arrays: N = 420 is 2e9 nonzeros). Column footprint: the rows'
// neighbours, [row0 - nx^2 - nx - 1, row0 + rows + nx^2 + nx + 1) clamped.
void load_shard_stencil(Shard& s, std::int64_t nx, std::int64_t row0, std::int64_t rows, double diag, double off,
                        int nranks) {
    const std::int64_t n = nx * nx * nx;
    s.row0 = row0;
    s.rows = rows;
    gen_stencil27_rows_device(nx, row0, row0 + rows, diag, off, s.row_ptr, s.col, s.val, rt().stream);
    s.nnz = stencil27_prefix_nnz(nx, row0 + rows) - stencil27_prefix_nnz(nx, row0);
    const std::int64_t halo = nx * nx + nx + 1;
    s.cmin = rows ? std::max<std::int64_t>(0, row0 - halo) : 0;
    s.cmax = rows ? std::min<std::int64_t>(n, row0 + rows + halo) : 0;
    CsrDev& A = s.A;
    A.rows = rows;
    A.nnz = s.nnz;
    A.cols = n;
    A.max_row = rows ? 27 : 0;
    A.row_ptr = s.row_ptr.as<std::int64_t>();
    A.col = s.col.ptr;
    A.col32 = true;
    A.val = s.val.as<double>();
    A.monotone = true;
    const CsrKernel pol = rt().kernel;
    if ((pol == CsrKernel::Auto && s.nnz >= (std::int64_t(16) << 20)) || pol == CsrKernel::Lane) {
        lrc_build_device(rows, A.row_ptr, A.col, true, A.val, s.nnz, n, s.lrc, rt().stream);
        A.lrc = &s.lrc.dev;
    }
    drop_plain(s);
    init_shard_vectors(s, n, nranks);
}

// nnz-balanced row bounds of the stencil over k shards (the rule of
// b200_partition_rows on the analytic row pointers).
std::vector<std::int64_t> stencil_bounds(std::int64_t nx, int k) {
    const std::int64_t n = nx * nx * nx, nnz = stencil27_prefix_nnz(nx, n);
    std::vector<std::int64_t> b(static_cast<std::size_t>(k) + 1, 0);
    for (int g = 1; g < k; ++g) {
        const std::int64_t target = (nnz * g + k - 1) / k;
        std::int64_t lo = b[g - 1], hi = n;  // first row r with prefix(r) >= target
        while (lo < hi) {
            const std::int64_t mid = lo + (hi - lo) / 2;
            if (stencil27_prefix_nnz(nx, mid) < target)
                lo = mid + 1;
            else
                hi = mid;
        }
        b[g] = lo;
    }
    b[k] = n;
    return b;
}

std::vector<ShardView> views(b200_dist_cg* d, cudaStream_t st) {
    std::vector<ShardView> vs;
    for (auto& s : d->shards) {
        ShardView v;
        v.row0 = s->row0;
        v.rows = s->rows;
        v.partial = reinterpret_cast<double*>(reinterpret_cast<char*>(s->v.sc) + offsetof(CgScalars, part));
        v.gathered = s->gathered.as<double>();
        v.stream = st;
        vs.push_back(v);
    }
    return vs;
}

void gather_scalars(b200_dist_cg* d, cudaStream_t st, int npart, CgFin fin, double shift) {
    auto vs = views(d, st);
    std::vector<CgScalars*> scs;
    for (auto& s : d->shards) scs.push_back(s->v.sc);
    if (d->ex->scalars_fin(vs, npart, fin, scs, shift)) return;  // pushed by the producers; wait + fin
    d->ex->exchange_scalars(vs, npart);
    for (auto& s : d->shards) cg_launch_fin(fin, s->v.sc, s->gathered.as<double>(), d->world, shift, st);
}

void gather_vector(b200_dist_cg* d, cudaStream_t st, bool z) {
    auto vs = views(d, st);
    std::vector<double*> fulls;
    for (auto& s : d->shards) fulls.push_back(z ? s->v.z_full : s->v.p_full);
    d->ex->exchange_vector(vs, fulls);
}


// Plain CG in steps over the shards (the stencil config): start from
// x = b = A 1, then one CG iteration per dist_step, dist_finish = |b - A z|.
void dist_init(b200_dist_cg* d, cudaStream_t st) {
    for (auto& s : d->shards) cg_launch_init(s->v, st);
    gather_scalars(d, st, 1, CgFin::Rho, 0.0);
    gather_vector(d, st, false);
}

void dist_start_rowsum(b200_dist_cg* d, cudaStream_t st) {
    for (auto& s : d->shards) {
        cg_launch_reset_x(s->v, st);  // x = 1 (owned rows)
        if (s->rows)
            B200_CUDA(cudaMemcpyAsync(s->v.p, s->v.x, sizeof(double) * static_cast<std::size_t>(s->rows),
                                      cudaMemcpyDeviceToDevice, st));
    }
    gather_vector(d, st, false);  // p replica = 1 over every footprint
    for (auto& s : d->shards) launch_spmv_csr(s->A, s->v.p_full, s->v.x, CsrKernel::Auto, st);  // b = A 1
    dist_init(d, st);
}

void dist_step(b200_dist_cg* d, cudaStream_t st) {
    for (auto& s : d->shards) cg_launch_spmv_dot(s->A, s->v, st);
    gather_scalars(d, st, 1, CgFin::Alpha, 0.0);
    for (auto& s : d->shards) cg_launch_update_zr(s->v, st);
    gather_scalars(d, st, 1, CgFin::Beta, 0.0);
    auto vs = views(d, st);
    std::vector<const CgVectors*> cv;
    for (auto& s : d->shards) cv.push_back(&s->v);
    if (!d->ex->update_p_exchange(vs, cv)) {
        for (auto& s : d->shards) cg_launch_update_p(s->v, st);
        gather_vector(d, st, false);
    }
}

void dist_finish(b200_dist_cg* d, cudaStream_t st) {
    gather_vector(d, st, true);
    for (auto& s : d->shards) {
        launch_spmv_csr(s->A, s->v.z_full, s->v.r, CsrKernel::Auto, st);
        cg_launch_resid_partial(s->v, st);
    }
    gather_scalars(d, st, 1, CgFin::Rnorm, 0.0);
}

// The fused sharded CG (k_cg_tiled_dist) needs the peer-memory exchange
// bound to every shard's producers and the tiled layout on every shard. Its
// slot table is uploaded here, outside any graph capture.
// LILAC_B200_DIST_FUSED=0 keeps the six kernels per step.
void prepare_fused(b200_dist_cg* d) {
    static const bool on = [] {
        const char* e = std::getenv("LILAC_B200_DIST_FUSED");
        return !(e && std::strcmp(e, "0") == 0);
    }();
    if (d->fused_ready || !on || !d->fused_on || d->transport != 2) return;
    for (auto& s : d->shards)
        if (!s->A.tiled) return;
    const std::size_t sb = dist_slot_bytes(), k = d->shards.size();
    d->fused_bars.ensure(sizeof(unsigned) * k);
    std::vector<char> host(sb * k);
    std::size_t smem = 0;
    for (std::size_t i = 0; i < k; ++i) {
        const Shard& sh = *d->shards[i];
        dist_slot_fill(host.data() + i * sb, *sh.A.tiled, sh.v, d->fused_bars.as<unsigned>() + i);
        smem = std::max(smem, tiled_smem_bytes(*sh.A.tiled));
    }
    d->fused_slots.ensure(host.size());
    B200_CUDA(cudaMemcpy(d->fused_slots.ptr, host.data(), host.size(), cudaMemcpyHostToDevice));
    d->fused_smem = smem;
    d->fused_ready = true;
}

bool dist_fused_steps(b200_dist_cg* d, int steps, cudaStream_t st) {
    d->fused_last = d->fused_ready && d->fused_on &&
                    launch_cg_tiled_dist(d->fused_slots.ptr, static_cast<int>(d->shards.size()), d->fused_smem,
                                         d->fused_bars.as<unsigned>(), steps, st);
    return d->fused_last;
}

void dist_outer(b200_dist_cg* d, int cgitmax, double shift, cudaStream_t st) {
    dist_init(d, st);  // q=z=0, r=p=x (owned slices), rho; p exchanged
    if (!dist_fused_steps(d, cgitmax, st))
        for (int it = 0; it < cgitmax; ++it) dist_step(d, st);
    dist_finish(d, st);  // residual r = A z needs all of z
    for (auto& s : d->shards) cg_launch_norms(s->v, shift, st);
    gather_scalars(d, st, 2, CgFin::Norms, shift);
    for (auto& s : d->shards) cg_launch_scale_x(s->v, st);
}

// Replays one outer iteration from a graph: at 8 shards a CG step is ~40 us
// of device work against ~10 launches + 3 collectives issued from the host,
// so launch overhead would otherwise bound the scaling. LILAC_B200_DIST_GRAPH=0
// issues the launches directly.
void dist_outer_graph(b200_dist_cg* d, int cgitmax, double shift, cudaStream_t st) {
    static const bool on = [] {
        const char* e = std::getenv("LILAC_B200_DIST_GRAPH");
        return !(e && std::strcmp(e, "0") == 0);
    }();
    if (!on) {
        dist_outer(d, cgitmax, shift, st);
        return;
    }
    if (!d->graph || d->graph_stream != st || d->graph_cgitmax != cgitmax || d->graph_shift != shift) {
        if (d->graph) {
            cudaGraphExecDestroy(d->graph);
            d->graph = nullptr;
        }
        cudaGraph_t g = nullptr;
        B200_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        try {
            dist_outer(d, cgitmax, shift, st);
        } catch (...) {
            cudaStreamEndCapture(st, &g);
            if (g) cudaGraphDestroy(g);
            throw;
        }
        B200_CUDA(cudaStreamEndCapture(st, &g));
        const cudaError_t e = cudaGraphInstantiate(&d->graph, g, 0);
        cudaGraphDestroy(g);
        if (e != cudaSuccess) throw_cuda(e, "cudaGraphInstantiate", __FILE__, __LINE__);
        d->graph_stream = st;
        d->graph_cgitmax = cgitmax;
        d->graph_shift = shift;
    }
    B200_CUDA(cudaGraphLaunch(d->graph, st));
}

b200_dist_cg* finish_create(std::unique_ptr<b200_dist_cg>& d) {
    d->stream = rt().stream;
    return d.release();
}

}  // namespace

extern "C" {

int b200_dist_nccl_id(void* out128) {
    return boundary("b200_dist_nccl_id", [&] { nccl_unique_id(out128); });
}

int b200_dist_cg_create_local(b200_dist_cg** out, int k, std::int64_t n, const std::int64_t* row_ptr,
                              const std::int64_t* col_ind, const double* val) {
    return boundary("b200_dist_cg_create_local", [&] {
        ensure_init();
        if (k < 1 || k > 64) throw Error(Errc::DataError, "shard count must be 1..64");
        auto d = std::make_unique<b200_dist_cg>();
        d->world = k;
        d->n = n;
        d->bounds.resize(k + 1);
        b200_partition_rows(n, row_ptr, k, d->bounds.data());
        for (int g = 0; g < k; ++g) {
            auto s = std::make_unique<Shard>();
            const std::int64_t r0 = d->bounds[g], r1 = d->bounds[g + 1];
            load_shard(*s, n, r0, r1 - r0, row_ptr + r0, col_ind, val, k);
            d->shards.push_back(std::move(s));
        }
        d->ex = std::make_unique<LocalExchange>(k);
        d->transport = 0;
        *out = finish_create(d);
    });
}

int b200_dist_cg_create_nccl(b200_dist_cg** out, int rank, int world, const void* nccl_id, std::int64_t n,
                             const std::int64_t* bounds, const std::int64_t* row_ptr, const std::int64_t* col_ind,
                             const double* val) {
    return boundary("b200_dist_cg_create_nccl", [&] {
        ensure_init();
        if (world < 1 || rank < 0 || rank >= world) throw Error(Errc::DataError, "bad rank/world");
        auto d = std::make_unique<b200_dist_cg>();
        d->world = world;
        d->n = n;
        d->bounds.assign(bounds, bounds + world + 1);
        if (d->bounds[0] != 0 || d->bounds[world] != n) throw Error(Errc::DataError, "bounds must span [0, n]");
        auto s = std::make_unique<Shard>();
        const std::int64_t r0 = d->bounds[rank], r1 = d->bounds[rank + 1];
        // row_ptr holds this rank's rows: r1 - r0 + 1 entries (absolute offsets into col_ind/val)
        load_shard(*s, n, r0, r1 - r0, row_ptr, col_ind, val, world);
        d->shards.push_back(std::move(s));
        d->ex = std::make_unique<NcclExchange>(rank, world, nccl_id, d->bounds, d->shards[0]->cmin,
                                               d->shards[0]->cmax);
        d->rank = rank;
        d->transport = 1;
        *out = finish_create(d);
    });
}

int b200_dist_cg_create_stencil27_nccl(b200_dist_cg** out, int rank, int world, const void* nccl_id, std::int64_t nx,
                                       double diag, double offdiag) {
    return boundary("b200_dist_cg_create_stencil27_nccl", [&] {
        ensure_init();
        if (world < 1 || rank < 0 || rank >= world) throw Error(Errc::DataError, "bad rank/world");
        if (nx < 1 || nx > 1290) throw Error(Errc::DataError, "nx must be 1..1290 (int32 columns)");
        auto d = std::make_unique<b200_dist_cg>();
        d->world = world;
        d->n = nx * nx * nx;
        d->bounds = stencil_bounds(nx, world);
        auto s = std::make_unique<Shard>();
        load_shard_stencil(*s, nx, d->bounds[rank], d->bounds[rank + 1] - d->bounds[rank], diag, offdiag, world);
        d->shards.push_back(std::move(s));
        d->ex = std::make_unique<NcclExchange>(rank, world, nccl_id, d->bounds, d->shards[0]->cmin,
                                               d->shards[0]->cmax);
        d->rank = rank;
        d->transport = 1;
        *out = finish_create(d);
    });
}

int b200_dist_cg_create_stencil27_local(b200_dist_cg** out, int k, std::int64_t nx, double diag, double offdiag) {
    return boundary("b200_dist_cg_create_stencil27_local", [&] {
        ensure_init();
        if (k < 1 || k > 64) throw Error(Errc::DataError, "shard count must be 1..64");
        if (nx < 1 || nx > 1290) throw Error(Errc::DataError, "nx must be 1..1290 (int32 columns)");
        auto d = std::make_unique<b200_dist_cg>();
        d->world = k;
        d->n = nx * nx * nx;
        d->bounds = stencil_bounds(nx, k);
        for (int g = 0; g < k; ++g) {
            auto s = std::make_unique<Shard>();
            load_shard_stencil(*s, nx, d->bounds[g], d->bounds[g + 1] - d->bounds[g], diag, offdiag, k);
            d->shards.push_back(std::move(s));
        }
        d->ex = std::make_unique<LocalExchange>(k);
        d->transport = 0;
        *out = finish_create(d);
    });
}

int b200_dist_cg_bounds(const b200_dist_cg* d, std::int64_t* bounds) {
    return boundary("b200_dist_cg_bounds", [&] { std::copy(d->bounds.begin(), d->bounds.end(), bounds); });
}

void b200_dist_cg_free(b200_dist_cg* d) {
    if (!d) return;
    device_quiesce();  // caller-stream work may still use the buffers (see b200_matrix_free)
    if (d->graph) cudaGraphExecDestroy(d->graph);
    for (auto& s : d->shards) s->release();
    delete d;
}

int b200_dist_cg_reset(b200_dist_cg* d, void* stream) {
    return boundary("b200_dist_cg_reset", [&] {
        cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : d->stream;
        for (auto& s : d->shards) cg_launch_reset_x(s->v, st);
    });
}

}  // extern "C"

namespace {

PeerExchange::ShardBufs bufs_of(const Shard& s) {
    PeerExchange::ShardBufs b;
    b.p_full = s.v.p_full;
    b.z_full = s.v.z_full;
    b.row0 = s.row0;
    b.rows = s.rows;
    b.fmin = s.cmin;
    b.fmax = s.cmax;
    return b;
}

void drop_graph(b200_dist_cg* d) {
    if (d->graph) cudaGraphExecDestroy(d->graph);
    d->graph = nullptr;
    d->fused_ready = false;  // the transport changed: the slot table is rebuilt on the next run
}

void check_peer_errors(b200_dist_cg* d) {
    if (d->transport != 2) return;
    if (static_cast<PeerExchange*>(d->ex.get())->timed_out())
        throw Error(Errc::DeviceError, "peer-memory exchange: a wait for a peer timed out");
}

}  // namespace

extern "C" {

int b200_dist_cg_use_p2p_local(b200_dist_cg* d) {
    return boundary("b200_dist_cg_use_p2p_local", [&] {
        if (d->transport != 0) throw Error(Errc::DataError, "peer memory between local shards only");
        std::vector<PeerExchange::ShardBufs> b;
        for (auto& s : d->shards) b.push_back(bufs_of(*s));
        B200_CUDA(cudaStreamSynchronize(d->stream));
        auto px = std::make_unique<PeerExchange>(b);
        std::vector<CgScalars*> scs;
        for (auto& s : d->shards) scs.push_back(s->v.sc);
        px->bind_producers(scs);
        d->ex = std::move(px);
        d->transport = 2;
        drop_graph(d);
    });
}

int b200_dist_cg_p2p_export(b200_dist_cg* d, void* out) {
    return boundary("b200_dist_cg_p2p_export", [&] {
        if (d->transport != 1 || d->shards.size() != 1)
            throw Error(Errc::DataError, "IPC export: one shard per process (the NCCL driver)");
        d->pending = std::make_unique<PeerExchange>(d->rank, d->world, bufs_of(*d->shards[0]));
        d->pending->export_handles(out);
    });
}

int b200_dist_cg_p2p_attach(b200_dist_cg* d, const void* handles) {
    return boundary("b200_dist_cg_p2p_attach", [&] {
        if (!d->pending) throw Error(Errc::DataError, "call b200_dist_cg_p2p_export first");
        d->pending->attach(handles);
        d->pending->bind_producers({d->shards[0]->v.sc});
        B200_CUDA(cudaDeviceSynchronize());
        d->ex = std::move(d->pending);
        d->transport = 2;
        drop_graph(d);
    });
}

int b200_dist_cg_transport(const b200_dist_cg* d) { return d ? d->transport : -1; }

int b200_dist_cg_set_fused(b200_dist_cg* d, int on) {
    return boundary("b200_dist_cg_set_fused", [&] {
        if (!d) throw Error(Errc::DataError, "NULL solver");
        d->fused_on = on != 0;
        drop_graph(d);
    });
}

int b200_dist_cg_fused(const b200_dist_cg* d) { return d && d->fused_last ? 1 : 0; }

int b200_dist_cg_load_x(b200_dist_cg* d, const double* x_host, void* stream) {
    return boundary("b200_dist_cg_load_x", [&] {
        cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : d->stream;
        std::int64_t off = 0;
        for (auto& s : d->shards) {
            const std::size_t bytes = sizeof(double) * static_cast<std::size_t>(s->rows);
            host_in(x_host + off, bytes);
            if (bytes) B200_CUDA(cudaMemcpyAsync(s->v.x, x_host + off, bytes, cudaMemcpyHostToDevice, st));
            off += s->rows;
        }
    });
}

int b200_dist_cg_outer(b200_dist_cg* d, int cgitmax, double shift, void* stream) {
    return boundary("b200_dist_cg_outer", [&] {
        prepare_fused(d);
        dist_outer_graph(d, cgitmax, shift, stream ? static_cast<cudaStream_t>(stream) : d->stream);
    });
}

int b200_dist_cg_start_rowsum(b200_dist_cg* d, void* stream) {
    return boundary("b200_dist_cg_start_rowsum", [&] {
        dist_start_rowsum(d, stream ? static_cast<cudaStream_t>(stream) : d->stream);
    });
}

int b200_dist_cg_start(b200_dist_cg* d, void* stream) {
    return boundary("b200_dist_cg_start", [&] { dist_init(d, stream ? static_cast<cudaStream_t>(stream) : d->stream); });
}

int b200_dist_cg_step(b200_dist_cg* d, void* stream) {
    return boundary("b200_dist_cg_step", [&] { dist_step(d, stream ? static_cast<cudaStream_t>(stream) : d->stream); });
}

int b200_dist_cg_finish(b200_dist_cg* d, void* stream) {
    return boundary("b200_dist_cg_finish", [&] {
        dist_finish(d, stream ? static_cast<cudaStream_t>(stream) : d->stream);
    });
}

int b200_dist_cg_scalars(b200_dist_cg* d, void* stream, double* rho, double* rnorm) {
    return boundary("b200_dist_cg_scalars", [&] {
        cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : d->stream;
        CgScalars sc;
        B200_CUDA(cudaMemcpyAsync(&sc, d->shards[0]->v.sc, sizeof sc, cudaMemcpyDeviceToHost, st));
        B200_CUDA(cudaStreamSynchronize(st));
        check_peer_errors(d);
        if (rho) *rho = sc.rho;
        if (rnorm) *rnorm = sc.rnorm;
    });
}

int b200_dist_cg_result(b200_dist_cg* d, double* zeta, double* rnorm) {
    return boundary("b200_dist_cg_result", [&] {
        CgScalars sc;
        B200_CUDA(cudaDeviceSynchronize());
        check_peer_errors(d);
        B200_CUDA(cudaMemcpy(&sc, d->shards[0]->v.sc, sizeof sc, cudaMemcpyDeviceToHost));
        if (zeta) *zeta = sc.zeta;
        if (rnorm) *rnorm = sc.rnorm;
    });
}

int b200_dist_npb(b200_dist_cg* d, int niter, double shift, double* zeta, double* rnorm) {
    return boundary("b200_dist_npb", [&] {
        cudaStream_t st = d->stream;
        prepare_fused(d);
        for (auto& s : d->shards) cg_launch_reset_x(s->v, st);
        dist_outer_graph(d, 25, shift, st);  // NPB's untimed warm-up iteration
        for (auto& s : d->shards) cg_launch_reset_x(s->v, st);
        for (int it = 0; it < niter; ++it) dist_outer_graph(d, 25, shift, st);
        B200_CUDA(cudaStreamSynchronize(st));
        check_peer_errors(d);
        CgScalars sc;
        B200_CUDA(cudaMemcpy(&sc, d->shards[0]->v.sc, sizeof sc, cudaMemcpyDeviceToHost));
        if (zeta) *zeta = sc.zeta;
        if (rnorm) *rnorm = sc.rnorm;
    });
}

int b200_dist_cg_info(const b200_dist_cg* d, int shard, std::int64_t* row0, std::int64_t* rows, std::int64_t* nnz,
                      int32_t* tiled) {
    return boundary("b200_dist_cg_info", [&] {
        if (shard < 0 || shard >= static_cast<int>(d->shards.size())) throw Error(Errc::DataError, "no such shard");
        const Shard& s = *d->shards[shard];
        if (row0) *row0 = s.row0;
        if (rows) *rows = s.rows;
        if (nnz) *nnz = s.nnz;
        if (tiled) *tiled = s.A.tiled ? 1 : 0;
    });
}

}  // extern "C"
