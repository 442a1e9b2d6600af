// tcsr.cu — tiled CSR SpMV for matrices whose x gathers have no locality.
//
// Why: with random columns (NPB CG) the plain vector kernel is bound by the
// L1TEX pipe, not HBM — every warp-wide x gather touches ~32 distinct sectors
// (32 wavefronts), ncu: l1tex 88.7% busy at 45% of HBM peak (profiles/). Here
// x is staged in shared memory one column slab at a time (cp.async.bulk into a
// double buffer, completion on an mbarrier), so a gather costs a few bank
// cycles instead of 32 L1 wavefronts, while val/key stream from HBM with
// fully coalesced 256-bit loads.
//
// One CTA (32 warps) per tile; warp w owns a contiguous row range of the tile.
// For each slab the warp streams its (slab, warp) run: each lane walks its own
// contiguous range of the run (layout in b200.hpp) chunk by chunk, gathers x
// from smem and sums rows in registers, flushing a row that began and ended
// inside the lane straight into a shared y buffer; the rows crossing lane
// boundaries are combined once per run by a shuffle-based segmented scan.
// Rows are owned by one warp: no atomics, deterministic order. y is written
// once per tile.

#include "b200.hpp"
#include "p2p.hpp"

#include <algorithm>
#include <cstdlib>
#include <cstring>

namespace b200 {

namespace {

constexpr unsigned kFull = 0xffffffffu;
#ifndef LILAC_CTA_TRACE
#define LILAC_CTA_TRACE 0
#endif
constexpr int kMaxTrace = 1024;
#if LILAC_CTA_TRACE
__device__ unsigned long long g_cta_trace[5 * kMaxTrace];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void trace_mark(int slot, bool cond = true) {
    if (cond && threadIdx.x == 0 && blockIdx.x < kMaxTrace) g_cta_trace[5 * blockIdx.x + slot] = gtimer();
}
// fused CG: [step][CTA][8] = step start, gate passed, first slab landed, walk
// end, after barrier 1, after barrier 2, p.q summed, z/p/r staged
constexpr int kCgTraceSteps = 32, kCgTraceCtas = 160;
__device__ unsigned long long g_cg_trace[kCgTraceSteps * kCgTraceCtas * 8];
__device__ unsigned g_cg_smid[kCgTraceCtas];
__device__ unsigned g_cg_rot;  // k_cg_tiled: CTA b takes tile (b + rot) % grid (trace builds)
__device__ __forceinline__ void cg_mark(int step, int slot) {
    if (threadIdx.x == 0 && step < kCgTraceSteps && blockIdx.x < kCgTraceCtas)
        g_cg_trace[(step * kCgTraceCtas + blockIdx.x) * 8 + slot] = gtimer();
}
#else
__device__ __forceinline__ void trace_mark(int, bool = true) {}
__device__ __forceinline__ void cg_mark(int, int) {}
#endif
#ifndef LILAC_PF_AHEAD
#define LILAC_PF_AHEAD 1
#endif
constexpr int kPfAhead = LILAC_PF_AHEAD;
// dynamic shared memory of a tiled launch: the matrix's slabs + y buffer
inline std::size_t tile_smem(const TcsrDev& T) { return tcsr_smem_bytes(T.slab_w, T.rows_max); }

__device__ __forceinline__ std::uint32_t smem_addr(const void* p) {
    return static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ std::uint32_t opaque_u32(std::uint32_t v) {
    asm volatile("mov.b32 %0, %0;" : "+r"(v));
    return v;
}

__device__ __forceinline__ void mbar_init(std::uint64_t* b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_arrive_tx(std::uint64_t* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(b)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(std::uint64_t* b, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra DONE_%=;\n\t"
        "bra WAIT_%=;\n"
        "DONE_%=:\n\t}" ::"r"(smem_addr(b)),
        "r"(parity)
        : "memory");
}

// x slabs are re-read by every tile: keep them in L2 (evict_last)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, std::uint64_t* b) {
    std::uint64_t pol;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(b)), "l"(pol)
        : "memory");
}

// 256-bit load (sm_100): one instruction moves a lane's 32 contiguous bytes,
// so a warp instruction covers 1 KB with every sector fully used. The matrix
// is read once: L2 evict_first once consumed, so it does not push out x or the
// runs prefetched for the next slab.
__device__ __forceinline__ void ld_stream_f64x4(const double* p, double2& a, double2& b, std::uint64_t pol) {
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f64 {%0, %1, %2, %3}, [%4], %5;"
        : "=d"(a.x), "=d"(a.y), "=d"(b.x), "=d"(b.y)
        : "l"(p), "l"(pol));
}

__device__ __forceinline__ uint2 ld_stream_u16x4(const std::uint16_t* p, std::uint64_t pol) {
    uint2 r;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0, %1}, [%2], %3;"
        : "=r"(r.x), "=r"(r.y)
        : "l"(p), "l"(pol));
    return r;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    return v;
}

__device__ __forceinline__ int slab_len(const TcsrDev& T, int k) {
    const long long rem = static_cast<long long>(T.cols - static_cast<std::int64_t>(k) * T.slab_w);
    return static_cast<int>(rem < T.slab_w ? rem : T.slab_w);
}

// Start the copy of slab k of x into `xs` through the bulk-copy engine
// (16-byte granules). An odd last column is stored by this thread before its
// arrive (release) on the slab's mbarrier, so every consumer's wait (acquire)
// sees it together with the bulk bytes. x is never read past cols.
__device__ __forceinline__ void issue_slab(const TcsrDev& T, const double* __restrict__ x, double* xs, int k,
                                           std::uint64_t* mbar, bool tiny = false) {
    const int len = tiny ? 2 : slab_len(T, k);
    const int even = len & ~1;
    const double* src = x + static_cast<std::int64_t>(k) * T.slab_w;
    if (len & 1) xs[even] = __ldcg(src + even);  // L2: x may have been written earlier in this kernel
    mbar_arrive_tx(mbar, static_cast<unsigned>(even) * 8u);
    if (even) bulk_g2s(xs, src, static_cast<unsigned>(even) * 8u, mbar);
}

// Asynchronous L2 prefetch of [p, p+bytes) by the bulk-copy engine: no
// registers, no completion tracking. Range widened to 16-byte granules.
__device__ __forceinline__ void prefetch_l2(const void* p, std::size_t bytes) {
    const std::uintptr_t a = reinterpret_cast<std::uintptr_t>(p) & ~std::uintptr_t(15);
    const std::uintptr_t e = (reinterpret_cast<std::uintptr_t>(p) + bytes + 15) & ~std::uintptr_t(15);
    if (e > a)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(static_cast<unsigned>(e - a))
                     : "memory");
}

// Prefetch a (slab, warp) run's val and key bytes into L2.
__device__ __forceinline__ void prefetch_run(const double* vb, const std::uint16_t* kb, int lo, int hi) {
    if (hi > lo) {
        prefetch_l2(vb + lo, static_cast<std::size_t>(hi - lo) * 8);
        prefetch_l2(kb + lo, static_cast<std::size_t>(hi - lo) * 2);
    }
}

__device__ __forceinline__ double lds_f64(std::uint32_t addr) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
    return v;
}

__device__ __forceinline__ void sts_add_f64(std::uint32_t addr, double v) {
    double o;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(o) : "r"(addr));
    asm volatile("st.shared.f64 [%0], %1;" ::"r"(addr), "d"(o + v));
}


// One chunk of a lane's range: 4 nonzeros, one 256-bit val load and one
// 64-bit key load (4 x 16-bit keys), both aligned (chunks are 32 B).
struct Chunk {
    double2 v0, v1;
    uint2 k;
};

__device__ __forceinline__ void load_chunk(Chunk& c, const double* vb, const std::uint16_t* kb, unsigned e,
                                           std::uint64_t pol) {
    ld_stream_f64x4(vb + e, c.v0, c.v1, pol);
    c.k = ld_stream_u16x4(kb + e, pol);
}

// A lane's walk state over its range: the row being summed, its partial sum,
// and whether a row began inside the lane.
struct Walk {
    unsigned row;
    double acc;
    bool split;
};

// MODE: 0 = the kernel. Timing probes (LILAC_B200_TILED_PROBE, wrong results,
// never on the CG path; tools/tiled_probes.sh): 1 no x gathers, 2 no row
// sums, 3 neither (loads only), 5 = 3 without slab copies/waits, 6 = 0
// without slab copies/waits, 8 / 9 = 3 / 0 with 16-byte slab copies, 10 / 11
// = 1 / 2 without slab copies/waits.
//
// At a row start the partial of the row before it is added into the shared y
// buffer at once (predicated, no branch). That row is either complete inside
// this lane or the lane's first row, continued from earlier lanes: those
// lanes' share arrives through the segmented scan after the walk, so no row
// is written by two lanes at the same time (rows are owned by one warp).
template <int MODE>
__device__ __forceinline__ double gather_x(unsigned key, std::uint32_t xb_s) {
    if (MODE == 12)  // probe: bank-conflict-free addresses (lane + 32 * start bit)
        return lds_f64(xb_s + (((threadIdx.x & 31u) + 32u * (key & 1u)) << 3));
    return (MODE == 1 || MODE == 3) ? 1.0 : lds_f64(xb_s + ((key & 0xfffeu) << 2));
}

template <int MODE>
__device__ __forceinline__ void walk_one(Walk& w, double v, double x, unsigned key, std::uint32_t yp_s) {
    if (MODE >= 2 && MODE != 12) {
        w.acc = fma(v, x, w.acc);
        return;
    }
    const bool st = (key & kKeyStart) != 0u;
    if (st) sts_add_f64(yp_s + 8u * w.row, w.acc);
    w.split = w.split || st;
    w.row += st ? 1u : 0u;
    w.acc = fma(v, x, st ? 0.0 : w.acc);
}

template <int MODE>
__device__ __forceinline__ void walk_chunk(Walk& w, const Chunk& c, std::uint32_t xb_s, std::uint32_t yp_s) {
    walk_one<MODE>(w, c.v0.x, gather_x<MODE>(c.k.x, xb_s), c.k.x, yp_s);
    walk_one<MODE>(w, c.v0.y, gather_x<MODE>(c.k.x >> 16, xb_s), c.k.x >> 16, yp_s);
    walk_one<MODE>(w, c.v1.x, gather_x<MODE>(c.k.y, xb_s), c.k.y, yp_s);
    walk_one<MODE>(w, c.v1.y, gather_x<MODE>(c.k.y >> 16, xb_s), c.k.y >> 16, yp_s);
}

// Combines the lanes' open rows once per run: lane l holds the partial of its
// last row (row k1, sum p1; the whole lane when no row began in it). Rows are
// non-decreasing across lanes. A segmented scan over the lanes sums each row
// continued across lanes, and the segment's last lane adds it into yp[row]
// (rows are owned by this warp: no atomics, fixed order). `cont`: the lane's
// first row began in an earlier lane; inactive lanes (no chunks) are segment
// heads that store nothing.
__device__ __forceinline__ void reduce_lanes(unsigned k1, double p1, bool split, bool cont, bool active, int lane,
                                             std::uint32_t yp_s) {
    double s = p1;
    const bool head = lane == 0 || split || !cont || !active;
    const unsigned hm = __ballot_sync(kFull, head);
    const int seg = 31 - __clz(hm & (kFull >> (31 - lane)));
    const int maxspan = static_cast<int>(__reduce_max_sync(kFull, static_cast<unsigned>(lane - seg + 1)));
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        if (d >= maxspan) break;
        const double t = __shfl_up_sync(kFull, s, d);
        if (lane - d >= seg) s += t;
    }
    if (active && (lane == 31 || ((hm >> (lane + 1)) & 1u))) sts_add_f64(yp_s + 8u * k1, s);
    __syncwarp();
}

#ifndef LILAC_TILE_PIPE
#define LILAC_TILE_PIPE 4
#endif
// chunks in flight per lane: a register ring, chunk i in slot i % kPipe
constexpr int kPipe = LILAC_TILE_PIPE;

// Lane `lane`'s first kPipe chunks of the run [lo, hi) (those it has: lane l
// gets m or m + 1 chunks, m = C / 32).
__device__ __forceinline__ void load_head_chunks(Chunk (&ring)[kPipe], const double* vb, const std::uint16_t* kb,
                                                 int lo, int hi, int lane, std::uint64_t pol) {
    const int C = (hi - lo) / kChunk;
    const int cnt = (C >> 5) + (lane < (C & 31) ? 1 : 0);
    const unsigned e0 = static_cast<unsigned>(lo + kChunk * lane);
#pragma unroll
    for (int u = 0; u < kPipe; ++u)
        if (cnt > u) load_chunk(ring[u], vb, kb, e0 + 128u * u, pol);
}

// Processes a (slab, warp) run [lo, hi) (tile-relative, multiples of kChunk)
// with lane descriptor `ld` against the slab in shared memory at xb_s. The
// run's bytes were prefetched into L2 one slab ahead; each ring slot is
// refilled with the chunk kPipe ahead as soon as it has been walked.
template <int MODE>
__device__ __forceinline__ void process_run(const double* vb, const std::uint16_t* kb, int lo, int hi, unsigned ld,
                                            Chunk (&ring)[kPipe], int next_lo, int next_hi, std::uint32_t xb_s,
                                            std::uint32_t yp_s, int lane) {
    std::uint64_t pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    const int C = (hi - lo) / kChunk, m = C >> 5, r = C & 31;
    const int cnt = m + (lane < r ? 1 : 0), iters = m + (r > 0 ? 1 : 0);
    const unsigned e0 = static_cast<unsigned>(lo + kChunk * lane);  // chunk i at e0 + 128 i
    Walk w{ld & 0x7fffu, 0.0, false};
    xb_s = opaque_u32(xb_s);  // one base register: a gather address is one LEA
    // the first kPipe chunks were loaded during the previous run
    for (int i = 0; i < iters; i += kPipe) {
#pragma unroll
        for (int u = 0; u < kPipe; ++u) {
            if (i + u >= iters) break;
            if (cnt > i + u) walk_chunk<MODE>(w, ring[u], xb_s, yp_s);
            if (cnt > i + u + kPipe) load_chunk(ring[u], vb, kb, e0 + 128u * (i + u + kPipe), pol);
        }
    }
    // the next run's first chunks stream in during this run's lane reduction
    // and the next slab wait (the matrix does not depend on x)
    load_head_chunks(ring, vb, kb, next_lo, next_hi, lane, pol);
    if (MODE >= 2 && MODE != 12) {  // probe: no row sums
        if (w.acc == 12345.678) sts_add_f64(yp_s, w.acc);
        return;
    }
    reduce_lanes(w.row, w.acc, w.split, (ld & kLaneCont) != 0u, cnt > 0, lane, yp_s);
}

// Shared-memory state of a tiled SpMV CTA (slab double buffer, row sums,
// mbarriers), carried across tiles and, in the fused CG kernel, across steps.
struct TileCta {
    double* xs;  // [2][stride]: slab + zero cell (stride = slab_w + 2)
    double* yp;  // [rows_max]
    int stride;
    std::uint64_t* mbar;
    unsigned* released;
    std::uint32_t xs_s, yp_s;
    unsigned phase0, phase1;
    int tstep;  // fused CG step (LILAC_CTA_TRACE builds)
    // fused CG: the tile's z, p, r rows (global, from st_row0, st_n of them)
    // are bulk-copied into the slab buffer that goes idle when the
    // penultimate slab is released, so they land during the last slab's walk
    // (st_n = 0: no staging)
    const double *st_z, *st_p, *st_r;
    std::int64_t st_row0;
    int st_n;
    int st_buf;            // the slab buffer the rows land in
    const double* st_ps;   // where the p rows land (shared memory): the p.q epilogue reads them
};

// Where the staged rows sit in the slab buffer: an array's rows start at an
// even offset (16-byte copies) plus the row-0 parity shift.
__device__ __forceinline__ int stage_pitch(int n) { return (n + 3) & ~1; }

// Issued by one thread: the three row ranges into buffer `dst` (a slab
// buffer no warp reads any more), completion on `mbar`.
__device__ __forceinline__ void issue_stage(const TileCta& c, double* dst, std::uint64_t* mbar) {
    const int sh = static_cast<int>(c.st_row0 & 1);
    const int len = (c.st_n + sh + 1) & ~1;  // even: whole 16-byte granules
    const int pitch = stage_pitch(c.st_n);
    const unsigned bytes = static_cast<unsigned>(len) * 8u;
    asm volatile("fence.proxy.async.global;" ::: "memory");  // rows written by generic stores last step
    mbar_arrive_tx(mbar, 3u * bytes);
    bulk_g2s(dst, c.st_z + (c.st_row0 - sh), bytes, mbar);
    bulk_g2s(dst + pitch, c.st_p + (c.st_row0 - sh), bytes, mbar);
    bulk_g2s(dst + 2 * pitch, c.st_r + (c.st_row0 - sh), bytes, mbar);
}

__device__ __forceinline__ void tile_cta_init(TileCta& c, const TcsrDev& T, double* smem, std::uint64_t* mbar,
                                              unsigned* released) {
    c.stride = T.slab_w + 2;
    c.xs = smem;
    c.yp = smem + 2 * c.stride;
    c.mbar = mbar;
    c.released = released;
    // opaque copies: kept in registers instead of being rebuilt from the
    // CTA id (S2R) at every use
    c.xs_s = opaque_u32(smem_addr(c.xs));
    c.yp_s = opaque_u32(smem_addr(c.yp));
    c.phase0 = c.phase1 = 0;
    c.tstep = 0;
    c.st_z = c.st_p = c.st_r = nullptr;
    c.st_row0 = 0;
    c.st_n = 0;
    c.st_buf = 0;
    c.st_ps = nullptr;
    if (threadIdx.x == 0) {
        released[0] = released[1] = 0;
        c.xs[T.slab_w] = c.xs[c.stride + T.slab_w] = 0.0;  // padding entries read these
        mbar_init(&mbar[0], 1);
        mbar_init(&mbar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
}

// y = A x over this CTA's tiles; with DOT, returns this thread's share of
// x.y over the tiles' rows (x read at dot_off + row). COHERENT: x may have been
// written earlier in the same kernel (fused CG): read it through L2 only.
// gate (fused CG): a grid barrier this CTA already arrived at; thread 0 waits
// for it only before the first slab copy of x, so the tile prologue (y
// buffer, L2 prefetch, descriptors, head chunks: nothing that depends on x)
// overlaps the barrier.
// A gate on peer flags (the sharded fused CG): every sender's flag must reach
// `epoch` (p slices pushed into this shard's replica) before x is read; a wait
// without progress for 5 s sets *err and gives up (a broken link fails the
// run instead of hanging the GPU).
struct FlagGate {
    const unsigned long long* flags;
    int n;
    unsigned long long epoch;
    int* err;
};

__device__ __forceinline__ unsigned long long gtime_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ void wait_flags(const unsigned long long* flags, int n, unsigned long long epoch, int* err) {
    if (*reinterpret_cast<volatile int*>(err)) return;
    const unsigned long long t0 = gtime_ns();
    for (int r = 0; r < n; ++r) {
        unsigned long long v;
        for (;;) {
            asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flags + r) : "memory");
            if (v >= epoch) break;
            if (gtime_ns() - t0 > 5000000000ull) {
                *reinterpret_cast<volatile int*>(err) = 1;
                return;
            }
        }
    }
}

// cta / ncta: this CTA's index among the CTAs sharing the matrix (-1: the
// whole grid; the sharded fused CG runs several shards' CTA groups in one grid)
template <bool DOT, int MODE, bool COHERENT>
__device__ __forceinline__ double spmv_tiles(const TcsrDev& T, const double* x, double* y, std::int64_t dot_off,
                                             TileCta& c, const unsigned* gate = nullptr, unsigned gate_target = 0,
                                             const FlagGate* fg = nullptr, int cta = -1, int ncta = -1) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    double* xs = c.xs;
    double* yp = c.yp;
    double pq = 0.0;
    const int P = T.parts;
    const std::int64_t items = T.ntiles * P;
    const std::int64_t my_cta = cta < 0 ? static_cast<std::int64_t>(blockIdx.x) : cta;
    const std::int64_t n_cta = ncta < 0 ? static_cast<std::int64_t>(gridDim.x) : ncta;
    for (std::int64_t item = my_cta; item < items; item += n_cta) {
        const std::int64_t t = item / P;
        const int part = static_cast<int>(item - t * P);
        const int k0 = part * T.nslabs / P, k1 = (part + 1) * T.nslabs / P;  // this part's slabs
        // Slab parts (small matrices, a few slabs per CTA) with no gate to
        // wait for: the first two slab copies start before anything else,
        // their arrival being the longest leg of the part's start (NPB C 1/8
        // block: 18.4 -> 16.5 us). With one part per tile (large matrices)
        // they wait behind the head chunk loads instead, which must lead
        // (whole NPB C: 72.2 vs 73.2 us issued first).
        bool issued = false;
        if (tid == 0 && P > 1 && !gate && !fg && k1 > k0 && (MODE < 5 || MODE == 8 || MODE == 9 || MODE == 12)) {
            if (COHERENT) asm volatile("fence.proxy.async.global;" ::: "memory");  // x: generic writes -> bulk reads
            issue_slab(T, x, xs, k0, &c.mbar[0], MODE == 8 || MODE == 9);
            if (k0 + 1 < k1) issue_slab(T, x, xs + c.stride, k0 + 1, &c.mbar[1], MODE == 8 || MODE == 9);
            issued = true;
        }
        const std::int64_t row0 = T.tile_row0[t];
        const int nrows = static_cast<int>(T.tile_row0[t + 1] - row0);
        const std::int64_t base = T.tile_base[t];
        const double* vb = T.val + base;
        const std::uint16_t* kb = T.key + base;
        const std::int32_t* wo = T.woff + t * (static_cast<std::int64_t>(T.nslabs) * kTileWarps + 1);
        const std::uint16_t* lr = T.lrow + t * (static_cast<std::int64_t>(T.nslabs) * kTileWarps) * 32 + lane;
        // this warp's run bounds, lane k holding slab k's (one coalesced load
        // per tile instead of a dependent L1 round trip at every run start)
        const int wlo = lane < T.nslabs ? __ldg(wo + lane * kTileWarps + warp) : 0;
        const int whi = lane < T.nslabs ? __ldg(wo + lane * kTileWarps + warp + 1) : 0;
        auto run_lo = [&](int k) { return k < 32 ? __shfl_sync(kFull, wlo, k) : __ldg(wo + k * kTileWarps + warp); };
        auto run_hi = [&](int k) {
            return k < 32 ? __shfl_sync(kFull, whi, k) : __ldg(wo + k * kTileWarps + warp + 1);
        };
        for (int r = tid; r < nrows; r += kTileThreads) yp[r] = 0.0;
        // No L2 prefetch of the first runs here (the loop prefetches from
        // k0 + 1 on): at a launch every CTA's first runs (33 MB on NPB C)
        // would queue ahead of the slab copies, which land ~2 us later that
        // way (CTA trace, tools/cta_trace.py; 72.8 -> 72.0 us, 505 -> 507 it/s).
        // lane descriptors and each run's first chunk are loaded one run ahead (registers)
        unsigned dnext = k1 > k0 ? __ldg(lr + (k0 * kTileWarps + warp) * 32) : 0u;
        Chunk ring[kPipe];
        if (k1 > k0) {
            std::uint64_t pol;
            asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
            load_head_chunks(ring, vb, kb, run_lo(k0), run_hi(k0), lane, pol);
        }
        if (tid == 0 && gate) {
            unsigned v;
            do {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(gate) : "memory");
            } while (v < gate_target);
            gate = nullptr;
        }
        if (tid == 0 && fg) wait_flags(fg->flags, fg->n, fg->epoch, fg->err);
        fg = nullptr;
        if (COHERENT) cg_mark(c.tstep, 1);
        if (tid == 0 && !issued && k1 > k0 && (MODE < 5 || MODE == 8 || MODE == 9 || MODE == 12)) {
            if (COHERENT) asm volatile("fence.proxy.async.global;" ::: "memory");  // x: generic writes -> bulk reads
            issue_slab(T, x, xs, k0, &c.mbar[0], MODE == 8 || MODE == 9);
            if (k0 + 1 < k1) issue_slab(T, x, xs + c.stride, k0 + 1, &c.mbar[1], MODE == 8 || MODE == 9);
        }
        // one slab: buffer 1 idles the whole SpMV, so the fused CG's rows of
        // this CTA (its own data) are staged there from the start
        if (COHERENT && tid == 0 && c.st_n > 0 && P == 1 && k1 - k0 == 1) issue_stage(c, xs + c.stride, &c.mbar[1]);
        __syncthreads();
        // Free-running slabs: a warp moves on as soon as the next slab has
        // landed; the last warp to release a buffer refills it (no CTA barrier).
        for (int k = k0; k < k1; ++k) {
            const int buf = (k - k0) & 1;
            if (MODE == 5 || MODE == 6 || MODE == 10 || MODE == 11) {
            } else if (buf == 0) {
                mbar_wait(&c.mbar[0], c.phase0);
                c.phase0 ^= 1;
            } else {
                mbar_wait(&c.mbar[1], c.phase1);
                c.phase1 ^= 1;
            }
            if (!DOT && !COHERENT && k == k0) trace_mark(2);
            if (COHERENT && k == k0) cg_mark(c.tstep, 2);
            const unsigned dcur = dnext;
            if (k + 1 < k1) {
                if (k + kPfAhead < k1) {
                    const int plo = run_lo(k + kPfAhead), phi = run_hi(k + kPfAhead);
                    if (lane == 0) prefetch_run(vb, kb, plo, phi);
                }
                dnext = __ldg(lr + ((k + 1) * kTileWarps + warp) * 32);
            }
            const bool more = k + 1 < k1;
            const int nlo = more ? run_lo(k + 1) : 0, nhi = more ? run_hi(k + 1) : 0;
            process_run<MODE == 5 || MODE == 8 ? 3 : (MODE == 6 || MODE == 9 ? 0 : (MODE == 10 || MODE == 11 ? MODE - 9 : MODE))>(
                vb, kb, run_lo(k), run_hi(k), dcur, ring, nlo, nhi,
                c.xs_s + 8u * static_cast<unsigned>(buf * c.stride), c.yp_s, lane);
            __syncwarp();
            if (lane == 0) {
                __threadfence_block();
                if (atomicAdd(&c.released[buf], 1u) == kTileWarps - 1) {
                    c.released[buf] = 0;
                    if (k + 2 < k1 && (MODE < 5 || MODE == 8 || MODE == 9 || MODE == 12)) {
                        if (COHERENT) asm volatile("fence.proxy.async.global;" ::: "memory");
                        issue_slab(T, x, xs + buf * c.stride, k + 2, &c.mbar[buf], MODE == 8 || MODE == 9);
                    } else if (COHERENT && c.st_n > 0 && P == 1 && k + 2 == k1) {
                        issue_stage(c, xs + buf * c.stride, &c.mbar[buf]);
                    }
                }
            }
        }
        __syncthreads();  // every row of the tile (this part's slabs) is complete
        if (!DOT && !COHERENT) trace_mark(3);
        if (COHERENT) cg_mark(c.tstep, 3);
        if (P == 1) {
            if (COHERENT && c.st_n > 0) {
                // the staged rows (issued at the penultimate slab) hold this
                // tile's p: the dot needs no global round trip
                if (c.st_buf == 0) {
                    mbar_wait(&c.mbar[0], c.phase0);
                    c.phase0 ^= 1;
                } else {
                    mbar_wait(&c.mbar[1], c.phase1);
                    c.phase1 ^= 1;
                }
                for (int r = tid; r < nrows; r += kTileThreads) {
                    const double v = yp[r];
                    y[row0 + r] = v;
                    if (DOT) pq += v * c.st_ps[r];
                }
            } else {
                for (int r = tid; r < nrows; r += kTileThreads) {
                    const double v = yp[r];
                    y[row0 + r] = v;
                    if (DOT) pq += v * (COHERENT ? __ldcg(x + dot_off + row0 + r) : __ldg(x + dot_off + row0 + r));
                }
            }
        } else {
            // this part's row sums out; the tile's last part adds all parts
            // in part order (the same bits whichever part finishes last)
            double* mine = T.ypart + static_cast<std::int64_t>(part) * T.rows + row0;
            for (int r = tid; r < nrows; r += kTileThreads) __stcg(mine + r, yp[r]);
            __syncthreads();
            // one fence after the barrier publishes the whole CTA's stores
            // (cumulative) before the ticket, as a per-thread fence would
            if (tid == 0) {
                __threadfence();
                c.released[2] = atomicAdd(&T.tile_done[t], 1u) == static_cast<unsigned>(P - 1) ? 1u : 0u;
            }
            __syncthreads();
            if (c.released[2]) {  // CTA-uniform
                __threadfence();
                double tpq = 0.0;
                for (int r = tid; r < nrows; r += kTileThreads) {
                    double v = __ldcg(T.ypart + row0 + r);
                    for (int q = 1; q < P; ++q) v += __ldcg(T.ypart + static_cast<std::int64_t>(q) * T.rows + row0 + r);
                    y[row0 + r] = v;
                    if (DOT) tpq += v * (COHERENT ? __ldcg(x + dot_off + row0 + r) : __ldg(x + dot_off + row0 + r));
                }
                if (DOT) {
                    // the tile's share of x.y by tile (not by CTA: which CTA
                    // finalises a tile varies run to run), summed later in
                    // tile order
                    __shared__ double tred[kTileWarps];
                    tpq = warp_sum(tpq);
                    if (lane == 0) tred[warp] = tpq;
                    __syncthreads();
                    if (warp == 0) {
                        tpq = warp_sum(lane < kTileWarps ? tred[lane] : 0.0);
                        if (lane == 0) T.tile_pq[t] = tpq;
                    }
                }
                if (tid == 0) T.tile_done[t] = 0u;  // next launch
            }
        }
        __syncthreads();  // yp reused by the next tile
    }
    return pq;
}

template <bool DOT, int MODE = 0>
__global__ void __launch_bounds__(kTileThreads, 1)
    k_spmv_tiled(TcsrDev T, const double* __restrict__ x, double* __restrict__ y, double* partials,
                 unsigned int* ticket, CgScalars* sc, std::int64_t dot_off) {
    extern __shared__ __align__(128) double smem[];
    __shared__ __align__(8) std::uint64_t mbar[2];
    __shared__ unsigned released[3];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    TileCta c;
#if LILAC_CTA_TRACE
    if (!DOT && tid == 0 && blockIdx.x < kMaxTrace) {
        unsigned smid;
        asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
        g_cta_trace[5 * blockIdx.x] = smid;
    }
    trace_mark(1, !DOT);
#endif
    tile_cta_init(c, T, smem, mbar, released);
    if (DOT) {  // CG step: launched programmatically after update_p
        pdl_trigger();
        if (lane == 0 && blockIdx.x < T.ntiles * T.parts && T.nslabs > 0) {  // the matrix does not depend on it
            const std::int64_t t = blockIdx.x / T.parts;
            const int k0 = static_cast<int>(blockIdx.x - t * T.parts) * T.nslabs / T.parts;
            const std::int32_t* wo = T.woff + t * (static_cast<std::int64_t>(T.nslabs) * kTileWarps + 1) +
                                     k0 * kTileWarps;
            prefetch_run(T.val + T.tile_base[t], T.key + T.tile_base[t], wo[warp], wo[warp + 1]);
        }
        pdl_wait();
    }
    __syncthreads();
    const double pq = spmv_tiles<DOT, MODE, false>(T, x, y, dot_off, c);
    trace_mark(4, !DOT);

    if (DOT) {
        __shared__ double red[kTileWarps];
        __shared__ bool last;
        double s = warp_sum(pq);
        if (lane == 0) red[warp] = s;
        __syncthreads();
        if (warp == 0) {
            s = warp_sum(lane < kTileWarps ? red[lane] : 0.0);
            if (lane == 0) partials[blockIdx.x] = s;
        }
        __syncthreads();
        if (tid == 0) {  // thread 0 wrote the partial: its fence orders it before the ticket
            __threadfence();
            last = atomicAdd(ticket, 1u) == gridDim.x - 1;
        }
        __syncthreads();
        if (last) {
            __threadfence();
            // per-CTA partials, or with slab parts the per-tile ones (CTA partials are 0)
            const double* src = T.parts > 1 ? T.tile_pq : partials;
            const unsigned n = T.parts > 1 ? static_cast<unsigned>(T.ntiles) : gridDim.x;
            double a = 0.0;
            for (unsigned i = tid; i < n; i += kTileThreads) a += __ldcg(src + i);
            a = warp_sum(a);
            __syncthreads();
            if (lane == 0) red[warp] = a;
            __syncthreads();
            if (warp == 0) {
                a = warp_sum(lane < kTileWarps ? red[lane] : 0.0);
                if (lane == 0) {
                    if (sc->nranks > 1) {
                        p2p_publish(sc, &a, 1);  // the shard's partial; alpha after the exchange
                    } else {
                        sc->d = a;
                        sc->rho0 = sc->rho;
                        sc->alpha = sc->rho / a;
                    }
                    *ticket = 0u;
                }
            }
        }
    }
}

// Grid-wide barrier of a co-resident (cooperative) grid: monotonic counter,
// `target` advances by gridDim.x per barrier.
__device__ __forceinline__ void grid_sync(unsigned* bar, unsigned& target) {
    __syncthreads();
    target += gridDim.x;
    if (threadIdx.x == 0) {
        // release: the CTA's writes (ordered before by __syncthreads) become
        // visible with the arrival; acquire on the poll below
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
        unsigned v;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
        } while (v < target);
    }
    __syncthreads();
}

// Arrival only (the wait is the gate of the next spmv_tiles).
__device__ __forceinline__ void grid_arrive(unsigned* bar, unsigned& target) {
    __syncthreads();
    target += gridDim.x;
    if (threadIdx.x == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
}

// Sum of every thread's v, returned to all threads (fixed tree).
__device__ __forceinline__ double cta_sum(double v, double* red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    if (warp == 0) {
        v = warp_sum(lane < kTileWarps ? red[lane] : 0.0);
        if (lane == 0) red[kTileWarps] = v;
    }
    __syncthreads();
    return red[kTileWarps];
}

// Sum of p[0..n) (the CTAs' partials) in a fixed order: the same bits in
// every CTA.
__device__ __forceinline__ double cta_sum_parts(const double* p, int n, double* red) {
    double a = 0.0;
    for (int i = threadIdx.x; i < n; i += kTileThreads) a += __ldcg(p + i);
    return cta_sum(a, red);
}

// `steps` NPB CG iterations (conj_grad's inner loop) on one GPU in one
// persistent cooperative kernel: per step q = A p with the p.q partials
// (spmv_tiles), grid barrier, alpha, z/r update of the CTA's own tile rows
// with the r.r partials, grid barrier, beta, p update of its own rows, grid
// barrier. Replaces 3 launches per step; dots are deterministic (fixed
// per-CTA partition, every CTA sums the partials in CTA order), updates use
// explicitly rounded mul/add like k_cg_update_zr/k_cg_update_p.
#ifndef LILAC_CG_PREFETCH
#define LILAC_CG_PREFETCH 1  // 0 / 1 / 2 / 3 slabs: 494.8 / 498.2 / 493.6 / 484.7 NPB C it/s
#endif
constexpr int kCgPrefetch = LILAC_CG_PREFETCH;  // slabs of the next step's runs prefetched during the barriers
#ifndef LILAC_CG_ASYNC_STAGE
#define LILAC_CG_ASYNC_STAGE 1
#endif
constexpr bool kCgAsyncStage = LILAC_CG_ASYNC_STAGE != 0;  // z, p, r rows staged by bulk copies during the last slab

__global__ void __launch_bounds__(kTileThreads, 1) k_cg_tiled(TcsrDev T, CgVectors v, int steps) {
    extern __shared__ __align__(128) double smem[];
    __shared__ __align__(8) std::uint64_t mbar[2];
    __shared__ unsigned released[3];
    __shared__ double red[kTileWarps + 1];
    const int tid = threadIdx.x;
#if LILAC_CTA_TRACE
    const unsigned me = (blockIdx.x + g_cg_rot) % gridDim.x;  // trace builds: which tile a CTA takes can rotate
#else
    const unsigned me = blockIdx.x;
#endif
    TileCta c;
    tile_cta_init(c, T, smem, mbar, released);
    __syncthreads();
    unsigned target = 0;
    unsigned* bar = &v.sc->bar;
    double rho = __ldcg(&v.sc->rho);
    double* pq_part = v.partials;
    double* rr_part = v.partials + 2 * kMaxParts;
    // the next step's first runs of this CTA's first item, loaded once
    __shared__ int pf_lo[kCgPrefetch > 0 ? kCgPrefetch : 1][kTileWarps], pf_hi[kCgPrefetch > 0 ? kCgPrefetch : 1][kTileWarps];
    __shared__ const double* pf_vb;
    __shared__ const std::uint16_t* pf_kb;
    const bool pf_on = kCgPrefetch > 0 && me < T.ntiles * T.parts;
    if (pf_on) {
        const std::int64_t t = me / T.parts;
        const int part = static_cast<int>(me - t * T.parts);
        const int k0 = part * T.nslabs / T.parts, k1 = (part + 1) * T.nslabs / T.parts;
        const std::int32_t* wo = T.woff + t * (static_cast<std::int64_t>(T.nslabs) * kTileWarps + 1);
        if (tid == 0) {
            pf_vb = T.val + T.tile_base[t];
            pf_kb = T.key + T.tile_base[t];
        }
        for (int e = tid; e < (kCgPrefetch > 0 ? kCgPrefetch : 1) * kTileWarps; e += kTileThreads) {
            const int q = e / kTileWarps, w = e - q * kTileWarps, k = k0 + q;
            pf_lo[q][w] = k < k1 ? wo[k * kTileWarps + w] : 0;
            pf_hi[q][w] = k < k1 ? wo[k * kTileWarps + w + 1] : 0;
        }
    }
    __syncthreads();
    // One tile per CTA: the tile's z, p, r rows are staged into a slab buffer
    // and q stays in the y buffer, so the updates below touch no global loads.
    // The staging is three bulk copies issued when the penultimate slab's
    // buffer is released (they land during the last slab's walk), or with a
    // single slab at the SpMV's start into the idle second buffer; loads after
    // the SpMV only when the rows do not fit one buffer.
    const bool one_tile = T.parts == 1 && T.ntiles <= gridDim.x && me < T.ntiles;
    const std::int64_t crow0 = one_tile ? T.tile_row0[me] : 0;
    const int cn = one_tile ? static_cast<int>(T.tile_row0[me + 1] - crow0) : 0;
    const bool async_stage = kCgAsyncStage && one_tile && T.nslabs >= 1 && 3 * stage_pitch(cn) <= c.stride;
    const bool cached = async_stage || (one_tile && 3 * cn <= 2 * c.stride);  // z, p, r rows fit the slab buffers
    const int sbuf = T.nslabs >= 2 ? (T.nslabs - 2) & 1 : 1;  // the buffer of slab nslabs - 2 (one slab: buffer 1)
    const int sh = static_cast<int>(crow0 & 1), pitch = stage_pitch(cn);
    double* zs = async_stage ? c.xs + sbuf * c.stride + sh : c.xs;
    double* ps = async_stage ? zs + pitch : c.xs + cn;
    double* rs = async_stage ? zs + 2 * pitch : c.xs + 2 * cn;
    if (async_stage) {
        c.st_z = v.z;
        c.st_p = v.p;
        c.st_r = v.r;
        c.st_row0 = crow0;
        c.st_n = cn;
        c.st_buf = sbuf;
        c.st_ps = ps;
    }
#if LILAC_CTA_TRACE
    if (tid == 0 && blockIdx.x < kCgTraceCtas) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        g_cg_smid[blockIdx.x] = smid;
    }
#endif
    for (int it = 0; it < steps; ++it) {
        c.tstep = it;
        cg_mark(it, 0);
        const double pq = cta_sum(spmv_tiles<true, 0, true>(T, v.p_full, v.q, 0, c, it > 0 ? bar : nullptr, target, nullptr,
                                                            static_cast<int>(me), -1),
                                  red);
        cg_mark(it, 6);
        if (tid == 0) pq_part[blockIdx.x] = pq;
        if (kCgPrefetch > 0 && it + 1 < steps && pf_on && (tid & 31) == 0) {
            // HBM is idle until the next step's SpMV (barriers, vector
            // updates, CTAs waiting for the slowest one): pull the runs of
            // this CTA's first slabs of the next step into L2 now (bounds
            // from shared memory: no global round trip before the barrier)
            const int warp = tid >> 5;
            for (int q = 0; q < kCgPrefetch; ++q)
                if (pf_lo[q][warp] < pf_hi[q][warp]) prefetch_run(pf_vb, pf_kb, pf_lo[q][warp], pf_hi[q][warp]);
        }
        if (async_stage) {
            // the staging copies landed: waited for in spmv_tiles' epilogue
        } else if (cached) {
            for (int r = tid; r < cn; r += kTileThreads) {
                zs[r] = __ldcg(v.z + crow0 + r);
                ps[r] = __ldcg(v.p + crow0 + r);
                rs[r] = __ldcg(v.r + crow0 + r);
            }
        }
        cg_mark(it, 7);
        grid_sync(bar, target);
        cg_mark(it, 4);
        const double d = T.parts > 1 ? cta_sum_parts(T.tile_pq, static_cast<int>(T.ntiles), red)
                                     : cta_sum_parts(pq_part, gridDim.x, red);
        const double alpha = rho / d;
        double rr = 0.0;
        if (cached) {
            for (int r = tid; r < cn; r += kTileThreads) {
                const double zi = __dadd_rn(zs[r], __dmul_rn(alpha, ps[r]));
                const double ri = __dsub_rn(rs[r], __dmul_rn(alpha, c.yp[r]));
                v.z[crow0 + r] = zi;
                v.r[crow0 + r] = ri;
                rs[r] = ri;
                rr += ri * ri;
            }
        } else {
            for (std::int64_t t = me; t < T.ntiles; t += gridDim.x) {
                const std::int64_t row0 = T.tile_row0[t], row1 = T.tile_row0[t + 1];
                for (std::int64_t i = row0 + tid; i < row1; i += kTileThreads) {
                    const double zi = __dadd_rn(v.z[i], __dmul_rn(alpha, v.p[i]));
                    const double ri = __dsub_rn(v.r[i], __dmul_rn(alpha, v.q[i]));
                    v.z[i] = zi;
                    v.r[i] = ri;
                    rr += ri * ri;
                }
            }
        }
        rr = cta_sum(rr, red);
        if (tid == 0) {
            rr_part[blockIdx.x] = rr;
            if (blockIdx.x == 0) {
                v.sc->d = d;
                v.sc->rho0 = rho;
                v.sc->alpha = alpha;
            }
        }
        grid_sync(bar, target);
        cg_mark(it, 5);
        const double rho_new = cta_sum_parts(rr_part, gridDim.x, red);
        const double beta = rho_new / rho;
        if (cached) {
            for (int r = tid; r < cn; r += kTileThreads) v.p[crow0 + r] = __dadd_rn(rs[r], __dmul_rn(beta, ps[r]));
            // the next step's slab copies (async proxy) overwrite these generic writes
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        } else {
            for (std::int64_t t = me; t < T.ntiles; t += gridDim.x) {
                const std::int64_t row0 = T.tile_row0[t], row1 = T.tile_row0[t + 1];
                for (std::int64_t i = row0 + tid; i < row1; i += kTileThreads)
                    v.p[i] = __dadd_rn(v.r[i], __dmul_rn(beta, v.p[i]));
            }
        }
        if (tid == 0 && blockIdx.x == 0) {
            v.sc->rho = rho_new;
            v.sc->beta = beta;
        }
        rho = rho_new;
        grid_arrive(bar, target);  // p complete before any CTA's slabs read it: waited on in spmv_tiles
    }
}

int g_sms = 0;

// ---- the sharded CG in one persistent kernel ------------------
//
// k_cg_tiled for a row shard whose p replica is filled by its peers over the
// peer-memory exchange (p2p.hpp): per CG step the tiled SpMV of the shard
// (gated on every sender's p flag), the p.q partial of the shard published
// into every peer's mailbox (NVLink stores + a release.sys flag), a wait for
// all shards' partials and alpha from their rank-order sum; the z/r update
// with r.r the same way; then the p update, each new value stored locally and
// into every peer's replica (only the rows in its column footprint), and this
// shard's flags raised. One launch replaces 6 kernels per CG step. The CTAs
// of a shard synchronise on a shard-local counter; shards only through the
// flags, so one process per GPU runs one slot, and k slots in one cooperative
// grid emulate k shards on one GPU (how it is tested here). Every wait gives
// up after 5 s and sets the mailbox error flag.
struct DistSlot {
    TcsrDev T;
    CgVectors v;
    unsigned* bar;  // the slot's barrier counter (zeroed before the launch)
};

__device__ __forceinline__ void slot_sync(unsigned* bar, unsigned& target, unsigned n, int* err) {
    __syncthreads();
    target += n;
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
        const unsigned long long t0 = gtime_ns();
        unsigned v;
        for (;;) {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
            if (v >= target) break;
            if (gtime_ns() - t0 > 5000000000ull) {
                *reinterpret_cast<volatile int*>(err) = 1;
                break;
            }
        }
    }
    __syncthreads();
}

// this shard's partial into slot (e & 1) of every peer's mailbox, then its flags
__device__ __forceinline__ void dist_publish(const P2pDesc& d, double val, unsigned long long e) {
    const unsigned long long slot = e & 1ull;
    for (int r = 0; r < d.world; ++r)
        d.peers[r].gathered[(slot * kP2pMaxWorld + d.rank) * kP2pMaxPart] = val;
    __threadfence_system();
    for (int r = 0; r < d.world; ++r)
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(d.peers[r].flags + d.rank), "l"(e) : "memory");
}

// every shard's partial of epoch e, summed in rank order (cg_fin_apply's order)
__device__ __forceinline__ double dist_gather_sum(const P2pDesc& d, unsigned long long e) {
    const unsigned long long slot = e & 1ull;
    double a = 0.0;
    for (int r = 0; r < d.world; ++r)
        a += *reinterpret_cast<volatile double*>(d.mb.gathered + (slot * kP2pMaxWorld + r) * kP2pMaxPart);
    return a;
}

__global__ void __launch_bounds__(kTileThreads, 1)
    k_cg_tiled_dist(const DistSlot* __restrict__ slots, int nslots, int steps) {
    extern __shared__ __align__(128) double smem[];
    __shared__ __align__(8) std::uint64_t mbar[2];
    __shared__ unsigned released[3];
    __shared__ double red[kTileWarps + 1];
    __shared__ unsigned long long epoch0;
    const int tid = threadIdx.x;
    const int cpr = static_cast<int>(gridDim.x) / nslots;
    const int slot = static_cast<int>(blockIdx.x) / cpr;
    if (slot >= nslots) return;
    const int cta = static_cast<int>(blockIdx.x) - slot * cpr;
    const DistSlot& S = slots[slot];
    const TcsrDev& T = S.T;
    const CgVectors& v = S.v;
    const P2pDesc& d = *static_cast<const P2pDesc*>(v.sc->p2p);
    TileCta c;
    tile_cta_init(c, T, smem, mbar, released);
    if (tid == 0) epoch0 = *d.mb.epoch;  // read by every CTA before any publish (the first needs all CTAs)
    __syncthreads();
    unsigned long long e = epoch0;
    unsigned target = 0;
    double rho = __ldcg(&v.sc->rho);
    double* pq_part = v.partials;
    double* rr_part = v.partials + 2 * kMaxParts;
    const std::int64_t* send = d.send;
    // One tile per CTA (one shard per GPU): the tile's z, p, r rows are
    // bulk-copied into the slab buffer that goes idle at the penultimate slab
    // (k_cg_tiled's staging), q stays in the y buffer, and the updates below
    // run from shared memory
    const bool one_tile = T.parts == 1 && T.ntiles <= cpr && cta < T.ntiles;
    const std::int64_t crow0 = one_tile ? T.tile_row0[cta] : 0;
    const int cn = one_tile ? static_cast<int>(T.tile_row0[cta + 1] - crow0) : 0;
    const bool staged = kCgAsyncStage && one_tile && T.nslabs >= 1 && 3 * stage_pitch(cn) <= c.stride;
    const int sbuf = T.nslabs >= 2 ? (T.nslabs - 2) & 1 : 1;
    double* zs = c.xs + sbuf * c.stride + static_cast<int>(crow0 & 1);
    double* ps = zs + stage_pitch(cn);
    double* rs = zs + 2 * stage_pitch(cn);
    // the next step's first runs of this CTA's first item (L2 prefetch
    // during the exchanges), bounds loaded once into shared memory
    __shared__ int pf_lo[kTileWarps], pf_hi[kTileWarps];
    __shared__ const double* pf_vb;
    __shared__ const std::uint16_t* pf_kb;
    const bool pf_on = kCgPrefetch > 0 && cta < T.ntiles * T.parts;
    if (pf_on) {
        const std::int64_t t = cta / T.parts;
        const int part = static_cast<int>(cta - t * T.parts);
        const int k0 = part * T.nslabs / T.parts, k1 = (part + 1) * T.nslabs / T.parts;
        const std::int32_t* wo = T.woff + t * (static_cast<std::int64_t>(T.nslabs) * kTileWarps + 1);
        if (tid == 0) {
            pf_vb = T.val + T.tile_base[t];
            pf_kb = T.key + T.tile_base[t];
        }
        if (tid < kTileWarps) {
            pf_lo[tid] = k0 < k1 ? wo[k0 * kTileWarps + tid] : 0;
            pf_hi[tid] = k0 < k1 ? wo[k0 * kTileWarps + tid + 1] : 0;
        }
    }
    __syncthreads();
    if (staged) {
        c.st_z = v.z;
        c.st_p = v.p;
        c.st_r = v.r;
        c.st_row0 = crow0;
        c.st_n = cn;
        c.st_buf = sbuf;
        c.st_ps = ps;
    }
    for (int it = 0; it < steps; ++it) {
        // q = A p over the shard once every sender's p slice (epoch e) is in
        const FlagGate fg{d.mb.flags, d.world, e, d.mb.err};
        const double pq = cta_sum(spmv_tiles<true, 0, true>(T, v.p_full, v.q, v.row0, c, nullptr, 0, &fg, cta, cpr),
                                  red);
        if (tid == 0) pq_part[cta] = pq;
        if (pf_on && it + 1 < steps && (tid & 31) == 0 && pf_lo[tid >> 5] < pf_hi[tid >> 5])
            prefetch_run(pf_vb, pf_kb, pf_lo[tid >> 5], pf_hi[tid >> 5]);
        slot_sync(S.bar, target, static_cast<unsigned>(cpr), d.mb.err);
        const double dpart = T.parts > 1 ? cta_sum_parts(T.tile_pq, static_cast<int>(T.ntiles), red)
                                         : cta_sum_parts(pq_part, cpr, red);
        ++e;
        if (cta == 0 && tid == 0) dist_publish(d, dpart, e);
        if (tid == 0) wait_flags(d.mb.flags, d.world, e, d.mb.err);
        __syncthreads();
        const double dsum = dist_gather_sum(d, e);
        const double alpha = rho / dsum;
        if (cta == 0 && tid == 0) {
            v.sc->d = dsum;
            v.sc->rho0 = rho;
            v.sc->alpha = alpha;
        }
        double rr = 0.0;
        if (staged) {
            for (int r = tid; r < cn; r += kTileThreads) {
                const double zi = __dadd_rn(zs[r], __dmul_rn(alpha, ps[r]));
                const double ri = __dsub_rn(rs[r], __dmul_rn(alpha, c.yp[r]));
                v.z[crow0 + r] = zi;
                v.r[crow0 + r] = ri;
                rs[r] = ri;
                rr += ri * ri;
            }
        } else {
            for (std::int64_t i = static_cast<std::int64_t>(cta) * kTileThreads + tid; i < v.n;
                 i += static_cast<std::int64_t>(cpr) * kTileThreads) {
                const double zi = __dadd_rn(__ldcg(v.z + i), __dmul_rn(alpha, __ldcg(v.p + i)));
                const double ri = __dsub_rn(__ldcg(v.r + i), __dmul_rn(alpha, __ldcg(v.q + i)));
                v.z[i] = zi;
                v.r[i] = ri;
                rr += ri * ri;
            }
        }
        rr = cta_sum(rr, red);
        if (tid == 0) rr_part[cta] = rr;
        slot_sync(S.bar, target, static_cast<unsigned>(cpr), d.mb.err);
        const double rpart = cta_sum_parts(rr_part, cpr, red);
        ++e;
        if (cta == 0 && tid == 0) dist_publish(d, rpart, e);
        if (tid == 0) wait_flags(d.mb.flags, d.world, e, d.mb.err);
        __syncthreads();
        const double rho_new = dist_gather_sum(d, e);
        const double beta = rho_new / rho;
        if (cta == 0 && tid == 0) {
            v.sc->rho = rho_new;
            v.sc->beta = beta;
        }
        rho = rho_new;
        // p = r + beta p on the owned rows, stored here and into every peer's
        // replica rows its SpMV reads
        bool pushed = false;  // this thread stored into a peer's replica
        if (staged) {
            for (int r = tid; r < cn; r += kTileThreads) {
                const std::int64_t i = crow0 + r;
                const double pv = __dadd_rn(rs[r], __dmul_rn(beta, ps[r]));
                v.p[i] = pv;
                for (int q = 0; q < d.world; ++q)
                    if (q != d.rank && i >= send[2 * q] && i < send[2 * q + 1]) {
                        d.peers[q].p_full[v.row0 + i] = pv;
                        pushed = true;
                    }
            }
            // the next step's slab copies (async proxy) overwrite the staged rows
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        } else {
            for (std::int64_t i = static_cast<std::int64_t>(cta) * kTileThreads + tid; i < v.n;
                 i += static_cast<std::int64_t>(cpr) * kTileThreads) {
                const double pv = __dadd_rn(__ldcg(v.r + i), __dmul_rn(beta, __ldcg(v.p + i)));
                v.p[i] = pv;
                for (int r = 0; r < d.world; ++r)
                    if (r != d.rank && i >= send[2 * r] && i < send[2 * r + 1]) {
                        d.peers[r].p_full[v.row0 + i] = pv;
                        pushed = true;
                    }
            }
        }
        // peer stores are made visible system-wide by their own thread before
        // the shard barrier; local stores are covered by the barrier and the
        // flag's release
        if (pushed) __threadfence_system();
        slot_sync(S.bar, target, static_cast<unsigned>(cpr), d.mb.err);
        ++e;
        if (cta == 0 && tid == 0) {
            __threadfence_system();
            for (int r = 0; r < d.world; ++r)
                asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(d.peers[r].flags + d.rank), "l"(e)
                             : "memory");
        }
    }
    if (cta == 0 && tid == 0) *d.mb.epoch = e;  // the host-side exchanges continue the sequence
}


}  // namespace

#if LILAC_CTA_TRACE
// Experiment builds only (tools/cta_trace.py): per CTA of the last standalone
// tiled SpMV launch: SM id, entry, first slab landed, walk done, exit (ns).
extern "C" int b200_debug_cg_rot(unsigned rot) {
    return cudaMemcpyToSymbol(g_cg_rot, &rot, sizeof rot) == cudaSuccess ? 0 : 1;
}
extern "C" int b200_debug_cg_smid(unsigned* out, int n) {
    return cudaMemcpyFromSymbol(out, g_cg_smid, sizeof(unsigned) * std::min(n, kCgTraceCtas)) == cudaSuccess ? 0 : 1;
}
extern "C" int b200_debug_cg_trace(unsigned long long* out, int n) {
    return cudaMemcpyFromSymbol(out, g_cg_trace,
                                sizeof(unsigned long long) * std::min(n, kCgTraceSteps * kCgTraceCtas * 8)) ==
                   cudaSuccess
               ? 0
               : 1;
}
extern "C" int b200_debug_cta_trace(unsigned long long* out, int n) {
    return cudaMemcpyFromSymbol(out, g_cta_trace, sizeof(unsigned long long) * std::min(n, 5 * kMaxTrace)) ==
                   cudaSuccess
               ? 0
               : 1;
}
#endif

template <int MODE>
void launch_variant(const TcsrDev& T, const double* x, double* y, double* partials, unsigned int* ticket,
                    CgScalars* sc, unsigned grid, cudaStream_t s, std::int64_t dot_off) {
    static std::uint64_t configured = 0;
    if (first_on_device(configured)) {
        B200_CUDA(cudaFuncSetAttribute(k_spmv_tiled<false, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       kTileSmemBudget));
        B200_CUDA(cudaFuncSetAttribute(k_spmv_tiled<true, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       kTileSmemBudget));
    }
    if (partials)
        launch_pdl(k_spmv_tiled<true, MODE>, dim3(std::min<unsigned>(grid, kMaxParts)), dim3(kTileThreads),
                   tile_smem(T), s, T, x, y, partials, ticket, sc, dot_off);
    else
        k_spmv_tiled<false, MODE><<<grid, kTileThreads, tile_smem(T), s>>>(T, x, y, nullptr, nullptr, nullptr, 0);
}

void launch_spmv_tiled(const TcsrDev& T, std::int64_t rows, const double* x, double* y, double* partials,
                       unsigned int* ticket, CgScalars* sc, cudaStream_t s, std::int64_t dot_off) {
    static int mode = -1;
    if (mode < 0) {
        int dev = 0;
        B200_CUDA(cudaGetDevice(&dev));
        B200_CUDA(cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev));
        const char* m = std::getenv("LILAC_B200_TILED_PROBE");  // timing probes only: wrong results
        mode = (m && *m) ? std::atoi(m) : 0;
    }
    if (rows <= 0 || T.ntiles <= 0) return;
    // The x slabs move by cp.async.bulk, which needs a 16-byte-aligned source.
    // A caller's x may be any 8-byte-aligned view (a torch slice, a sub-range
    // of a device mirror): stage it once into an aligned scratch vector on the
    // same stream (8*cols extra bytes, only in that case).
    if (reinterpret_cast<std::uintptr_t>(x) & 15u) {
        static DevBuf xalign;  // one per process; calls are stream-ordered per caller
        const std::size_t xb = static_cast<std::size_t>(T.cols) * sizeof(double);
        if (xalign.bytes < xb) {
            B200_CUDA(cudaStreamSynchronize(s));
            xalign.ensure(xb, false);
        }
        B200_CUDA(cudaMemcpyAsync(xalign.ptr, x, xb, cudaMemcpyDeviceToDevice, s));
        x = xalign.as<const double>();
    }
    const unsigned grid = static_cast<unsigned>(std::min<std::int64_t>(T.ntiles * T.parts, g_sms));
    switch (partials ? 0 : mode) {  // probes never on the fused CG path
    case 1: launch_variant<1>(T, x, y, partials, ticket, sc, grid, s, dot_off); break;
    case 2: launch_variant<2>(T, x, y, partials, ticket, sc, grid, s, dot_off); break;
    case 5: launch_variant<5>(T, x, y, partials, ticket, sc, grid, s, dot_off); break;
    case 6: launch_variant<6>(T, x, y, partials, ticket, sc, grid, s, dot_off); break;
    case 8: launch_variant<8>(T, x, y, partials, ticket, sc, grid, s, dot_off); break;
    case 9: launch_variant<9>(T, x, y, partials, ticket, sc, grid, s, dot_off); break;
    case 10: launch_variant<10>(T, x, y, partials, ticket, sc, grid, s, dot_off); break;
    case 11: launch_variant<11>(T, x, y, partials, ticket, sc, grid, s, dot_off); break;
    case 12: launch_variant<12>(T, x, y, partials, ticket, sc, grid, s, dot_off); break;
    default: launch_variant<0>(T, x, y, partials, ticket, sc, grid, s, dot_off); break;
    }
    B200_CUDA(cudaGetLastError());
}

bool launch_cg_tiled(const TcsrDev& T, const CgVectors& v, int steps, cudaStream_t s) {
    static int enabled = -1;
    static int max_grid = 0;
    if (enabled < 0) {
        const char* e = std::getenv("LILAC_B200_CG_FUSED");
        enabled = (e && std::strcmp(e, "0") == 0) ? 0 : 1;
        int dev = 0, coop = 0, per_sm = 0, sms = 0;
        B200_CUDA(cudaGetDevice(&dev));
        B200_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
        B200_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        B200_CUDA(cudaFuncSetAttribute(k_cg_tiled, cudaFuncAttributeMaxDynamicSharedMemorySize, kTileSmemBudget));
        B200_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_cg_tiled, kTileThreads, kTileSmemBudget));
        max_grid = coop ? per_sm * sms : 0;
        if (max_grid <= 0) enabled = 0;
    }
    static std::uint64_t configured = 0;
    if (enabled && first_on_device(configured))
        B200_CUDA(cudaFuncSetAttribute(k_cg_tiled, cudaFuncAttributeMaxDynamicSharedMemorySize, kTileSmemBudget));
    if (!enabled || steps <= 0 || T.ntiles <= 0 || v.row0 != 0 || v.p != v.p_full) return false;
    const unsigned grid = static_cast<unsigned>(std::min<std::int64_t>({T.ntiles * T.parts, max_grid, kMaxParts}));
    B200_CUDA(cudaMemsetAsync(&v.sc->bar, 0, sizeof(unsigned), s));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kTileThreads);
    cfg.dynamicSmemBytes = tile_smem(T);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    B200_CUDA(cudaLaunchKernelEx(&cfg, k_cg_tiled, T, v, steps));
    return true;
}


// Host: k slots (device array of DistSlot) in one cooperative launch, each
// slot's CTAs one per SM; bars: nslots counters. false when the grid cannot
// give every slot a CTA.
bool launch_cg_tiled_dist(const void* slots_dev, int nslots, std::size_t smem, unsigned* bars, int steps,
                          cudaStream_t s) {
    static int max_grid = -1;
    if (max_grid < 0) {
        int dev = 0, coop = 0, per_sm = 0, sms = 0;
        B200_CUDA(cudaGetDevice(&dev));
        B200_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
        B200_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        B200_CUDA(
            cudaFuncSetAttribute(k_cg_tiled_dist, cudaFuncAttributeMaxDynamicSharedMemorySize, kTileSmemBudget));
        B200_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_cg_tiled_dist, kTileThreads,
                                                                 kTileSmemBudget));
        max_grid = coop ? per_sm * sms : 0;
    }
    static std::uint64_t configured = 0;
    if (first_on_device(configured))
        B200_CUDA(
            cudaFuncSetAttribute(k_cg_tiled_dist, cudaFuncAttributeMaxDynamicSharedMemorySize, kTileSmemBudget));
    if (nslots <= 0 || steps <= 0) return false;
    const int cpr = std::min(max_grid / nslots, kMaxParts);
    if (cpr <= 0) return false;
    B200_CUDA(cudaMemsetAsync(bars, 0, sizeof(unsigned) * static_cast<std::size_t>(nslots), s));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(cpr * nslots));
    cfg.blockDim = dim3(kTileThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    B200_CUDA(cudaLaunchKernelEx(&cfg, k_cg_tiled_dist, static_cast<const DistSlot*>(slots_dev), nslots, steps));
    return true;
}

std::size_t dist_slot_bytes() { return sizeof(DistSlot); }
void dist_slot_fill(void* out, const TcsrDev& T, const CgVectors& v, unsigned* bar) {
    DistSlot d{T, v, bar};
    std::memcpy(out, &d, sizeof d);
}
std::size_t tiled_smem_bytes(const TcsrDev& T) { return tile_smem(T); }

}  // namespace b200
