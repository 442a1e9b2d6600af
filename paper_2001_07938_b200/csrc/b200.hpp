#pragma once
// b200.hpp — internal declarations shared by the host runtime (.cpp) and the
// sm_100a kernels (.cu). Nothing here is part of the C ABI (include/lilac_b200.h).

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <string>
#include <utility>

#include "lilac/marshal.hpp"

namespace b200 {

using lilac::marshal::Errc;
using lilac::marshal::Error;

[[noreturn]] void throw_cuda(cudaError_t e, const char* what, const char* file, int line);
#define B200_CUDA(call)                                                     \
    do {                                                                    \
        cudaError_t e_ = (call);                                            \
        if (e_ != cudaSuccess) ::b200::throw_cuda(e_, #call, __FILE__, __LINE__); \
    } while (0)

// Programmatic dependent launch for the CG step kernels (k_spmv_tiled's p.q
// variant, k_cg_update_zr, k_cg_update_p): each is launched with programmatic
// stream serialization, lets its successor launch early
// (griddepcontrol.launch_dependents) and waits for its predecessor's
// completion and memory (griddepcontrol.wait) before touching anything the
// predecessor wrote, so the launch and prologue overlap the predecessor's
// tail. LILAC_B200_PDL=0 turns it off.
bool pdl_enabled();

template <typename... KArgs, typename... Args>
void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, std::size_t smem, cudaStream_t s, Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    B200_CUDA(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
}

#ifdef __CUDACC__
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
#endif

// ---------------------------------------------------------------------------
// Device memory
// ---------------------------------------------------------------------------

// Every device array is over-allocated by kPadBytes so vector loads that run
// past a row end (masked, never used) stay inside the allocation.
constexpr std::size_t kPadBytes = 256;

struct DevBuf {
    void* ptr = nullptr;
    std::size_t bytes = 0;  // usable bytes (without padding)
    std::size_t cap = 0;    // allocated bytes
    int device = -1;

    // grow-only; contents not preserved. zero_tail: clear the padding past n
    // (index arrays: masked over-reads must stay in range)
    void ensure(std::size_t n, bool zero_tail = true);
    void release();
    template <typename T>
    T* as() const { return static_cast<T*>(ptr); }
};
void pool_trim();  // return every cached block to CUDA
// True the first time it is called for the current device (function
// attributes such as the dynamic shared-memory limit are per device).
inline bool first_on_device(std::uint64_t& mask) {
    int d = 0;
    if (cudaGetDevice(&d) != cudaSuccess) return false;
    const std::uint64_t bit = 1ull << (d & 63);
    if (mask & bit) return false;
    mask |= bit;
    return true;
}
// Wait for all work on the current device (errors ignored: teardown paths)
// before buffers that caller streams may still use go back to the pool.
void device_quiesce();

// ---------------------------------------------------------------------------
// Resident sparse matrices (device layout)
// ---------------------------------------------------------------------------

enum class CsrKernel : int { Auto = 0, Vector = 1, Merge = 2, Exact = 3, Tiled = 4, Split = 5, Lane = 6 };
const char* csr_kernel_name(CsrKernel k);
// Keep a resident matrix's plain CSR (col / val) once a derived layout (tiled,
// lane-range) serves it? Default no: the derived layout alone is used and the
// plain arrays' HBM is freed (NPB class C 0.80 -> 0.42 GB, stencil N=420
// 48 -> 24 GB). LILAC_B200_KEEP_CSR=1 keeps them (any kernel stays selectable).
bool keep_plain_csr();
CsrKernel parse_csr_kernel(const std::string& s);

// Tiled CSR (upload-time cached invariant, tcsr_build.cpp): rows cut into
// tiles (one CTA each), columns into slabs of kSlabW that fit shared memory.
// Inside a tile the nonzeros are ordered slab-major, then by the owning warp's
// contiguous row range, then by row, so each (slab, warp) is one run. A run's
// nonzeros (in that order) are cut into 4-nonzero chunks and the chunks into
// 32 contiguous lane ranges (lane l gets chunks [l*m + min(l, r), ...), m or
// m + 1 of them); chunk i of lane l is stored at run offset (32 i + l) * 4, so
// every warp-wide chunk load is one contiguous 1 KB burst while each lane
// walks its own range in order, summing rows in registers. Each nonzero has a
// 2-byte key = slab-local column << 1 | kKeyStart when it opens a row (never set on
// a lane's first nonzero); each lane has a 2-byte descriptor = tile-local row
// of its first nonzero | kLaneCont when that row began in an earlier lane.
// HBM cost: 10 bytes per stored nonzero + 64 bytes per run.
// 16 warps per tile with 4 chunks in flight per lane (116 registers) beat 32
// warps with 2 (64 registers): NPB C 73.8 -> 71.6 us, 479 -> 502 it/s
// (sweep: 1024/2, 1024/3, 768/3, 768/4, 512/2, 512/4, 512/5, 384/6, 256/8)
#ifndef LILAC_TILE_THREADS
#define LILAC_TILE_THREADS 512
#endif
constexpr int kTileThreads = LILAC_TILE_THREADS;
constexpr int kTileWarps = kTileThreads / 32;
constexpr int kSlabW = 12288;            // columns per slab: 2 x 96 KB double-buffered in smem
constexpr int kSlabStride = kSlabW + 2;  // + a zero cell (column kSlabW) read by padding entries
constexpr int kMaxTileRows = 4096;       // tile-local rows fit a descriptor and the smem y buffer
constexpr int kChunk = 4;                // nonzeros per lane per load (one 256-bit val load)
// key = slab-local column << 1 | start: the gather address is one mask + one
// shifted add (xs + (key & ~1) * 4), the start bit one test
constexpr std::uint16_t kKeyStart = 1u;
constexpr std::uint16_t kKeyColMask = (1u << 14) - 1u;
constexpr std::uint16_t kLaneCont = 1u << 15;
constexpr std::uint16_t tcsr_key(int col, bool start) {
    return static_cast<std::uint16_t>((static_cast<unsigned>(col) << 1) | (start ? kKeyStart : 0u));
}
constexpr int tcsr_key_col(unsigned key) { return static_cast<int>((key >> 1) & kKeyColMask); }
// padding entry: value 0 times the zero cell (never an Inf or NaN of x)
constexpr std::uint16_t kPadKey = tcsr_key(kSlabW, false);
static_assert(kSlabW <= static_cast<int>(kKeyColMask), "slab columns and the zero cell must fit the key");
// The builder widens the slab to what shared memory leaves after the tile's
// y buffer: 2 (slab_w + 2) + rows_max doubles within kTileSmemBudget (NPB
// class C: tiles of <= 1030 rows -> 13,946-column slabs, 11 instead of 13).
constexpr int kTileSmemBudget = 227 * 1024 - 1024;  // dynamic smem, 1 KB left for static
constexpr int kSlabWMax = kKeyColMask - 1;           // the zero cell (column slab_w) must fit the key
inline std::size_t tcsr_smem_bytes(int slab_w, int rows_max) {
    return sizeof(double) * (2 * static_cast<std::size_t>(slab_w + 2) + static_cast<std::size_t>(rows_max));
}

struct TcsrDev {
    std::int64_t ntiles = 0;
    int nslabs = 0;
    std::int64_t cols = 0;
    int slab_w = kSlabW;                      // columns per slab (even)
    int rows_max = kMaxTileRows;              // tallest tile (y buffer rows)
    const std::int64_t* tile_row0 = nullptr;  // ntiles + 1 row bounds
    const std::int64_t* tile_base = nullptr;  // ntiles + 1 element offsets
    const std::int32_t* woff = nullptr;       // ntiles x (nslabs*kTileWarps + 1): run element offsets, tile-relative
    const std::uint16_t* lrow = nullptr;      // ntiles x nslabs*kTileWarps x 32 lane descriptors
    const double* val = nullptr;              // stored nonzeros (+ pads), tiled order
    const std::uint16_t* key = nullptr;       // same: tcsr_key(slab-local column, row start)
    // Slab parts: with parts > 1 a tile's slabs are cut into `parts`
    // contiguous ranges, one CTA each (work item t * parts + part). Each part
    // stores its row sums in ypart[part * rows + row]; the part that finishes
    // last (tile_done ticket) adds the parts in part order into y. Fewer,
    // taller tiles then stage fewer x slabs per CTA (small matrices with
    // random columns, where re-staging all of x per tile dominates).
    int parts = 1;
    std::int64_t rows = 0;
    double* ypart = nullptr;        // parts x rows (parts > 1)
    unsigned* tile_done = nullptr;  // ntiles tickets, zero between launches
    double* tile_pq = nullptr;      // ntiles: each tile's x.y share (DOT), summed in tile order
};

// Merge-path plan (merge.cu): per-CTA start coordinates on the merge of row
// ends and nonzeros, plus one carry slot per CTA. Cached invariant of row_ptr.
struct MergeDev {
    std::int64_t nctas = 0;
    const std::int64_t* coord_row = nullptr;  // nctas + 1
    const std::int64_t* coord_nz = nullptr;   // nctas + 1 (relative to row_ptr[0])
    std::int64_t* carry_row = nullptr;        // nctas
    double* carry_val = nullptr;              // nctas
};

// Split plan (split.cu) for skewed rows: rows longer than short_max leave the
// vector kernel and are cut into chunks of <= kSplitChunk nonzeros, one warp
// each; chunk partials are summed per row in chunk order (deterministic).
constexpr std::int64_t kSplitChunk = 2048;
struct SplitDev {
    std::int64_t short_max = 0;            // longest row the vector kernel keeps
    std::int64_t nlong = 0, nchunks = 0;
    std::int64_t nnz_short = 0;            // nonzeros in the short rows
    const std::int64_t* long_rows = nullptr;  // nlong
    const std::int64_t* long_first = nullptr; // nlong + 1: first chunk of each long row
    const std::int64_t* chunk_lo = nullptr;   // nchunks: absolute nonzero range
    const std::int64_t* chunk_hi = nullptr;
    const std::int64_t* chunk_row = nullptr;  // nchunks: index into long_rows
    double* partial = nullptr;                // nchunks
    unsigned* done = nullptr;                 // nlong: chunks finished this call (reset by the last)
    unsigned long long* work = nullptr;       // work-unit counter (zeroed before each launch)
};

// Lane-range CSR (upload-time cached invariant, lrcsr_build.cpp; kernel in
// lrcsr.cu) for matrices whose x gathers must go to global memory (skewed
// graphs): the nonzeros, in CSR order with empty rows compacted away, are cut
// into units of kLrcUnit = 32 lanes x kLrcChunks chunks x 4; lane l of a unit
// owns a contiguous range of 4 kLrcChunks nonzeros and chunk i of lane l is
// stored at unit offset (32 i + l) * 4, so each warp-wide chunk load is a
// contiguous 1 KB (val) + 512 B (col) burst, independent of row lengths (no
// row_ptr -> col -> x dependence chain, no per-row imbalance). col is a u32:
// bit 31 = a row starts here, bit 30 = the column is one of the `hot` most
// frequent columns and the low bits are its slot in a shared-memory copy of
// their x values (the gathers that would dominate the L1TEX queue become
// LDS), else the global column. A lane descriptor holds the compact row of its
// first nonzero | kLrcCont when that row began before the lane. Rows complete
// inside a unit are stored directly; the row in progress at each unit's start
// and end goes to a per-unit carry; a fix-up pass sums every row that crossed
// units from a structural plan built with the layout (one thread per short
// crossing, one warp per long one: a fixed order, deterministic). HBM: 12 bytes per nonzero + 4 per 4 kLrcChunks nonzeros.
// units of 32 x 16 x 4 = 2048 nonzeros: Kronecker-22 231 -> 225 us, stencil
// N=420 SpMV 0.92 -> 0.945 of copy (4: 247 us; 32: 271 us — fewer, longer
// units under-fill the tail)
#ifndef LILAC_LRC_CHUNKS
#define LILAC_LRC_CHUNKS 16
#endif
constexpr int kLrcChunks = LILAC_LRC_CHUNKS;
constexpr int kLrcLaneNnz = 4 * kLrcChunks;
constexpr int kLrcUnit = 32 * kLrcLaneNnz;
constexpr std::uint32_t kLrcStart = 1u << 31;
constexpr std::uint32_t kLrcHot = 1u << 30;
constexpr std::uint32_t kLrcColMask = kLrcHot - 1u;
constexpr std::uint32_t kLrcCont = 1u << 31;
constexpr int kLrcHotMax = 27 * 1024 - 1;  // + the zero cell: 216 KB of shared memory
// Per unit, per call: the partial of the row open at the unit's start (when
// lane 0 continues a row) and of the row open at its end.
struct LrcCarry {
    double head_val, tail_val;
};
// A row crossing units (structural, built with the layout): it begins in unit
// u and ends in unit e >= u; y[row] = tail_val[u] + head_val[u+1..e].
struct LrcFix {
    std::int32_t u, e, row, pad;
};
struct LrcDev {
    std::int64_t units = 0, nnz = 0;
    std::int64_t rows_c = 0;                  // nonempty rows
    int hot = 0;                              // hot columns (slot `hot` is a zero cell)
    bool has_empty = false;                   // some rows are empty
    const double* val = nullptr;              // units * kLrcUnit
    const std::uint32_t* col = nullptr;       // units * kLrcUnit
    const std::uint32_t* desc = nullptr;      // units * 32
    const std::int32_t* rmap = nullptr;       // rows_c: compact -> original row (null: identity)
    const std::int32_t* empty = nullptr;      // rows - rows_c empty rows (the fix-up pass zeroes them)
    std::int64_t nempty = 0;
    const std::int32_t* hot_cols = nullptr;   // hot
    double* x_hot = nullptr;                  // hot + 1, gathered per call
    LrcCarry* carry = nullptr;                // units
    const LrcFix* fix = nullptr;              // nfix_short entries (e - u <= kLrcFixShort), then nfix_long
    std::int64_t nfix_short = 0, nfix_long = 0;
};
constexpr int kLrcFixShort = 16;  // longer crossings are summed by a warp

struct CsrDev {
    std::int64_t rows = 0;      // number of rows computed
    std::int64_t nnz = 0;       // extent of val/col (row_ptr[rows] for the ABI)
    std::int64_t cols = 0;      // 1 + max(col_ind), ReadableMax semantics
    std::int64_t max_row = 0;   // longest row
    const std::int64_t* row_ptr = nullptr;  // rows+1, int64 (ABI width)
    const void* col = nullptr;              // nnz, int32 if col32 else int64
    bool col32 = true;
    const double* val = nullptr;            // nnz
    bool monotone = true;                   // row_ptr non-decreasing
    const TcsrDev* tiled = nullptr;         // present when the tiled layout was built
    const MergeDev* merge = nullptr;        // present when the merge plan was built
    const SplitDev* split = nullptr;        // present when the split plan was built
    const LrcDev* lrc = nullptr;            // present when the lane-range layout was built
};

// Segmented JDS (k_jds_seg): a jagged row of L nonzeros is served by
// G = ceil(L / kJdsSegD) consecutive lanes of one warp, lane s holding
// diagonals [s * kJdsSegD, (s + 1) * kJdsSegD); the row's sum is carried lane
// to lane in k order (bit-identical to the reference). Rows are length-sorted
// in JDS, so rows of equal G form contiguous zones; zone z packs 32 / G rows
// per warp. nzones == 0: the layout does not qualify (nzcnt not
// non-increasing, or a row longer than 32 * kJdsSegD) and k_jds serves it.
#ifndef LILAC_JDS_SEG_D
#define LILAC_JDS_SEG_D 10
#endif
constexpr int kJdsSegD = LILAC_JDS_SEG_D;
constexpr int kJdsMaxZones = 32;
struct JdsSeg {
    int nzones = 0;
    int g[kJdsMaxZones] = {};                  // lanes per row in zone z
    std::int64_t row0[kJdsMaxZones + 1] = {};  // zone z = jagged rows [row0[z], row0[z + 1])
    std::int64_t warp0[kJdsMaxZones + 1] = {};  // first warp of zone z; warp0[nzones] = warps in all
};
// Host: the zone table of a JDS nzcnt (rows entries, jagged order).
JdsSeg jds_segments(const std::int64_t* nzcnt, std::int64_t rows);

struct JdsDev {
    std::int64_t rows = 0;
    std::int64_t nnz = 0;
    std::int64_t cols = 0;
    std::int64_t njd = 0;                      // max_nz + 1 entries of jd_ptr
    const std::int64_t* nzcnt = nullptr;       // rows, jagged order
    const std::int64_t* perm = nullptr;        // rows, original -> jagged
    const std::int64_t* inv_perm = nullptr;    // rows, jagged -> original (null: perm not a bijection)
    const std::int64_t* jd_ptr = nullptr;      // njd
    const void* col = nullptr;
    bool col32 = true;
    const double* val = nullptr;
    JdsSeg seg;  // k_jds_seg zones (nzones 0: k_jds)
};

// ---------------------------------------------------------------------------
// Kernel launchers (kernels.cu). All asynchronous on `s`.
// ---------------------------------------------------------------------------

// Chooses the CSR kernel for a matrix shape.
CsrKernel choose_csr_kernel(const CsrDev& A, CsrKernel requested);
int csr_vector_width(const CsrDev& A);  // lanes per row for the vector kernel

void launch_spmv_csr(const CsrDev& A, const double* x, double* y, CsrKernel k, cudaStream_t s);
struct CgScalars;
// Merge-path kernel (merge.cu) for skewed rows.
std::int64_t merge_ctas(std::int64_t rows, std::int64_t nnz);
void launch_merge_plan(const std::int64_t* row_ptr, std::int64_t rows, std::int64_t nnz, std::int64_t* coord_row,
                       std::int64_t* coord_nz, cudaStream_t s);
void launch_spmv_merge(const CsrDev& A, const double* x, double* y, cudaStream_t s);
// Split kernel (kernels.cu): vector rows + warp-per-chunk long rows in one launch.
void launch_spmv_split(const CsrDev& A, const double* x, double* y, cudaStream_t s);
// y = A x on the lane-range layout (lrcsr.cu): hot-x gather, main kernel, carry fix-up.
void launch_spmv_lrc(const LrcDev& L, std::int64_t rows, const double* x, double* y, cudaStream_t s);
// One PageRank step on the lane-range layout, the update fused into the row
// stores: y = d * (A x) + (1 - d) / rows, the same bits as the SpMV followed by
// launch_pagerank_update. y must not alias x. false: not applicable (no units).
bool launch_pagerank_lrc(const LrcDev& L, std::int64_t rows, const double* x, double* y, double d, cudaStream_t s);
// p.q of a finished SpMV into the CG scalars (alpha, or the shard partial).
void launch_cg_dot_scalars(const double* p, const double* q, std::int64_t n, double* partials, unsigned int* ticket,
                           CgScalars* sc, cudaStream_t s);

// Tiled kernel (tcsr.cu); partials/ticket/sc non-null = fused p.q for CG.
void launch_spmv_tiled(const TcsrDev& T, std::int64_t rows, const double* x, double* y, double* partials,
                       unsigned int* ticket, struct CgScalars* sc, cudaStream_t s, std::int64_t dot_off = 0);
void launch_spmv_jds(const JdsDev& A, const double* x, double* y, cudaStream_t s);
bool jds_segmented(const JdsDev& A);  // launch_spmv_jds takes k_jds_seg

struct CgScalars;
// Fused CG kernel: q = A p and d = p.q in one pass; the last CTA sets
// sc->d, sc->rho0 = sc->rho, sc->alpha = rho / d.
// `dot_off`: global index of local row 0 (the dot reads p[dot_off + row]).
void launch_spmv_csr_dot(const CsrDev& A, const double* p, double* q, double* partials,
                         unsigned int* ticket, CgScalars* sc, cudaStream_t s, std::int64_t dot_off = 0);

// Upload-time validation / narrowing (one pass each, device side).
//  * narrow_cols: col64[nnz] -> col32 (if col32 != null), max into *d_max, any
//    negative index into *d_bad.
void launch_scan_cols(const std::int64_t* col64, std::int64_t nnz, std::int32_t* col32,
                      unsigned long long* d_max, int* d_bad, cudaStream_t s);
//  * check_row_ptr: rows whose nonempty range leaves [0, nnz) set *d_bad;
//    the longest row goes to *d_max.
void launch_check_row_ptr(const std::int64_t* row_ptr, std::int64_t rows, std::int64_t nnz,
                          unsigned long long* d_max, int* d_bad, cudaStream_t s);
//  * invert_perm: inv[perm[i]] = i; out-of-range or repeated targets set *d_bad.
void launch_invert_perm(const std::int64_t* perm, std::int64_t rows, std::int64_t* inv, int* d_bad,
                        cudaStream_t s);
//  * check_jds: every (k < nzcnt[p]) offset jd_ptr[k]+p inside [0,nnz).
void launch_check_jds(const std::int64_t* nzcnt, const std::int64_t* jd_ptr, std::int64_t rows,
                      std::int64_t njd, std::int64_t nnz, int* d_bad, cudaStream_t s);

// BLAS-1 companions (deterministic: fixed partition and fixed-order sums).
int dot_parts_for(std::int64_t n);
// Host-mapped scalar slot: a reducing kernel also writes its result there and
// then `seq` to `flag` (device pointers of pinned mapped memory), so the host
// can spin on the flag instead of a D2H copy + stream sync. value==nullptr: off.
struct HostSlot {
    double* value = nullptr;
    unsigned* flag = nullptr;
    unsigned seq = 0;
};
void launch_dot(const double* a, const double* b, std::int64_t n, double* result, double* partials,
                unsigned int* ticket, cudaStream_t s, HostSlot slot = {});
void launch_dot_exact(const double* a, const double* b, std::int64_t n, double* result, cudaStream_t s,
                      HostSlot slot = {});
void launch_axpy(std::int64_t n, double* y, double alpha, const double* x, cudaStream_t s);
void launch_xpay(std::int64_t n, double* y, double beta, const double* x, cudaStream_t s);
// out-of-place forms (out may alias y): the harness writes its output binding
// straight from the input binding's device bytes
// gemm (gemm.cu): c = a b, row-major; exact = the reference's k order
void launch_gemm(std::int64_t n, std::int64_t m, std::int64_t p, const double* a, const double* b, double* c,
                 bool exact, cudaStream_t s);
void launch_axpy_to(std::int64_t n, double* out, const double* y, double alpha, const double* x, cudaStream_t s);
void launch_xpay_to(std::int64_t n, double* out, const double* y, double beta, const double* x, cudaStream_t s);

// ---------------------------------------------------------------------------
// NPB CG device step kernels (cg.cu)
// ---------------------------------------------------------------------------

struct CgScalars {  // device-resident, one per solver (shard)
    double rho, rho0, d, alpha, beta, rnorm, t1, t2, zeta;
    unsigned int ticket[4];
    int nranks;     // > 1: sharded mode — reductions stop at this shard's partial (part[]); exchange + fin_* follow
    unsigned int bar;  // grid barrier counter of the fused CG kernel (zeroed before each launch)
    double part[4];
    // peer-memory exchange (p2p.hpp P2pDesc, device memory) or null: when set,
    // the kernel that produces the partials also pushes them to the peers
    const void* p2p;
};

struct CgVectors {
    std::int64_t n;          // rows owned (all rows on one GPU)
    double *x, *z, *p, *q, *r;  // owned slices; p/z point into p_full/z_full at row0
    double *p_full, *z_full;    // full-length replicas the SpMV reads
    std::int64_t row0;
    double* partials;  // 4 * kMaxParts
    int nparts;
    CgScalars* sc;
};

constexpr int kMaxParts = 2048;

void cg_launch_init(const CgVectors& v, cudaStream_t s);            // q=z=0, r=p=x, rho=r.r
void cg_launch_iteration(const CsrDev& A, const CgVectors& v, cudaStream_t s);
// `steps` CG iterations: one persistent fused kernel (tcsr.cu k_cg_tiled) for
// a tiled matrix on one GPU, else cg_launch_iteration per step.
void cg_launch_iterations(const CsrDev& A, const CgVectors& v, int steps, cudaStream_t s);
// Fused single-GPU CG steps over the tiled layout; false if not available.
bool launch_cg_tiled(const TcsrDev& T, const CgVectors& v, int steps, cudaStream_t s);
// Sharded fused CG steps over the tiled layout (tcsr.cu k_cg_tiled_dist): a
// device array of `nslots` slots (dist_slot_fill), each a shard with its
// peer-memory exchange bound (CgScalars::p2p); false if not available.
bool launch_cg_tiled_dist(const void* slots_dev, int nslots, std::size_t smem, unsigned* bars, int steps,
                          cudaStream_t s);
std::size_t dist_slot_bytes();
void dist_slot_fill(void* out, const TcsrDev& T, const CgVectors& v, unsigned* bar);
std::size_t tiled_smem_bytes(const TcsrDev& T);
void cg_launch_residual(const CsrDev& A, const CgVectors& v, cudaStream_t s);  // r=A z, rnorm
void cg_launch_outer_update(const CgVectors& v, double shift, cudaStream_t s);  // zeta, x = z/|z|
void cg_launch_reset_x(const CgVectors& v, cudaStream_t s);

// Workload pieces (workloads_dev.cu): the 27-point stencil matrix generated in
// HBM (int32 columns) and the PageRank update x = d*ax + (1-d)/n.
std::int64_t stencil27_nnz(std::int64_t nx);
// nonzeros of rows [0, r) of the stencil (exact, O(nx))
std::int64_t stencil27_prefix_nnz(std::int64_t nx, std::int64_t r);
// rows [r0, r1) generated in HBM: rebased int64 row_ptr, int32 col, f64 val
void gen_stencil27_rows_device(std::int64_t nx, std::int64_t r0, std::int64_t r1, double diag, double off,
                               DevBuf& row_ptr, DevBuf& col, DevBuf& val, cudaStream_t s);
void gen_stencil27_device(std::int64_t nx, double diag, double off, DevBuf& row_ptr, DevBuf& col, DevBuf& val,
                          cudaStream_t s);
void launch_pagerank_update(std::int64_t n, double* x, const double* ax, double d, cudaStream_t s);

// Single steps (the sharded driver interleaves exchanges between them).
void cg_launch_spmv_dot(const CsrDev& A, const CgVectors& v, cudaStream_t s);
void cg_launch_update_zr(const CgVectors& v, cudaStream_t s);
void cg_launch_update_p(const CgVectors& v, cudaStream_t s);
void cg_launch_norms(const CgVectors& v, double shift, cudaStream_t s);
void cg_launch_scale_x(const CgVectors& v, cudaStream_t s);
void cg_launch_resid_partial(const CgVectors& v, cudaStream_t s);

// Sharded CG (nranks > 1): finalize scalars from the rank-ordered gathered
// partials of all shards (`gathered` holds nranks * stride doubles).
enum class CgFin : int { Rho = 0, Alpha = 1, Beta = 2, Rnorm = 3, Norms = 4 };
void cg_launch_fin(CgFin what, CgScalars* sc, const double* gathered, int nranks, double shift, cudaStream_t s);

}  // namespace b200
