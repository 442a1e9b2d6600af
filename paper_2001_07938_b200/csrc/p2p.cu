// p2p.cu — the sharded CG driver's exchange step over peer memory (SURVEY
// §8(e) phase 2): every shard pushes its data straight into its peers'
// buffers (NVLink stores through CUDA IPC mappings between processes, plain
// device stores between shards of one process) and raises a per-sender flag
// with the exchange's epoch; receivers wait on the flags. No collective
// library and no host round trip: the exchange is two small kernels per step
// and captures into the outer iteration's CUDA graph.
//
// Ordering: data stores, __threadfence_system(), then the flag (an
// epoch number, monotonically increasing and identical on every shard since
// all shards run the same exchange sequence). A receiver's wait kernel
// observes every sender's flag >= its own epoch before the stream moves on.
// Scalar slots are double-buffered by epoch parity: a sender can run at most
// one exchange ahead of the slowest receiver (every exchange waits for all
// senders), so it never overwrites a slot that is still being read. Vector
// slices need one buffer: the next push of a p slice happens two scalar
// exchanges after the receiver's SpMV consumed it.
// A wait that sees no progress for 5 s records an error and lets the stream
// continue; later waits then return at once (a broken peer link must fail
// the run, not hang the box).

#include "b200.hpp"
#include "p2p.hpp"
#include "cg_fin.cuh"

namespace b200 {

namespace {

__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ void raise_flags(const PeerPtrs* peers, int world, int rank, Mailbox mb) {
    const unsigned long long e = *mb.epoch + 1;
    *mb.epoch = e;
    __threadfence_system();
    for (int r = 0; r < world; ++r) st_release_sys(peers[r].flags + rank, e);
}

__global__ void k_push_scalars(const double* __restrict__ partial, int npart, const PeerPtrs* __restrict__ peers,
                               int world, int rank, Mailbox mb) {
    if (threadIdx.x != 0) return;
    const unsigned long long slot = (*mb.epoch + 1) & 1ull;
    for (int r = 0; r < world; ++r)
        for (int k = 0; k < npart; ++k)
            peers[r].gathered[(slot * kP2pMaxWorld + rank) * kP2pMaxPart + k] = partial[k];
    raise_flags(peers, world, rank, mb);
}

// one CTA copies the slice to every peer (grid-stride), the last CTA raises
// the flags
__global__ void k_push_vector(const double* __restrict__ src, std::int64_t rows, std::int64_t row0,
                              const PeerPtrs* __restrict__ peers, int world, int rank, int which, Mailbox mb,
                              const std::int64_t* __restrict__ send) {
    const std::int64_t stride = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
    for (int r = 0; r < world; ++r) {
        if (r == rank) continue;  // src is this shard's own slice of the same buffer
        double* dst = (which ? peers[r].z_full : peers[r].p_full) + row0;
        const std::int64_t lo = send[2 * r], hi = send[2 * r + 1];
        for (std::int64_t i = lo + static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < hi; i += stride)
            dst[i] = src[i];
    }
    (void)rows;
    __threadfence_system();
    __syncthreads();
    __shared__ bool last;
    if (threadIdx.x == 0) last = atomicAdd(mb.ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last || threadIdx.x != 0) return;
    *mb.ticket = 0u;
    raise_flags(peers, world, rank, mb);
}

// p = r + beta*p over this shard's rows, each new value stored locally and
// into every peer's replica in the same pass (the CG p update fused with its
// exchange); the last CTA raises the flags
__global__ void k_update_p_push(CgVectors v, const PeerPtrs* __restrict__ peers, int world, int rank, Mailbox mb,
                                const std::int64_t* __restrict__ send) {
    const double beta = v.sc->beta;
    const std::int64_t stride = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
    for (std::int64_t i = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < v.n; i += stride) {
        const double pv = __dadd_rn(v.r[i], __dmul_rn(beta, v.p[i]));
        v.p[i] = pv;
        for (int r = 0; r < world; ++r)
            if (r != rank && i >= send[2 * r] && i < send[2 * r + 1]) peers[r].p_full[v.row0 + i] = pv;
    }
    __threadfence_system();
    __syncthreads();
    __shared__ bool last;
    if (threadIdx.x == 0) last = atomicAdd(mb.ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last || threadIdx.x != 0) return;
    *mb.ticket = 0u;
    raise_flags(peers, world, rank, mb);
}

// waits for every sender's flag to reach this shard's epoch; for a scalar
// exchange copies the epoch's slot into `out` (rank-major, npart each)
__global__ void k_wait(int world, Mailbox mb, int npart, double* __restrict__ out) {
    if (threadIdx.x != 0) return;
    if (*reinterpret_cast<volatile int*>(mb.err)) return;  // already failed: do not wait again
    const unsigned long long e = *mb.epoch;
    const unsigned long long t0 = globaltimer_ns();
    for (int r = 0; r < world; ++r) {
        while (ld_acquire_sys(mb.flags + r) < e) {
            if (globaltimer_ns() - t0 > 5000000000ull) {
                *mb.err = 1;
                break;
            }
        }
    }
    const unsigned long long slot = e & 1ull;
    for (int r = 0; r < world; ++r)
        for (int k = 0; k < npart; ++k)
            out[r * npart + k] = *reinterpret_cast<volatile double*>(
                mb.gathered + (slot * kP2pMaxWorld + r) * kP2pMaxPart + k);
}

__global__ void k_wait_fin(int world, Mailbox mb, int npart, int fin, CgScalars* sc, double shift) {
    if (threadIdx.x != 0) return;
    const unsigned long long e = *mb.epoch;
    if (!*reinterpret_cast<volatile int*>(mb.err)) {
        const unsigned long long t0 = globaltimer_ns();
        for (int r = 0; r < world; ++r) {
            while (ld_acquire_sys(mb.flags + r) < e) {
                if (globaltimer_ns() - t0 > 5000000000ull) {
                    *mb.err = 1;
                    break;
                }
            }
        }
    }
    double g[kP2pMaxWorld * kP2pMaxPart];
    const unsigned long long slot = e & 1ull;
    for (int r = 0; r < world; ++r)
        for (int k = 0; k < npart; ++k)
            g[r * npart + k] = *reinterpret_cast<volatile double*>(
                mb.gathered + (slot * kP2pMaxWorld + r) * kP2pMaxPart + k);
    cg_fin_apply(fin, sc, g, world, shift);
}

}  // namespace

void p2p_wait_fin(int world, Mailbox mb, int npart, int fin, CgScalars* sc, double shift, cudaStream_t s) {
    k_wait_fin<<<1, 32, 0, s>>>(world, mb, npart, fin, sc, shift);
    B200_CUDA(cudaGetLastError());
}

void p2p_push_scalars(const double* partial, int npart, const PeerPtrs* peers, int world, int rank, Mailbox mb,
                      cudaStream_t s) {
    k_push_scalars<<<1, 32, 0, s>>>(partial, npart, peers, world, rank, mb);
    B200_CUDA(cudaGetLastError());
}

void p2p_push_vector(const double* src, std::int64_t rows, std::int64_t row0, const PeerPtrs* peers, int world,
                     int rank, bool z, Mailbox mb, const std::int64_t* send, cudaStream_t s) {
    const unsigned grid =
        static_cast<unsigned>(std::max<std::int64_t>(1, std::min<std::int64_t>((rows + 255) / 256, 148)));
    k_push_vector<<<grid, 256, 0, s>>>(src, rows, row0, peers, world, rank, z ? 1 : 0, mb, send);
    B200_CUDA(cudaGetLastError());
}

void p2p_update_p_push(const CgVectors& v, const PeerPtrs* peers, int world, int rank, Mailbox mb,
                       const std::int64_t* send, cudaStream_t s) {
    const unsigned grid =
        static_cast<unsigned>(std::max<std::int64_t>(1, std::min<std::int64_t>((v.n + 511) / 512, 148 * 4)));
    k_update_p_push<<<grid, 256, 0, s>>>(v, peers, world, rank, mb, send);
    B200_CUDA(cudaGetLastError());
}

void p2p_wait(int world, Mailbox mb, int npart, double* out, cudaStream_t s) {
    k_wait<<<1, 32, 0, s>>>(world, mb, npart, out);
    B200_CUDA(cudaGetLastError());
}

}  // namespace b200
