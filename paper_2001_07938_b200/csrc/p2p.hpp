#pragma once
// p2p.hpp — peer-memory exchange of the sharded CG driver (p2p.cu).

#include "b200.hpp"

#include <cstdint>

namespace b200 {

constexpr int kP2pMaxWorld = 64;
constexpr std::size_t kP2pRecord = 3 * 64 + 2 * sizeof(std::int64_t);  // IPC handles + footprint
constexpr int kP2pMaxPart = 2;

// Where a shard receives: its p / z replicas and its mailbox (scalar slots +
// one flag per sender). A PeerPtrs table (device memory) lists every shard's,
// as this shard sees them (IPC mappings for other processes).
struct PeerPtrs {
    double* p_full;
    double* z_full;
    double* gathered;             // [2][kP2pMaxWorld][kP2pMaxPart]
    unsigned long long* flags;    // [kP2pMaxWorld]
};

// This shard's own mailbox words (device memory).
struct Mailbox {
    double* gathered;
    unsigned long long* flags;
    unsigned long long* epoch;    // exchanges done by this shard
    unsigned int* ticket;         // last-CTA detection of the vector push
    int* err;                     // set when a wait timed out
};

// Mailbox block layout (one allocation, exported by CUDA IPC).
constexpr std::size_t kMboxGathered = 0;
constexpr std::size_t kMboxFlags = sizeof(double) * 2 * kP2pMaxWorld * kP2pMaxPart;
constexpr std::size_t kMboxEpoch = kMboxFlags + sizeof(unsigned long long) * kP2pMaxWorld;
constexpr std::size_t kMboxTicket = kMboxEpoch + sizeof(unsigned long long);
constexpr std::size_t kMboxErr = kMboxTicket + sizeof(unsigned int);
constexpr std::size_t kMboxBytes = 4096;
static_assert(kMboxErr + sizeof(int) <= kMboxBytes, "mailbox layout");

// What a producing kernel needs to push its partials itself (device memory;
// CgScalars::p2p points here while the peer-memory exchange is attached).
struct P2pDesc {
    const PeerPtrs* peers;
    Mailbox mb;
    int world;
    int rank;
    const std::int64_t* send;  // world x {lo, hi}: the part of this shard's slice each peer reads
};

#ifdef __CUDACC__
// Called by the one thread that finalises a shard's partials: stores them in
// sc->part and, with a peer-memory exchange attached, into every peer's
// mailbox slot for the next epoch, then raises this shard's flags.
__device__ __forceinline__ void p2p_publish(CgScalars* sc, const double* vals, int npart) {
    for (int k = 0; k < npart; ++k) sc->part[k] = vals[k];
    const P2pDesc* d = static_cast<const P2pDesc*>(sc->p2p);
    if (!d) return;
    const unsigned long long e = *d->mb.epoch + 1;
    const unsigned long long slot = e & 1ull;
    for (int r = 0; r < d->world; ++r)
        for (int k = 0; k < npart; ++k)
            d->peers[r].gathered[(slot * kP2pMaxWorld + d->rank) * kP2pMaxPart + k] = vals[k];
    *d->mb.epoch = e;
    __threadfence_system();
    for (int r = 0; r < d->world; ++r)
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(d->peers[r].flags + d->rank), "l"(e) : "memory");
}
#endif

// waits for the epoch's partials of every shard, then applies the CG
// finalisation `fin` (cg.cu CgFin) to sc — the exchange's receive side and
// fin_* in one kernel
void p2p_wait_fin(int world, Mailbox mb, int npart, int fin, CgScalars* sc, double shift, cudaStream_t s);

void p2p_push_scalars(const double* partial, int npart, const PeerPtrs* peers, int world, int rank, Mailbox mb,
                      cudaStream_t s);
// send: world x {lo, hi} offsets into this shard's slice — the rows of it in
// each peer's column footprint (banded / stencil operators: a halo)
void p2p_push_vector(const double* src, std::int64_t rows, std::int64_t row0, const PeerPtrs* peers, int world,
                     int rank, bool z, Mailbox mb, const std::int64_t* send, cudaStream_t s);
void p2p_wait(int world, Mailbox mb, int npart, double* out, cudaStream_t s);
// the CG p update (p = r + beta*p, own rows) fused with the push of the slice
void p2p_update_p_push(const CgVectors& v, const PeerPtrs* peers, int world, int rank, Mailbox mb,
                       const std::int64_t* send, cudaStream_t s);

}  // namespace b200
