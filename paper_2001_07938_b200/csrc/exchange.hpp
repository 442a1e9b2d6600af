#pragma once
// exchange.hpp — the one exchange step of the row-sharded driver (SURVEY
// §8(e)): gather every shard's scalar partials and all-gather the p (or z)
// vector slices. Two implementations:
//  * NcclExchange: one shard per process/GPU, NCCL over NVLink (libnccl.so.2
//    loaded at run time, so the library also loads where NCCL is absent);
//  * LocalExchange: k shards driven by one host thread on one GPU, exchanged
//    with device-to-device copies — the same sharded algorithm, used to test
//    it on a single GPU (no kernel ever waits on another).

#include "b200.hpp"

#include <cstdint>
#include <vector>

#include "p2p.hpp"

namespace b200 {

struct ShardView {
    std::int64_t row0 = 0, rows = 0;  // owned global rows
    double* full = nullptr;           // full-length vector replica (p or z)
    double* partial = nullptr;        // this shard's scalar partials (npart doubles)
    double* gathered = nullptr;       // [nshards * npart] after exchange_scalars
    cudaStream_t stream = nullptr;
};

class Exchange {
public:
    virtual ~Exchange() = default;
    virtual int nshards() const = 0;
    // gathered[r*npart + i] = partial_r[i] on every shard, rank order.
    virtual void exchange_scalars(std::vector<ShardView>& shards, int npart) = 0;
    // every shard's full[row0_r .. row0_r+rows_r) = shard r's slice.
    virtual void exchange_vector(std::vector<ShardView>& shards, std::vector<double*> fulls) = 0;
    // The CG p update fused with its exchange, if this transport can; false =
    // the caller runs the update and exchange_vector.
    virtual bool update_p_exchange(std::vector<ShardView>& shards, const std::vector<const CgVectors*>& v) {
        (void)shards;
        (void)v;
        return false;
    }
    // Receive side of a scalar exchange whose partials the producing kernels
    // already pushed, fused with the finalisation, if this transport can;
    // false = the caller runs exchange_scalars + fin.
    virtual bool scalars_fin(std::vector<ShardView>& shards, int npart, CgFin fin, const std::vector<CgScalars*>& sc,
                             double shift) {
        (void)shards;
        (void)npart;
        (void)fin;
        (void)sc;
        (void)shift;
        return false;
    }
};

class LocalExchange : public Exchange {
public:
    explicit LocalExchange(int k) : k_(k) {}
    int nshards() const override { return k_; }
    void exchange_scalars(std::vector<ShardView>& shards, int npart) override;
    void exchange_vector(std::vector<ShardView>& shards, std::vector<double*> fulls) override;

private:
    int k_;
};

// NCCL communicator wrapper (dlopen'ed). One shard (this rank).
class NcclExchange : public Exchange {
public:
    // fmin/fmax: this shard's column footprint; the communicator all-gathers
    // every rank's, and a vector exchange then moves only the ranges each rank
    // reads (grouped send/recv: a halo for banded rows, everything for NPB)
    NcclExchange(int rank, int world, const void* unique_id, const std::vector<std::int64_t>& bounds,
                 std::int64_t fmin, std::int64_t fmax);
    ~NcclExchange() override;
    int nshards() const override { return 1; }
    int rank() const { return rank_; }
    int world() const { return world_; }
    void exchange_scalars(std::vector<ShardView>& shards, int npart) override;
    void exchange_vector(std::vector<ShardView>& shards, std::vector<double*> fulls) override;

private:
    int rank_, world_;
    void* comm_ = nullptr;
    std::vector<std::int64_t> bounds_;
    std::vector<std::int64_t> send_, recv_;  // world x {lo, hi}: slice-relative ranges to / from each rank
    bool full_ = true;                       // every rank reads every slice: grouped broadcasts
};

// Peer-memory exchange (p2p.cu): each shard pushes into its peers' replicas
// and mailboxes and waits on per-sender epoch flags. Either k shards of this
// process (peers addressed directly) or one shard per process (peers mapped
// with CUDA IPC: export() this shard's three handles, attach() everyone's).
class PeerExchange : public Exchange {
public:
    struct ShardBufs {
        double* p_full;
        double* z_full;
        std::int64_t row0, rows;
        std::int64_t fmin, fmax;  // column footprint: the replica entries this shard's SpMV reads
    };
    // k local shards, ranks 0..k-1
    explicit PeerExchange(const std::vector<ShardBufs>& local);
    // one shard of `world` (this process), peers attached later
    PeerExchange(int rank, int world, const ShardBufs& mine);
    ~PeerExchange() override;
    int nshards() const override { return static_cast<int>(shards_.size()); }
    void exchange_scalars(std::vector<ShardView>& shards, int npart) override;
    void exchange_vector(std::vector<ShardView>& shards, std::vector<double*> fulls) override;
    bool update_p_exchange(std::vector<ShardView>& shards, const std::vector<const CgVectors*>& v) override;
    bool scalars_fin(std::vector<ShardView>& shards, int npart, CgFin fin, const std::vector<CgScalars*>& sc,
                     double shift) override;
    // point each shard's CgScalars::p2p at its descriptor: its producing
    // kernels then push their partials themselves
    void bind_producers(const std::vector<CgScalars*>& sc);
    // IPC: this shard's record — three 64-byte handles (p_full, z_full,
    // mailbox) and its column footprint (2 x int64): kP2pRecord bytes
    void export_handles(void* out) const;
    // records of all `world` ranks (rank-major); maps the others
    void attach(const void* handles);
    // a wait timed out somewhere (checked after a run)
    bool timed_out() const;

private:
    struct Local {
        int rank = 0;
        ShardBufs bufs{};
        DevBuf mbox;
        DevBuf table;  // world PeerPtrs
        DevBuf desc;   // P2pDesc
        DevBuf send;   // world x {lo, hi}: the part of my slice each peer reads
    };
    void upload_send(Local& l, const std::vector<std::int64_t>& fmin, const std::vector<std::int64_t>& fmax);
    void upload_table(Local& l, const std::vector<PeerPtrs>& peers);
    Mailbox mailbox(const Local& l) const;
    std::vector<Local> shards_;
    int world_ = 1;
    std::vector<void*> opened_;  // IPC mappings to close
};

// The part of shard [row0, row0+rows) that each rank r reads: its column
// footprint [fmin[r], fmax[r]) intersected with the shard, as slice-relative
// {lo, hi} pairs ({0, 0}: nothing). Host logic shared by the peer exchange and
// b200_dist_send_ranges (the CPU-checkable exchange plan).
std::vector<std::int64_t> send_ranges(std::int64_t row0, std::int64_t rows, const std::vector<std::int64_t>& fmin,
                                      const std::vector<std::int64_t>& fmax);

void nccl_unique_id(void* out128);
int nccl_version();

}  // namespace b200
