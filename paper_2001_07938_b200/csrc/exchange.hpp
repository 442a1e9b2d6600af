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
    NcclExchange(int rank, int world, const void* unique_id, const std::vector<std::int64_t>& bounds);
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
};

void nccl_unique_id(void* out128);
int nccl_version();

}  // namespace b200
