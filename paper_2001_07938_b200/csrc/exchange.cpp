// exchange.cpp — NCCL (dlopen) and single-GPU local exchange for the sharded
// CG driver. See exchange.hpp.

#include "exchange.hpp"

#include <nccl.h>

#include <dlfcn.h>

#include <mutex>
#include <string>

namespace b200 {

namespace {

struct NcclApi {
    void* handle = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    ncclResult_t (*GetVersion)(int*) = nullptr;
};

NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        // the process may already hold a libnccl (torch's); reuse it if so
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            api.handle = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
            if (api.handle) break;
        }
        if (!api.handle) return;
        auto sym = [](const char* n) { return dlsym(api.handle, n); };
        api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
        api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
        api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
        api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
        api.Broadcast = reinterpret_cast<decltype(api.Broadcast)>(sym("ncclBroadcast"));
        api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
        api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
        api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
        api.GetVersion = reinterpret_cast<decltype(api.GetVersion)>(sym("ncclGetVersion"));
    });
    if (!api.handle || !api.CommInitRank || !api.AllGather || !api.Broadcast)
        throw Error(Errc::DeviceError, "NCCL (libnccl.so.2) is not loadable: the multi-GPU driver needs it");
    return api;
}

void check_nccl(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw Error(Errc::DeviceError, std::string(what) + ": " +
                                           (nccl().GetErrorString ? nccl().GetErrorString(r) : "nccl error"));
}

}  // namespace

void nccl_unique_id(void* out128) {
    ncclUniqueId id;
    check_nccl(nccl().GetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(out128, &id, sizeof id);
}

int nccl_version() {
    int v = 0;
    if (nccl().GetVersion) nccl().GetVersion(&v);
    return v;
}

// ---- LocalExchange ----------------------------------------------------------------

void LocalExchange::exchange_scalars(std::vector<ShardView>& shards, int npart) {
    // all shards live on this GPU and stream: stream order makes the copies
    // follow the producing kernels
    for (auto& dst : shards)
        for (std::size_t r = 0; r < shards.size(); ++r)
            B200_CUDA(cudaMemcpyAsync(dst.gathered + r * npart, shards[r].partial, sizeof(double) * npart,
                                      cudaMemcpyDeviceToDevice, dst.stream));
}

void LocalExchange::exchange_vector(std::vector<ShardView>& shards, std::vector<double*> fulls) {
    for (std::size_t d = 0; d < shards.size(); ++d)
        for (std::size_t r = 0; r < shards.size(); ++r) {
            if (r == d || shards[r].rows == 0) continue;
            B200_CUDA(cudaMemcpyAsync(fulls[d] + shards[r].row0, fulls[r] + shards[r].row0,
                                      sizeof(double) * shards[r].rows, cudaMemcpyDeviceToDevice,
                                      shards[d].stream));
        }
}

// ---- NcclExchange --------------------------------------------------------------------

NcclExchange::NcclExchange(int rank, int world, const void* unique_id, const std::vector<std::int64_t>& bounds)
    : rank_(rank), world_(world), bounds_(bounds) {
    ncclUniqueId id;
    std::memcpy(&id, unique_id, sizeof id);
    ncclComm_t c = nullptr;
    check_nccl(nccl().CommInitRank(&c, world, id, rank), "ncclCommInitRank");
    comm_ = c;
}

NcclExchange::~NcclExchange() {
    if (comm_) nccl().CommDestroy(static_cast<ncclComm_t>(comm_));
}

void NcclExchange::exchange_scalars(std::vector<ShardView>& shards, int npart) {
    ShardView& s = shards[0];
    check_nccl(nccl().AllGather(s.partial, s.gathered, static_cast<size_t>(npart), ncclDouble,
                                static_cast<ncclComm_t>(comm_), s.stream),
               "ncclAllGather");
}

void NcclExchange::exchange_vector(std::vector<ShardView>& shards, std::vector<double*> fulls) {
    // variable-size all-gather: one broadcast per owner, fused in a group
    ShardView& s = shards[0];
    double* full = fulls[0];
    check_nccl(nccl().GroupStart(), "ncclGroupStart");
    for (int r = 0; r < world_; ++r) {
        const std::int64_t lo = bounds_[r], n = bounds_[r + 1] - bounds_[r];
        if (n == 0) continue;
        check_nccl(nccl().Broadcast(full + lo, full + lo, static_cast<size_t>(n), ncclDouble, r,
                                    static_cast<ncclComm_t>(comm_), s.stream),
                   "ncclBroadcast");
    }
    check_nccl(nccl().GroupEnd(), "ncclGroupEnd");
}

}  // namespace b200
