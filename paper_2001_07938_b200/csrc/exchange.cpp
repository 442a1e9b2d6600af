// exchange.cpp — NCCL (dlopen) and single-GPU local exchange for the sharded
// CG driver. See exchange.hpp.

#include "exchange.hpp"
#include "runtime.hpp"

#include <nccl.h>

#include <dlfcn.h>

#include <cstddef>
#include <cstring>

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
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
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
        api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
        api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
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

NcclExchange::NcclExchange(int rank, int world, const void* unique_id, const std::vector<std::int64_t>& bounds,
                           std::int64_t fmin, std::int64_t fmax)
    : rank_(rank), world_(world), bounds_(bounds) {
    ncclUniqueId id;
    std::memcpy(&id, unique_id, sizeof id);
    ncclComm_t c = nullptr;
    check_nccl(nccl().CommInitRank(&c, world, id, rank), "ncclCommInitRank");
    comm_ = c;
    // every rank's footprint, then this rank's send/recv ranges
    DevBuf fp;
    fp.ensure(sizeof(std::int64_t) * 2 * static_cast<std::size_t>(world + 1));
    const std::int64_t mine[2] = {fmin, fmax};
    cudaStream_t st = rt().stream;
    B200_CUDA(cudaMemcpyAsync(fp.as<std::int64_t>() + 2 * world, mine, sizeof mine, cudaMemcpyHostToDevice, st));
    check_nccl(nccl().AllGather(fp.as<std::int64_t>() + 2 * world, fp.as<std::int64_t>(), 2, ncclInt64, c, st),
               "ncclAllGather(footprints)");
    std::vector<std::int64_t> all(2 * static_cast<std::size_t>(world));
    B200_CUDA(cudaMemcpyAsync(all.data(), fp.ptr, sizeof(std::int64_t) * all.size(), cudaMemcpyDeviceToHost, st));
    B200_CUDA(cudaStreamSynchronize(st));
    fp.release();
    std::vector<std::int64_t> lo(world), hi(world);
    for (int r = 0; r < world; ++r) {
        lo[r] = all[2 * r];
        hi[r] = all[2 * r + 1];
    }
    send_ = send_ranges(bounds_[rank], bounds_[rank + 1] - bounds_[rank], lo, hi);
    recv_.assign(2 * static_cast<std::size_t>(world), 0);
    for (int src = 0; src < world; ++src) {
        const std::vector<std::int64_t> sr = send_ranges(bounds_[src], bounds_[src + 1] - bounds_[src], lo, hi);
        recv_[2 * src] = sr[2 * rank];
        recv_[2 * src + 1] = sr[2 * rank + 1];
        for (int r = 0; r < world; ++r)  // full: every slice goes whole to every rank
            if (r != src && sr[2 * r + 1] - sr[2 * r] != bounds_[src + 1] - bounds_[src]) full_ = false;
    }
    if (!nccl().Send || !nccl().Recv) full_ = true;
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
    ShardView& s = shards[0];
    double* full = fulls[0];
    check_nccl(nccl().GroupStart(), "ncclGroupStart");
    if (full_) {
        // every rank reads every slice (NPB's random columns): a variable-size
        // all-gather as one broadcast per owner, fused in a group
        for (int r = 0; r < world_; ++r) {
            const std::int64_t lo = bounds_[r], n = bounds_[r + 1] - bounds_[r];
            if (n == 0) continue;
            check_nccl(nccl().Broadcast(full + lo, full + lo, static_cast<size_t>(n), ncclDouble, r,
                                        static_cast<ncclComm_t>(comm_), s.stream),
                       "ncclBroadcast");
        }
    } else {
        // footprint-limited (banded / stencil rows): each rank gets only the
        // part of each slice its SpMV reads — the halo, not the whole vector
        const std::int64_t mine = bounds_[rank_];
        for (int r = 0; r < world_; ++r) {
            if (r == rank_) continue;
            const std::int64_t slo = send_[2 * r], shi = send_[2 * r + 1];
            if (shi > slo)
                check_nccl(nccl().Send(full + mine + slo, static_cast<size_t>(shi - slo), ncclDouble, r,
                                       static_cast<ncclComm_t>(comm_), s.stream),
                           "ncclSend");
            const std::int64_t rlo = recv_[2 * r], rhi = recv_[2 * r + 1];
            if (rhi > rlo)
                check_nccl(nccl().Recv(full + bounds_[r] + rlo, static_cast<size_t>(rhi - rlo), ncclDouble, r,
                                       static_cast<ncclComm_t>(comm_), s.stream),
                           "ncclRecv");
        }
    }
    check_nccl(nccl().GroupEnd(), "ncclGroupEnd");
}

// ---- PeerExchange --------------------------------------------------------------------

namespace {

PeerPtrs peer_of(double* p_full, double* z_full, char* mbox) {
    PeerPtrs pp;
    pp.p_full = p_full;
    pp.z_full = z_full;
    pp.gathered = reinterpret_cast<double*>(mbox + kMboxGathered);
    pp.flags = reinterpret_cast<unsigned long long*>(mbox + kMboxFlags);
    return pp;
}

}  // namespace

Mailbox PeerExchange::mailbox(const Local& l) const {
    char* b = l.mbox.as<char>();
    Mailbox mb;
    mb.gathered = reinterpret_cast<double*>(b + kMboxGathered);
    mb.flags = reinterpret_cast<unsigned long long*>(b + kMboxFlags);
    mb.epoch = reinterpret_cast<unsigned long long*>(b + kMboxEpoch);
    mb.ticket = reinterpret_cast<unsigned int*>(b + kMboxTicket);
    mb.err = reinterpret_cast<int*>(b + kMboxErr);
    return mb;
}

void PeerExchange::upload_table(Local& l, const std::vector<PeerPtrs>& peers) {
    l.table.ensure(sizeof(PeerPtrs) * peers.size());
    B200_CUDA(cudaMemcpyAsync(l.table.ptr, peers.data(), sizeof(PeerPtrs) * peers.size(), cudaMemcpyHostToDevice,
                              rt().stream));
    B200_CUDA(cudaStreamSynchronize(rt().stream));
}

std::vector<std::int64_t> send_ranges(std::int64_t row0, std::int64_t rows, const std::vector<std::int64_t>& fmin,
                                      const std::vector<std::int64_t>& fmax) {
    const std::size_t world = fmin.size();
    std::vector<std::int64_t> send(2 * world, 0);
    const std::int64_t a = row0, b = row0 + rows;
    for (std::size_t r = 0; r < world; ++r) {
        const std::int64_t lo = std::max(a, fmin[r]), hi = std::min(b, fmax[r]);
        if (hi > lo) {
            send[2 * r] = lo - a;
            send[2 * r + 1] = hi - a;
        }
    }
    return send;
}

void PeerExchange::upload_send(Local& l, const std::vector<std::int64_t>& fmin, const std::vector<std::int64_t>& fmax) {
    const std::vector<std::int64_t> send = send_ranges(l.bufs.row0, l.bufs.rows, fmin, fmax);
    l.send.ensure(sizeof(std::int64_t) * send.size());
    B200_CUDA(cudaMemcpyAsync(l.send.ptr, send.data(), sizeof(std::int64_t) * send.size(), cudaMemcpyHostToDevice,
                              rt().stream));
    B200_CUDA(cudaStreamSynchronize(rt().stream));
}

PeerExchange::PeerExchange(const std::vector<ShardBufs>& local) : world_(static_cast<int>(local.size())) {
    if (world_ < 1 || world_ > kP2pMaxWorld) throw Error(Errc::DataError, "peer exchange: 1..64 shards");
    shards_.resize(local.size());
    std::vector<PeerPtrs> peers;
    for (int i = 0; i < world_; ++i) {
        Local& l = shards_[i];
        l.rank = i;
        l.bufs = local[i];
        l.mbox.ensure(kMboxBytes);
        B200_CUDA(cudaMemsetAsync(l.mbox.ptr, 0, kMboxBytes, rt().stream));
        peers.push_back(peer_of(l.bufs.p_full, l.bufs.z_full, l.mbox.as<char>()));
    }
    std::vector<std::int64_t> fmin, fmax;
    for (const ShardBufs& b : local) {
        fmin.push_back(b.fmin);
        fmax.push_back(b.fmax);
    }
    for (Local& l : shards_) {
        upload_table(l, peers);
        upload_send(l, fmin, fmax);
    }
}

PeerExchange::PeerExchange(int rank, int world, const ShardBufs& mine) : world_(world) {
    if (world < 1 || world > kP2pMaxWorld || rank < 0 || rank >= world)
        throw Error(Errc::DataError, "peer exchange: bad rank/world");
    shards_.resize(1);
    Local& l = shards_[0];
    l.rank = rank;
    l.bufs = mine;
    l.mbox.ensure(kMboxBytes);
    B200_CUDA(cudaMemsetAsync(l.mbox.ptr, 0, kMboxBytes, rt().stream));
    B200_CUDA(cudaStreamSynchronize(rt().stream));
}

PeerExchange::~PeerExchange() {
    for (void* p : opened_) cudaIpcCloseMemHandle(p);
    for (Local& l : shards_) {
        l.mbox.release();
        l.table.release();
        l.desc.release();
        l.send.release();
    }
}

void PeerExchange::export_handles(void* out) const {
    if (shards_.size() != 1) throw Error(Errc::DataError, "IPC export needs one shard per process");
    const Local& l = shards_[0];
    auto* o = static_cast<char*>(out);
    std::memcpy(o + 192, &l.bufs.fmin, sizeof(std::int64_t));
    std::memcpy(o + 200, &l.bufs.fmax, sizeof(std::int64_t));
    cudaIpcMemHandle_t h;
    for (int k = 0; k < 3; ++k) {
        void* base = k == 0 ? static_cast<void*>(l.bufs.p_full)
                            : (k == 1 ? static_cast<void*>(l.bufs.z_full) : l.mbox.ptr);
        B200_CUDA(cudaIpcGetMemHandle(&h, base));
        static_assert(sizeof h == 64, "cudaIpcMemHandle_t is 64 bytes");
        std::memcpy(o + 64 * k, &h, sizeof h);
    }
}

void PeerExchange::attach(const void* handles) {
    if (shards_.size() != 1) throw Error(Errc::DataError, "IPC attach needs one shard per process");
    Local& l = shards_[0];
    const auto* in = static_cast<const char*>(handles);
    std::vector<PeerPtrs> peers;
    std::vector<std::int64_t> fmin(world_), fmax(world_);
    for (int r = 0; r < world_; ++r) {
        std::memcpy(&fmin[r], in + kP2pRecord * r + 192, sizeof(std::int64_t));
        std::memcpy(&fmax[r], in + kP2pRecord * r + 200, sizeof(std::int64_t));
    }
    for (int r = 0; r < world_; ++r) {
        if (r == l.rank) {
            peers.push_back(peer_of(l.bufs.p_full, l.bufs.z_full, l.mbox.as<char>()));
            continue;
        }
        void* m[3];
        for (int k = 0; k < 3; ++k) {
            cudaIpcMemHandle_t h;
            std::memcpy(&h, in + kP2pRecord * r + 64 * k, sizeof h);
            B200_CUDA(cudaIpcOpenMemHandle(&m[k], h, cudaIpcMemLazyEnablePeerAccess));
            opened_.push_back(m[k]);
        }
        peers.push_back(peer_of(static_cast<double*>(m[0]), static_cast<double*>(m[1]), static_cast<char*>(m[2])));
    }
    upload_table(l, peers);
    upload_send(l, fmin, fmax);
}

void PeerExchange::exchange_scalars(std::vector<ShardView>& views, int npart) {
    if (npart > kP2pMaxPart) throw Error(Errc::DataError, "peer exchange: too many scalars");
    for (std::size_t i = 0; i < shards_.size(); ++i)
        p2p_push_scalars(views[i].partial, npart, shards_[i].table.as<PeerPtrs>(), world_, shards_[i].rank,
                         mailbox(shards_[i]), views[i].stream);
    for (std::size_t i = 0; i < shards_.size(); ++i)
        p2p_wait(world_, mailbox(shards_[i]), npart, views[i].gathered, views[i].stream);
}

void PeerExchange::exchange_vector(std::vector<ShardView>& views, std::vector<double*> fulls) {
    for (std::size_t i = 0; i < shards_.size(); ++i) {
        const Local& l = shards_[i];
        const bool z = fulls[i] == l.bufs.z_full;
        p2p_push_vector(fulls[i] + l.bufs.row0, l.bufs.rows, l.bufs.row0, l.table.as<PeerPtrs>(), world_, l.rank, z,
                        mailbox(l), l.send.as<std::int64_t>(), views[i].stream);
    }
    for (std::size_t i = 0; i < shards_.size(); ++i)
        p2p_wait(world_, mailbox(shards_[i]), 0, nullptr, views[i].stream);
}

bool PeerExchange::update_p_exchange(std::vector<ShardView>& views, const std::vector<const CgVectors*>& v) {
    for (std::size_t i = 0; i < shards_.size(); ++i)
        p2p_update_p_push(*v[i], shards_[i].table.as<PeerPtrs>(), world_, shards_[i].rank, mailbox(shards_[i]),
                          shards_[i].send.as<std::int64_t>(), views[i].stream);
    for (std::size_t i = 0; i < shards_.size(); ++i)
        p2p_wait(world_, mailbox(shards_[i]), 0, nullptr, views[i].stream);
    return true;
}

bool PeerExchange::scalars_fin(std::vector<ShardView>& views, int npart, CgFin fin, const std::vector<CgScalars*>& sc,
                               double shift) {
    for (std::size_t i = 0; i < shards_.size(); ++i)
        p2p_wait_fin(world_, mailbox(shards_[i]), npart, static_cast<int>(fin), sc[i], shift, views[i].stream);
    return true;
}

void PeerExchange::bind_producers(const std::vector<CgScalars*>& sc) {
    for (std::size_t i = 0; i < shards_.size(); ++i) {
        Local& l = shards_[i];
        P2pDesc d;
        d.peers = l.table.as<PeerPtrs>();
        d.mb = mailbox(l);
        d.world = world_;
        d.rank = l.rank;
        d.send = l.send.as<std::int64_t>();
        l.desc.ensure(sizeof d);
        B200_CUDA(cudaMemcpyAsync(l.desc.ptr, &d, sizeof d, cudaMemcpyHostToDevice, rt().stream));
        const void* dp = l.desc.ptr;
        B200_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(sc[i]) + offsetof(CgScalars, p2p), &dp, sizeof dp,
                                  cudaMemcpyHostToDevice, rt().stream));
    }
    B200_CUDA(cudaStreamSynchronize(rt().stream));
}

bool PeerExchange::timed_out() const {
    for (const Local& l : shards_) {
        int e = 0;
        B200_CUDA(cudaMemcpy(&e, mailbox(l).err, sizeof e, cudaMemcpyDeviceToHost));
        if (e) return true;
    }
    return false;
}

}  // namespace b200
