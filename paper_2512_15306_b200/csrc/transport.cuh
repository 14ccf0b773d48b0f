// Cross-rank transports of the training session.
//
// The session's collectives (src/trainer.cpp:90-110 and the ZeRO-1 optimizer,
// src/optim.cpp:112-176) reduce to four operations on buffers whose layout is
// identical on every rank (same config/plan => same arena layout):
//   allreduce_max_u32  per-tensor absmax bit patterns (StepContext scales)
//   allreduce_sum_f64  the gradient sum of squares (global_grad_norm)
//   allgather          in place: rank r's chunk at base + r*chunk on every rank
//   alltoall           rank j receives send_base + j*send_stride of every rank i
//                      into recv_base + i*recv_stride (the ZeRO-1 shard exchange)
//
// Two implementations:
//   NcclTransport   one process per GPU, NCCL over NVLink/NVSwitch
//                   (send/recv all-to-all, AllReduce, in-place AllGather).
//   PeerTransport   the paper's copy-engine collectives (PAPER.md:235-356,
//                   src/comms.cpp:185-293): ranks are threads of ONE process
//                   (the reference's WorkerGroup, src/comms.cpp:19-38), each
//                   driving its own session and stream, on one GPU or several.
//                   Every operation PULLS the bytes it needs straight out of
//                   the peers' arenas with cudaMemcpyAsync (DMA copy engines,
//                   no SM work), ordered by CUDA events and a host barrier:
//                     record ready -> barrier -> wait peers' ready -> copies ->
//                     record done -> barrier -> wait peers' done
//                   so a rank never reads a peer buffer before the peer wrote
//                   it, and never overwrites its own buffer while a peer still
//                   reads it.  Reductions sum the pulled rows in ascending rank
//                   order on every rank, so every rank gets identical bits.
#pragma once
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <algorithm>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "nccl_dl.h"

namespace qtb {

struct TransportError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

struct AllGatherItem {
    void* base;       // this rank's buffer; chunk r at base + r*chunk_bytes
    size_t chunk_bytes;
};
struct GatherItem {
    const void* src;  // this rank's chunk (same offset in every rank's arena)
    void* dst;        // rank r's chunk lands at dst + r*chunk_bytes
    size_t chunk_bytes;
};
struct AllToAllItem {
    const void* send_base;  // chunk destined to rank j at send_base + j*send_stride
    size_t send_stride;
    void* recv_base;        // chunk from rank i lands at recv_base + i*recv_stride
    size_t recv_stride;
    size_t bytes;           // per chunk
};

class Transport {
   public:
    int rank = 0, world = 1;
    virtual ~Transport() = default;
    virtual const char* kind() const = 0;
    virtual void allreduce_max_u32(uint32_t* buf, size_t n, cudaStream_t s) = 0;
    virtual void allreduce_sum_f64(double* buf, size_t n, cudaStream_t s) = 0;
    virtual void allgather(const std::vector<AllGatherItem>& items, cudaStream_t s) = 0;
    // out of place: dst + r*chunk = rank r's src, on every rank
    virtual void allgather_to(const std::vector<GatherItem>& items, cudaStream_t s) = 0;
    virtual void alltoall(const std::vector<AllToAllItem>& items, cudaStream_t s) = 0;
    // Outside the step: dst[r*chunk .. ] = rank r's chunk at `src` (same offset on every rank)
    // (the peer group reads idle peers' arenas directly; NCCL: a collective all ranks enter)
    virtual void gather_idle(const void* src, size_t chunk_bytes, void* dst, cudaStream_t s) = 0;
    // bytes this rank moved through the transport (sent + received), for the bench line
    double bytes_moved = 0.0;
};

// ---------------------------------------------------------------------------
// NCCL (one process per GPU)
// ---------------------------------------------------------------------------
class NcclTransport final : public Transport {
   public:
    ncclComm_t comm = nullptr;
    NcclTransport(int rk, int ws, const void* nccl_id) {
        rank = rk;
        world = ws;
        auto& api = NcclApi::get();
        if (!api.ok) throw TransportError("world > 1 needs NCCL (libnccl.so.2 not loadable)");
        if (!nccl_id) throw TransportError("world > 1 needs an NCCL unique id");
        ncclUniqueId id;
        std::memcpy(&id, nccl_id, sizeof(id));
        ncclResult_t r = api.CommInitRank(&comm, world, id, rank);
        if (r != ncclSuccess) throw TransportError(std::string("ncclCommInitRank: ") + api.GetErrorString(r));
    }
    ~NcclTransport() override {
        if (comm) NcclApi::get().CommDestroy(comm);
    }
    const char* kind() const override { return "nccl"; }
    static void check(ncclResult_t r, const char* what) {
        if (r != ncclSuccess) throw TransportError(std::string("NCCL ") + what + ": " + NcclApi::get().GetErrorString(r));
    }
    void allreduce_max_u32(uint32_t* buf, size_t n, cudaStream_t s) override {
        check(NcclApi::get().AllReduce(buf, buf, n, ncclUint32, ncclMax, comm, s), "allreduce max");
    }
    void allreduce_sum_f64(double* buf, size_t n, cudaStream_t s) override {
        check(NcclApi::get().AllReduce(buf, buf, n, ncclFloat64, ncclSum, comm, s), "allreduce sum");
    }
    void allgather(const std::vector<AllGatherItem>& items, cudaStream_t s) override {
        auto& api = NcclApi::get();
        api.GroupStart();
        for (auto& it : items) {
            uint8_t* b = static_cast<uint8_t*>(it.base);
            api.AllGather(b + (size_t)rank * it.chunk_bytes, b, it.chunk_bytes, ncclUint8, comm, s);
            bytes_moved += 2.0 * (world - 1) * it.chunk_bytes;
        }
        check(api.GroupEnd(), "all-gather");
    }
    void allgather_to(const std::vector<GatherItem>& items, cudaStream_t s) override {
        auto& api = NcclApi::get();
        api.GroupStart();
        for (auto& it : items) {
            api.AllGather(it.src, it.dst, it.chunk_bytes, ncclUint8, comm, s);
            bytes_moved += 2.0 * (world - 1) * it.chunk_bytes;
        }
        check(api.GroupEnd(), "all-gather");
    }
    void alltoall(const std::vector<AllToAllItem>& items, cudaStream_t s) override {
        auto& api = NcclApi::get();
        api.GroupStart();
        for (auto& it : items) {
            const uint8_t* sb = static_cast<const uint8_t*>(it.send_base);
            uint8_t* rb = static_cast<uint8_t*>(it.recv_base);
            for (int j = 0; j < world; ++j) {
                if (j == rank) {
                    cudaMemcpyAsync(rb + (size_t)rank * it.recv_stride, sb + (size_t)rank * it.send_stride, it.bytes,
                                    cudaMemcpyDeviceToDevice, s);
                } else {
                    api.Send(sb + (size_t)j * it.send_stride, it.bytes, ncclUint8, j, comm, s);
                    api.Recv(rb + (size_t)j * it.recv_stride, it.bytes, ncclUint8, j, comm, s);
                    bytes_moved += 2.0 * it.bytes;
                }
            }
        }
        check(api.GroupEnd(), "shard exchange");
    }
    void gather_idle(const void* src, size_t chunk_bytes, void* dst, cudaStream_t s) override {
        check(NcclApi::get().AllGather(src, dst, chunk_bytes, ncclUint8, comm, s), "gather");
        cudaStreamSynchronize(s);
    }
};

// ---------------------------------------------------------------------------
// Copy-engine peer transport (ranks = threads of one process)
// ---------------------------------------------------------------------------
// Host barrier with a timeout and a broken state: a rank that fails (or a peer
// that never arrives) breaks the group instead of hanging the others.
class HostBarrier {
   public:
    explicit HostBarrier(int n) : n_(n) {}
    void wait(double timeout_s) {
        std::unique_lock<std::mutex> lk(m_);
        if (broken_) throw TransportError("peer group is broken (a rank failed earlier)");
        const uint64_t gen = gen_;
        if (++count_ == n_) {
            count_ = 0;
            ++gen_;
            cv_.notify_all();
            return;
        }
        const bool ok = cv_.wait_for(lk, std::chrono::duration<double>(timeout_s),
                                     [&] { return gen_ != gen || broken_; });
        if (gen_ != gen) return;  // this barrier completed (even if the group broke afterwards)
        if (broken_) throw TransportError("peer group is broken (a rank failed during a collective)");
        if (!ok) {
            broken_ = true;
            cv_.notify_all();
            throw TransportError("peer group barrier timed out (a rank did not enter the collective)");
        }
    }
    void break_all() {
        std::lock_guard<std::mutex> lk(m_);
        broken_ = true;
        cv_.notify_all();
    }
    bool broken() {
        std::lock_guard<std::mutex> lk(m_);
        return broken_;
    }

   private:
    std::mutex m_;
    std::condition_variable cv_;
    int n_, count_ = 0;
    uint64_t gen_ = 0;
    bool broken_ = false;
};

// The group: W member slots, each filled by one rank's session at creation.
struct PeerGroup {
    int world;
    HostBarrier bar;
    std::mutex reg_m;
    struct Member {
        const uint8_t* arena = nullptr;
        const uint8_t* host = nullptr;  // the rank's pinned host region (offload tiers), or null
        int device = -1;
        cudaEvent_t ready = nullptr, done = nullptr;
    };
    std::vector<Member> mem;
    double timeout_s;
    explicit PeerGroup(int w) : world(w), bar(w), mem((size_t)w) {
        const char* e = getenv("QTB_PEER_TIMEOUT_S");
        timeout_s = e ? atof(e) : 300.0;
    }
};

__global__ void peer_max_u32_kernel(const uint32_t* __restrict__ rows, int W, size_t n, uint32_t* __restrict__ out) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        uint32_t m = rows[i];
        for (int w = 1; w < W; ++w) m = max(m, rows[(size_t)w * n + i]);
        out[i] = m;
    }
}
__global__ void peer_sum_f64_kernel(const double* __restrict__ rows, int W, size_t n, double* __restrict__ out) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        double s = rows[i];
        for (int w = 1; w < W; ++w) s = __dadd_rn(s, rows[(size_t)w * n + i]);  // ascending rank order
        out[i] = s;
    }
}

class PeerTransport final : public Transport {
   public:
    std::shared_ptr<PeerGroup> g;  // shared: the group outlives every member whatever the release order
    int device;
    const uint8_t* arena;  // this rank's arena (peers' buffers are at the same offsets in theirs)
    size_t arena_bytes;
    const uint8_t* host = nullptr;  // this rank's pinned host region (same layout on every rank)
    size_t host_bytes = 0;
    uint8_t* stage = nullptr;  // W x kStage bytes for the small reductions
    static constexpr size_t kStage = 64 * 1024;
    bool peers_ready = false;

    PeerTransport(std::shared_ptr<PeerGroup> grp, int rk, int dev, const uint8_t* arena_base, size_t bytes,
                  const uint8_t* host_base = nullptr, size_t hbytes = 0)
        : g(grp), device(dev), arena(arena_base), arena_bytes(bytes), host(host_base), host_bytes(hbytes) {
        rank = rk;
        world = grp->world;
        if (cudaMalloc(&stage, (size_t)world * kStage) != cudaSuccess)
            throw TransportError("peer transport: staging allocation failed");
        std::lock_guard<std::mutex> lk(g->reg_m);
        auto& m = g->mem[(size_t)rank];
        if (m.arena) throw TransportError("peer group: rank " + std::to_string(rank) + " already joined");
        m.arena = arena_base;
        m.host = host_base;
        m.device = dev;
        cudaEventCreateWithFlags(&m.ready, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&m.done, cudaEventDisableTiming);
    }
    ~PeerTransport() override {
        {
            std::lock_guard<std::mutex> lk(g->reg_m);
            auto& m = g->mem[(size_t)rank];
            if (m.ready) cudaEventDestroy(m.ready);
            if (m.done) cudaEventDestroy(m.done);
            m = PeerGroup::Member{};
        }
        if (stage) cudaFree(stage);
    }
    const char* kind() const override { return "peer-copy"; }

    // a peer's address of the buffer at `local` in this rank's arena
    const uint8_t* peer_addr(int p, const void* local) const {
        const uint8_t* l = static_cast<const uint8_t*>(local);
        if (l >= arena && l < arena + arena_bytes) return g->mem[(size_t)p].arena + (l - arena);
        if (host && l >= host && l < host + host_bytes) return g->mem[(size_t)p].host + (l - host);
        throw TransportError("peer transport: buffer outside the arena");
    }
    void first_use() {
        if (peers_ready) return;
        // every member has joined once the first barrier passes; enable P2P between devices
        g->bar.wait(g->timeout_s);
        for (int p = 0; p < world; ++p) {
            const int pd = g->mem[(size_t)p].device;
            if (pd != device) {
                int can = 0;
                cudaDeviceCanAccessPeer(&can, device, pd);
                if (can) {
                    cudaError_t e = cudaDeviceEnablePeerAccess(pd, 0);
                    if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
                }
            }
        }
        peers_ready = true;
    }
    // record ready -> barrier -> wait for every peer's ready
    void enter(cudaStream_t s) {
        first_use();
        cudaEventRecord(g->mem[(size_t)rank].ready, s);
        g->bar.wait(g->timeout_s);
        for (int p = 0; p < world; ++p)
            if (p != rank) cudaStreamWaitEvent(s, g->mem[(size_t)p].ready, 0);
    }
    // record done -> barrier -> wait for every peer's done (their reads of my buffers finished)
    void leave(cudaStream_t s) {
        cudaEventRecord(g->mem[(size_t)rank].done, s);
        g->bar.wait(g->timeout_s);
        for (int p = 0; p < world; ++p)
            if (p != rank) cudaStreamWaitEvent(s, g->mem[(size_t)p].done, 0);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) throw TransportError(std::string("peer transport: ") + cudaGetErrorString(e));
    }
    void pull(void* dst, int p, const void* local_src, size_t bytes, cudaStream_t s) {
        if (!bytes) return;
        cudaMemcpyAsync(dst, peer_addr(p, local_src), bytes, cudaMemcpyDefault, s);
        if (p != rank) bytes_moved += (double)bytes;
    }
    template <typename T, typename K>
    void allreduce_small(T* buf, size_t n, cudaStream_t s, K kernel) {
        if (n * sizeof(T) > kStage) throw TransportError("peer transport: reduction larger than the staging area");
        enter(s);
        T* rows = reinterpret_cast<T*>(stage);
        for (int p = 0; p < world; ++p) pull(rows + (size_t)p * n, p, buf, n * sizeof(T), s);
        leave(s);  // every peer has read my (unreduced) buf before I overwrite it
        kernel<<<(unsigned)std::max<size_t>(1, std::min<size_t>((n + 255) / 256, 1024)), 256, 0, s>>>(rows, world, n,
                                                                                                     buf);
    }
    void allreduce_max_u32(uint32_t* buf, size_t n, cudaStream_t s) override {
        allreduce_small(buf, n, s, peer_max_u32_kernel);
    }
    void allreduce_sum_f64(double* buf, size_t n, cudaStream_t s) override {
        allreduce_small(buf, n, s, peer_sum_f64_kernel);
    }
    void allgather(const std::vector<AllGatherItem>& items, cudaStream_t s) override {
        enter(s);
        for (auto& it : items)
            for (int p = 0; p < world; ++p)
                if (p != rank) {
                    uint8_t* b = static_cast<uint8_t*>(it.base) + (size_t)p * it.chunk_bytes;
                    pull(b, p, b, it.chunk_bytes, s);
                }
        leave(s);
    }
    void gather_idle(const void* src, size_t chunk_bytes, void* dst, cudaStream_t s) override {
        first_use_nobarrier();
        for (int p = 0; p < world; ++p)
            cudaMemcpyAsync(static_cast<uint8_t*>(dst) + (size_t)p * chunk_bytes, peer_addr(p, src), chunk_bytes,
                            cudaMemcpyDefault, s);
        cudaStreamSynchronize(s);
    }
    void allgather_to(const std::vector<GatherItem>& items, cudaStream_t s) override {
        enter(s);
        for (auto& it : items)
            for (int p = 0; p < world; ++p)
                pull(static_cast<uint8_t*>(it.dst) + (size_t)p * it.chunk_bytes, p, it.src, it.chunk_bytes, s);
        leave(s);
    }
    void first_use_nobarrier() {
        for (int p = 0; p < world; ++p)
            if (!g->mem[(size_t)p].arena) throw TransportError("peer group: not every rank has joined yet");
    }
    void alltoall(const std::vector<AllToAllItem>& items, cudaStream_t s) override {
        enter(s);
        for (auto& it : items) {
            const uint8_t* sb = static_cast<const uint8_t*>(it.send_base) + (size_t)rank * it.send_stride;
            uint8_t* rb = static_cast<uint8_t*>(it.recv_base);
            for (int p = 0; p < world; ++p) pull(rb + (size_t)p * it.recv_stride, p, sb, it.bytes, s);
        }
        leave(s);
    }
};

}  // namespace qtb
