// nccl_loopback.h -- in-process loopback implementation of the NcclApi table (TEST TRANSPORT).
//
// Every rank of a job lives in this process on the same device, one host thread per rank, each
// with its own stream.  The x-slab driver then runs exactly the code it runs over NCCL -- the
// communicator cache (comm_acquire), the grouped ncclSend/ncclRecv halo exchange (transfer) and
// the ncclAllReduce counters (gsum / gmax) -- so the GPU suite executes the NCCL path on one GPU
// (DESIGN.md §8).  Selected with cg_nccl_loopback(1) (include/colgraph.h, test hook).
//
// Semantics (a subset of NCCL's, enough for this library):
//   send/recv inside groupStart/groupEnd: at groupEnd every send is posted with an event recorded
//   on the sender's stream; every recv waits (host) for its matching post, makes its stream wait
//   on that event and copies device-to-device on the receiver's stream, recording a done event;
//   every sender then makes its stream wait on the done event (the send buffer stays untouched
//   until the copy has run).  Posts between a pair of ranks are matched in order.
//   allReduce (int32 / int64, sum / max): the caller's stream is synchronised, the values are
//   combined on the host under a generation barrier, and the result is copied back on the stream.
#pragma once

#include <condition_variable>
#include <cstring>
#include <deque>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "nccl_shim.h"

namespace cg {
namespace loopback {

struct Post {
    const void *buf = nullptr;
    size_t bytes = 0;
    cudaEvent_t ready = nullptr, done = nullptr;
    bool copied = false;
};

struct Group {
    std::mutex mu;
    std::condition_variable cv;
    int nranks = 0;
    std::map<std::pair<int, int>, std::deque<std::shared_ptr<Post>>> box;  // (src, dst) -> posts in order
    // allreduce generation barrier
    int arrived = 0;
    uint64_t gen = 0;
    std::vector<int64_t> acc;
    std::shared_ptr<std::vector<int64_t>> result;
};

struct Comm {
    std::shared_ptr<Group> grp;
    int rank;
};

struct Op {
    bool send;
    void *buf;
    size_t bytes;
    int peer;
    Comm *comm;
    cudaStream_t stream;
};

inline std::mutex &reg_mu() {
    static std::mutex m;
    return m;
}
inline std::map<std::string, std::shared_ptr<Group>> &registry() {
    static std::map<std::string, std::shared_ptr<Group>> r;
    return r;
}
inline thread_local int t_depth = 0;
inline thread_local std::vector<Op> t_ops;

inline size_t type_size(ncclDataType_t t) {
    switch (t) {
        case ncclInt8: case ncclUint8: return 1;
        case ncclInt32: case ncclUint32: case ncclFloat32: return 4;
        case ncclInt64: case ncclUint64: case ncclFloat64: return 8;
        default: return 0;
    }
}

inline ncclResult_t getUniqueId(ncclUniqueId *id) {
    static std::mutex m;
    static uint64_t counter = 0;
    std::lock_guard<std::mutex> lk(m);
    memset(id, 0, sizeof(*id));
    const uint64_t c = ++counter;
    const uint64_t tag = 0x6c6f6f706261636bull;  // "loopback"
    memcpy(id->internal, &tag, 8);
    memcpy(id->internal + 8, &c, 8);
    const void *self = &counter;
    memcpy(id->internal + 16, &self, sizeof(self));
    return ncclSuccess;
}

inline ncclResult_t commInitRank(ncclComm_t *out, int nranks, ncclUniqueId id, int rank) {
    if (nranks < 1 || rank < 0 || rank >= nranks) return ncclInvalidArgument;
    std::lock_guard<std::mutex> lk(reg_mu());
    std::shared_ptr<Group> &g = registry()[std::string(id.internal, sizeof(id.internal))];
    if (!g) {
        g = std::make_shared<Group>();
        g->nranks = nranks;
    }
    if (g->nranks != nranks) return ncclInvalidArgument;
    *out = reinterpret_cast<ncclComm_t>(new Comm{g, rank});
    return ncclSuccess;
}

inline ncclResult_t commDestroy(ncclComm_t c) {
    delete reinterpret_cast<Comm *>(c);
    return ncclSuccess;
}

inline ncclResult_t run_group(std::vector<Op> &ops) {
    std::vector<std::pair<std::shared_ptr<Post>, Op *>> mine;
    // 1. post every send (event recorded on the sender's stream)
    for (Op &o : ops) {
        if (!o.send) continue;
        auto p = std::make_shared<Post>();
        p->buf = o.buf;
        p->bytes = o.bytes;
        if (cudaEventCreateWithFlags(&p->ready, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&p->done, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventRecord(p->ready, o.stream) != cudaSuccess)
            return ncclUnhandledCudaError;
        Group &g = *o.comm->grp;
        {
            std::lock_guard<std::mutex> lk(g.mu);
            g.box[{o.comm->rank, o.peer}].push_back(p);
        }
        g.cv.notify_all();
        mine.push_back({p, &o});
    }
    // 2. every recv: wait for the matching post, copy on the receiver's stream
    for (Op &o : ops) {
        if (o.send) continue;
        Group &g = *o.comm->grp;
        std::shared_ptr<Post> p;
        {
            std::unique_lock<std::mutex> lk(g.mu);
            auto &q = g.box[{o.peer, o.comm->rank}];
            g.cv.wait(lk, [&] { return !q.empty(); });
            p = q.front();
            q.pop_front();
        }
        if (p->bytes != o.bytes) return ncclInvalidArgument;
        if (cudaStreamWaitEvent(o.stream, p->ready, 0) != cudaSuccess ||
            cudaMemcpyAsync(o.buf, p->buf, o.bytes, cudaMemcpyDeviceToDevice, o.stream) != cudaSuccess ||
            cudaEventRecord(p->done, o.stream) != cudaSuccess)
            return ncclUnhandledCudaError;
        {
            std::lock_guard<std::mutex> lk(g.mu);
            p->copied = true;
        }
        g.cv.notify_all();
    }
    // 3. senders: the send buffer is reusable once the receiver's copy has run
    for (auto &pr : mine) {
        Group &g = *pr.second->comm->grp;
        {
            std::unique_lock<std::mutex> lk(g.mu);
            g.cv.wait(lk, [&] { return pr.first->copied; });
        }
        if (cudaStreamWaitEvent(pr.second->stream, pr.first->done, 0) != cudaSuccess) return ncclUnhandledCudaError;
        cudaEventDestroy(pr.first->ready);
        cudaEventDestroy(pr.first->done);
    }
    return ncclSuccess;
}

inline ncclResult_t p2p(bool send, const void *buf, size_t count, ncclDataType_t t, int peer, ncclComm_t c,
                        cudaStream_t s) {
    Comm *comm = reinterpret_cast<Comm *>(c);
    const size_t ts = type_size(t);
    if (!comm || !ts || peer < 0 || peer >= comm->grp->nranks) return ncclInvalidArgument;
    t_ops.push_back(Op{send, const_cast<void *>(buf), count * ts, peer, comm, s});
    if (t_depth == 0) {  // outside a group: a group of one
        std::vector<Op> ops;
        ops.swap(t_ops);
        return run_group(ops);
    }
    return ncclSuccess;
}
inline ncclResult_t send(const void *b, size_t n, ncclDataType_t t, int peer, ncclComm_t c, cudaStream_t s) {
    return p2p(true, b, n, t, peer, c, s);
}
inline ncclResult_t recv(void *b, size_t n, ncclDataType_t t, int peer, ncclComm_t c, cudaStream_t s) {
    return p2p(false, b, n, t, peer, c, s);
}
inline ncclResult_t groupStart() {
    ++t_depth;
    return ncclSuccess;
}
inline ncclResult_t groupEnd() {
    if (t_depth <= 0) return ncclInvalidUsage;
    if (--t_depth > 0) return ncclSuccess;
    std::vector<Op> ops;
    ops.swap(t_ops);
    return run_group(ops);
}

inline ncclResult_t allReduce(const void *sb, void *rb, size_t count, ncclDataType_t t, ncclRedOp_t op, ncclComm_t c,
                              cudaStream_t s) {
    Comm *comm = reinterpret_cast<Comm *>(c);
    const size_t ts = type_size(t);
    const bool i64 = t == ncclInt64, i32 = t == ncclInt32;
    if (!comm || !(i64 || i32) || !(op == ncclSum || op == ncclMax)) return ncclInvalidArgument;
    std::vector<int64_t> v(count);
    std::vector<char> raw(count * ts);
    if (cudaMemcpyAsync(raw.data(), sb, count * ts, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
        return ncclUnhandledCudaError;
    for (size_t i = 0; i < count; i++)
        v[i] = i64 ? reinterpret_cast<int64_t *>(raw.data())[i] : reinterpret_cast<int32_t *>(raw.data())[i];
    Group &g = *comm->grp;
    std::shared_ptr<std::vector<int64_t>> res;
    {
        std::unique_lock<std::mutex> lk(g.mu);
        if (g.arrived == 0) {
            g.acc = v;
        } else {
            if (g.acc.size() != count) return ncclInvalidArgument;
            for (size_t i = 0; i < count; i++) g.acc[i] = op == ncclSum ? g.acc[i] + v[i] : std::max(g.acc[i], v[i]);
        }
        const uint64_t my_gen = g.gen;
        if (++g.arrived == g.nranks) {
            g.result = std::make_shared<std::vector<int64_t>>(g.acc);
            g.arrived = 0;
            g.gen++;
            g.cv.notify_all();
        } else {
            g.cv.wait(lk, [&] { return g.gen != my_gen; });
        }
        res = g.result;
    }
    for (size_t i = 0; i < count; i++) {
        if (i64) reinterpret_cast<int64_t *>(raw.data())[i] = (*res)[i];
        else reinterpret_cast<int32_t *>(raw.data())[i] = (int32_t)(*res)[i];
    }
    if (cudaMemcpyAsync(rb, raw.data(), count * ts, cudaMemcpyHostToDevice, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
        return ncclUnhandledCudaError;
    return ncclSuccess;
}

inline NcclApi api() {
    NcclApi a;
    a.getUniqueId = getUniqueId;
    a.commInitRank = commInitRank;
    a.commDestroy = commDestroy;
    a.send = send;
    a.recv = recv;
    a.allReduce = allReduce;
    a.groupStart = groupStart;
    a.groupEnd = groupEnd;
    a.ok = true;
    return a;
}

}  // namespace loopback
}  // namespace cg
