// nccl_emu.cu -- TEST INFRASTRUCTURE: an in-process stand-in for libnccl.so.2 so the
// NCCL branches of the slab decomposition (csrc/petto_dev.cu "teams": all-reduce,
// send/recv halos, the REPLICA chain, broadcast) run with several ranks on ONE GPU.
//
// Real NCCL refuses two ranks on one device ("Duplicate GPU detected"), so the
// multi-rank NCCL path could otherwise only run on a multi-GPU node.  Here every
// rank is a host thread of one process driving its own context; the library is
// loaded through PETTO_NCCL_LIB.  Semantics kept from NCCL:
//   * calls never block the host (except ncclCommInitRank, a rendezvous);
//   * every operation is ordered on the caller's stream: at call time the rank
//     records an event on its stream and makes the stream wait (cuStreamWaitValue32)
//     on a device flag; once every participant has posted, the data movement is
//     enqueued on the communicator's stream after all participants' events, then
//     every participant's flag is released (cuStreamWriteValue32);
//   * collectives match by per-rank call order, point-to-point by the k-th message
//     between a (sender, receiver) pair; inside ncclGroupStart/End the stream waits
//     are deferred to ncclGroupEnd and the group's operations count as one step of
//     the rank's program (NCCL progresses a group's sends and receives together).
// Operations are enqueued on the communicator's ONE stream in an order consistent
// with every rank's program order (an operation waits until each participant's
// earlier operations are enqueued), so that FIFO stream never holds an operation
// behind one it depends on.  Stream waits block the hardware work queue a stream is
// mapped to, so the process needs CUDA_DEVICE_MAX_CONNECTIONS=32 (one queue per
// stream) and CUDA_MODULE_LOADING=EAGER (a lazy module load synchronises the
// device).  Only streams wait (stream memory operations), no kernel waits on a rank.
#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <condition_variable>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

namespace {

typedef CUresult (*StreamValueFn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

StreamValueFn drv(const char* name) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) == cudaSuccess && q == cudaDriverEntryPointSuccess)
        return reinterpret_cast<StreamValueFn>(p);
    return nullptr;
}

bool trace_on() {
    static const bool on = std::getenv("EMU_TRACE") && std::getenv("EMU_TRACE")[0] == '1';
    return on;
}

size_t type_size(ncclDataType_t t) {
    switch (t) {
        case ncclInt8: case ncclUint8: return 1;
        case ncclFloat16: case ncclBfloat16: return 2;
        case ncclInt32: case ncclUint32: case ncclFloat32: return 4;
        default: return 8;
    }
}

struct Post {
    int rank = -1;
    long long seq = 0;          // the rank's program step of this operation
    const void* send = nullptr;
    void* recv = nullptr;
    cudaEvent_t ev = nullptr;   // the caller's stream reached the operation
    unsigned* flag = nullptr;   // the caller's stream waits for it
};

struct Op {
    int kind = 0;               // 0 all-reduce, 1 broadcast, 2 send/recv
    size_t count = 0;
    ncclDataType_t type = ncclFloat64;
    ncclRedOp_t red = ncclSum;
    int root = 0;
    int needed = 0;             // participants
    std::vector<Post> posts;    // send/recv: [0] sender, [1] receiver
    int posted = 0;
};

struct Shared {
    int nranks = 0, joined = 0;
    std::mutex m;
    std::condition_variable cv;
    cudaStream_t stream = nullptr;  // where the data movement runs (FIFO)
    unsigned* flags = nullptr;      // stream flags, preallocated (no allocation once ranks wait)
    long long next_flag = 0;
    static constexpr long long NFLAGS = 1 << 22;
    char* tmp = nullptr;            // reduction scratch ring
    static constexpr long long TMP_SLOT = 4096, NTMP = 4096;
    long long next_tmp = 0;
    // matching
    long long next_id = 0;
    std::map<long long, Op> ops;                          // id -> op (not yet enqueued)
    std::vector<long long> coll_seq;                      // per rank: collectives posted
    std::map<long long, long long> coll_id;               // collective index -> op id
    std::map<std::pair<int, int>, long long> sent, recvd; // (src, dst) -> messages posted
    std::map<std::tuple<int, int, long long>, long long> p2p_id;
    // program order
    std::vector<long long> seq;                           // per rank: next program step
    std::vector<std::map<long long, int>> pending;        // per rank: step -> ops not yet enqueued
};

std::mutex g_m;
std::map<std::string, std::shared_ptr<Shared>> g_comms;
long long g_ids = 0;

struct Inputs {
    const void* p[8];
};

// in rank order (the emulator's own deterministic reduction order)
template <class T>
__global__ void k_reduce(Inputs in, int n, size_t count, int op, T* out) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
        T a = static_cast<const T*>(in.p[0])[i];
        for (int r = 1; r < n; ++r) {
            const T b = static_cast<const T*>(in.p[r])[i];
            a = op == ncclSum ? a + b : op == ncclMax ? (a > b ? a : b) : (a < b ? a : b);
        }
        out[i] = a;
    }
}

// the data movement of a fully posted operation, on the communicator's stream
ncclResult_t execute(Shared& s, Op& op) {
    static StreamValueFn wr = drv("cuStreamWriteValue32");
    for (const Post& p : op.posts) cudaStreamWaitEvent(s.stream, p.ev, 0);
    const size_t bytes = op.count * type_size(op.type);
    if (op.kind == 2) {
        cudaMemcpyAsync(op.posts[1].recv, op.posts[0].send, bytes, cudaMemcpyDefault, s.stream);
    } else if (op.kind == 1) {
        const void* src = nullptr;
        for (const Post& p : op.posts)
            if (p.rank == op.root) src = p.send;
        for (const Post& p : op.posts)
            if (p.recv != src) cudaMemcpyAsync(p.recv, src, bytes, cudaMemcpyDefault, s.stream);
    } else {
        const int n = (int)op.posts.size();
        if (n > 8 || bytes > (size_t)Shared::TMP_SLOT) return ncclInvalidArgument;
        Inputs in{};
        for (const Post& p : op.posts) in.p[p.rank] = p.send;
        void* tmp = s.tmp + (s.next_tmp++ % Shared::NTMP) * Shared::TMP_SLOT;
        const int blocks = (int)std::min<size_t>(1024, (op.count + 255) / 256 + 1);
        switch (op.type) {
            case ncclFloat64:
                k_reduce<double><<<blocks, 256, 0, s.stream>>>(in, n, op.count, op.red, static_cast<double*>(tmp));
                break;
            case ncclInt64:
                k_reduce<long long><<<blocks, 256, 0, s.stream>>>(in, n, op.count, op.red,
                                                                  static_cast<long long*>(tmp));
                break;
            case ncclUint64:
                k_reduce<unsigned long long><<<blocks, 256, 0, s.stream>>>(in, n, op.count, op.red,
                                                                           static_cast<unsigned long long*>(tmp));
                break;
            case ncclUint32:
                k_reduce<unsigned><<<blocks, 256, 0, s.stream>>>(in, n, op.count, op.red, static_cast<unsigned*>(tmp));
                break;
            default:
                return ncclInvalidArgument;
        }
        for (const Post& p : op.posts) cudaMemcpyAsync(p.recv, tmp, bytes, cudaMemcpyDeviceToDevice, s.stream);
    }
    for (const Post& p : op.posts)
        if (wr(reinterpret_cast<CUstream>(s.stream), reinterpret_cast<CUdeviceptr>(p.flag), 1, 0) != CUDA_SUCCESS)
            return ncclSystemError;
    if (trace_on()) std::fprintf(stderr, "emu execute kind %d count %zu\n", op.kind, op.count);
    return cudaGetLastError() == cudaSuccess ? ncclSuccess : ncclUnhandledCudaError;
}

// enqueue every fully posted operation whose participants' earlier program steps
// are all enqueued (repeat until nothing moves); caller holds s.m
ncclResult_t drain(Shared& s) {
    for (bool moved = true; moved;) {
        moved = false;
        for (auto it = s.ops.begin(); it != s.ops.end();) {
            Op& op = it->second;
            bool ready = op.posted == op.needed;
            for (int i = 0; ready && i < (int)op.posts.size(); ++i) {
                const Post& p = op.posts[i];
                ready = s.pending[p.rank].begin()->first == p.seq;  // the rank's lowest pending step
            }
            if (!ready) {
                ++it;
                continue;
            }
            if (ncclResult_t r = execute(s, op)) return r;
            for (const Post& p : op.posts) {
                auto& pend = s.pending[p.rank];
                if (--pend[p.seq] == 0) pend.erase(p.seq);
            }
            it = s.ops.erase(it);
            moved = true;
        }
    }
    return ncclSuccess;
}

// Inside ncclGroupStart/End the stream waits are deferred to ncclGroupEnd and the
// group's operations share one program step per (communicator, rank).
thread_local int g_depth = 0;
thread_local std::vector<std::pair<cudaStream_t, unsigned*>> g_waits;
thread_local std::map<Shared*, long long> g_group_seq;

ncclResult_t stream_wait(cudaStream_t stream, unsigned* flag) {
    static StreamValueFn wt = drv("cuStreamWaitValue32");
    return wt(reinterpret_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(flag), 1, 0x0 /*GEQ*/) == CUDA_SUCCESS
               ? ncclSuccess
               : ncclSystemError;
}

// the caller's side of any operation: event + (deferred) stream wait on a fresh
// flag, and its program step; caller holds s.m
ncclResult_t post(Shared& s, Post& p, int rank, const void* send, void* recv, cudaStream_t stream) {
    p.rank = rank;
    p.send = send;
    p.recv = recv;
    if (s.next_flag >= Shared::NFLAGS) return ncclSystemError;
    p.flag = s.flags + s.next_flag++;
    if (g_depth > 0) {
        auto it = g_group_seq.find(&s);
        if (it == g_group_seq.end()) it = g_group_seq.emplace(&s, s.seq[rank]++).first;
        p.seq = it->second;
    } else {
        p.seq = s.seq[rank]++;
    }
    s.pending[rank][p.seq]++;
    if (cudaEventCreateWithFlags(&p.ev, cudaEventDisableTiming) != cudaSuccess) return ncclSystemError;
    cudaEventRecord(p.ev, stream);
    if (g_depth > 0) {
        g_waits.emplace_back(stream, p.flag);
        return ncclSuccess;
    }
    return stream_wait(stream, p.flag);
}

}  // namespace

struct ncclComm {
    std::shared_ptr<Shared> s;
    int rank;
};

namespace {

ncclResult_t collective(ncclComm_t c, int kind, const void* send, void* recv, size_t count, ncclDataType_t t,
                        ncclRedOp_t red, int root, cudaStream_t stream) {
    Shared& s = *c->s;
    std::lock_guard<std::mutex> lk(s.m);
    Post p;
    if (ncclResult_t r = post(s, p, c->rank, send, recv, stream)) return r;
    const long long k = s.coll_seq[c->rank]++;
    if (trace_on()) std::fprintf(stderr, "emu rank %d collective %d #%lld\n", c->rank, kind, k);
    auto idit = s.coll_id.find(k);
    if (idit == s.coll_id.end()) idit = s.coll_id.emplace(k, s.next_id++).first;
    Op& op = s.ops[idit->second];
    if (op.posted == 0) {
        op.kind = kind;
        op.count = count;
        op.type = t;
        op.red = red;
        op.root = root;
        op.needed = s.nranks;
    } else if (op.kind != kind || op.count != count || op.type != t) {
        return ncclInvalidUsage;  // mismatched collective order across ranks
    }
    op.posts.push_back(p);
    if (++op.posted == op.needed) s.coll_id.erase(k);
    return drain(s);
}

ncclResult_t p2p(ncclComm_t c, bool is_send, void* buf, size_t count, ncclDataType_t t, int peer,
                 cudaStream_t stream) {
    Shared& s = *c->s;
    std::lock_guard<std::mutex> lk(s.m);
    Post p;
    if (ncclResult_t r = post(s, p, c->rank, is_send ? buf : nullptr, is_send ? nullptr : buf, stream)) return r;
    const int src = is_send ? c->rank : peer, dst = is_send ? peer : c->rank;
    const long long k = is_send ? s.sent[{src, dst}]++ : s.recvd[{src, dst}]++;
    if (trace_on())
        std::fprintf(stderr, "emu rank %d %s %d->%d #%lld\n", c->rank, is_send ? "send" : "recv", src, dst, k);
    const auto key = std::make_tuple(src, dst, k);
    auto idit = s.p2p_id.find(key);
    if (idit == s.p2p_id.end()) idit = s.p2p_id.emplace(key, s.next_id++).first;
    Op& op = s.ops[idit->second];
    if (op.posted == 0) {
        op.kind = 2;
        op.count = count;
        op.type = t;
        op.needed = 2;
        op.posts.resize(2);
    } else if (op.count != count || op.type != t) {
        return ncclInvalidUsage;
    }
    op.posts[is_send ? 0 : 1] = p;
    if (++op.posted == op.needed) s.p2p_id.erase(key);
    return drain(s);
}

}  // namespace

extern "C" {

ncclResult_t ncclGetUniqueId(ncclUniqueId* id) {
    std::lock_guard<std::mutex> lk(g_m);
    std::memset(id, 0, sizeof(*id));
    std::snprintf(id->internal, sizeof(id->internal), "nccl-emu-%lld", ++g_ids);
    return ncclSuccess;
}

ncclResult_t ncclCommInitRank(ncclComm_t* comm, int nranks, ncclUniqueId id, int rank) {
    std::shared_ptr<Shared> s;
    {
        std::lock_guard<std::mutex> lk(g_m);
        std::shared_ptr<Shared>& e = g_comms[std::string(id.internal)];
        if (!e) {
            e = std::make_shared<Shared>();
            e->nranks = nranks;
            e->coll_seq.assign(nranks, 0);
            e->seq.assign(nranks, 0);
            e->pending.resize(nranks);
            if (cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking) != cudaSuccess ||
                cudaMalloc(&e->flags, sizeof(unsigned) * Shared::NFLAGS) != cudaSuccess ||
                cudaMemset(e->flags, 0, sizeof(unsigned) * Shared::NFLAGS) != cudaSuccess ||
                cudaMalloc(&e->tmp, Shared::TMP_SLOT * Shared::NTMP) != cudaSuccess)
                return ncclSystemError;
            // load the reduction kernels now (lazy module loading may synchronise)
            cudaFuncAttributes fa;
            cudaFuncGetAttributes(&fa, k_reduce<double>);
            cudaFuncGetAttributes(&fa, k_reduce<long long>);
            cudaFuncGetAttributes(&fa, k_reduce<unsigned long long>);
            cudaFuncGetAttributes(&fa, k_reduce<unsigned>);
            cudaDeviceSynchronize();
        }
        s = e;
    }
    if (rank < 0 || rank >= nranks || s->nranks != nranks) return ncclInvalidArgument;
    std::unique_lock<std::mutex> lk(s->m);
    ++s->joined;
    s->cv.notify_all();
    s->cv.wait(lk, [&] { return s->joined >= s->nranks; });
    *comm = new ncclComm{s, rank};
    return ncclSuccess;
}

ncclResult_t ncclCommDestroy(ncclComm_t comm) {
    delete comm;
    return ncclSuccess;
}

ncclResult_t ncclAllReduce(const void* send, void* recv, size_t count, ncclDataType_t t, ncclRedOp_t op,
                           ncclComm_t comm, cudaStream_t stream) {
    return collective(comm, 0, send, recv, count, t, op, 0, stream);
}

ncclResult_t ncclBroadcast(const void* send, void* recv, size_t count, ncclDataType_t t, int root, ncclComm_t comm,
                           cudaStream_t stream) {
    return collective(comm, 1, send, recv, count, t, ncclSum, root, stream);
}

ncclResult_t ncclSend(const void* buf, size_t count, ncclDataType_t t, int peer, ncclComm_t comm,
                      cudaStream_t stream) {
    return p2p(comm, true, const_cast<void*>(buf), count, t, peer, stream);
}

ncclResult_t ncclRecv(void* buf, size_t count, ncclDataType_t t, int peer, ncclComm_t comm, cudaStream_t stream) {
    return p2p(comm, false, buf, count, t, peer, stream);
}

ncclResult_t ncclGroupStart() {
    ++g_depth;
    return ncclSuccess;
}

ncclResult_t ncclGroupEnd() {
    if (g_depth == 0) return ncclInvalidUsage;
    if (--g_depth > 0) return ncclSuccess;
    for (const auto& w : g_waits)
        if (ncclResult_t r = stream_wait(w.first, w.second)) return r;
    g_waits.clear();
    g_group_seq.clear();
    return ncclSuccess;
}

const char* ncclGetErrorString(ncclResult_t r) { return r == ncclSuccess ? "success" : "nccl-emu error"; }

}  // extern "C"
