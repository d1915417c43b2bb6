// nccl_emu_mp.cu -- TEST INFRASTRUCTURE: a multi-PROCESS stand-in for libnccl.so.2,
// so that the deployment shape of the slab decomposition -- one process per rank
// under torchrun, bench.py --gpus N included -- runs with N ranks on ONE GPU
// (real NCCL refuses two ranks on one device: "Duplicate GPU detected").
//
// Loaded through PETTO_NCCL_LIB.  The ranks share one file mapping (under /tmp,
// named by the unique id) that holds, per rank, a collective slot and, per
// (sender, receiver) pair, a mailbox; sequence / acknowledgement counters are
// lock-free atomics in that mapping.  Unlike the in-process emulator
// (nccl_emu.cu), the calls are host-blocking: an operation synchronises the
// caller's stream, moves its bytes through the mapping and returns once its
// result is on the device -- stream order is kept (everything enqueued after the
// call runs after it) at the price of overlap, which is not what these runs
// measure.  Collectives match by per-communicator call order, point-to-point by
// the k-th message of a (sender, receiver) pair (a ring of NMSG messages per
// pair); inside ncclGroupStart/End the sends run first, so paired exchanges of up
// to NMSG messages per peer cannot deadlock.  Reductions combine the
// ranks' contributions in rank order (the same bits on every rank).
#include <cuda_runtime.h>
#include <fcntl.h>
#include <nccl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <time.h>
#include <unistd.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

namespace {

constexpr int MAXR = 8;
constexpr size_t SLOT = 1 << 20;   // bytes of one rank's collective contribution
constexpr int NMSG = 8;            // messages in flight per (sender, receiver) pair
constexpr size_t MSG = 4 << 20;    // bytes of one point-to-point message

struct Slot {
    std::atomic<uint64_t> seq;   // collective number posted
    std::atomic<uint64_t> ack;   // collective number whose inputs this rank has read
    unsigned char data[SLOT];
};
struct Box {                     // a ring of NMSG messages
    std::atomic<uint64_t> seq;   // messages posted
    std::atomic<uint64_t> ack;   // messages consumed
    uint64_t bytes[NMSG];
    unsigned char data[NMSG][MSG];
};
struct Shared {
    std::atomic<int> arrived;
    Slot slot[MAXR];
    Box box[MAXR][MAXR];   // [sender][receiver]
};

struct Comm {
    int rank = 0, n = 0;
    Shared* sh = nullptr;
    std::string path;
    uint64_t cseq = 0;               // collectives issued
    uint64_t sent[MAXR] = {}, recvd[MAXR] = {};
    std::vector<unsigned char> tmp;  // reduction result
};

struct Pending {
    int kind;  // 0 send, 1 recv, 2 all-reduce, 3 broadcast
    const void* sbuf;
    void* rbuf;
    size_t bytes;
    ncclDataType_t type;
    ncclRedOp_t op;
    int peer;
    Comm* comm;
    cudaStream_t stream;
};
thread_local int group_depth = 0;
thread_local std::vector<Pending> group_ops;

size_t type_size(ncclDataType_t t) {
    switch (t) {
        case ncclInt8: case ncclUint8: return 1;
        case ncclFloat16: case ncclBfloat16: return 2;
        case ncclInt32: case ncclUint32: case ncclFloat32: return 4;
        default: return 8;
    }
}

void spin_until(const std::atomic<uint64_t>& a, uint64_t v) {
    const time_t t0 = time(nullptr);
    int k = 0;
    while (a.load(std::memory_order_acquire) < v) {
        if (++k > 64) usleep(20);
        if (time(nullptr) - t0 > 120) {
            fprintf(stderr, "nccl_emu_mp: a peer did not arrive within 120 s\n");
            abort();
        }
    }
}

template <class T>
void combine(T* acc, const T* x, size_t n, ncclRedOp_t op) {
    for (size_t i = 0; i < n; ++i) {
        switch (op) {
            case ncclSum: acc[i] = acc[i] + x[i]; break;
            case ncclProd: acc[i] = acc[i] * x[i]; break;
            case ncclMax: acc[i] = acc[i] < x[i] ? x[i] : acc[i]; break;
            case ncclMin: acc[i] = x[i] < acc[i] ? x[i] : acc[i]; break;
            default: break;
        }
    }
}

void reduce_into(void* acc, const void* x, size_t count, ncclDataType_t t, ncclRedOp_t op) {
    switch (t) {
        case ncclInt8: combine((int8_t*)acc, (const int8_t*)x, count, op); break;
        case ncclUint8: combine((uint8_t*)acc, (const uint8_t*)x, count, op); break;
        case ncclInt32: combine((int32_t*)acc, (const int32_t*)x, count, op); break;
        case ncclUint32: combine((uint32_t*)acc, (const uint32_t*)x, count, op); break;
        case ncclInt64: combine((int64_t*)acc, (const int64_t*)x, count, op); break;
        case ncclUint64: combine((uint64_t*)acc, (const uint64_t*)x, count, op); break;
        case ncclFloat32: combine((float*)acc, (const float*)x, count, op); break;
        default: combine((double*)acc, (const double*)x, count, op); break;
    }
}

ncclResult_t cuda_ok(cudaError_t e) {
    if (e == cudaSuccess) return ncclSuccess;
    fprintf(stderr, "nccl_emu_mp: %s\n", cudaGetErrorString(e));
    return ncclUnhandledCudaError;
}

// a copy on the caller's stream, complete on return (a plain cudaMemcpy from
// pageable memory returns before its DMA lands and is not ordered with a
// non-blocking stream)
ncclResult_t copy(void* dst, const void* src, size_t bytes, cudaMemcpyKind kind, cudaStream_t s) {
    if (ncclResult_t e = cuda_ok(cudaMemcpyAsync(dst, src, bytes, kind, s))) return e;
    return cuda_ok(cudaStreamSynchronize(s));
}

// all-reduce (kind 2) and broadcast (kind 3, peer = root): post, wait for every
// rank, combine in rank order, acknowledge
ncclResult_t collective(const Pending& p) {
    Comm* c = p.comm;
    if (p.bytes > SLOT) return ncclInvalidArgument;
    const uint64_t s = ++c->cseq;
    // this rank's slot is free once every rank has read the previous collective
    for (int r = 0; r < c->n; ++r) spin_until(c->sh->slot[r].ack, s - 1);
    if (ncclResult_t e = cuda_ok(cudaStreamSynchronize(p.stream))) return e;
    Slot& mine = c->sh->slot[c->rank];
    if (p.kind == 2 || c->rank == p.peer)
        if (ncclResult_t e = copy(mine.data, p.sbuf, p.bytes, cudaMemcpyDeviceToHost, p.stream)) return e;
    mine.seq.store(s, std::memory_order_release);
    for (int r = 0; r < c->n; ++r) spin_until(c->sh->slot[r].seq, s);
    c->tmp.resize(p.bytes);
    if (p.kind == 3) {
        memcpy(c->tmp.data(), c->sh->slot[p.peer].data, p.bytes);
    } else {
        memcpy(c->tmp.data(), c->sh->slot[0].data, p.bytes);
        for (int r = 1; r < c->n; ++r)
            reduce_into(c->tmp.data(), c->sh->slot[r].data, p.bytes / type_size(p.type), p.type, p.op);
    }
    mine.ack.store(s, std::memory_order_release);
    return copy(p.rbuf, c->tmp.data(), p.bytes, cudaMemcpyHostToDevice, p.stream);
}

ncclResult_t send(const Pending& p) {
    Comm* c = p.comm;
    if (p.bytes > MSG || p.peer < 0 || p.peer >= c->n) return ncclInvalidArgument;
    Box& b = c->sh->box[c->rank][p.peer];
    const uint64_t s = ++c->sent[p.peer];
    if (s > NMSG) spin_until(b.ack, s - NMSG);  // the ring slot is free
    const int k = (int)((s - 1) % NMSG);
    if (ncclResult_t e = copy(b.data[k], p.sbuf, p.bytes, cudaMemcpyDeviceToHost, p.stream)) return e;
    b.bytes[k] = p.bytes;
    b.seq.store(s, std::memory_order_release);
    return ncclSuccess;
}

ncclResult_t recv(const Pending& p) {
    Comm* c = p.comm;
    if (p.peer < 0 || p.peer >= c->n) return ncclInvalidArgument;
    Box& b = c->sh->box[p.peer][c->rank];
    const uint64_t s = ++c->recvd[p.peer];
    spin_until(b.seq, s);
    const int k = (int)((s - 1) % NMSG);
    if (b.bytes[k] != p.bytes) {
        fprintf(stderr, "nccl_emu_mp: rank %d expected %zu bytes from %d, got %llu\n", c->rank, p.bytes, p.peer,
                (unsigned long long)b.bytes[k]);
        return ncclInvalidUsage;
    }
    if (ncclResult_t e = copy(p.rbuf, b.data[k], p.bytes, cudaMemcpyHostToDevice, p.stream)) return e;
    b.ack.store(s, std::memory_order_release);
    return ncclSuccess;
}

ncclResult_t run(const Pending& p) {
    switch (p.kind) {
        case 0: return send(p);
        case 1: return recv(p);
        default: return collective(p);
    }
}

ncclResult_t submit(const Pending& p) {
    if (group_depth > 0) {
        group_ops.push_back(p);
        return ncclSuccess;
    }
    return run(p);
}

}  // namespace

extern "C" {

ncclResult_t ncclGetUniqueId(ncclUniqueId* id) {
    memset(id, 0, sizeof(*id));
    timespec ts;
    clock_gettime(CLOCK_REALTIME, &ts);
    snprintf(id->internal, sizeof(id->internal), "petto_emu_mp_%d_%lld_%ld", (int)getpid(), (long long)ts.tv_sec,
             ts.tv_nsec);
    return ncclSuccess;
}

ncclResult_t ncclCommInitRank(ncclComm_t* out, int nranks, ncclUniqueId id, int rank) {
    if (nranks < 1 || nranks > MAXR || rank < 0 || rank >= nranks) return ncclInvalidArgument;
    Comm* c = new Comm;
    c->rank = rank;
    c->n = nranks;
    const char* dir = std::getenv("NCCL_EMU_DIR");
    c->path = std::string(dir ? dir : "/tmp") + "/" + std::string(id.internal, strnlen(id.internal, 120));
    const int fd = open(c->path.c_str(), O_RDWR | O_CREAT, 0600);
    if (fd < 0) {
        delete c;
        return ncclSystemError;
    }
    // every rank extends the (sparse) file to the same size; fresh pages read zero,
    // which is the initial state of every counter
    if (ftruncate(fd, sizeof(Shared)) != 0) {
        close(fd);
        delete c;
        return ncclSystemError;
    }
    void* m = mmap(nullptr, sizeof(Shared), PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (m == MAP_FAILED) {
        delete c;
        return ncclSystemError;
    }
    c->sh = static_cast<Shared*>(m);
    c->sh->arrived.fetch_add(1);
    const time_t t0 = time(nullptr);
    while (c->sh->arrived.load() < nranks) {
        usleep(100);
        if (time(nullptr) - t0 > 120) return ncclSystemError;
    }
    // every rank has mapped the file: drop its name (nothing is left in /tmp, even
    // when a rank process exits without destroying its communicator)
    if (rank == 0) unlink(c->path.c_str());
    *out = reinterpret_cast<ncclComm_t>(c);
    return ncclSuccess;
}

ncclResult_t ncclCommDestroy(ncclComm_t comm) {
    Comm* c = reinterpret_cast<Comm*>(comm);
    if (!c) return ncclSuccess;
    munmap(c->sh, sizeof(Shared));
    delete c;
    return ncclSuccess;
}

ncclResult_t ncclSend(const void* buf, size_t count, ncclDataType_t t, int peer, ncclComm_t comm, cudaStream_t s) {
    return submit({0, buf, nullptr, count * type_size(t), t, ncclSum, peer, reinterpret_cast<Comm*>(comm), s});
}

ncclResult_t ncclRecv(void* buf, size_t count, ncclDataType_t t, int peer, ncclComm_t comm, cudaStream_t s) {
    return submit({1, nullptr, buf, count * type_size(t), t, ncclSum, peer, reinterpret_cast<Comm*>(comm), s});
}

ncclResult_t ncclAllReduce(const void* sb, void* rb, size_t count, ncclDataType_t t, ncclRedOp_t op,
                           ncclComm_t comm, cudaStream_t s) {
    return submit({2, sb, rb, count * type_size(t), t, op, -1, reinterpret_cast<Comm*>(comm), s});
}

ncclResult_t ncclBroadcast(const void* sb, void* rb, size_t count, ncclDataType_t t, int root, ncclComm_t comm,
                           cudaStream_t s) {
    return submit({3, sb, rb, count * type_size(t), t, ncclSum, root, reinterpret_cast<Comm*>(comm), s});
}

ncclResult_t ncclGroupStart() {
    ++group_depth;
    return ncclSuccess;
}

ncclResult_t ncclGroupEnd() {
    if (group_depth == 0) return ncclInvalidUsage;
    if (--group_depth > 0) return ncclSuccess;
    std::vector<Pending> ops;
    ops.swap(group_ops);
    int per_peer[MAXR] = {};
    for (const Pending& p : ops)
        if (p.kind == 0 && p.peer >= 0 && p.peer < MAXR && ++per_peer[p.peer] > NMSG) return ncclInvalidUsage;
    ncclResult_t rc = ncclSuccess;
    for (const Pending& p : ops)  // sends first: a group's receives never wait on its own sends
        if (p.kind == 0 && rc == ncclSuccess) rc = run(p);
    for (const Pending& p : ops)
        if (p.kind != 0 && rc == ncclSuccess) rc = run(p);
    return rc;
}

const char* ncclGetErrorString(ncclResult_t r) {
    switch (r) {
        case ncclSuccess: return "no error (nccl_emu_mp)";
        case ncclInvalidArgument: return "invalid argument (nccl_emu_mp)";
        case ncclInvalidUsage: return "invalid usage (nccl_emu_mp)";
        case ncclSystemError: return "system error (nccl_emu_mp)";
        default: return "CUDA error (nccl_emu_mp)";
    }
}

}  // extern "C"
