// nccl_shim.cu -- TEST INFRASTRUCTURE: the subset of the NCCL ABI the z-slab
// transport uses (csrc/slab.cu, namespace nccl), for 2..8 ranks that are
// processes on ONE GPU, so the distributed data plane (send/recv halo rows
// with one or two neighbours, foreign-plane zeroing, all-reduces of plane
// sums / max / min / histograms, the eager retry loop) runs end to end
// without a multi-GPU box.
//
// Transport: every rank owns a device staging buffer exported by CUDA IPC;
// the handshake lives in a POSIX shared-memory segment named by the unique
// id.  All synchronisation is on the host: a group end (or an all-reduce)
// synchronises the caller's stream, copies the rank's sends into its own
// staging buffer (with a table of (destination, offset, bytes)), publishes a
// sequence number, waits for the sequence number of every rank it receives
// from, and copies the matching sends out of their staging buffers.  No
// kernel ever waits on another process, so ranks sharing a GPU cannot
// deadlock it.  Semantics follow NCCL: within a group the k-th send from a
// rank to a peer matches the peer's k-th receive from that rank; all-reduce
// combines the ranks in rank order (identical bits on every rank).  Every
// rank must issue the same sequence of group ends and all-reduces (the slab
// transport does: the same plan structure on every rank).
//
// Exported: ncclGetUniqueId, ncclCommInitRank, ncclCommDestroy, ncclSend,
// ncclRecv, ncclAllReduce, ncclGroupStart, ncclGroupEnd, ncclGetErrorString.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <random>
#include <thread>
#include <vector>

namespace {

constexpr int kMaxRanks = 8;
constexpr size_t kStage = 128ull << 20;  // staging bytes per rank
constexpr int kMaxOps = 256;

struct OpDesc {
    int dst;
    uint64_t off, bytes;
};

struct Shared {
    std::atomic<int> joined;
    cudaIpcMemHandle_t stage[kMaxRanks];
    std::atomic<uint64_t> posted[kMaxRanks];    // last published op sequence of rank r
    std::atomic<uint64_t> consumed[kMaxRanks];  // last op sequence rank r has finished reading
    int nsend[kMaxRanks];
    OpDesc send[kMaxRanks][kMaxOps];            // rank r's sends of its last published op
};

}  // namespace

// the communicator (external linkage: it appears in the exported C ABI)
struct ncclComm {
    int rank = 0, nranks = 0;
    Shared* sh = nullptr;
    char name[64] = {};
    void* stage = nullptr;               // own staging buffer
    void* peer_stage[kMaxRanks] = {};    // the others', opened by IPC
    uint64_t seq = 0;
    void* tmp = nullptr;                 // all-reduce scratch (one slot per rank)
    cudaStream_t copy = nullptr;         // the shim's copy stream (D2D cudaMemcpy does not block the host)
};
typedef ncclComm Comm;

namespace {

struct PendingOp {
    bool send;
    void* buf;
    size_t bytes;
    int peer;
    cudaStream_t stream;
};

thread_local int g_group_depth = 0;
thread_local std::vector<PendingOp> g_pending;
thread_local Comm* g_group_comm = nullptr;

size_t dtype_size(int dt) {
    switch (dt) {
        case 0: case 1: return 1;          // int8, uint8
        case 2: case 3: case 7: return 4;  // int32, uint32, float32
        case 4: case 5: case 8: return 8;  // int64, uint64, float64
        case 6: return 2;                  // float16
        default: return 0;
    }
}

void spin_until(const std::atomic<uint64_t>& a, uint64_t v) {
    auto t0 = std::chrono::steady_clock::now();
    while (a.load(std::memory_order_acquire) < v) {
        std::this_thread::yield();
        if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(120)) {
            std::fprintf(stderr, "nccl_shim: a peer did not arrive within 120 s\n");
            std::abort();
        }
    }
}

int check(cudaError_t e) {
    if (e != cudaSuccess) {
        std::fprintf(stderr, "nccl_shim: %s\n", cudaGetErrorString(e));
        return 1;
    }
    return 0;
}

// One exchange step: publish `sends` (copied back to back into the own
// staging buffer), then copy each peer's sends addressed to this rank, in
// their issue order, into this rank's receives from that peer.
int exchange(Comm* c, cudaStream_t s, const std::vector<PendingOp>& sends, const std::vector<PendingOp>& recvs) {
    const int me = c->rank;
    if (check(cudaStreamSynchronize(s))) return 1;
    const uint64_t seq = ++c->seq;
    // every rank has finished reading our previous op's staging
    for (int r = 0; r < c->nranks; ++r)
        if (r != me) spin_until(c->sh->consumed[r], seq - 1);
    if ((int)sends.size() > kMaxOps) return 1;
    uint64_t off = 0;
    for (size_t k = 0; k < sends.size(); ++k) {
        if (off + sends[k].bytes > kStage) return 1;
        if (check(cudaMemcpyAsync((char*)c->stage + off, sends[k].buf, sends[k].bytes, cudaMemcpyDeviceToDevice,
                                  c->copy)))
            return 1;
        c->sh->send[me][k] = OpDesc{sends[k].peer, off, sends[k].bytes};
        off += (sends[k].bytes + 255) & ~255ull;
    }
    if (check(cudaStreamSynchronize(c->copy))) return 1;  // staged before it is published
    c->sh->nsend[me] = (int)sends.size();
    c->sh->posted[me].store(seq, std::memory_order_release);
    // receives, matched per source in issue order
    int next[kMaxRanks] = {0};
    for (const PendingOp& rv : recvs) {
        const int src = rv.peer;
        spin_until(c->sh->posted[src], seq);
        int k = next[src];
        while (k < c->sh->nsend[src] && c->sh->send[src][k].dst != me) ++k;
        if (k >= c->sh->nsend[src]) {
            std::fprintf(stderr, "nccl_shim: rank %d receives more from %d than it sent\n", me, src);
            return 1;
        }
        const OpDesc d = c->sh->send[src][k];
        next[src] = k + 1;
        if (d.bytes != rv.bytes) {
            std::fprintf(stderr, "nccl_shim: recv of %zu bytes matches a send of %llu\n", rv.bytes,
                         (unsigned long long)d.bytes);
            return 1;
        }
        if (check(cudaMemcpyAsync(rv.buf, (char*)c->peer_stage[src] + d.off, d.bytes, cudaMemcpyDeviceToDevice,
                                  c->copy)))
            return 1;
    }
    if (check(cudaStreamSynchronize(c->copy))) return 1;  // read before the peers may reuse their staging
    c->sh->consumed[me].store(seq, std::memory_order_release);
    return 0;
}

// out = op over ranks 0..nr-1 of in[r] (rank order), element-wise
template <class T>
__global__ void k_reduce(const T* in, size_t stride, int nr, T* out, size_t n, int op) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        T acc = in[i];
        for (int r = 1; r < nr; ++r) {
            const T y = in[r * stride + i];
            acc = op == 0 ? (T)(acc + y) : op == 2 ? (acc > y ? acc : y) : (acc < y ? acc : y);
        }
        out[i] = acc;
    }
}

}  // namespace

extern "C" {

typedef struct {
    char internal[128];
} ncclUniqueId;

int ncclGetUniqueId(ncclUniqueId* id) {
    std::memset(id->internal, 0, 128);
    std::random_device rd;
    std::snprintf(id->internal, 64, "/wlm_nccl_shim_%d_%08x", (int)getpid(), (unsigned)rd());
    return 0;
}

int ncclCommInitRank(Comm** out, int nranks, ncclUniqueId id, int rank) {
    if (nranks < 1 || nranks > kMaxRanks || rank < 0 || rank >= nranks) return 4;
    Comm* c = new Comm();
    c->rank = rank;
    c->nranks = nranks;
    std::strncpy(c->name, id.internal, sizeof(c->name) - 1);
    int fd = -1;
    if (rank == 0) {
        fd = shm_open(c->name, O_CREAT | O_RDWR, 0600);
        if (fd < 0 || ftruncate(fd, sizeof(Shared)) != 0) return 2;
    } else {
        for (int i = 0; i < 12000 && fd < 0; ++i) {
            fd = shm_open(c->name, O_RDWR, 0600);
            if (fd < 0) std::this_thread::sleep_for(std::chrono::milliseconds(10));
        }
        if (fd < 0) return 2;
        // wait for rank 0's ftruncate
        for (int i = 0; i < 12000 && lseek(fd, 0, SEEK_END) < (off_t)sizeof(Shared); ++i)
            std::this_thread::sleep_for(std::chrono::milliseconds(10));
    }
    void* p = mmap(nullptr, sizeof(Shared), PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (p == MAP_FAILED) return 2;
    c->sh = static_cast<Shared*>(p);
    if (check(cudaMalloc(&c->stage, kStage)) || check(cudaMalloc(&c->tmp, kStage))) return 1;
    if (check(cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking))) return 1;
    if (check(cudaIpcGetMemHandle(&c->sh->stage[rank], c->stage))) return 1;
    c->sh->joined.fetch_add(1);
    for (int i = 0; i < 12000 && c->sh->joined.load() < nranks; ++i)
        std::this_thread::sleep_for(std::chrono::milliseconds(10));
    if (c->sh->joined.load() < nranks) return 2;
    for (int r = 0; r < nranks; ++r)
        if (r != rank &&
            check(cudaIpcOpenMemHandle(&c->peer_stage[r], c->sh->stage[r], cudaIpcMemLazyEnablePeerAccess)))
            return 1;
    *out = c;
    return 0;
}

int ncclCommDestroy(Comm* c) {
    if (!c) return 0;
    // leave after every rank has read our last op
    for (int r = 0; r < c->nranks; ++r)
        if (r != c->rank) spin_until(c->sh->consumed[r], c->seq);
    for (int r = 0; r < c->nranks; ++r)
        if (c->peer_stage[r]) cudaIpcCloseMemHandle(c->peer_stage[r]);
    cudaFree(c->stage);
    cudaFree(c->tmp);
    cudaStreamDestroy(c->copy);
    const bool owner = c->rank == 0;
    munmap(c->sh, sizeof(Shared));
    if (owner) shm_unlink(c->name);
    delete c;
    return 0;
}

int ncclGroupStart() {
    ++g_group_depth;
    return 0;
}

static int flush(cudaStream_t s) {
    std::vector<PendingOp> sends, recvs;
    for (const PendingOp& o : g_pending) (o.send ? sends : recvs).push_back(o);
    const int r = g_group_comm ? exchange(g_group_comm, s, sends, recvs) : 0;
    g_pending.clear();
    g_group_comm = nullptr;
    return r;
}

int ncclGroupEnd() {
    if (--g_group_depth > 0) return 0;
    if (g_pending.empty()) return 0;
    return flush(g_pending.front().stream);
}

static int queue(bool send, void* buf, size_t count, int dt, int peer, Comm* c, cudaStream_t s) {
    if (peer < 0 || peer >= c->nranks || peer == c->rank) return 4;
    g_group_comm = c;
    g_pending.push_back(PendingOp{send, buf, count * dtype_size(dt), peer, s});
    if (g_group_depth == 0) return flush(s);
    return 0;
}

int ncclSend(const void* buf, size_t count, int dt, int peer, Comm* c, cudaStream_t s) {
    return queue(true, const_cast<void*>(buf), count, dt, peer, c, s);
}

int ncclRecv(void* buf, size_t count, int dt, int peer, Comm* c, cudaStream_t s) {
    return queue(false, buf, count, dt, peer, c, s);
}

// Deterministic all-reduce: out = op(rank 0's, rank 1's, ...) on every rank.
int ncclAllReduce(const void* sendbuf, void* recvbuf, size_t count, int dt, int op, Comm* c, cudaStream_t s) {
    const size_t bytes = count * dtype_size(dt);
    const size_t slot = (bytes + 255) & ~size_t(255);
    if (bytes == 0 || slot * c->nranks > kStage) return 4;
    std::vector<PendingOp> sends, recvs;
    for (int r = 0; r < c->nranks; ++r) {
        if (r == c->rank) continue;
        sends.push_back(PendingOp{true, const_cast<void*>(sendbuf), bytes, r, s});
        recvs.push_back(PendingOp{false, (char*)c->tmp + r * slot, bytes, r, s});
    }
    if (check(cudaMemcpyAsync((char*)c->tmp + c->rank * slot, sendbuf, bytes, cudaMemcpyDeviceToDevice, s)))
        return 1;
    if (exchange(c, s, sends, recvs)) return 1;
    const int grid = (int)std::min<size_t>(1024, (count + 255) / 256);
    const size_t st = slot / dtype_size(dt);
    switch (dt) {
        case 2: k_reduce<int><<<grid, 256, 0, s>>>((const int*)c->tmp, st, c->nranks, (int*)recvbuf, count, op); break;
        case 3: k_reduce<unsigned><<<grid, 256, 0, s>>>((const unsigned*)c->tmp, st, c->nranks, (unsigned*)recvbuf,
                                                        count, op); break;
        case 5: k_reduce<unsigned long long><<<grid, 256, 0, s>>>((const unsigned long long*)c->tmp, st, c->nranks,
                                                                  (unsigned long long*)recvbuf, count, op); break;
        case 7: k_reduce<float><<<grid, 256, 0, s>>>((const float*)c->tmp, st, c->nranks, (float*)recvbuf, count,
                                                     op); break;
        case 8: k_reduce<double><<<grid, 256, 0, s>>>((const double*)c->tmp, st, c->nranks, (double*)recvbuf,
                                                      count, op); break;
        default: return 4;
    }
    return check(cudaStreamSynchronize(s));
}

const char* ncclGetErrorString(int r) {
    switch (r) {
        case 0: return "ncclSuccess (shim)";
        case 1: return "unhandled cuda error (shim)";
        case 2: return "system error (shim: shared memory / rendezvous)";
        case 4: return "invalid argument (shim: 1..8 ranks, a peer other than itself)";
        default: return "error (shim)";
    }
}

}  // extern "C"
