// slab.cu -- z-slab decomposition of one registration (config 5).
//
// A volume is split along z into P slabs of >= kHalo planes.  Each slab is a
// wlm_engine whose per-voxel buffers hold its owned planes plus kHalo halo
// planes; F and M are whole-volume (the warp gathers M up to max|u| planes
// away, so M is replicated rather than haloed).  One LM attempt runs the
// stages of every slab with a halo exchange after each producer stage:
//
//   K2 (+Adam) -> exchange g (R_u planes) -> K3 -> max over slabs
//   -> exchange dU_s (R_w) -> K4 -> exchange u' (R_w + 1, >= 2)
//   -> [Jacobian, min over slabs] -> K1a/K1b: per-plane sum(rho)
//   -> sum of plane arrays over slabs -> K5 (identical state machine on every
//   slab) -> exchange A, B, E (2 planes)
//
// Every voxel's arithmetic is the single-domain arithmetic (direct z sums,
// global faces) and sum(rho) is reduced per plane then over planes in z
// order, so any P gives bit-identical losses, decisions and warps.
//
// The exchange schedule is one host-computed plan (slab_plan, exported as
// wlm_slab_halo_plan) executed by one of two transports:
//   * local: all slabs on the context's device; the plan's rows become
//     device-to-device copies captured in the attempt graph, the plane sums
//     share one array, the max/min is a one-thread combine kernel;
//   * nccl: one slab per process/GPU; the rows become ncclSend/ncclRecv in
//     one group per exchange, the plane sums an ncclAllReduce(sum) over
//     arrays that are zero on foreign planes (x + 0 is exact, so still
//     bit-identical), the max/min an ncclAllReduce on the ordered bits.
// libnccl is dlopen'ed (the one torch loaded), so the library has no link
// dependency on it.
#include <dlfcn.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <array>
#include <vector>

#include <cstdlib>

#include "internal.cuh"

using namespace wlm;

// ---- minimal NCCL ABI (nccl.h 2.x; resolved at run time) ----
namespace nccl {
typedef struct ncclComm* Comm;
struct UniqueId {
    char internal[128];
};
enum { Uint8 = 1, Int32 = 2, Uint32 = 3, Uint64 = 5, Float32 = 7, Float64 = 8 };
enum { Sum = 0, Max = 2, Min = 3 };
typedef int (*GetUniqueId_t)(UniqueId*);
typedef int (*CommInitRank_t)(Comm*, int, UniqueId, int);
typedef int (*CommDestroy_t)(Comm);
typedef int (*Send_t)(const void*, size_t, int, int, Comm, cudaStream_t);
typedef int (*Recv_t)(void*, size_t, int, int, Comm, cudaStream_t);
typedef int (*AllReduce_t)(const void*, void*, size_t, int, int, Comm, cudaStream_t);
typedef int (*Group_t)();
typedef const char* (*ErrStr_t)(int);

struct Api {
    void* h = nullptr;
    GetUniqueId_t get_unique_id = nullptr;
    CommInitRank_t comm_init_rank = nullptr;
    CommDestroy_t comm_destroy = nullptr;
    Send_t send = nullptr;
    Recv_t recv = nullptr;
    AllReduce_t all_reduce = nullptr;
    Group_t group_start = nullptr, group_end = nullptr;
    ErrStr_t err = nullptr;
};

Api g_api;

bool load(const char* path, std::string* why) {
    if (g_api.h) return true;
    void* h = dlopen(path && *path ? path : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
        *why = std::string("dlopen libnccl: ") + dlerror();
        return false;
    }
    Api a;
    a.h = h;
#define SYM(field, name)                                              \
    a.field = reinterpret_cast<decltype(a.field)>(dlsym(h, name));  \
    if (!a.field) {                                                   \
        *why = std::string("libnccl lacks ") + name;                  \
        return false;                                                 \
    }
    SYM(get_unique_id, "ncclGetUniqueId");
    SYM(comm_init_rank, "ncclCommInitRank");
    SYM(comm_destroy, "ncclCommDestroy");
    SYM(send, "ncclSend");
    SYM(recv, "ncclRecv");
    SYM(all_reduce, "ncclAllReduce");
    SYM(group_start, "ncclGroupStart");
    SYM(group_end, "ncclGroupEnd");
    SYM(err, "ncclGetErrorString");
#undef SYM
    g_api = a;
    return true;
}
}  // namespace nccl

namespace {

int cdiv_host(int a, int b) { return (a + b - 1) / b; }

constexpr int kHalo = 4;  // minimum halo depth: >= max(R_u, R_w + 1, 2) for sigma <= 1

// Halo planes a slab keeps: K3 reads g R_u planes out, K4 composes R_w
// planes out from a warp ring one plane wider, K1 reads Mw 2 planes out.
int slab_halo(int Ru, int Rw) { return std::max(kHalo, std::max(Ru, Rw + 1)); }
int slab_halo(const wlm_reg_config* cfg) {
    return slab_halo(smooth_radius(cfg->sigma_update), smooth_radius(cfg->sigma_warp));
}

enum Buffer { BUF_G = 0, BUF_V = 1, BUF_U = 2, BUF_ABE = 3, BUF_TM = 4 };

// Owned planes of slab k; with tiled LM (align = k of Eq. 5) the boundaries
// sit on tile boundaries so no k^3 tile straddles two slabs.
void partition(int nz, int nslabs, int k, int* zs, int* ze, int align = 1) {
    auto bound = [&](int i) {
        if (i >= nslabs) return nz;
        const int z = (int)((long long)i * nz / nslabs);
        return align > 1 ? z / align * align : z;
    };
    *zs = bound(k);
    *ze = bound(k + 1);
}

int halo_depth(int buffer, int Ru, int Rw) {
    switch (buffer) {
        case BUF_G: return Ru;
        case BUF_V: return Rw;
        case BUF_U: return std::max(Rw + 1, 2);
        default: return 2;  // A, B, E: the LNCC window radius
    }
}

// Rows of slab k's exchanges, in a fixed order: per buffer, the lower
// neighbour then the upper one, receive before send.  A slab receives its
// halo planes [z0, z1) from the neighbour owning them and sends the
// neighbour's halo planes out of its own owned planes; the two rows of one
// transfer name the same [z0, z1) on both sides.
// Tiled LM: the step matrices of the k^3 tiles covering the R_u halo planes
// come from the neighbour that owns them (rows in planes, whole tile-planes).
std::vector<wlm_halo_xfer> slab_plan(wlm_dims d, int nslabs, int k, int Ru, int Rw, int tk = 1) {
    std::vector<wlm_halo_xfer> rows;
    int zs, ze;
    partition(d.nz, nslabs, k, &zs, &ze, tk);
    auto down = [&](int z) { return std::max(0, (z >= 0 ? z : z - tk + 1) / tk * tk); };
    auto up = [&](int z) { return std::min(d.nz, (z + tk - 1) / tk * tk); };
    if (tk > 1) {
        if (k > 0) {
            rows.push_back({BUF_TM, k - 1, 0, down(zs - Ru), zs});
            rows.push_back({BUF_TM, k - 1, 1, zs, up(zs + Ru)});
        }
        if (k + 1 < nslabs) {
            rows.push_back({BUF_TM, k + 1, 0, ze, up(ze + Ru)});
            rows.push_back({BUF_TM, k + 1, 1, down(ze - Ru), ze});
        }
    }
    for (int b = BUF_G; b <= BUF_ABE; ++b) {
        const int h = halo_depth(b, Ru, Rw);
        if (h <= 0) continue;
        if (k > 0) {
            rows.push_back({b, k - 1, 0, std::max(0, zs - h), zs});
            rows.push_back({b, k - 1, 1, zs, std::min(ze, zs + h)});
        }
        if (k + 1 < nslabs) {
            rows.push_back({b, k + 1, 0, ze, std::min(d.nz, ze + h)});
            rows.push_back({b, k + 1, 1, std::max(zs, ze - h), ze});
        }
    }
    return rows;
}

__global__ void k_group_combine(PairState** sts, int n, int jac) {
    unsigned mx = 0u;
    int mn = 0x7f800000;
    for (int i = 0; i < n; ++i) {
        mx = max(mx, sts[i]->max_bits);
        mn = min(mn, sts[i]->jac_bits);
    }
    for (int i = 0; i < n; ++i) {
        sts[i]->max_bits = mx;
        if (jac) sts[i]->jac_bits = mn;
    }
}

// Copy `count` voxels per channel of the attempt warp buffer (1 - cur) from
// one slab engine's local planes to another's (same device).
__global__ void k_copy_attempt_warp(float* dst, long long dn, long long doff, const float* src, long long sn,
                                    long long soff, long long count, const PairState* st) {
    const int buf = 1 - st->cur;
    for (int c = 0; c < 3; ++c) {
        float* d = dst + (long long)(buf * 3 + c) * dn + doff;
        const float* s = src + (long long)(buf * 3 + c) * sn + soff;
        for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
             i += (long long)gridDim.x * blockDim.x)
            d[i] = s[i];
    }
}

__global__ void k_set_cur0(PairState* st) { st->cur = 0; }

// MI: sum of the slabs' fixed-point joint histograms, written back to every
// slab (integer sums: exact and order-independent).
__global__ void k_hist_allreduce(unsigned long long** h, int n, int bins2) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < bins2; i += gridDim.x * blockDim.x) {
        unsigned long long t = 0ull;
        for (int k = 0; k < n; ++k) t += h[k][i];
        for (int k = 0; k < n; ++k) h[k][i] = t;
    }
}

__global__ void k_group_cond(const PairState* st, cudaGraphConditionalHandle h) {
    cudaGraphSetConditional(h, st->done ? 0u : 1u);
}

}  // namespace

struct wlm_slab_group {
    wlm_ctx* ctx = nullptr;
    wlm_dims dims{};
    Geo gfull{};
    int nslabs = 0;  // slabs of the whole decomposition
    int first = 0;   // global index of eng[0] (nccl: this process's rank)
    wlm_reg_config cfg{};
    std::vector<wlm_engine*> eng;
    std::vector<std::vector<wlm_halo_xfer>> plan;  // per local engine
    DevBuf<float> F, M;        // local transport: whole volume, shared
    DevBuf<double> plane_sum;  // local transport: shared per-plane sums
    DevBuf<PairState*> sts;
    DevBuf<unsigned long long*> hists;  // MI: every slab's histogram (in-process)
    nccl::Comm comm = nullptr;  // nccl transport
    cudaGraphExec_t step_exec = nullptr, loop_exec = nullptr;
    cudaGraph_t step_graph = nullptr, loop_graph = nullptr;
    int body_kernels = 0;

    // interior / boundary overlap (see body_overlap)
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;

    // fused halo stores (see setup_fused): per buffer kind, whether the
    // producing kernel stores the neighbours' halo planes itself
    bool fused[4] = {false, false, false, false};
    std::vector<void*> ipc_open;  // neighbour buffers mapped by CUDA IPC (nccl)
    DevBuf<int> token;            // [send, recv lower, recv upper] ordering tokens (nccl)

    ~wlm_slab_group() {
        for (void* q : ipc_open) cudaIpcCloseMemHandle(q);
        if (side) cudaStreamDestroy(side);
        if (ev_fork) cudaEventDestroy(ev_fork);
        if (ev_join) cudaEventDestroy(ev_join);
        if (step_exec) cudaGraphExecDestroy(step_exec);
        if (loop_exec) cudaGraphExecDestroy(loop_exec);
        if (step_graph) cudaGraphDestroy(step_graph);
        if (loop_graph) cudaGraphDestroy(loop_graph);
        for (auto* e : eng) delete e;
        if (comm) nccl::g_api.comm_destroy(comm);
    }

    bool distributed() const { return comm != nullptr; }
    long long nxy() const { return (long long)dims.nx * dims.ny; }
    wlm_engine* local(int global) const { return eng[global - first]; }

    void nccl_check(int r, const char* what) {
        if (r != 0) {
            set_err(ctx, std::string(what) + ": " + nccl::g_api.err(r));
            throw Fail{WLM_CUDA};
        }
    }

    // Channel stacks of one buffer kind: base, element size, channel stride
    // (elements), channel count.
    struct Chan {
        char* base;
        size_t esz;
        long long stride;
        int nch;
    };
    static std::vector<Chan> channels(wlm_engine* e, int b) {
        const long long n = e->g.n;
        switch (b) {
            case BUF_G: return {{(char*)e->G.p, 4, n, 3}};
            case BUF_V: return {{(char*)e->B.VS, 4, n, 3}};  // inside ABE (one pair)
            case BUF_U: return {{(char*)e->U.p, 4, n, 6}};  // both ping-pong buffers (nccl)
            default: return {{(char*)e->ABE.p, 4, n, 2}, {(char*)(e->ABE.p + 2 * n), 8, n, 1}};
        }
    }

    // Tile step matrices: global tile-plane indexing on every slab, so a row
    // [z0, z1) (tile-aligned planes) is the same byte range on both sides.
    void tm_range(const wlm_halo_xfer& r, size_t* off, size_t* cnt) const {
        const LmParams& P = eng[0]->P;
        const int k = P.tile_k;
        const size_t plane = (size_t)eng[0]->B.tkx * eng[0]->B.tky * 6;
        const int b0 = r.z0 / k, b1 = (r.z1 + k - 1) / k;
        *off = (size_t)b0 * plane;
        *cnt = (size_t)(b1 - b0) * plane;
    }

    void exchange(int b, cudaStream_t s) {
        if (b == BUF_TM) {
            if (!distributed()) {
                for (size_t li = 0; li < eng.size(); ++li)
                    for (const wlm_halo_xfer& r : plan[li]) {
                        if (r.buffer != BUF_TM || r.send) continue;
                        size_t off, cnt;
                        tm_range(r, &off, &cnt);
                        CK(cudaMemcpyAsync(eng[li]->B.TM + off, local(r.peer)->B.TM + off, sizeof(double) * cnt,
                                           cudaMemcpyDeviceToDevice, s));
                    }
                return;
            }
            nccl_check(nccl::g_api.group_start(), "ncclGroupStart");
            for (const wlm_halo_xfer& r : plan[0]) {
                if (r.buffer != BUF_TM) continue;
                size_t off, cnt;
                tm_range(r, &off, &cnt);
                double* p = eng[0]->B.TM + off;
                if (r.send) nccl_check(nccl::g_api.send(p, cnt, nccl::Float64, r.peer, comm, s), "ncclSend");
                else nccl_check(nccl::g_api.recv(p, cnt, nccl::Float64, r.peer, comm, s), "ncclRecv");
            }
            nccl_check(nccl::g_api.group_end(), "ncclGroupEnd");
            return;
        }
        if (!distributed()) {
            for (size_t li = 0; li < eng.size(); ++li) {
                wlm_engine* d = eng[li];
                for (const wlm_halo_xfer& r : plan[li]) {
                    if (r.buffer != b || r.send) continue;
                    wlm_engine* src = local(r.peer);
                    const long long cnt = (long long)(r.z1 - r.z0) * nxy();
                    const long long doff = (r.z0 - d->g.zlo) * nxy(), soff = (r.z0 - src->g.zlo) * nxy();
                    if (b == BUF_U) {
                        const int grid = (int)std::min<long long>(148 * 4, (cnt + 255) / 256);
                        k_copy_attempt_warp<<<grid, 256, 0, s>>>(d->U.p, d->g.n, doff, src->U.p, src->g.n,
                                                                 soff, cnt, src->st.p);
                        ++g_kernel_launches;
                        continue;
                    }
                    const auto dc = channels(d, b), sc = channels(src, b);
                    for (size_t q = 0; q < dc.size(); ++q)
                        for (int c = 0; c < dc[q].nch; ++c)
                            CK(cudaMemcpyAsync(dc[q].base + (c * dc[q].stride + doff) * dc[q].esz,
                                               sc[q].base + (c * sc[q].stride + soff) * sc[q].esz,
                                               cnt * dc[q].esz, cudaMemcpyDeviceToDevice, s));
                }
            }
            return;
        }
        // nccl: this process holds exactly one slab.  The warp sends both
        // ping-pong buffers (the accepted one's halo is unchanged, so
        // overwriting it with the owner's identical values is harmless and
        // the host need not know which buffer the device selected).
        wlm_engine* e = eng[0];
        const auto ch = channels(e, b);
        nccl_check(nccl::g_api.group_start(), "ncclGroupStart");
        for (const wlm_halo_xfer& r : plan[0]) {
            if (r.buffer != b) continue;
            const long long cnt = (long long)(r.z1 - r.z0) * nxy();
            const long long off = (r.z0 - e->g.zlo) * nxy();
            for (const Chan& q : ch)
                for (int c = 0; c < q.nch; ++c) {
                    char* p = q.base + (c * q.stride + off) * q.esz;
                    const int dt = q.esz == 8 ? nccl::Float64 : nccl::Float32;
                    if (r.send)
                        nccl_check(nccl::g_api.send(p, (size_t)cnt, dt, r.peer, comm, s), "ncclSend");
                    else
                        nccl_check(nccl::g_api.recv(p, (size_t)cnt, dt, r.peer, comm, s), "ncclRecv");
                }
        }
        nccl_check(nccl::g_api.group_end(), "ncclGroupEnd");
    }

    // Fused halo stores.  K2 (g), K3 (dU_s),
    // K4 (the attempt warp) and K1b (A, B, E) store each output plane that a
    // neighbour keeps as halo straight into the neighbour's buffer as well:
    // the same device in-process; peer memory mapped by CUDA IPC (NVLink on
    // a multi-GPU node) with one process per GPU.  The exchange after such a
    // stage then moves no data: in-process the single stream already orders
    // the neighbour's consumer after every producer; across processes a
    // 4-byte ncclSend/ncclRecv with each neighbour, queued behind the
    // producer, orders it (the neighbour's consumer waits for the token,
    // which is sent after the producer kernel completed).  Each producer
    // writes only planes the receiver does not itself write, into the buffer
    // the receiver reads next, and every write happens after the receiver's
    // last read of the previous contents (its previous stage chain precedes
    // the token the producer waited for), so the result is bit-identical to
    // the copy exchange.  Kinds whose producer is not a fused kernel (Adam's
    // g, MSE/MI, tiled LM's step, the generic paths) keep the exchange.
    // WLM_SLAB_FUSED=0 keeps every exchange.
    void setup_fused() {
        const char* v = std::getenv("WLM_SLAB_FUSED");
        if ((v && std::atoi(v) == 0) || nslabs < 2) return;
        const LmParams& P = eng[0]->P;
        const bool lncc2 = P.metric == WLM_METRIC_LNCC && P.radius == 2;
        fused[BUF_G] = lncc2 && P.optimizer != WLM_OPT_ADAM && P.tile_k <= 1;
        fused[BUF_V] = P.Ru <= 6 && P.tile_k <= 1;
        fused[BUF_U] = P.Rw <= 6;
        fused[BUF_ABE] = lncc2;
        if (!any_fused()) return;  // the same decision on every rank (same config)
        struct Info {
            cudaIpcMemHandle_t h[4];
            long long n;
            int zlo, pad;
        };
        // this process's (or engine's) buffers as a neighbour sees them
        // (dU_s lives inside ABE: one allocation, one mapping for both)
        auto bases = [](wlm_engine* e, void* out[4]) {
            out[0] = e->G.p; out[1] = e->B.VS; out[2] = e->U.p; out[3] = e->ABE.p;
        };
        std::vector<std::array<void*, 4>> nb_base(2 * eng.size(), {nullptr, nullptr, nullptr, nullptr});
        std::vector<long long> nb_n(2 * eng.size(), 0);
        std::vector<int> nb_zlo(2 * eng.size(), 0);
        if (!distributed()) {
            for (size_t li = 0; li < eng.size(); ++li)
                for (int sd = 0; sd < 2; ++sd) {
                    const int k = first + (int)li + (sd == 0 ? -1 : 1);
                    if (k < first || k >= first + (int)eng.size()) continue;
                    wlm_engine* o = local(k);
                    void* b4[4];
                    bases(o, b4);
                    for (int q = 0; q < 4; ++q) nb_base[2 * li + sd][q] = b4[q];
                    nb_n[2 * li + sd] = o->g.n;
                    nb_zlo[2 * li + sd] = o->g.zlo;
                }
        } else {
            wlm_engine* e = eng[0];
            Info mine{};
            void* b4[4];
            bases(e, b4);
            for (int q = 0; q < 4; ++q)
                if (q != 1) CK(cudaIpcGetMemHandle(&mine.h[q], b4[q]));
            mine.n = e->g.n;
            mine.zlo = e->g.zlo;
            DevBuf<unsigned char> buf(ctx, 3 * sizeof(Info));
            cudaStream_t st = ctx->stream;
            CK(cudaMemcpyAsync(buf.p, &mine, sizeof(Info), cudaMemcpyHostToDevice, st));
            nccl_check(nccl::g_api.group_start(), "ncclGroupStart");
            for (int sd = 0; sd < 2; ++sd) {
                const int k = first + (sd == 0 ? -1 : 1);
                if (k < 0 || k >= nslabs) continue;
                nccl_check(nccl::g_api.send(buf.p, sizeof(Info), nccl::Uint8, k, comm, st), "ncclSend");
                nccl_check(nccl::g_api.recv(buf.p + (1 + sd) * sizeof(Info), sizeof(Info), nccl::Uint8, k, comm, st),
                           "ncclRecv");
            }
            nccl_check(nccl::g_api.group_end(), "ncclGroupEnd");
            Info theirs[2];
            CK(cudaMemcpyAsync(theirs, buf.p + sizeof(Info), 2 * sizeof(Info), cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            int ok = 1;
            for (int sd = 0; sd < 2 && ok; ++sd) {
                const int k = first + (sd == 0 ? -1 : 1);
                if (k < 0 || k >= nslabs) continue;
                for (int q = 0; q < 4 && ok; ++q) {
                    if (q == 1) continue;  // dU_s: the ABE mapping (set below)
                    void* ptr = nullptr;
                    if (cudaIpcOpenMemHandle(&ptr, theirs[sd].h[q], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
                        cudaGetLastError();
                        ok = 0;  // no peer mapping (GPUs without P2P): every rank keeps the copy exchange
                        break;
                    }
                    ipc_open.push_back(ptr);
                    nb_base[sd][q] = ptr;
                }
                nb_base[sd][1] = nb_base[sd][3];
                nb_n[sd] = theirs[sd].n;
                nb_zlo[sd] = theirs[sd].zlo;
            }
            // the decision must be the same on every rank (tokens and copies
            // do not match each other): min over the communicator
            token = DevBuf<int>(ctx, 3);
            CK(cudaMemcpyAsync(token.p, &ok, sizeof(int), cudaMemcpyHostToDevice, st));
            nccl_check(nccl::g_api.all_reduce(token.p, token.p, 1, nccl::Int32, nccl::Min, comm, st),
                       "ncclAllReduce(min)");
            CK(cudaMemcpyAsync(&ok, token.p, sizeof(int), cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            CK(cudaMemsetAsync(token.p, 0, sizeof(int) * 3, st));
            if (!ok) {
                for (void* q : ipc_open) cudaIpcCloseMemHandle(q);
                ipc_open.clear();
                for (bool& f : fused) f = false;
                return;
            }
        }
        for (size_t li = 0; li < eng.size(); ++li) {
            wlm_engine* e = eng[li];
            HaloPeer hp{};
            for (int sd = 0; sd < 2; ++sd) {
                hp.g[sd] = static_cast<float*>(nb_base[2 * li + sd][0]);
                hp.v[sd] = static_cast<float*>(nb_base[2 * li + sd][1]);
                hp.u[sd] = static_cast<float*>(nb_base[2 * li + sd][2]);
                hp.abe[sd] = static_cast<float*>(nb_base[2 * li + sd][3]);
                hp.n[sd] = nb_n[2 * li + sd];
                hp.zlo[sd] = nb_zlo[2 * li + sd];
            }
            for (int k = 0; k < 4; ++k) {
                hp.lo_end[k] = e->g.zs;  // empty unless a fused send row says otherwise
                hp.hi_begin[k] = e->g.ze;
            }
            for (const wlm_halo_xfer& r : plan[li]) {
                if (!r.send || r.buffer > BUF_ABE || !fused[r.buffer]) continue;
                if (r.peer < first + (int)li) hp.lo_end[r.buffer] = r.z1;  // [zs, z1) to the lower neighbour
                else hp.hi_begin[r.buffer] = r.z0;                        // [z0, ze) to the upper one
            }
            e->B.peer = hp;
            e->B.peer_on = 1;
        }
    }
    bool any_fused() const { return fused[0] || fused[1] || fused[2] || fused[3]; }

    // The halo step after a producer stage of buffer kind b: the copy
    // exchange, or (fused) only the ordering token across processes.
    void halo(int b, cudaStream_t s) {
        if (b > BUF_ABE || !fused[b]) {
            exchange(b, s);
            return;
        }
        if (!distributed()) return;
        nccl_check(nccl::g_api.group_start(), "ncclGroupStart");
        for (int sd = 0; sd < 2; ++sd) {
            const int k = first + (sd == 0 ? -1 : 1);
            if (k < 0 || k >= nslabs) continue;
            nccl_check(nccl::g_api.send(token.p, 1, nccl::Int32, k, comm, s), "ncclSend(token)");
            nccl_check(nccl::g_api.recv(token.p + 1 + sd, 1, nccl::Int32, k, comm, s), "ncclRecv(token)");
        }
        nccl_check(nccl::g_api.group_end(), "ncclGroupEnd");
    }

    void reduce_max(int jac, cudaStream_t s) {
        if (!distributed()) {
            k_group_combine<<<1, 1, 0, s>>>(sts.p, (int)eng.size(), jac);
            ++g_kernel_launches;
            return;
        }
        PairState* st = eng[0]->st.p;
        if (!jac)
            nccl_check(nccl::g_api.all_reduce(&st->max_bits, &st->max_bits, 1, nccl::Uint32, nccl::Max, comm, s),
                       "ncclAllReduce(max)");
        else
            nccl_check(nccl::g_api.all_reduce(&st->jac_bits, &st->jac_bits, 1, nccl::Int32, nccl::Min, comm, s),
                       "ncclAllReduce(min)");
    }

    void reduce_planes(cudaStream_t s) {
        if (eng[0]->P.metric == WLM_METRIC_MI) {  // the loss is the whole-volume histogram
            const int bins2 = eng[0]->P.mi_bins * eng[0]->P.mi_bins;
            if (!distributed()) {
                k_hist_allreduce<<<cdiv_host(bins2, 256), 256, 0, s>>>(hists.p, (int)eng.size(), bins2);
                ++g_kernel_launches;
            } else {
                unsigned long long* h = eng[0]->B.HIST;
                nccl_check(nccl::g_api.all_reduce(h, h, (size_t)bins2, nccl::Uint64, nccl::Sum, comm, s),
                           "ncclAllReduce(histogram)");
            }
            return;
        }
        if (!distributed()) return;  // one shared plane array
        double* ps = eng[0]->B.plane_sum;
        nccl_check(nccl::g_api.all_reduce(ps, ps, (size_t)dims.nz, nccl::Float64, nccl::Sum, comm, s),
                   "ncclAllReduce(planes)");
    }

    void evaluate(int mode, cudaStream_t s) {
        for (auto* e : eng) e->stage_eval(mode, s);
        reduce_planes(s);
        for (auto* e : eng) e->stage_finalize(mode, s);
        halo(BUF_ABE, s);
    }

    // Interior / boundary split: every stage whose output a
    // neighbour needs runs first on the planes it sends (the plan's send
    // rows), the exchange is queued behind those, and the remaining interior
    // planes run on a side stream meanwhile; the streams join before the
    // next stage.  Every voxel's arithmetic is independent of the launch
    // range (z sums are direct sums over the ring), so the split is bit-
    // identical to one launch.  Fused LNCC (radius 2) path with pointwise
    // steps; WLM_SLAB_OVERLAP=0 keeps the serial body.
    bool overlap_enabled() const {
        const LmParams& P = eng[0]->P;
        const char* v = std::getenv("WLM_SLAB_OVERLAP");
        if ((v && std::atoi(v) == 0) || any_fused()) return false;  // fused stores need no split
        return P.metric == WLM_METRIC_LNCC && P.radius == 2 && P.tile_k <= 1 && P.Ru <= 6 && P.Rw <= 6;
    }

    // Boundary views (the planes engine li sends of buffer b) and the
    // interior view of its owned planes.
    void views(size_t li, int b, std::vector<std::pair<wlm_engine*, Batch>>& bnd,
               std::vector<std::pair<wlm_engine*, Batch>>& inner) const {
        wlm_engine* e = eng[li];
        const int zs = e->g.zs, ze = e->g.ze;
        int lo = zs, hi = ze;  // interior [lo, hi)
        for (const wlm_halo_xfer& r : plan[li]) {
            if (r.buffer != b || !r.send) continue;
            if (r.z0 == zs) lo = std::max(lo, r.z1);
            if (r.z1 == ze) hi = std::min(hi, r.z0);
        }
        auto view = [&](int z0, int z1) {
            Batch v = e->B;
            v.g.zs = z0;
            v.g.ze = z1;
            return v;
        };
        if (lo >= hi) {  // thin slab: everything is boundary
            bnd.push_back({e, e->B});
            return;
        }
        if (lo > zs) bnd.push_back({e, view(zs, lo)});
        if (hi < ze) bnd.push_back({e, view(hi, ze)});
        inner.push_back({e, view(lo, hi)});
    }

    template <class Fn>
    void staged(int b, Fn fn, cudaStream_t s) {
        std::vector<std::pair<wlm_engine*, Batch>> bnd, inner;
        for (size_t li = 0; li < eng.size(); ++li) views(li, b, bnd, inner);
        CK(cudaEventRecord(ev_fork, s));
        CK(cudaStreamWaitEvent(side, ev_fork, 0));
        for (auto& v : bnd) fn(v.first, v.second, s);
        exchange(b, s);
        for (auto& v : inner) fn(v.first, v.second, side);
        CK(cudaEventRecord(ev_join, side));
        CK(cudaStreamWaitEvent(s, ev_join, 0));
    }

    void body_overlap(cudaStream_t s) {
        if (!side) {
            CK(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
            CK(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
        }
        staged(BUF_G, [](wlm_engine* e, const Batch& v, cudaStream_t st) { e->stage_grad(v, st); }, s);
        staged(BUF_V, [](wlm_engine* e, const Batch& v, cudaStream_t st) { launch_step_smooth(v, e->P, st); }, s);
        reduce_max(0, s);
        staged(BUF_U, [](wlm_engine* e, const Batch& v, cudaStream_t st) { launch_compose_smooth(v, e->P, st); },
               s);
        if (eng[0]->P.log_jacobian) {
            for (auto* e : eng) launch_jacobian_diag(e->B, e->P, s);
            reduce_max(1, s);
        }
        // evaluate(1): K1a on the owned planes + halo, K1b split, then the
        // per-plane sums and the loss on the whole slab
        for (auto* e : eng) launch_lncc_warp(e->B, e->P, 1, s);
        staged(BUF_ABE, [](wlm_engine*, const Batch& v, cudaStream_t st) { launch_lncc_window(v, st); }, s);
        for (auto* e : eng) launch_plane_sums(e->B, s);
        reduce_planes(s);
        for (auto* e : eng) e->stage_finalize(1, s);
    }

    void body(cudaStream_t s) {
        if (overlap_enabled()) {
            body_overlap(s);
            return;
        }
        for (auto* e : eng) e->stage_grad(s);
        halo(BUF_G, s);
        if (eng[0]->P.optimizer == WLM_OPT_LM && eng[0]->P.tile_k > 1) {
            for (auto* e : eng) launch_tile_matrix(e->B, e->P, s);  // owned tiles
            exchange(BUF_TM, s);                                   // halo tiles
            for (auto* e : eng) launch_step_smooth(e->B, e->P, s);
        } else {
            for (auto* e : eng) e->stage_step(s);
        }
        reduce_max(0, s);
        halo(BUF_V, s);
        for (auto* e : eng) launch_compose_smooth(e->B, e->P, s);
        halo(BUF_U, s);
        if (eng[0]->P.log_jacobian) {
            for (auto* e : eng) launch_jacobian_diag(e->B, e->P, s);
            reduce_max(1, s);
        }
        evaluate(1, s);
    }

    void build_step_graph() {
        if (step_exec) return;
        const uint64_t saved = g_kernel_launches;
        CK(cudaStreamBeginCapture(ctx->capture, cudaStreamCaptureModeThreadLocal));
        body(ctx->capture);
        CK(cudaStreamEndCapture(ctx->capture, &step_graph));
        body_kernels = (int)(g_kernel_launches - saved);
        g_kernel_launches = saved;
        CK(cudaGraphInstantiate(&step_exec, step_graph, 0));
    }

    void build_loop_graph() {
        if (loop_exec) return;
        CK(cudaGraphCreate(&loop_graph, 0));
        cudaGraphConditionalHandle h;
        CK(cudaGraphConditionalHandleCreate(&h, loop_graph, 1, cudaGraphCondAssignDefault));
        alignas(cudaGraphNodeParams) unsigned char raw[sizeof(cudaGraphNodeParams)] = {};
        cudaGraphNodeParams& cp = *reinterpret_cast<cudaGraphNodeParams*>(raw);
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = h;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        cudaGraphNode_t node;
        CK(cudaGraphAddNode(&node, loop_graph, nullptr, 0, &cp));
        const uint64_t saved = g_kernel_launches;
        CK(cudaStreamBeginCaptureToGraph(ctx->capture, cp.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                         cudaStreamCaptureModeThreadLocal));
        body(ctx->capture);
        k_group_cond<<<1, 1, 0, ctx->capture>>>(eng[0]->st.p, h);
        cudaGraph_t out = nullptr;
        CK(cudaStreamEndCapture(ctx->capture, &out));
        g_kernel_launches = saved;
        CK(cudaGraphInstantiate(&loop_exec, loop_graph, 0));
    }

    // nccl transport without rejection: the attempt (kernels, halo
    // send/recv groups and all-reduces) is captured once as a CUDA graph
    // (NCCL supports stream capture) and launched per iteration.  A transport
    // that cannot be captured (a capture error, e.g. a host-synchronising
    // NCCL stand-in) leaves the group on eager launches.
    int graph_state = 0;  // 0 untried, 1 captured, -1 not capturable
    bool try_step_graph() {
        if (graph_state != 0) return graph_state > 0;
        const uint64_t saved = g_kernel_launches;
        cudaGraph_t gr = nullptr;
        bool ok = cudaStreamBeginCapture(ctx->capture, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
        if (ok) {
            try {
                body(ctx->capture);
            } catch (const Fail&) {
                ok = false;
            }
            const cudaError_t e = cudaStreamEndCapture(ctx->capture, &gr);
            ok = ok && e == cudaSuccess && gr != nullptr;
        }
        body_kernels = (int)(g_kernel_launches - saved);
        g_kernel_launches = saved;
        if (ok && cudaGraphInstantiate(&step_exec, gr, 0) == cudaSuccess) {
            step_graph = gr;
            graph_state = 1;
        } else {
            if (gr) cudaGraphDestroy(gr);
            step_exec = nullptr;
            graph_state = -1;
        }
        cudaGetLastError();  // clear a failed capture's sticky-free error state
        return graph_state > 0;
    }

    // nccl transport with rejection (or when capture failed): attempts are
    // launched eagerly (collectives inside conditional graph bodies are not
    // relied on).  Attempts of a finished registration are no-ops on the
    // device, so with rejection the host launches the lower bound of
    // remaining attempts, then re-reads the state.
    void iterate_eager(int iters) {
        cudaStream_t s = ctx->stream;
        if (!eng[0]->P.rejection) {
            for (int i = 0; i < iters; ++i) body(s);
            return;
        }
        for (;;) {
            const PairState st = read_states(eng[0])[0];
            if (st.done) return;
            const int left = std::max(1, st.iters_target - st.iter);
            for (int i = 0; i < left; ++i) body(s);
        }
    }

    void attach(wlm_engine* e) {
        if (!distributed()) {
            e->shared_fm = true;
            e->shared_plane_sum = true;
            e->B.F = F.p;
            e->B.M = M.p;
            e->B.plane_sum = plane_sum.p;
        }
        engine_alloc(e);
        if (distributed()) e->B.zero_foreign_planes = 1;
    }

    float* fp() const { return distributed() ? eng[0]->F.p : F.p; }
    float* mp() const { return distributed() ? eng[0]->M.p : M.p; }
};

namespace {

wlm_status make_group(wlm_ctx* ctx, wlm_dims d, int nslabs, int first, int count, const wlm_reg_config* cfg,
                      nccl::Comm comm, wlm_slab_group** out) {
    wlm_slab_group* grp = new wlm_slab_group();
    grp->ctx = ctx;
    grp->dims = d;
    grp->gfull = make_geo(d);
    grp->nslabs = nslabs;
    grp->first = first;
    grp->cfg = *cfg;
    grp->comm = comm;  // owned (destroyed with the group) from here on
    wlm_status s = run(ctx, [&] {
        if (!comm) {
            grp->F = DevBuf<float>(ctx, (size_t)grp->gfull.nfull);
            grp->M = DevBuf<float>(ctx, (size_t)grp->gfull.nfull);
            grp->plane_sum = DevBuf<double>(ctx, (size_t)d.nz);
            CK(cudaMemsetAsync(grp->plane_sum.p, 0, sizeof(double) * d.nz, ctx->stream));
        }
        std::vector<PairState*> hst;
        for (int k = first; k < first + count; ++k) {
            wlm_engine* e = new wlm_engine();
            grp->eng.push_back(e);
            const wlm_status es = engine_init(e, ctx, d, 1, cfg);
            if (es != WLM_OK) throw Fail{es};
            int zs, ze;
            const int tk = std::max(1, cfg->lm.tile_size);
            partition(d.nz, nslabs, k, &zs, &ze, tk);
            e->g = make_slab_geo(d, zs, ze, slab_halo(e->P.Ru, e->P.Rw));
            grp->attach(e);
            grp->plan.push_back(slab_plan(d, nslabs, k, e->P.Ru, e->P.Rw, tk));
            hst.push_back(e->st.p);
        }
        grp->setup_fused();
        grp->sts = DevBuf<PairState*>(ctx, hst.size());
        CK(cudaMemcpyAsync(grp->sts.p, hst.data(), sizeof(PairState*) * hst.size(), cudaMemcpyHostToDevice,
                           ctx->stream));
        if (cfg->metric == WLM_METRIC_MI) {
            std::vector<unsigned long long*> hh;
            for (auto* e : grp->eng) hh.push_back(e->B.HIST);
            grp->hists = DevBuf<unsigned long long*>(ctx, hh.size());
            CK(cudaMemcpyAsync(grp->hists.p, hh.data(), sizeof(unsigned long long*) * hh.size(),
                               cudaMemcpyHostToDevice, ctx->stream));
        }
        CK(cudaStreamSynchronize(ctx->stream));
    });
    if (s != WLM_OK) {
        delete grp;
        return s;
    }
    *out = grp;
    return WLM_OK;
}

wlm_status check_split(wlm_ctx* ctx, wlm_dims d, int nslabs, const wlm_reg_config* cfg) {
    if (nslabs < 1 || !valid_dims(d)) return WLM_INVALID_ARG;  // ctx may be null (host-only helpers)
    // slabs run the fused kernels only (LNCC radius 2, smoothing radius <= 6);
    // the generic paths (generic.cu) are single-domain
    if ((cfg->metric == WLM_METRIC_LNCC && cfg->lncc_radius != 2) || smooth_radius(cfg->sigma_update) > 6 ||
        smooth_radius(cfg->sigma_warp) > 6) {
        set_err(ctx, "slab_group: LNCC radius 2 and sigma <= 2 only (the generic paths are single-domain)");
        return WLM_UNSUPPORTED;
    }
    // every slab (tile-aligned when tiled) holds at least the halo depth and,
    // with tiles, the R_u + k planes its halo tiles can reach into
    const int tk = std::max(1, cfg->lm.tile_size);
    const int halo = slab_halo(cfg);
    const int need = tk > 1 ? std::max(halo, smooth_radius(cfg->sigma_update) + tk) : halo;
    for (int k = 0; k < nslabs; ++k) {
        int zs, ze;
        partition(d.nz, nslabs, k, &zs, &ze, tk);
        if (ze - zs < need) {
            set_err(ctx, "slab_group: every slab needs at least " + std::to_string(need) +
                             " planes (halo depth" + (tk > 1 ? " + tile" : "") + ")");
            return WLM_INVALID_ARG;
        }
    }
    return WLM_OK;
}

}  // namespace

extern "C" {

wlm_status wlm_slab_partition(int nz, int nslabs, int slab, int* zs, int* ze) {
    if (nz < 1 || nslabs < 1 || slab < 0 || slab >= nslabs || !zs || !ze) return WLM_INVALID_ARG;
    partition(nz, nslabs, slab, zs, ze);
    return nz / nslabs >= kHalo ? WLM_OK : WLM_INVALID_ARG;
}

wlm_status wlm_slab_halo_plan(wlm_dims d, int nslabs, int slab, const wlm_reg_config* cfg, wlm_halo_xfer* rows,
                              size_t cap, size_t* len) {
    if (!cfg || !len || nslabs < 1 || slab < 0 || slab >= nslabs || !valid_dims(d)) return WLM_INVALID_ARG;
    // the same per-slab test as wlm_slab_group_create (tile-aligned splits,
    // R_u + k planes with tiles): no plan for a split a group would refuse
    const wlm_status ok = check_split(nullptr, d, nslabs, cfg);
    if (ok != WLM_OK) return ok;
    const auto p = slab_plan(d, nslabs, slab, smooth_radius(cfg->sigma_update), smooth_radius(cfg->sigma_warp),
                             std::max(1, cfg->lm.tile_size));
    *len = p.size();
    if (rows) std::memcpy(rows, p.data(), sizeof(wlm_halo_xfer) * std::min(cap, p.size()));
    return WLM_OK;
}

wlm_status wlm_slab_group_create(wlm_ctx* ctx, wlm_dims d, int nslabs, const wlm_reg_config* cfg,
                                 wlm_slab_group** out) {
    if (!out || !cfg) return WLM_INVALID_ARG;
    *out = nullptr;
    if (!ctx) return WLM_INVALID_ARG;
    const wlm_status s = check_split(ctx, d, nslabs, cfg);
    if (s != WLM_OK) return s;
    return make_group(ctx, d, nslabs, 0, nslabs, cfg, nullptr, out);
}

wlm_status wlm_nccl_unique_id(const char* nccl_lib, unsigned char id[128]) {
    std::string why;
    if (!id) return WLM_INVALID_ARG;
    if (!nccl::load(nccl_lib, &why)) return WLM_UNSUPPORTED;
    nccl::UniqueId u;
    if (nccl::g_api.get_unique_id(&u) != 0) return WLM_CUDA;
    std::memcpy(id, u.internal, 128);
    return WLM_OK;
}

wlm_status wlm_slab_group_create_nccl(wlm_ctx* ctx, wlm_dims d, int rank, int nranks, const unsigned char id[128],
                                      const char* nccl_lib, const wlm_reg_config* cfg, wlm_slab_group** out) {
    if (!ctx || !out || !cfg || !id || rank < 0 || rank >= nranks) return WLM_INVALID_ARG;
    *out = nullptr;
    wlm_status s = check_split(ctx, d, nranks, cfg);
    if (s != WLM_OK) return s;
    std::string why;
    if (!nccl::load(nccl_lib, &why)) {
        set_err(ctx, why);
        return WLM_UNSUPPORTED;
    }
    nccl::Comm comm = nullptr;
    s = run(ctx, [&] {
        nccl::UniqueId u;
        std::memcpy(u.internal, id, 128);
        const int r = nccl::g_api.comm_init_rank(&comm, nranks, u, rank);
        if (r != 0) {
            set_err(ctx, std::string("ncclCommInitRank: ") + nccl::g_api.err(r));
            throw Fail{WLM_CUDA};
        }
    });
    if (s != WLM_OK) return s;
    return make_group(ctx, d, nranks, rank, 1, cfg, comm, out);
}

void wlm_slab_group_destroy(wlm_slab_group* g) {
    if (!g) return;
    cudaSetDevice(g->ctx->device);
    cudaStreamSynchronize(g->ctx->stream);
    delete g;
}

wlm_status wlm_slab_group_load(wlm_slab_group* g, const float* F, const float* M, int is_host) {
    if (!g || !F || !M) return WLM_INVALID_ARG;
    wlm_ctx* ctx = g->ctx;
    return run(ctx, [&] {
        const size_t bytes = sizeof(float) * (size_t)g->gfull.nfull;
        const cudaMemcpyKind k = is_host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
        CK(cudaMemcpyAsync(g->fp(), F, bytes, k, ctx->stream));
        CK(cudaMemcpyAsync(g->mp(), M, bytes, k, ctx->stream));
        for (auto* e : g->eng) launch_shifts(e->B, ctx->stream);
    });
}

wlm_status wlm_slab_group_set_warp(wlm_slab_group* g, const float* u, int is_host) {
    if (!g) return WLM_INVALID_ARG;
    wlm_ctx* ctx = g->ctx;
    return run(ctx, [&] {
        const long long nxy = g->nxy();
        for (auto* e : g->eng) {
            k_set_cur0<<<1, 1, 0, ctx->stream>>>(e->st.p);
            ++g_kernel_launches;
            CK(cudaMemsetAsync(e->U.p, 0, sizeof(float) * 6 * (size_t)e->g.n, ctx->stream));
            if (!u) continue;
            for (int c = 0; c < 3; ++c)
                CK(cudaMemcpyAsync(e->U.p + (size_t)c * e->g.n, u + (size_t)c * g->gfull.nfull + e->g.zlo * nxy,
                                   sizeof(float) * (size_t)e->g.n,
                                   is_host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, ctx->stream));
        }
        CK(cudaStreamSynchronize(ctx->stream));
    });
}

wlm_status wlm_slab_group_get_warp(wlm_slab_group* g, float* u, int is_host) {
    if (!g || !u) return WLM_INVALID_ARG;
    wlm_ctx* ctx = g->ctx;
    return run(ctx, [&] {
        const long long nxy = g->nxy();
        for (auto* e : g->eng) {
            const int buf = read_states(e)[0].cur;
            for (int c = 0; c < 3; ++c)
                CK(cudaMemcpyAsync(u + (size_t)c * g->gfull.nfull + (size_t)e->g.zs * nxy,
                                   e->U.p + (size_t)(buf * 3 + c) * e->g.n + (size_t)(e->g.zs - e->g.zlo) * nxy,
                                   sizeof(float) * (size_t)(e->g.ze - e->g.zs) * nxy,
                                   is_host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, ctx->stream));
        }
        CK(cudaStreamSynchronize(ctx->stream));
    });
}

wlm_status wlm_slab_group_fused_halos(const wlm_slab_group* g, int* mask) {
    if (!g || !mask) return WLM_INVALID_ARG;
    *mask = 0;
    for (int k = 0; k < 4; ++k)
        if (g->fused[k]) *mask |= 1 << k;
    return WLM_OK;
}

wlm_status wlm_slab_group_owned(const wlm_slab_group* g, int* zs, int* ze) {
    if (!g || !zs || !ze) return WLM_INVALID_ARG;
    *zs = g->eng.front()->g.zs;
    *ze = g->eng.back()->g.ze;
    return WLM_OK;
}

wlm_status wlm_slab_group_reset(wlm_slab_group* g) {
    if (!g) return WLM_INVALID_ARG;
    wlm_ctx* ctx = g->ctx;
    return run(ctx, [&] {
        for (auto* e : g->eng) {
            launch_begin_level(e->B, e->P, 0, 1, e->cfg.lm.lambda0, ctx->stream);
            clear_adam_moments(e, ctx->stream);
        }
    });
}

wlm_status wlm_slab_group_begin_level(wlm_slab_group* g, int level) {
    if (!g) return WLM_INVALID_ARG;
    wlm_ctx* ctx = g->ctx;
    return run(ctx, [&] {
        for (auto* e : g->eng) launch_begin_level(e->B, e->P, level, 0, e->cfg.lm.lambda0, ctx->stream);
        g->evaluate(0, ctx->stream);
    });
}

wlm_status wlm_slab_group_iterate(wlm_slab_group* g, int iters) {
    if (!g || iters < 0) return WLM_INVALID_ARG;
    wlm_ctx* ctx = g->ctx;
    return run(ctx, [&] {
        for (auto* e : g->eng) launch_set_targets(e->B, iters, ctx->stream);
        if (iters == 0) return;
        if (g->distributed()) {
            if (!g->eng[0]->P.rejection && g->try_step_graph()) {
                for (int i = 0; i < iters; ++i) CK(cudaGraphLaunch(g->step_exec, ctx->stream));
                g_kernel_launches += (uint64_t)iters * g->body_kernels;
            } else {
                g->iterate_eager(iters);
            }
        } else if (!g->eng[0]->P.rejection) {
            g->build_step_graph();
            for (int i = 0; i < iters; ++i) CK(cudaGraphLaunch(g->step_exec, ctx->stream));
            g_kernel_launches += (uint64_t)iters * g->body_kernels;
        } else {
            g->build_loop_graph();
            CK(cudaGraphLaunch(g->loop_exec, ctx->stream));
            g_kernel_launches += (uint64_t)g->body_kernels + 1;
        }
    });
}

wlm_status wlm_slab_group_trace(wlm_slab_group* g, wlm_step_log* rows, size_t cap, size_t* len) {
    if (!g) return WLM_INVALID_ARG;
    wlm_status s = wlm_engine_trace(g->eng[0], 0, rows, cap, len);
    if (s != WLM_OK) return s;
    std::vector<wlm_step_log> other(cap);
    for (size_t k = 1; k < g->eng.size(); ++k) {
        size_t n2 = 0;
        s = wlm_engine_trace(g->eng[k], 0, other.data(), cap, &n2);
        if (s != WLM_OK) return s;
        if (n2 != *len || (rows && std::memcmp(other.data(), rows, sizeof(wlm_step_log) * n2) != 0)) {
            set_err(g->ctx, "slab_group: slabs diverged (state machines disagree)");
            return WLM_CUDA;
        }
    }
    return WLM_OK;
}

wlm_status wlm_slab_group_state(wlm_slab_group* g, wlm_lm_state* st, double* r, double* lncc, int* iters) {
    if (!g) return WLM_INVALID_ARG;
    return wlm_engine_state(g->eng[0], 0, st, r, lncc, iters);
}

}  // extern "C"
