// slab.cu -- z-slab decomposition of one registration (config 5).
//
// A volume is split along z into P slabs of >= kHalo planes.  Each slab is a
// wlm_engine whose per-voxel buffers hold its owned planes plus kHalo halo
// planes; F and M are whole-volume and shared.  One LM attempt runs the
// stages of every slab with a halo exchange after each producer stage:
//
//   K2 (+Adam) -> exchange g (R_u planes) -> K3 -> max over slabs
//   -> exchange dU_s (R_w) -> K4 -> exchange u' of the attempt buffer
//   (R_w + 1, >= 2) -> [Jacobian, min over slabs] -> K1a/K1b (per-plane
//   sum(rho) into the shared plane array) -> K5 on every slab (identical
//   state machines) -> exchange A, B, E (2 planes)
//
// Every voxel's arithmetic is the single-domain arithmetic (direct z sums,
// global faces) and sum(rho) is reduced per plane then over planes in z
// order, so any P gives bit-identical losses, decisions and warps -- the
// P-invariance the tests check.  Here the slabs share one device and the
// exchange is device-to-device copies inside the captured attempt graph; on
// P GPUs the same schedule maps to NCCL send/recv of the same plane ranges
// and an all-reduce of the plane sums and of the max.
#include <algorithm>
#include <cstring>
#include <vector>

#include "internal.cuh"

using namespace wlm;

namespace {

constexpr int kHalo = 4;  // >= max(R_u, R_w + 1, 2) for sigma <= 1

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
__global__ void k_copy_attempt_warp(float* dst, long long dn, int doff, const float* src, long long sn,
                                    int soff, int count, const PairState* st) {
    const int buf = 1 - st->cur;
    for (int c = 0; c < 3; ++c) {
        float* d = dst + (long long)(buf * 3 + c) * dn + doff;
        const float* s = src + (long long)(buf * 3 + c) * sn + soff;
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x) d[i] = s[i];
    }
}

__global__ void k_set_cur0(PairState* st) { st->cur = 0; }

__global__ void k_group_cond(const PairState* st, cudaGraphConditionalHandle h) {
    cudaGraphSetConditional(h, st->done ? 0u : 1u);
}

}  // namespace

struct wlm_slab_group {
    wlm_ctx* ctx = nullptr;
    wlm_dims dims{};
    Geo gfull{};
    int nslabs = 0;
    wlm_reg_config cfg{};
    std::vector<wlm_engine*> eng;
    DevBuf<float> F, M;
    DevBuf<double> plane_sum;
    DevBuf<PairState*> sts;
    cudaGraphExec_t step_exec = nullptr, loop_exec = nullptr;
    cudaGraph_t step_graph = nullptr, loop_graph = nullptr;
    int body_kernels = 0;

    ~wlm_slab_group() {
        if (step_exec) cudaGraphExecDestroy(step_exec);
        if (loop_exec) cudaGraphExecDestroy(loop_exec);
        if (step_graph) cudaGraphDestroy(step_graph);
        if (loop_graph) cudaGraphDestroy(loop_graph);
        for (auto* e : eng) delete e;
    }

    long long nxy() const { return (long long)dims.nx * dims.ny; }

    // Fill slab k's halo planes of a single (non-ping-pong) buffer of `ch`
    // channels x `esz` bytes from its neighbours' owned planes.
    void exchange_fixed(cudaStream_t s, int h, int ch, size_t esz, char* (*base)(wlm_engine*)) {
        for (int k = 0; k < nslabs; ++k) {
            wlm_engine* d = eng[k];
            for (int side = 0; side < 2; ++side) {
                const int nb = side == 0 ? k - 1 : k + 1;
                if (nb < 0 || nb >= nslabs) continue;
                wlm_engine* src = eng[nb];
                const int z0 = side == 0 ? std::max(0, d->g.zs - h) : d->g.ze;
                const int z1 = side == 0 ? d->g.zs : std::min(dims.nz, d->g.ze + h);
                if (z1 <= z0) continue;
                const size_t cnt = (size_t)(z1 - z0) * nxy();
                for (int c = 0; c < ch; ++c) {
                    char* dp = base(d) + ((size_t)c * d->g.n + (size_t)(z0 - d->g.zlo) * nxy()) * esz;
                    const char* sp = base(src) + ((size_t)c * src->g.n + (size_t)(z0 - src->g.zlo) * nxy()) * esz;
                    CK(cudaMemcpyAsync(dp, sp, cnt * esz, cudaMemcpyDeviceToDevice, s));
                }
            }
        }
    }

    void exchange_attempt_warp(cudaStream_t s, int h) {
        for (int k = 0; k < nslabs; ++k) {
            wlm_engine* d = eng[k];
            for (int side = 0; side < 2; ++side) {
                const int nb = side == 0 ? k - 1 : k + 1;
                if (nb < 0 || nb >= nslabs) continue;
                wlm_engine* src = eng[nb];
                const int z0 = side == 0 ? std::max(0, d->g.zs - h) : d->g.ze;
                const int z1 = side == 0 ? d->g.zs : std::min(dims.nz, d->g.ze + h);
                if (z1 <= z0) continue;
                const int cnt = (int)((z1 - z0) * nxy());
                k_copy_attempt_warp<<<std::min(148 * 4, (cnt + 255) / 256), 256, 0, s>>>(
                    d->U.p, d->g.n, (int)((z0 - d->g.zlo) * nxy()), src->U.p, src->g.n,
                    (int)((z0 - src->g.zlo) * nxy()), cnt, src->st.p);
                ++g_kernel_launches;
            }
        }
    }

    void xchg_g(cudaStream_t s) {
        exchange_fixed(s, eng[0]->P.Ru, 3, sizeof(float), [](wlm_engine* e) { return (char*)e->G.p; });
    }
    void xchg_v(cudaStream_t s) {
        exchange_fixed(s, eng[0]->P.Rw, 3, sizeof(float), [](wlm_engine* e) { return (char*)e->VS.p; });
    }
    void xchg_abe(cudaStream_t s) {
        // A, B: two fp32 planes-stacks; E: one fp64 stack stored after them
        exchange_fixed(s, 2, 2, sizeof(float), [](wlm_engine* e) { return (char*)e->ABE.p; });
        exchange_fixed(s, 2, 1, sizeof(double),
                       [](wlm_engine* e) { return (char*)(e->ABE.p + 2 * e->g.n); });
    }

    void body(cudaStream_t s) {
        for (auto* e : eng) e->stage_grad(s);
        xchg_g(s);
        for (auto* e : eng) e->stage_step(s);
        const int jac = eng[0]->P.log_jacobian;
        k_group_combine<<<1, 1, 0, s>>>(sts.p, nslabs, 0);
        ++g_kernel_launches;
        xchg_v(s);
        for (auto* e : eng) launch_compose_smooth(e->B, e->P, s);
        exchange_attempt_warp(s, std::max(eng[0]->P.Rw + 1, 2));
        if (jac) {
            for (auto* e : eng) launch_jacobian_diag(e->B, e->P, s);
            k_group_combine<<<1, 1, 0, s>>>(sts.p, nslabs, 1);
            ++g_kernel_launches;
        }
        for (auto* e : eng) e->stage_eval(1, s);
        for (auto* e : eng) e->stage_finalize(1, s);
        xchg_abe(s);
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
};

extern "C" {

wlm_status wlm_slab_group_create(wlm_ctx* ctx, wlm_dims d, int nslabs, const wlm_reg_config* cfg,
                                 wlm_slab_group** out) {
    if (!ctx || !out || !cfg || nslabs < 1 || !valid_dims(d)) return WLM_INVALID_ARG;
    *out = nullptr;
    if (d.nz / nslabs < kHalo) {
        set_err(ctx, "slab_group: every slab needs at least 4 planes (halo depth)");
        return WLM_INVALID_ARG;
    }
    wlm_slab_group* grp = new wlm_slab_group();
    grp->ctx = ctx;
    grp->dims = d;
    grp->gfull = make_geo(d);
    grp->nslabs = nslabs;
    grp->cfg = *cfg;
    wlm_status s = run(ctx, [&] {
        grp->F = DevBuf<float>(ctx, (size_t)grp->gfull.nfull);
        grp->M = DevBuf<float>(ctx, (size_t)grp->gfull.nfull);
        grp->plane_sum = DevBuf<double>(ctx, (size_t)d.nz);
        CK(cudaMemsetAsync(grp->plane_sum.p, 0, sizeof(double) * d.nz, ctx->stream));
        std::vector<PairState*> hst;
        for (int k = 0; k < nslabs; ++k) {
            wlm_engine* e = new wlm_engine();
            grp->eng.push_back(e);
            const wlm_status es = engine_init(e, ctx, d, 1, cfg);
            if (es != WLM_OK) throw Fail{es};
            const int zs = (int)((long long)k * d.nz / nslabs), ze = (int)((long long)(k + 1) * d.nz / nslabs);
            e->g = make_slab_geo(d, zs, ze, kHalo);
            e->shared_fm = true;
            e->shared_plane_sum = true;
            e->B.F = grp->F.p;
            e->B.M = grp->M.p;
            e->B.plane_sum = grp->plane_sum.p;
            engine_alloc(e);
            hst.push_back(e->st.p);
        }
        grp->sts = DevBuf<PairState*>(ctx, nslabs);
        CK(cudaMemcpyAsync(grp->sts.p, hst.data(), sizeof(PairState*) * nslabs, cudaMemcpyHostToDevice,
                           ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    });
    if (s != WLM_OK) {
        delete grp;
        return s;
    }
    *out = grp;
    return WLM_OK;
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
        CK(cudaMemcpyAsync(g->F.p, F, bytes, k, ctx->stream));
        CK(cudaMemcpyAsync(g->M.p, M, bytes, k, ctx->stream));
        for (auto* e : g->eng) launch_shifts(e->B, ctx->stream);
    });
}

// u: whole-volume SoA [3][nz][ny][nx] (host or device), or null for identity.
// Each slab receives its owned planes and its halo planes.
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
            const std::vector<PairState> st = read_states(e);
            const int buf = st[0].cur;
            for (int c = 0; c < 3; ++c)
                CK(cudaMemcpyAsync(u + (size_t)c * g->gfull.nfull + (size_t)e->g.zs * nxy,
                                   e->U.p + (size_t)(buf * 3 + c) * e->g.n + (size_t)(e->g.zs - e->g.zlo) * nxy,
                                   sizeof(float) * (size_t)(e->g.ze - e->g.zs) * nxy,
                                   is_host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, ctx->stream));
        }
        CK(cudaStreamSynchronize(ctx->stream));
    });
}

wlm_status wlm_slab_group_begin_level(wlm_slab_group* g, int level) {
    if (!g) return WLM_INVALID_ARG;
    wlm_ctx* ctx = g->ctx;
    return run(ctx, [&] {
        for (auto* e : g->eng) launch_begin_level(e->B, e->P, level, 0, e->cfg.lm.lambda0, ctx->stream);
        for (auto* e : g->eng) e->stage_eval(0, ctx->stream);
        for (auto* e : g->eng) e->stage_finalize(0, ctx->stream);
        g->xchg_abe(ctx->stream);
    });
}

wlm_status wlm_slab_group_iterate(wlm_slab_group* g, int iters) {
    if (!g || iters < 0) return WLM_INVALID_ARG;
    wlm_ctx* ctx = g->ctx;
    return run(ctx, [&] {
        for (auto* e : g->eng) launch_set_targets(e->B, iters, ctx->stream);
        if (iters == 0) return;
        if (!g->eng[0]->P.rejection) {
            g->build_step_graph();
            for (int i = 0; i < iters; ++i) CK(cudaGraphLaunch(g->step_exec, ctx->stream));
            g_kernel_launches += (uint64_t)iters * g->body_kernels;
        } else {
            g->build_loop_graph();
            CK(cudaGraphLaunch(g->loop_exec, ctx->stream));
        }
    });
}

// Trace of slab 0; WLM_INTERNAL-style consistency: every slab must have run
// the identical state machine (returns WLM_CUDA with a message otherwise).
wlm_status wlm_slab_group_trace(wlm_slab_group* g, wlm_step_log* rows, size_t cap, size_t* len) {
    if (!g) return WLM_INVALID_ARG;
    wlm_status s = wlm_engine_trace(g->eng[0], 0, rows, cap, len);
    if (s != WLM_OK) return s;
    std::vector<wlm_step_log> other(cap);
    for (int k = 1; k < g->nslabs; ++k) {
        size_t n2 = 0;
        s = wlm_engine_trace(g->eng[k], 0, other.data(), cap, &n2);
        if (s != WLM_OK) return s;
        if (n2 != *len || std::memcmp(other.data(), rows, sizeof(wlm_step_log) * n2) != 0) {
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
