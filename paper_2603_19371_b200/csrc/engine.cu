// engine.cu -- device-resident LM engine, register() driver and the C-ABI.
//
// Host code here only orchestrates: allocations, uploads, CUDA-graph capture
// and launch.  Every per-voxel operation and the per-iteration scalar state
// machine run on the GPU; within a pyramid level there is no host
// synchronisation at all.  There is no CPU fallback: without a
// CUDA device every entry point fails with WLM_CUDA.
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "internal.cuh"

using namespace wlm;

namespace wlm {

wlm_status engine_init(wlm_engine* e, wlm_ctx* ctx, wlm_dims d, int pairs, const wlm_reg_config* c) {
    e->ctx = ctx;
    e->dims = d;
    e->g = make_geo(d);
    e->pairs = pairs;
    e->cfg = *c;
    // pair groups of the attempt graph; WLM_PAIR_GROUPS=1
    // captures the whole batch as one chain
    {
        const char* v = std::getenv("WLM_PAIR_GROUPS");
        const int n = v ? std::atoi(v) : 0;
        e->pair_groups = (n >= 1 && n <= wlm_engine::kMaxGroups) ? n : 2;
    }
    if (c->lm.tile_size < 1) {
        set_err(ctx, "lm.tile_size must be >= 1 (SPEC.md:259)");
        return WLM_INVALID_ARG;
    }
    if (c->metric != WLM_METRIC_LNCC && c->metric != WLM_METRIC_MSE && c->metric != WLM_METRIC_MI) {
        set_err(ctx, "metric: LNCC, MSE or MI");
        return WLM_INVALID_ARG;
    }
    if (c->metric == WLM_METRIC_MI && (c->mi_bins < 2 || c->mi_bins > 64 || !(c->mi_sigma > 0.0) ||
                                       c->mi_sigma > 2.0)) {
        set_err(ctx, "MI: mi_bins in [2, 64] (SPEC.md:124), mi_sigma in (0, 2] bin widths");
        return WLM_INVALID_ARG;
    }
    if (c->optimizer < WLM_OPT_LM || c->optimizer > WLM_OPT_DEMONS) {
        set_err(ctx, "optimizer: LM, ADAM, GD or DEMONS");
        return WLM_INVALID_ARG;
    }
    if (c->optimizer == WLM_OPT_DEMONS && (c->metric != WLM_METRIC_MSE || !(c->demons_alpha > 0.0))) {
        set_err(ctx, "DEMONS needs metric = MSE (per-voxel residual, SPEC.md:166) and alpha > 0 (SPEC.md:243)");
        return WLM_INVALID_ARG;
    }
    if (c->metric == WLM_METRIC_LNCC && c->lncc_radius < 1) {
        set_err(ctx, "lncc_radius must be >= 1 (SPEC.md:123)");
        return WLM_INVALID_ARG;
    }
    if ((long long)d.nx * d.ny * d.nz >= (1ll << 31)) {
        set_err(ctx, "volumes of 2^31 voxels or more are not supported (io.cpp:13 cap)");
        return WLM_UNSUPPORTED;
    }
    if (c->metric == WLM_METRIC_LNCC &&
        (d.nx <= 2 * c->lncc_radius || d.ny <= 2 * c->lncc_radius || d.nz <= 2 * c->lncc_radius)) {
        set_err(ctx, "residual_lncc: dims must exceed 2*radius (SPEC.md:138)");
        return WLM_INVALID_ARG;
    }
    if (!(c->target_max_disp > 0.0 && c->target_max_disp < 0.5)) {
        set_err(ctx, "normalize_step: target_max_disp must lie in (0, 0.5)");
        return WLM_INVALID_ARG;
    }
    LmParams& P = e->P;
    std::memset(&P, 0, sizeof(P));
    P.mu_plus = c->lm.mu_plus;
    P.mu_minus = c->lm.mu_minus;
    P.lambda_max = c->lm.lambda_max;
    P.tau = c->lm.tau;
    P.target = c->target_max_disp;
    P.step_floor = c->step_floor;
    P.adam_b1 = c->adam.beta1; P.adam_b2 = c->adam.beta2;
    P.adam_eps = c->adam.eps_hat; P.adam_lr = c->adam.lr;
    P.gd_lr = c->gd_lr;
    P.rejection = c->lm.rejection;
    P.max_retries = c->lm.max_retries;
    P.optimizer = c->optimizer;
    P.log_jacobian = c->log_jacobian;
    P.radius = c->lncc_radius;
    P.metric = c->metric;
    P.demons_alpha = c->demons_alpha;
    P.tile_k = c->lm.tile_size;
    P.mi_bins = c->mi_bins;
    P.mi_sigma = c->mi_sigma;
    // memory layout: K2 re-gathers grad M(x+u) (fused LNCC path only)
    P.lean = c->low_memory && c->metric == WLM_METRIC_LNCC && c->lncc_radius == 2 ? 1 : 0;
    P.Ru = smooth_radius(c->sigma_update);
    P.Rw = smooth_radius(c->sigma_warp);
    // radius <= 6 (sigma <= 2): the fused K3 / K4; larger: generic.cu
    // half-kernels of the fused K3 / K4 (radius <= 6; LmParams holds 8 taps)
    if (P.Ru <= 6) {
        fill_half_kernel(c->sigma_update, P.Ru, P.wu, &P.wu_full);
        fill_half_kernel(c->sigma_update, P.Ru, P.wud, &P.wud_full);
    }
    if (P.Rw <= 6) {
        fill_half_kernel(c->sigma_warp, P.Rw, P.wwd, &P.wwd_full);
        fill_half_kernel(c->sigma_warp, P.Rw, P.ww, &P.ww_full);
    }
    int maxit = 0;
    for (int i = 0; i < c->nlevels && i < WLM_MAX_LEVELS; ++i) maxit = std::max(maxit, c->iters[i]);
    P.trace_cap = std::max(1024, maxit + 1);
    return WLM_OK;
}

// A new registration starts from zero Adam moments: k_adam's bias correction
// restarts at t = 1 with the iteration counter, and stale m, v would be
// amplified by it.
void clear_adam_moments(wlm_engine* e, cudaStream_t s) {
    if (e->P.optimizer != WLM_OPT_ADAM) return;
    wlm_ctx* ctx = e->ctx;
    const size_t bytes = sizeof(float) * (size_t)e->pairs * 3 * (size_t)e->g.n;
    CK(cudaMemsetAsync(e->AM.p, 0, bytes, s));
    CK(cudaMemsetAsync(e->AV.p, 0, bytes, s));
}

void engine_alloc(wlm_engine* e) {
    wlm_ctx* ctx = e->ctx;
    const size_t n = (size_t)e->g.n, B = (size_t)e->pairs;
    if (!e->shared_fm) {  // slab groups share one whole-volume F, M
        e->F = DevBuf<float>(ctx, B * (size_t)e->g.nfull);
        e->M = DevBuf<float>(ctx, B * (size_t)e->g.nfull);
    }
    e->U = DevBuf<float>(ctx, B * 6 * n);
    e->ABE = DevBuf<float>(ctx, B * 4 * n);  // A, B fp32 + E fp64
    e->MW = DevBuf<double>(ctx, B * n);
    if (e->P.metric == WLM_METRIC_LNCC && !e->P.lean) e->GM = DevBuf<double>(ctx, B * 3 * n);  // K1a -> K2
    e->shift_part = DevBuf<double>(ctx, B * 2 * 256 * 3);  // sums + (min, max)
    init_constants();
    e->G = DevBuf<float>(ctx, B * 3 * n);
    // dU_s (K3 -> K4, the Jacobian) shares ABE's memory: A, B, E are written by
    // K1b and last read by K2, so they are dead exactly while dU_s lives
    // (12 B/voxel less)
    if (e->P.optimizer == WLM_OPT_ADAM) {
        e->AM = DevBuf<float>(ctx, B * 3 * n);
        e->AV = DevBuf<float>(ctx, B * 3 * n);
        CK(cudaMemsetAsync(e->AM.p, 0, sizeof(float) * B * 3 * n, ctx->stream));
        CK(cudaMemsetAsync(e->AV.p, 0, sizeof(float) * B * 3 * n, ctx->stream));
        // bias corrections 1 - beta^t with the host's std::pow (the oracle's)
        const int nt = e->P.trace_cap + 1;
        std::vector<double> bc(2 * (size_t)nt);
        for (int t = 1; t <= nt; ++t) {
            bc[t - 1] = 1.0 - std::pow(e->P.adam_b1, t);
            bc[nt + t - 1] = 1.0 - std::pow(e->P.adam_b2, t);
        }
        e->ABC = DevBuf<double>(ctx, bc.size());
        CK(cudaMemcpy(e->ABC.p, bc.data(), sizeof(double) * bc.size(), cudaMemcpyHostToDevice));
        e->P.adam_bc = e->ABC.p;
        e->P.adam_bc_n = nt;
    }
    // generic paths (generic.cu): fp64 scratch and device Gaussian taps
    const bool gen_lncc = e->P.metric == WLM_METRIC_LNCC && e->P.radius != 2;
    if (gen_lncc || e->P.Ru > 6 || e->P.Rw > 6) e->X64 = DevBuf<double>(ctx, B * generic_scratch_doubles(e->g));
    auto taps = [&](double sigma, int R, DevBuf<double>& buf) -> const double* {
        if (R <= 6) return nullptr;
        int r = 0;
        const std::vector<double> w = gaussian_taps64(sigma, &r);
        buf = DevBuf<double>(ctx, w.size());
        CK(cudaMemcpy(buf.p, w.data(), sizeof(double) * w.size(), cudaMemcpyHostToDevice));
        return buf.p;
    };
    e->P.taps_u = taps(e->cfg.sigma_update, e->P.Ru, e->TAPU);
    e->P.taps_w = taps(e->cfg.sigma_warp, e->P.Rw, e->TAPW);
    e->st = DevBuf<PairState>(ctx, B);
    CK(cudaMemsetAsync(e->st.p, 0, sizeof(PairState) * B, ctx->stream));
    const int tiles = plane_tiles(e->g);
    e->partials = DevBuf<double>(ctx, B * (size_t)e->g.nz * tiles * 8);
    if (!e->shared_plane_sum) e->plane_sum = DevBuf<double>(ctx, B * (size_t)e->g.nz);
    if (e->P.tile_k > 1) {  // tiled LM (Eq. 5): one matrix per k^3 tile
        const int k = e->P.tile_k;
        e->B.tkx = (e->g.nx + k - 1) / k;
        e->B.tky = (e->g.ny + k - 1) / k;
        e->B.tkz = (e->g.nz + k - 1) / k;
        e->TM = DevBuf<double>(ctx, B * 6 * (size_t)e->B.tkx * e->B.tky * e->B.tkz);
    }
    if (e->P.metric == WLM_METRIC_MI) {
        const size_t bb = (size_t)e->P.mi_bins * e->P.mi_bins;
        e->HIST = DevBuf<unsigned long long>(ctx, B * bb);
        e->MIT = DevBuf<double>(ctx, B * bb);
        CK(cudaMemsetAsync(e->HIST.p, 0, sizeof(unsigned long long) * B * bb, ctx->stream));
    }
    e->trace = DevBuf<wlm_step_log>(ctx, B * (size_t)e->P.trace_cap);
    e->P.trace = e->trace.p;
    Batch& b = e->B;
    b.g = e->g;
    b.pairs = e->pairs;
    if (!e->shared_fm) { b.F = e->F.p; b.M = e->M.p; }
    b.U = e->U.p; b.ABE = e->ABE.p; b.G = e->G.p;
    b.VS = e->ABE.p;
    b.vs_ps = 4 * (long long)n;
    b.AM = e->AM.p; b.AV = e->AV.p;
    b.MW = e->MW.p;
    b.GM = e->GM.p;
    b.st = e->st.p;
    b.partials = e->partials.p;
    if (!e->shared_plane_sum) b.plane_sum = e->plane_sum.p;
    b.zero_foreign_planes = 0;
    b.peer_on = 0;  // a slab group turns on its fused halo stores after allocation
    std::memset(&b.peer, 0, sizeof(b.peer));
    b.shift_part = e->shift_part.p;
    b.TM = e->TM.p;
    b.HIST = e->HIST.p;
    b.MIT = e->MIT.p;
    b.X64 = e->X64.p;
    b.max_blocks = tiles;
    make_tma_u(b, e->P.Rw);
    CK(cudaMemsetAsync(e->U.p, 0, sizeof(float) * B * 6 * n, ctx->stream));
    launch_begin_level(b, e->P, 0, 1, e->cfg.lm.lambda0, ctx->stream);
}

std::vector<PairState> read_states(wlm_engine* e) {
    wlm_ctx* ctx = e->ctx;
    std::vector<PairState> s(e->pairs);
    CK(cudaMemcpyAsync(s.data(), e->st.p, sizeof(PairState) * e->pairs, cudaMemcpyDeviceToHost,
                       ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return s;
}

namespace {
__global__ void k_reset_cur(PairState* st, int pairs) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < pairs) st[i].cur = 0;
}

}  // namespace

void copy_warps_in(wlm_engine* e, const float* u, int is_host) {
    wlm_ctx* ctx = e->ctx;
    const size_t n3 = 3 * (size_t)e->g.n;
    k_reset_cur<<<(e->pairs + 127) / 128, 128, 0, ctx->stream>>>(e->st.p, e->pairs);
    ++g_kernel_launches;
    if (!u) {
        CK(cudaMemsetAsync(e->U.p, 0, sizeof(float) * 2 * n3 * e->pairs, ctx->stream));
        return;
    }
    CK(cudaMemcpy2DAsync(e->U.p, sizeof(float) * 2 * n3, u, sizeof(float) * n3, sizeof(float) * n3,
                         e->pairs, is_host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice,
                         ctx->stream));
}

}  // namespace wlm

// ===========================================================================
// C-ABI
extern "C" {

const char* wlm_version(void) { return "warplm-b200 0.1 (sm_100a)"; }

void wlm_default_reg_config(wlm_reg_config* c) {
    std::memset(c, 0, sizeof(*c));
    c->lncc_radius = 2;
    c->optimizer = WLM_OPT_LM;
    c->lm.lambda0 = 0.006; c->lm.mu_plus = 1.5; c->lm.mu_minus = 0.975;
    c->lm.tile_size = 1; c->lm.rejection = 0; c->lm.tau = 1.0; c->lm.lambda_max = 1.0;
    c->lm.max_retries = 10;
    c->adam.beta1 = 0.9; c->adam.beta2 = 0.999; c->adam.eps_hat = 1e-8; c->adam.lr = 0.5;
    c->gd_lr = 1.0;
    c->nlevels = 3;
    c->factors[0] = 4; c->factors[1] = 2; c->factors[2] = 1;
    c->iters[0] = 100; c->iters[1] = 75; c->iters[2] = 50;
    c->target_max_disp = 0.4; c->step_floor = 1e-12;
    c->sigma_update = 1.0; c->sigma_warp = 0.5;
    c->log_jacobian = 0;
    c->metric = WLM_METRIC_LNCC;
    c->demons_alpha = 1.0;
    c->mi_bins = 32;
    c->mi_sigma = 1.0;
    c->low_memory = 0;
}

wlm_status wlm_ctx_create(int device, wlm_ctx** out) {
    if (!out) return WLM_INVALID_ARG;
    *out = nullptr;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) return WLM_CUDA;
    if (device < 0 || device >= n) return WLM_INVALID_ARG;
    if (cudaSetDevice(device) != cudaSuccess) return WLM_CUDA;
    wlm_ctx* c = new wlm_ctx();
    c->device = device;
    if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&c->capture, cudaStreamNonBlocking) != cudaSuccess) {
        delete c;
        return WLM_CUDA;
    }
    *out = c;
    return WLM_OK;
}

void wlm_ctx_destroy(wlm_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    if (c->stream && c->own_stream) cudaStreamDestroy(c->stream);
    if (c->capture) cudaStreamDestroy(c->capture);
    delete c;
}

const char* wlm_last_error(const wlm_ctx* c) { return c ? c->err.c_str() : "null context"; }
void* wlm_ctx_stream(wlm_ctx* c) { return c ? (void*)c->stream : nullptr; }

wlm_status wlm_ctx_set_stream(wlm_ctx* c, void* s) {
    if (!c) return WLM_INVALID_ARG;
    if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
    c->stream = (cudaStream_t)s;
    c->own_stream = false;
    return WLM_OK;
}

wlm_status wlm_ctx_synchronize(wlm_ctx* ctx) {
    return run(ctx, [&] { CK(cudaStreamSynchronize(ctx->stream)); });
}

uint64_t wlm_ctx_launch_count(const wlm_ctx* c) { return c ? c->launches : 0; }
size_t wlm_ctx_peak_bytes(const wlm_ctx* c) { return c ? c->peak_bytes : 0; }

wlm_status wlm_engine_create(wlm_ctx* ctx, wlm_dims d, int pairs, const wlm_reg_config* cfg,
                             wlm_engine** out) {
    if (!ctx || !out || !cfg || pairs < 1 || !valid_dims(d)) return WLM_INVALID_ARG;
    *out = nullptr;
    wlm_engine* e = new wlm_engine();
    wlm_status s = guard(ctx);
    if (s == WLM_OK) s = engine_init(e, ctx, d, pairs, cfg);
    if (s == WLM_OK) s = run(ctx, [&] { engine_alloc(e); });
    if (s != WLM_OK) {
        delete e;
        return s;
    }
    *out = e;
    return WLM_OK;
}

void wlm_engine_destroy(wlm_engine* e) {
    if (!e) return;
    cudaSetDevice(e->ctx->device);
    cudaStreamSynchronize(e->ctx->stream);
    delete e;
}

wlm_status wlm_engine_load(wlm_engine* e, const float* F, const float* M, int is_host) {
    if (!e || !F || !M) return WLM_INVALID_ARG;
    wlm_ctx* ctx = e->ctx;
    return run(ctx, [&] {
        const size_t bytes = sizeof(float) * (size_t)e->g.nfull * e->pairs;
        const cudaMemcpyKind k = is_host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
        CK(cudaMemcpyAsync(e->F.p, F, bytes, k, ctx->stream));
        CK(cudaMemcpyAsync(e->M.p, M, bytes, k, ctx->stream));
        launch_shifts(e->B, ctx->stream);
    });
}

wlm_status wlm_engine_set_warp(wlm_engine* e, const float* u, int is_host) {
    if (!e) return WLM_INVALID_ARG;
    wlm_ctx* ctx = e->ctx;
    return run(ctx, [&] { copy_warps_in(e, u, is_host); });
}

wlm_status wlm_engine_get_warp(wlm_engine* e, float* u, int is_host) {
    if (!e || !u) return WLM_INVALID_ARG;
    wlm_ctx* ctx = e->ctx;
    return run(ctx, [&] {
        const std::vector<PairState> s = read_states(e);
        const size_t n3 = 3 * (size_t)e->g.n;
        for (int p = 0; p < e->pairs; ++p)
            CK(cudaMemcpyAsync(u + (size_t)p * n3, e->U.p + ((size_t)p * 2 + s[p].cur) * n3,
                               sizeof(float) * n3,
                               is_host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice,
                               ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    });
}

wlm_status wlm_engine_reset(wlm_engine* e) {
    if (!e) return WLM_INVALID_ARG;
    wlm_ctx* ctx = e->ctx;
    return run(ctx, [&] {
        launch_begin_level(e->B, e->P, 0, 1, e->cfg.lm.lambda0, ctx->stream);
        clear_adam_moments(e, ctx->stream);
    });
}

wlm_status wlm_engine_begin_level(wlm_engine* e, int level) {
    if (!e) return WLM_INVALID_ARG;
    wlm_ctx* ctx = e->ctx;
    return run(ctx, [&] {
        launch_begin_level(e->B, e->P, level, 0, e->cfg.lm.lambda0, ctx->stream);
        e->stage_eval(0, ctx->stream);
        e->stage_finalize(0, ctx->stream);
    });
}

wlm_status wlm_engine_iterate(wlm_engine* e, int iters) {
    if (!e || iters < 0) return WLM_INVALID_ARG;
    wlm_ctx* ctx = e->ctx;
    return run(ctx, [&] {
        launch_set_targets(e->B, iters, ctx->stream);
        if (iters == 0) return;
        if (!e->P.rejection && e->grouped()) {
            e->launch_grouped(iters, ctx->stream);
            g_kernel_launches += (uint64_t)iters * e->group_kernels;
        } else if (!e->P.rejection) {
            e->build_step_graph();
            for (int i = 0; i < iters; ++i) CK(cudaGraphLaunch(e->step_exec, ctx->stream));
            g_kernel_launches += (uint64_t)iters * e->body_kernels;
        } else if (e->grouped()) {
            e->launch_grouped_loop(ctx->stream);
            g_kernel_launches += (uint64_t)e->group_kernels + e->ngroups();  // at least one trip
        } else {
            e->build_loop_graph();
            CK(cudaGraphLaunch(e->loop_exec, ctx->stream));
            g_kernel_launches += (uint64_t)e->body_kernels + 1;  // at least one trip
        }
    });
}

wlm_status wlm_engine_step(wlm_engine* e) {
    if (!e) return WLM_INVALID_ARG;
    if (e->P.rejection) return WLM_UNSUPPORTED;
    wlm_ctx* ctx = e->ctx;
    return run(ctx, [&] {
        if (e->grouped()) {
            e->launch_grouped(1, ctx->stream);
            g_kernel_launches += e->group_kernels;
        } else {
            e->build_step_graph();
            CK(cudaGraphLaunch(e->step_exec, ctx->stream));
            g_kernel_launches += e->body_kernels;
        }
    });
}

wlm_status wlm_engine_set_pair_groups(wlm_engine* e, int groups) {
    if (!e || groups < 1 || groups > wlm_engine::kMaxGroups) return WLM_INVALID_ARG;
    if (e->pair_groups != groups) {
        wlm_ctx* ctx = e->ctx;
        wlm_status s = run(ctx, [&] { CK(cudaStreamSynchronize(ctx->stream)); });
        if (s != WLM_OK) return s;
        e->invalidate_graphs();
        e->pair_groups = groups;
    }
    return WLM_OK;
}

wlm_status wlm_engine_stage(wlm_engine* e, int stage) {
    if (!e || stage < 0 || stage > 4) return WLM_INVALID_ARG;
    wlm_ctx* ctx = e->ctx;
    return run(ctx, [&] {
        switch (stage) {
            case 0: e->stage_eval(1, ctx->stream); e->stage_finalize(1, ctx->stream); break;
            case 1: launch_lncc_bwd(e->B, e->P, ctx->stream); break;
            case 2: launch_step_smooth(e->B, e->P, ctx->stream); break;
            case 3: launch_compose_smooth(e->B, e->P, ctx->stream); break;
            default: e->stage_eval(0, ctx->stream); e->stage_finalize(0, ctx->stream); break;
        }
    });
}

wlm_status wlm_engine_state(wlm_engine* e, int pair, wlm_lm_state* st, double* r, double* lncc,
                            int* iters_done) {
    if (!e || pair < 0 || pair >= e->pairs) return WLM_INVALID_ARG;
    wlm_ctx* ctx = e->ctx;
    wlm_status status = WLM_OK;
    wlm_status s = run(ctx, [&] {
        const std::vector<PairState> v = read_states(e);
        const PairState& p = v[pair];
        if (st) { st->lambda = p.lambda; st->hist_n = p.hist_n; st->L1 = p.L1; st->L2 = p.L2; }
        if (r) *r = p.r_cur;
        if (lncc) *lncc = p.lncc_cur;
        if (iters_done) *iters_done = p.iter;
        status = (wlm_status)p.status;
    });
    if (s != WLM_OK) return s;
    if (status != WLM_OK) set_err(ctx, "non-finite loss: iteration aborted (SPEC.md:287)");
    return status;
}

wlm_status wlm_engine_trace(wlm_engine* e, int pair, wlm_step_log* rows, size_t cap, size_t* len) {
    if (!e || pair < 0 || pair >= e->pairs) return WLM_INVALID_ARG;
    wlm_ctx* ctx = e->ctx;
    return run(ctx, [&] {
        const std::vector<PairState> v = read_states(e);
        const size_t n = std::min((size_t)v[pair].trace_len, cap);
        if (n && rows)
            CK(cudaMemcpy(rows, e->trace.p + (size_t)pair * e->P.trace_cap, sizeof(wlm_step_log) * n,
                          cudaMemcpyDeviceToHost));
        if (len) *len = n;
    });
}

wlm_status wlm_engine_buffers(wlm_engine* e, const float** F, const float** M, float** u_cur,
                              float** g, float** vs, float** abe) {
    if (!e) return WLM_INVALID_ARG;
    wlm_ctx* ctx = e->ctx;
    return run(ctx, [&] {
        if (F) *F = e->F.p;
        if (M) *M = e->M.p;
        if (g) *g = e->G.p;
        if (vs) *vs = e->B.VS;  // pair stride 4 n (inside ABE)
        if (abe) *abe = e->ABE.p;
        if (u_cur) {
            const std::vector<PairState> v = read_states(e);
            *u_cur = e->U.p + (size_t)v[0].cur * 3 * (size_t)e->g.n;
        }
    });
}

wlm_status wlm_engine_read_buffer(wlm_engine* e, int which, int pair, float* host, size_t count) {
    if (!e || !host || pair < 0 || pair >= e->pairs || which < 0 || which > 5) return WLM_INVALID_ARG;
    wlm_ctx* ctx = e->ctx;
    const size_t n = (size_t)e->g.n;
    const size_t nch = which < 2 ? 1 : which == 5 ? 4 : 3;
    if (count > nch * n) return WLM_INVALID_ARG;
    return run(ctx, [&] {
        const float* src = nullptr;
        switch (which) {
            case 0: src = e->F.p + pair * n; break;
            case 1: src = e->M.p + pair * n; break;
            case 2: {
                const std::vector<PairState> v = read_states(e);
                src = e->U.p + ((size_t)pair * 2 + v[pair].cur) * 3 * n;
                break;
            }
            case 3: src = e->G.p + pair * 3 * n; break;
            case 4: src = e->B.VS + (size_t)pair * e->B.vs_ps; break;
            default: src = e->ABE.p + pair * 4 * n; break;
        }
        CK(cudaMemcpyAsync(host, src, sizeof(float) * count, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    });
}

wlm_status wlm_engine_script_losses(wlm_engine* e, const double* losses, int n) {
    if (!e || n < 0) return WLM_INVALID_ARG;
    wlm_ctx* ctx = e->ctx;
    return run(ctx, [&] {
        e->invalidate_graphs();
        if (n == 0) {
            e->P.script = nullptr;
            e->P.script_n = 0;
            e->script.release();
            return;
        }
        e->script = DevBuf<double>(ctx, (size_t)n * e->pairs);
        CK(cudaMemcpyAsync(e->script.p, losses, sizeof(double) * n * e->pairs, cudaMemcpyHostToDevice,
                           ctx->stream));
        e->P.script = e->script.p;
        e->P.script_n = n;
    });
}

}  // extern "C"
