// ops.cu -- host-buffer mirror of the reference API (fp64 AoS in/out, like a
// by-value warplm:: call) and the register() pyramid driver.  The `field`
// mirrors (warp_volume, sample_field, compose_warp, max_abs_component,
// normalize_step, jacobian_det_min, gaussian_smooth, lm_step_pointwise,
// downsample, upsample_warp) keep the caller's fp64 AoS data and run the
// reference's arithmetic in its operation order on the device (field64.cu),
// so they return the reference's bits.  The residual mirrors run the
// engine's own hot kernels.  No CPU compute path exists.
#include <cmath>
#include <limits>
#include <vector>

#include "internal.cuh"

using namespace wlm;

namespace {

// fp64 AoS host -> fp32 SoA device.
DevBuf<float> upload_soa(wlm_ctx* ctx, const double* host, size_t n, int nchan) {
    DevBuf<double> tmp(ctx, n * nchan);
    CK(cudaMemcpyAsync(tmp.p, host, sizeof(double) * n * nchan, cudaMemcpyHostToDevice, ctx->stream));
    DevBuf<float> out(ctx, n * nchan);
    launch_aos_to_soa(tmp.p, out.p, (long long)n, nchan, ctx->stream);
    CK(cudaStreamSynchronize(ctx->stream));
    return out;
}

__global__ void k_soa_to_aos_range(const float* __restrict__ in, long long n, long long off, long long cnt, int nchan,
                                   double* __restrict__ out) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < cnt * nchan;
         i += (long long)gridDim.x * blockDim.x)
        out[i] = (double)in[(i % nchan) * n + off + i / nchan];
}

// fp32 SoA device -> fp64 AoS host through a bounded device staging buffer
// (at most 2^20 voxels at a time), so the result download does not raise the
// peak device memory by 8 B per voxel and channel.
void download_aos(wlm_ctx* ctx, const float* dev, size_t n, int nchan, double* host) {
    const size_t chunk = std::min<size_t>(n, (size_t)1 << 20);
    DevBuf<double> tmp(ctx, chunk * nchan);
    for (size_t off = 0; off < n; off += chunk) {
        const size_t cnt = std::min(chunk, n - off);
        const int grid = (int)std::min<size_t>(148 * 8, (cnt * nchan + 255) / 256);
        k_soa_to_aos_range<<<grid, 256, 0, ctx->stream>>>(dev, (long long)n, (long long)off, (long long)cnt, nchan,
                                                          tmp.p);
        ++g_kernel_launches;
        CK(cudaMemcpyAsync(host + off * nchan, tmp.p, sizeof(double) * cnt * nchan, cudaMemcpyDeviceToHost,
                           ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    }
}



DevBuf<double> upload64(wlm_ctx* ctx, const double* host, size_t count) {
    DevBuf<double> d(ctx, count);
    CK(cudaMemcpyAsync(d.p, host, sizeof(double) * count, cudaMemcpyHostToDevice, ctx->stream));
    return d;
}

void download64(wlm_ctx* ctx, const double* dev, size_t count, double* host) {
    CK(cudaMemcpyAsync(host, dev, sizeof(double) * count, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
}

double read_max64(wlm_ctx* ctx, const double* v, long long count) {
    DevBuf<unsigned long long> bits(ctx, 1);
    CK(cudaMemsetAsync(bits.p, 0, sizeof(unsigned long long), ctx->stream));
    launch_max_abs64(v, count, bits.p, ctx->stream);
    unsigned long long h = 0;
    CK(cudaMemcpyAsync(&h, bits.p, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    double m;
    std::memcpy(&m, &h, 8);
    return m;
}

// jacobian_det_min of an fp64 AoS device field (field.cpp:172-201)
double read_jacdet64(wlm_ctx* ctx, const double* u, wlm_dims d, const float* u_soa32 = nullptr) {
    DevBuf<unsigned long long> o(ctx, 1);
    const unsigned long long init = jacobian_key_init();
    CK(cudaMemcpyAsync(o.p, &init, sizeof(init), cudaMemcpyHostToDevice, ctx->stream));
    if (u_soa32) launch_jacobian_min64_soa32(u_soa32, d, o.p, ctx->stream);
    else launch_jacobian_min64(u, d, o.p, ctx->stream);
    unsigned long long h = 0;
    CK(cudaMemcpyAsync(&h, o.p, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return jacobian_key_to_double(h);
}

// gaussian_smooth of an fp64 AoS device array in place (field.cpp:253-269)
void smooth_aos64(wlm_ctx* ctx, double* data, wlm_dims d, int nchan, double sigma) {
    if (sigma <= 0.0) return;  // field.cpp:254, :263
    int R = 0;
    const std::vector<double> w = gaussian_taps64(sigma, &R);
    DevBuf<double> dw = upload64(ctx, w.data(), w.size()), tmp(ctx, nvox(d) * nchan);
    smooth64(data, tmp.p, dw.p, R, d, nchan, 1, nchan, ctx->stream);
    CK(cudaStreamSynchronize(ctx->stream));
}

wlm_status bad(wlm_ctx* ctx, wlm_status s, const char* msg) {
    set_err(ctx, msg);
    return s;
}

}  // namespace

extern "C" {

wlm_status wlm_warp_volume(wlm_ctx* ctx, const double* M, const double* u, wlm_dims d, double* Mw,
                           double* gradM) {
    if (!M || !u || !Mw || !valid_dims(d)) return bad(ctx, WLM_INVALID_ARG, "warp_volume: bad args");
    return run(ctx, [&] {
        const size_t n = nvox(d);
        DevBuf<double> dM = upload64(ctx, M, n), du = upload64(ctx, u, 3 * n);
        DevBuf<double> dw(ctx, n), dg(ctx, gradM ? 3 * n : 0);
        launch_warp_volume64(dM.p, du.p, d, dw.p, gradM ? dg.p : nullptr, ctx->stream);
        download64(ctx, dw.p, n, Mw);
        if (gradM) download64(ctx, dg.p, 3 * n, gradM);
    });
}

// sample_trilinear / sample_trilinear_grad at arbitrary points
// (field.cpp:43-90): value and analytic interpolant gradient, fp64.
wlm_status wlm_sample_trilinear_grad_points(wlm_ctx* ctx, const double* vol, wlm_dims d, const double* pts,
                                            size_t npts, double* val, double* grad) {
    if (!vol || !pts || !val || !valid_dims(d)) return bad(ctx, WLM_INVALID_ARG, "sample_trilinear: bad args");
    return run(ctx, [&] {
        DevBuf<double> dv = upload64(ctx, vol, nvox(d)), dp = upload64(ctx, pts, 3 * npts);
        DevBuf<double> dval(ctx, npts), dg(ctx, grad ? 3 * npts : 0);
        launch_sample_grad_points64(dv.p, d, dp.p, (long long)npts, dval.p, grad ? dg.p : nullptr, ctx->stream);
        download64(ctx, dval.p, npts, val);
        if (grad) download64(ctx, dg.p, 3 * npts, grad);
    });
}

wlm_status wlm_sample_field_points(wlm_ctx* ctx, const double* u, wlm_dims d, const double* pts,
                                   size_t npts, double* out) {
    if (!u || !pts || !out || !valid_dims(d)) return bad(ctx, WLM_INVALID_ARG, "sample_field: bad args");
    return run(ctx, [&] {
        const size_t n = nvox(d);
        DevBuf<double> du = upload64(ctx, u, 3 * n), dp = upload64(ctx, pts, 3 * npts), dout(ctx, 3 * npts);
        launch_sample_points64(du.p, d, dp.p, (long long)npts, dout.p, ctx->stream);
        download64(ctx, dout.p, 3 * npts, out);
    });
}

// compose_warp (field.cpp:123-142): dimension mismatch -> WLM_DIM_MISMATCH
// (the reference throws std::invalid_argument, field.cpp:124-126).
wlm_status wlm_compose_warp(wlm_ctx* ctx, const double* u, wlm_dims du, const double* v, wlm_dims dv,
                            double eps, double* out) {
    if (!u || !v || !out || !valid_dims(du) || !valid_dims(dv))
        return bad(ctx, WLM_INVALID_ARG, "compose_warp: bad args");
    if (!same_dims(du, dv)) return bad(ctx, WLM_DIM_MISMATCH, "compose_warp: dimension mismatch");
    return run(ctx, [&] {
        const size_t n = nvox(du);
        DevBuf<double> a = upload64(ctx, u, 3 * n), b = upload64(ctx, v, 3 * n), o(ctx, 3 * n);
        launch_compose64(a.p, b.p, eps, du, o.p, ctx->stream);
        download64(ctx, o.p, 3 * n, out);
    });
}

wlm_status wlm_max_abs_component(wlm_ctx* ctx, const double* v, wlm_dims d, double* out) {
    if (!v || !out || !valid_dims(d)) return bad(ctx, WLM_INVALID_ARG, "max_abs_component: bad args");
    return run(ctx, [&] {
        const size_t n = nvox(d);
        DevBuf<double> a = upload64(ctx, v, 3 * n);
        *out = read_max64(ctx, a.p, (long long)(3 * n));
    });
}

// normalize_step (field.cpp:150-155): target outside (0, 0.5) -> INVALID_ARG.
wlm_status wlm_normalize_step(wlm_ctx* ctx, const double* v, wlm_dims d, double target, double floor_,
                              double* eps) {
    if (!(target > 0.0 && target < 0.5))
        return bad(ctx, WLM_INVALID_ARG, "normalize_step: target_max_disp must lie in (0, 0.5)");
    double m = 0.0;
    wlm_status s = wlm_max_abs_component(ctx, v, d, &m);
    if (s != WLM_OK) return s;
    *eps = target / std::max(m, floor_);
    return WLM_OK;
}

wlm_status wlm_jacobian_det_min(wlm_ctx* ctx, const double* u, wlm_dims d, double* out) {
    if (!u || !out || !valid_dims(d)) return bad(ctx, WLM_INVALID_ARG, "jacobian_det_min: bad args");
    if (d.nx < 2 || d.ny < 2 || d.nz < 2)
        return bad(ctx, WLM_INVALID_ARG, "jacobian_det_min: dims must be >= 2 per axis");
    return run(ctx, [&] {
        DevBuf<double> a = upload64(ctx, u, 3 * nvox(d));
        *out = read_jacdet64(ctx, a.p, d);
    });
}

static wlm_status smooth_common(wlm_ctx* ctx, const double* in, wlm_dims d, double sigma, double* out,
                                int nchan) {
    if (!in || !out || !valid_dims(d)) return bad(ctx, WLM_INVALID_ARG, "gaussian_smooth: bad args");
    return run(ctx, [&] {
        const size_t n = nvox(d) * nchan;
        DevBuf<double> a = upload64(ctx, in, n);
        smooth_aos64(ctx, a.p, d, nchan, sigma);  // any sigma (radius ceil(3 sigma), field.cpp:206)
        download64(ctx, a.p, n, out);
    });
}

wlm_status wlm_gaussian_smooth_vol(wlm_ctx* ctx, const double* in, wlm_dims d, double sigma, double* out) {
    return smooth_common(ctx, in, d, sigma, out, 1);
}
wlm_status wlm_gaussian_smooth_field(wlm_ctx* ctx, const double* in, wlm_dims d, double sigma, double* out) {
    return smooth_common(ctx, in, d, sigma, out, 3);
}

namespace {
__global__ void k_nonfinite_d(const double* v, long long n, int* flag) {
    int bad_ = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        bad_ |= !isfinite(v[i]);
    bad_ = __syncthreads_or(bad_);
    if (threadIdx.x == 0 && bad_) atomicOr(flag, 1);
}
}  // namespace

wlm_status wlm_all_finite(wlm_ctx* ctx, const double* data, size_t count, int* out) {
    if (!data || !out) return bad(ctx, WLM_INVALID_ARG, "all_finite: bad args");
    return run(ctx, [&] {
        DevBuf<double> a(ctx, count);
        DevBuf<int> f(ctx, 1);
        CK(cudaMemcpyAsync(a.p, data, sizeof(double) * count, cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaMemsetAsync(f.p, 0, sizeof(int), ctx->stream));
        const long long blocks = std::min<long long>(148 * 16, std::max<long long>(1, ((long long)count + 255) / 256));
        k_nonfinite_d<<<(int)blocks, 256, 0, ctx->stream>>>(a.p, (long long)count, f.p);
        ++g_kernel_launches;
        int h = 0;
        CK(cudaMemcpyAsync(&h, f.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        *out = h ? 0 : 1;
    });
}

// residual_lncc: the engine's own K1/K2 kernels on a one-pair
// batch, so this entry point exercises exactly the hot-path code.
wlm_status wlm_residual_lncc(wlm_ctx* ctx, const double* F, const double* M, const double* u, wlm_dims d,
                             int radius, double* r, double* lncc, double* g) {
    if (!F || !M || !u || !valid_dims(d)) return bad(ctx, WLM_INVALID_ARG, "residual_lncc: bad args");
    wlm_reg_config cfg;
    wlm_default_reg_config(&cfg);
    cfg.lncc_radius = radius;
    cfg.nlevels = 1; cfg.factors[0] = 1; cfg.iters[0] = 0;
    wlm_engine* e = nullptr;
    wlm_status s = wlm_engine_create(ctx, d, 1, &cfg, &e);
    if (s != WLM_OK) return s;
    s = run(ctx, [&] {
        const size_t n = nvox(d);
        std::vector<float> hf(n), hm(n);
        for (size_t i = 0; i < n; ++i) { hf[i] = (float)F[i]; hm[i] = (float)M[i]; }
        CK(cudaMemcpyAsync(e->F.p, hf.data(), sizeof(float) * n, cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaMemcpyAsync(e->M.p, hm.data(), sizeof(float) * n, cudaMemcpyHostToDevice, ctx->stream));
        launch_shifts(e->B, ctx->stream);
        DevBuf<float> du = upload_soa(ctx, u, n, 3);
        copy_warps_in(e, du.p, 0);
        launch_begin_level(e->B, e->P, 0, 1, cfg.lm.lambda0, ctx->stream);
        e->stage_eval(0, ctx->stream);
        e->stage_finalize(0, ctx->stream);
        if (g) {
            launch_lncc_bwd(e->B, e->P, ctx->stream);
            download_aos(ctx, e->G.p, n, 3, g);
        }
        const std::vector<PairState> st = read_states(e);
        if (r) *r = st[0].r_cur;
        if (lncc) *lncc = st[0].lncc_cur;
        if (st[0].status) throw Fail{(wlm_status)st[0].status};
    });
    wlm_engine_destroy(e);
    return s;
}

wlm_status wlm_residual_mi(wlm_ctx* ctx, const double* F, const double* M, const double* u, wlm_dims d, int bins,
                           double sigma, double* r, double* mi, double* g) {
    if (!F || !M || !u || !valid_dims(d)) return bad(ctx, WLM_INVALID_ARG, "residual_mi: bad args");
    wlm_reg_config cfg;
    wlm_default_reg_config(&cfg);
    cfg.metric = WLM_METRIC_MI;
    cfg.mi_bins = bins;
    cfg.mi_sigma = sigma;
    cfg.nlevels = 1; cfg.factors[0] = 1; cfg.iters[0] = 0;
    wlm_engine* e = nullptr;
    wlm_status s = wlm_engine_create(ctx, d, 1, &cfg, &e);
    if (s != WLM_OK) return s;
    s = run(ctx, [&] {
        const size_t n = nvox(d);
        std::vector<float> hf(n), hm(n);
        for (size_t i = 0; i < n; ++i) { hf[i] = (float)F[i]; hm[i] = (float)M[i]; }
        CK(cudaMemcpyAsync(e->F.p, hf.data(), sizeof(float) * n, cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaMemcpyAsync(e->M.p, hm.data(), sizeof(float) * n, cudaMemcpyHostToDevice, ctx->stream));
        launch_shifts(e->B, ctx->stream);
        DevBuf<float> du = upload_soa(ctx, u, n, 3);
        copy_warps_in(e, du.p, 0);
        launch_begin_level(e->B, e->P, 0, 1, cfg.lm.lambda0, ctx->stream);
        e->stage_eval(0, ctx->stream);
        e->stage_finalize(0, ctx->stream);
        if (g) {
            launch_mi_grad(e->B, e->P, ctx->stream);
            download_aos(ctx, e->G.p, n, 3, g);
        }
        const std::vector<PairState> st = read_states(e);
        if (r) *r = st[0].r_cur;
        if (mi) *mi = st[0].lncc_cur;
        if (st[0].status) throw Fail{(wlm_status)st[0].status};
    });
    wlm_engine_destroy(e);
    return s;
}

wlm_status wlm_residual_mse(wlm_ctx* ctx, const double* F, const double* M, const double* u, wlm_dims d,
                            double* r, double* g) {
    if (!F || !M || !u || !valid_dims(d)) return bad(ctx, WLM_INVALID_ARG, "residual_mse: bad args");
    wlm_reg_config cfg;
    wlm_default_reg_config(&cfg);
    cfg.metric = WLM_METRIC_MSE;
    cfg.nlevels = 1; cfg.factors[0] = 1; cfg.iters[0] = 0;
    wlm_engine* e = nullptr;
    wlm_status s = wlm_engine_create(ctx, d, 1, &cfg, &e);
    if (s != WLM_OK) return s;
    s = run(ctx, [&] {
        const size_t n = nvox(d);
        std::vector<float> hf(n), hm(n);
        for (size_t i = 0; i < n; ++i) { hf[i] = (float)F[i]; hm[i] = (float)M[i]; }
        CK(cudaMemcpyAsync(e->F.p, hf.data(), sizeof(float) * n, cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaMemcpyAsync(e->M.p, hm.data(), sizeof(float) * n, cudaMemcpyHostToDevice, ctx->stream));
        DevBuf<float> du = upload_soa(ctx, u, n, 3);
        copy_warps_in(e, du.p, 0);
        launch_begin_level(e->B, e->P, 0, 1, cfg.lm.lambda0, ctx->stream);
        e->stage_eval(0, ctx->stream);
        e->stage_finalize(0, ctx->stream);
        if (g) {
            launch_mse_grad(e->B, e->P, ctx->stream);
            download_aos(ctx, e->G.p, n, 3, g);
        }
        const std::vector<PairState> st = read_states(e);
        if (r) *r = st[0].r_cur;
        if (st[0].status) throw Fail{(wlm_status)st[0].status};
    });
    wlm_engine_destroy(e);
    return s;
}

wlm_status wlm_lm_step_tiled(wlm_ctx* ctx, double r, const double* g, wlm_dims d, double lambda, int k,
                             double* out) {
    if (!g || !out || !valid_dims(d) || !(lambda > 0.0) || k < 1)
        return bad(ctx, WLM_INVALID_ARG, "lm_step_tiled: bad args (lambda > 0, k >= 1)");
    return run(ctx, [&] {
        const size_t N = nvox(d);
        DevBuf<double> dg(ctx, 3 * N), dout(ctx, 3 * N);
        CK(cudaMemcpyAsync(dg.p, g, sizeof(double) * 3 * N, cudaMemcpyHostToDevice, ctx->stream));
        launch_lm_tiled_fp64(r, dg.p, make_geo(d), lambda, k, nullptr, dout.p, ctx->stream);
        CK(cudaMemcpyAsync(out, dout.p, sizeof(double) * 3 * N, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    });
}

wlm_status wlm_demons_step_mse(wlm_ctx* ctx, const double* r, const double* n, wlm_dims d, double alpha,
                               double* out) {
    if (!r || !n || !out || !valid_dims(d) || !(alpha > 0.0))
        return bad(ctx, WLM_INVALID_ARG, "demons_step_mse: bad args (alpha > 0, SPEC.md:243)");
    return run(ctx, [&] {
        const size_t N = nvox(d);
        DevBuf<double> dr(ctx, N), dn(ctx, 3 * N), dout(ctx, 3 * N);
        CK(cudaMemcpyAsync(dr.p, r, sizeof(double) * N, cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaMemcpyAsync(dn.p, n, sizeof(double) * 3 * N, cudaMemcpyHostToDevice, ctx->stream));
        launch_demons_pointwise(dr.p, dn.p, (long long)N, alpha, dout.p, ctx->stream);
        CK(cudaMemcpyAsync(out, dout.p, sizeof(double) * 3 * N, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    });
}

wlm_status wlm_lm_step_pointwise(wlm_ctx* ctx, double r, const double* g, wlm_dims d, double lambda,
                                 double* out) {
    if (!g || !out || !valid_dims(d) || !(lambda > 0.0))
        return bad(ctx, WLM_INVALID_ARG, "lm_step_pointwise: bad args (lambda > 0)");
    return run(ctx, [&] {
        const size_t n = nvox(d);
        DevBuf<double> a = upload64(ctx, g, 3 * n), o(ctx, 3 * n);
        launch_lm_step64(r, a.p, (long long)n, lambda, o.p, ctx->stream);
        download64(ctx, o.p, 3 * n, out);
    });
}

// Scalar state updates: the same fp64 arithmetic the
// device state machine runs inside the evaluation kernel.
void wlm_update_damping(wlm_lm_state* s, double loss_new, const wlm_lm_config* c) {
    const bool badstep = s->hist_n == 0 || loss_new > s->L1;
    double lam = badstep ? c->mu_plus * s->lambda : c->mu_minus * s->lambda;
    if (c->lambda_max > 0.0 && std::isfinite(c->lambda_max)) lam = std::min(lam, c->lambda_max);
    s->lambda = std::max(lam, 1e-12);
    s->L2 = s->L1;
    s->L1 = loss_new;
    s->hist_n = std::min(s->hist_n + 1, 2);
}

int wlm_rejection_test(double loss_new, double L1, double L2, double tau) {
    return (loss_new - L1) > tau * std::fabs(L1 - L2) ? 1 : 0;
}

static wlm_dims level_dims(wlm_dims d, int f) {
    return wlm_dims{(d.nx + f - 1) / f, (d.ny + f - 1) / f, (d.nz + f - 1) / f};
}

// downsample: Gaussian sigma = 0.5 f, then stride f.
wlm_status wlm_downsample(wlm_ctx* ctx, const double* vol, wlm_dims d, int factor, double* out,
                          wlm_dims* out_dims) {
    if (!vol || !out || !valid_dims(d)) return bad(ctx, WLM_INVALID_ARG, "downsample: bad args");
    if (factor < 1) return bad(ctx, WLM_INVALID_ARG, "downsample: factor < 1");
    const wlm_dims nd = level_dims(d, factor);
    if (out_dims) *out_dims = nd;
    return run(ctx, [&] {
        const size_t n = nvox(d);
        DevBuf<double> a = upload64(ctx, vol, n);
        if (factor == 1) { download64(ctx, a.p, n, out); return; }
        smooth_aos64(ctx, a.p, d, 1, 0.5 * factor);  // Gaussian sigma = 0.5 f
        DevBuf<double> o(ctx, nvox(nd));
        launch_stride64(a.p, d, factor, o.p, nd, ctx->stream);
        download64(ctx, o.p, nvox(nd), out);
    });
}

// upsample_warp: trilinear at x / scale, values * scale.
wlm_status wlm_upsample_warp(wlm_ctx* ctx, const double* u, wlm_dims d, wlm_dims nd, double scale,
                             double* out) {
    if (!u || !out || !valid_dims(d) || !valid_dims(nd) || !(scale > 0.0))
        return bad(ctx, WLM_INVALID_ARG, "upsample_warp: invalid dims");
    return run(ctx, [&] {
        DevBuf<double> a = upload64(ctx, u, 3 * nvox(d)), o(ctx, 3 * nvox(nd));
        launch_upsample64(a.p, d, nd, scale, o.p, ctx->stream);
        download64(ctx, o.p, 3 * nvox(nd), out);
    });
}

size_t wlm_state_bytes(int optimizer, wlm_dims d, int elem_bytes) {
    if (optimizer == WLM_OPT_ADAM) return 2 * 3 * nvox(d) * (size_t)elem_bytes;  // m, v fields
    if (optimizer == WLM_OPT_LM) return sizeof(wlm_lm_state) + sizeof(wlm_lm_config);
    return 0;
}

// register: coarse -> fine on the device.  Level
// images are Gaussian-downsampled from the full-resolution device copies, the
// warp is inherited with upsample_warp, lambda carries over, the loss history
// resets.  Within a level the iterations run as CUDA graphs with no host
// synchronisation; the trace is read back once per level.
wlm_status wlm_register(wlm_ctx* ctx, const float* F, const float* M, wlm_dims d, const wlm_reg_config* cfg,
                        double* warp_out, wlm_step_log* trace, size_t cap, size_t* len, double* jac_final) {
    if (!F || !M || !cfg || !warp_out || !valid_dims(d)) return bad(ctx, WLM_INVALID_ARG, "register: bad args");
    if (cfg->nlevels < 1 || cfg->nlevels > WLM_MAX_LEVELS || cfg->factors[cfg->nlevels - 1] != 1)
        return bad(ctx, WLM_INVALID_ARG, "register: schedule must end at factor 1");
    for (int l = 0; l < cfg->nlevels; ++l) {
        if (cfg->factors[l] < 1 || cfg->iters[l] < 0 || (l > 0 && cfg->factors[l] >= cfg->factors[l - 1]))
            return bad(ctx, WLM_INVALID_ARG, "register: factors must strictly decrease to 1");
        if (cfg->factors[l] > 42) return bad(ctx, WLM_UNSUPPORTED, "register: factor > 42");
    }
    if (len) *len = 0;
    ctx->peak_bytes = ctx->cur_bytes;
    size_t used = 0;
    wlm_status result = WLM_OK;
    wlm_status s = run(ctx, [&] {
        const size_t n = nvox(d);
        const Geo g0 = make_geo(d);
        DevBuf<float> F0(ctx, n), M0(ctx, n);
        CK(cudaMemcpyAsync(F0.p, F, sizeof(float) * n, cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaMemcpyAsync(M0.p, M, sizeof(float) * n, cudaMemcpyHostToDevice, ctx->stream));
        wlm_engine* prev = nullptr;
        for (int l = 0; l < cfg->nlevels; ++l) {
            const int f = cfg->factors[l];
            const wlm_dims ld = level_dims(d, f);
            wlm_engine* e = nullptr;
            wlm_status es = wlm_engine_create(ctx, ld, 1, cfg, &e);
            if (es != WLM_OK) { if (prev) wlm_engine_destroy(prev); throw Fail{es}; }
            if (f == 1) {
                CK(cudaMemcpyAsync(e->F.p, F0.p, sizeof(float) * n, cudaMemcpyDeviceToDevice, ctx->stream));
                CK(cudaMemcpyAsync(e->M.p, M0.p, sizeof(float) * n, cudaMemcpyDeviceToDevice, ctx->stream));
            } else {
                launch_downsample_gauss(F0.p, g0, f, e->F.p, e->g, ctx->stream);
                launch_downsample_gauss(M0.p, g0, f, e->M.p, e->g, ctx->stream);
            }
            launch_shifts(e->B, ctx->stream);
            if (prev) {
                const std::vector<PairState> ps = read_states(prev);
                const float* up = prev->U.p + (size_t)ps[0].cur * 3 * (size_t)prev->g.n;
                launch_upsample(up, prev->g, e->g, (float)cfg->factors[l - 1] / (float)f, e->U.p, ctx->stream);
                // carry lambda: copy the whole state, then reset history
                CK(cudaMemcpyAsync(e->st.p, prev->st.p, sizeof(PairState), cudaMemcpyDeviceToDevice, ctx->stream));
                CK(cudaStreamSynchronize(ctx->stream));
                wlm_engine_destroy(prev);
                prev = nullptr;
                // the upsampled warp is in buffer 0
                PairState hs = ps[0];
                hs.cur = 0;
                CK(cudaMemcpyAsync(e->st.p, &hs, sizeof(PairState), cudaMemcpyHostToDevice, ctx->stream));
                launch_shifts(e->B, ctx->stream);
                launch_begin_level(e->B, e->P, l, 0, cfg->lm.lambda0, ctx->stream);
            } else {
                launch_begin_level(e->B, e->P, l, 1, cfg->lm.lambda0, ctx->stream);
            }
            e->stage_eval(0, ctx->stream);
            e->stage_finalize(0, ctx->stream);
            const uint64_t before = g_kernel_launches;
            es = wlm_engine_iterate(e, cfg->iters[l]);
            (void)before;
            if (es != WLM_OK) { wlm_engine_destroy(e); throw Fail{es}; }
            const std::vector<PairState> ps = read_states(e);
            const size_t rows = std::min((size_t)ps[0].trace_len, cap > used ? cap - used : 0);
            if (rows && trace)
                CK(cudaMemcpy(trace + used, e->trace.p, sizeof(wlm_step_log) * rows, cudaMemcpyDeviceToHost));
            used += rows;
            if (len) *len = used;
            if (ps[0].status != 0) {
                result = (wlm_status)ps[0].status;
                set_err(ctx, "register: non-finite loss, aborted with partial trace (SPEC.md:366)");
                wlm_engine_destroy(e);
                return;
            }
            prev = e;
        }
        const std::vector<PairState> ps = read_states(prev);
        const float* uf = prev->U.p + (size_t)ps[0].cur * 3 * n;
        download_aos(ctx, uf, n, 3, warp_out);
        if (jac_final) {
            if (d.nx >= 2 && d.ny >= 2 && d.nz >= 2) {
                // the reference's fp64 jacobian_det_min of the (fp32) final warp
                *jac_final = read_jacdet64(ctx, nullptr, d, uf);
            } else {
                *jac_final = std::numeric_limits<double>::quiet_NaN();
            }
        }
        wlm_engine_destroy(prev);
    });
    if (s != WLM_OK) return s;
    return result;
}

}  // extern "C"
