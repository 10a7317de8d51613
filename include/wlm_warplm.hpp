// wlm_warplm.hpp -- header-only C++ adapter: the reference `warplm` call
// signatures (value types in, value types out, exceptions on error) on top of
// the C ABI in wlm.h.  A reference caller swaps
//     warplm::compose_warp(u, v, eps)      ->  wlm_warplm::compose_warp(u, v, eps)
// and links libwarplm_b200.so.  The templates accept the reference's own
// value types (proj/include/warplm/field.hpp:18-70): anything with
// `dims.{nx,ny,nz}`, `dims.voxels()`, a `std::vector<double> data` and a
// constructor from dims -- i.e. warplm::Volume3 / warplm::DispField3 -- so no
// reference header is needed to build this adapter.
//
//   reference (field.hpp / SPEC.md)            adapter                      errors
//   compose_warp              field.hpp:96     compose_warp                 invalid_argument (dims)
//   max_abs_component         field.hpp:99     max_abs_component
//   normalize_step            field.hpp:104    normalize_step               invalid_argument (target)
//   jacobian_det_min          field.hpp:108    jacobian_det_min             invalid_argument (dims < 2)
//   gaussian_smooth (vol/fld) field.hpp:113-114 gaussian_smooth
//   all_finite                field.hpp:116-117 all_finite
//   residual_mse              SPEC.md:127      residual_mse -> ResidualReport
//   residual_lncc             SPEC.md:136      residual_lncc -> ResidualReport
//   residual_mi               SPEC.md:145      residual_mi -> ResidualReport
//   lm_step_tiled             SPEC.md:256      lm_step_tiled
//   demons_step_mse           SPEC.md:301      demons_step_mse
//   register                  SPEC.md:362      register_pair -> RegResult   runtime_error (non-finite)
#pragma once

#include <array>
#include <cstddef>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "wlm.h"

namespace wlm_warplm {

// Device failure (no GPU, OOM, CUDA error): there is no CPU fallback.
struct device_error : std::runtime_error {
    wlm_status status;
    device_error(wlm_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};

class Context {
public:
    explicit Context(int device = 0) {
        wlm_ctx* c = nullptr;
        const wlm_status s = wlm_ctx_create(device, &c);
        if (s != WLM_OK) throw device_error(s, "wlm_ctx_create failed (no usable CUDA device)");
        ctx_.reset(c);
    }
    wlm_ctx* get() const { return ctx_.get(); }

private:
    struct Del { void operator()(wlm_ctx* c) const { wlm_ctx_destroy(c); } };
    std::unique_ptr<wlm_ctx, Del> ctx_;
};

inline Context& default_context() {
    static thread_local Context c(0);
    return c;
}

inline void check(wlm_status s, const Context& c) {
    if (s == WLM_OK) return;
    const std::string m = wlm_last_error(c.get());
    if (s == WLM_INVALID_ARG || s == WLM_DIM_MISMATCH) throw std::invalid_argument(m);
    throw device_error(s, m);
}

template <class D>
wlm_dims dims_of(const D& d) {
    return wlm_dims{d.nx, d.ny, d.nz};
}

// sample_trilinear / sample_trilinear_grad (field.hpp:82-90) at one point;
// Vec3 is std::array<double, 3> (field.hpp:10), SampleGrad {value, grad}.
struct SampleGrad {
    double value = 0.0;
    std::array<double, 3> grad{0.0, 0.0, 0.0};
};

template <class Volume>
SampleGrad sample_trilinear_grad(const Volume& vol, double px, double py, double pz,
                                 Context& c = default_context()) {
    const double p[3] = {px, py, pz};
    SampleGrad s;
    check(wlm_sample_trilinear_grad_points(c.get(), vol.data.data(), dims_of(vol.dims), p, 1, &s.value,
                                           s.grad.data()),
          c);
    return s;
}

template <class Volume>
double sample_trilinear(const Volume& vol, double px, double py, double pz, Context& c = default_context()) {
    return sample_trilinear_grad(vol, px, py, pz, c).value;
}

// sample_field (field.hpp:93): the three components at one point.
template <class Field>
std::array<double, 3> sample_field(const Field& u, double px, double py, double pz, Context& c = default_context()) {
    const double p[3] = {px, py, pz};
    std::array<double, 3> out{};
    check(wlm_sample_field_points(c.get(), u.data.data(), dims_of(u.dims), p, 1, out.data()), c);
    return out;
}

template <class Field>
Field compose_warp(const Field& u, const Field& v, double eps, Context& c = default_context()) {
    Field out(u.dims);
    check(wlm_compose_warp(c.get(), u.data.data(), dims_of(u.dims), v.data.data(), dims_of(v.dims), eps,
                           out.data.data()),
          c);
    return out;
}

template <class Field>
double max_abs_component(const Field& v, Context& c = default_context()) {
    double m = 0.0;
    check(wlm_max_abs_component(c.get(), v.data.data(), dims_of(v.dims), &m), c);
    return m;
}

template <class Field, class StepScale>
double normalize_step(const Field& v, const StepScale& s, Context& c = default_context()) {
    double eps = 0.0;
    check(wlm_normalize_step(c.get(), v.data.data(), dims_of(v.dims), s.target_max_disp, s.floor, &eps), c);
    return eps;
}

template <class Field>
double jacobian_det_min(const Field& u, Context& c = default_context()) {
    double m = 0.0;
    check(wlm_jacobian_det_min(c.get(), u.data.data(), dims_of(u.dims), &m), c);
    return m;
}

// Volume3 or DispField3, told apart by the payload size (field.hpp:42, :55).
template <class T>
T gaussian_smooth(const T& a, double sigma, Context& c = default_context()) {
    T out(a.dims);
    if (a.data.size() == a.dims.voxels())
        check(wlm_gaussian_smooth_vol(c.get(), a.data.data(), dims_of(a.dims), sigma, out.data.data()), c);
    else
        check(wlm_gaussian_smooth_field(c.get(), a.data.data(), dims_of(a.dims), sigma, out.data.data()), c);
    return out;
}

template <class T>
bool all_finite(const T& a, Context& c = default_context()) {
    int ok = 0;
    check(wlm_all_finite(c.get(), a.data.data(), a.data.size(), &ok), c);
    return ok != 0;
}

// ResidualReport.
template <class Field>
struct ResidualReport {
    double r = 0.0;
    Field g;
    double loss_raw = 0.0;
};

template <class Volume, class Field>
ResidualReport<Field> residual_lncc(const Volume& F, const Volume& M, const Field& u, int radius = 2,
                                    Context& c = default_context()) {
    ResidualReport<Field> rep;
    rep.g = Field(u.dims);
    check(wlm_residual_lncc(c.get(), F.data.data(), M.data.data(), u.data.data(), dims_of(F.dims), radius,
                            &rep.r, &rep.loss_raw, rep.g.data.data()),
          c);
    return rep;
}

template <class Volume, class Field>
ResidualReport<Field> residual_mse(const Volume& F, const Volume& M, const Field& u,
                                   Context& c = default_context()) {
    ResidualReport<Field> rep;
    rep.g = Field(u.dims);
    check(wlm_residual_mse(c.get(), F.data.data(), M.data.data(), u.data.data(), dims_of(F.dims), &rep.r,
                           rep.g.data.data()),
          c);
    rep.loss_raw = rep.r;
    return rep;
}

// MetricConfig{kind = mi, mi_bins, mi_parzen_sigma}.
template <class Volume, class Field>
ResidualReport<Field> residual_mi(const Volume& F, const Volume& M, const Field& u, int bins = 32,
                                  double sigma = 1.0, Context& c = default_context()) {
    ResidualReport<Field> rep;
    rep.g = Field(u.dims);
    check(wlm_residual_mi(c.get(), F.data.data(), M.data.data(), u.data.data(), dims_of(F.dims), bins, sigma,
                          &rep.r, &rep.loss_raw, rep.g.data.data()),
          c);
    return rep;
}

// lm_step_pointwise: -r g / (|g|^2 + lambda) per voxel.
template <class Field>
Field lm_step_pointwise(double r, const Field& g, double lambda, Context& c = default_context()) {
    Field out(g.dims);
    check(wlm_lm_step_pointwise(c.get(), r, g.data.data(), dims_of(g.dims), lambda, out.data.data()), c);
    return out;
}

// update_damping / rejection_test: host scalar state, the
// arithmetic the device state machine runs.
inline void update_damping(wlm_lm_state& s, double loss_new, const wlm_lm_config& cfg) {
    wlm_update_damping(&s, loss_new, &cfg);
}
inline bool rejection_test(double loss_new, double loss_prev, double loss_prev2, double tau) {
    return wlm_rejection_test(loss_new, loss_prev, loss_prev2, tau) != 0;
}

// downsample: Gaussian sigma 0.5 f, stride f, dims ceil(n / f).
template <class Volume>
Volume downsample(const Volume& vol, int factor, Context& c = default_context()) {
    wlm_dims nd{};
    const int f = factor < 1 ? 1 : factor;
    std::vector<double> tmp(((std::size_t)(vol.dims.nx + f - 1) / f) * ((vol.dims.ny + f - 1) / f) *
                            ((vol.dims.nz + f - 1) / f));
    check(wlm_downsample(c.get(), vol.data.data(), dims_of(vol.dims), factor, tmp.data(), &nd), c);
    decltype(vol.dims) od = vol.dims;
    od.nx = nd.nx;
    od.ny = nd.ny;
    od.nz = nd.nz;
    Volume out(od);
    out.data = std::move(tmp);
    return out;
}

// upsample_warp: trilinear at x / scale, values * scale.
template <class Field, class Dims>
Field upsample_warp(const Field& u, const Dims& new_dims, double scale, Context& c = default_context()) {
    Field out(new_dims);
    check(wlm_upsample_warp(c.get(), u.data.data(), dims_of(u.dims), dims_of(new_dims), scale, out.data.data()), c);
    return out;
}

template <class Field>
Field lm_step_tiled(double r, const Field& g, double lambda, int k, Context& c = default_context()) {
    Field out(g.dims);
    check(wlm_lm_step_tiled(c.get(), r, g.data.data(), dims_of(g.dims), lambda, k, out.data.data()), c);
    return out;
}

template <class Volume, class Field>
Field demons_step_mse(const Volume& per_voxel_r, const Field& moving_grad, double alpha,
                      Context& c = default_context()) {
    Field out(moving_grad.dims);
    check(wlm_demons_step_mse(c.get(), per_voxel_r.data.data(), moving_grad.data.data(),
                              dims_of(moving_grad.dims), alpha, out.data.data()),
          c);
    return out;
}

// RegResult.
template <class Field>
struct RegResult {
    Field final_warp;
    std::vector<wlm_step_log> loss_trace;
    double jac_det_min_final = 0.0;
};

// register(fixed, moving, RegConfig).  `register` is a C++
// keyword, hence register_pair.  Level images are fp32 (the VOL3 payload).
template <class Volume, class Field>
RegResult<Field> register_pair(const Volume& F, const Volume& M, const wlm_reg_config& cfg,
                               Context& c = default_context()) {
    const std::size_t n = F.data.size();
    std::vector<float> f(n), m(n);
    for (std::size_t i = 0; i < n; ++i) {
        f[i] = (float)F.data[i];
        m[i] = (float)M.data[i];
    }
    RegResult<Field> res;
    res.final_warp = Field(F.dims);
    std::size_t cap = 1, len = 0;
    for (int l = 0; l < cfg.nlevels; ++l) cap += (std::size_t)cfg.iters[l];
    res.loss_trace.resize(cap);
    const wlm_status s = wlm_register(c.get(), f.data(), m.data(), dims_of(F.dims), &cfg,
                                      res.final_warp.data.data(), res.loss_trace.data(), cap, &len,
                                      &res.jac_det_min_final);
    res.loss_trace.resize(len);
    if (s == WLM_NONFINITE) throw std::runtime_error("register: non-finite loss (SPEC.md:366)");
    check(s, c);
    return res;
}

inline wlm_reg_config default_reg_config() {
    wlm_reg_config c;
    wlm_default_reg_config(&c);
    return c;
}

}  // namespace wlm_warplm
