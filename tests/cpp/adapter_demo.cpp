// adapter_demo.cpp -- a reference-style caller of the B200 path through the
// C++ adapter (include/wlm_warplm.hpp).  The two structs below have the
// reference's shapes (proj/include/warplm/field.hpp:18-70, minimal subset) so
// this compiles without /root/reference; with the reference headers on the
// include path, `warplm::Volume3` / `warplm::DispField3` drop in unchanged.
//
// Build: g++ -std=c++17 -I include tests/cpp/adapter_demo.cpp \
//            -L paper_2603_19371_b200 -lwarplm_b200 -Wl,-rpath,...
#include <cmath>
#include <cstdio>
#include <vector>

#include "wlm_warplm.hpp"

namespace ref_shape {
struct Dims3 {
    int nx = 0, ny = 0, nz = 0;
    std::size_t voxels() const { return (std::size_t)nx * ny * nz; }
};
struct Volume3 {
    Dims3 dims;
    std::vector<double> data;
    Volume3() = default;
    explicit Volume3(Dims3 d) : dims(d), data(d.voxels(), 0.0) {}
};
struct DispField3 {
    Dims3 dims;
    std::vector<double> data;
    DispField3() = default;
    explicit DispField3(Dims3 d) : dims(d), data(3 * d.voxels(), 0.0) {}
};
struct StepScale {
    double target_max_disp = 0.4;
    double floor = 1e-12;
};
}  // namespace ref_shape

int main() {
    using namespace ref_shape;
    const Dims3 d{12, 10, 8};
    DispField3 u(d), v(d);
    for (std::size_t i = 0; i < v.data.size(); ++i) v.data[i] = std::sin(0.37 * (double)i);
    // compose_warp(0, v, eps) == eps v
    const DispField3 w = wlm_warplm::compose_warp(u, v, 0.25);
    double err = 0.0;  // the field mirrors return the reference's bits: exact here
    for (std::size_t i = 0; i < w.data.size(); ++i) err = std::fmax(err, std::fabs(w.data[i] - 0.25 * v.data[i]));
    const double eps = wlm_warplm::normalize_step(v, StepScale{});
    bool threw = false;
    try {
        wlm_warplm::compose_warp(u, DispField3(Dims3{12, 10, 9}), 0.1);
    } catch (const std::invalid_argument&) {
        threw = true;  // field.cpp:124-126
    }
    const double jac = wlm_warplm::jacobian_det_min(u);
    // SPEC.md:132-133 (MSE KATs) and :307 (Demons KAT) through the adapter
    Volume3 F(d), M(d);
    for (std::size_t i = 0; i < F.data.size(); ++i) M.data[i] = 1.0;
    const auto mse = wlm_warplm::residual_mse(F, M, u);
    Volume3 r1(Dims3{1, 1, 1});
    r1.data[0] = 1.0;
    DispField3 n1(Dims3{1, 1, 1});
    n1.data[0] = 2.0;
    const DispField3 dm = wlm_warplm::demons_step_mse(r1, n1, 1.0);
    const DispField3 t1 = wlm_warplm::lm_step_tiled(0.5, v, 0.1, 3);
    // point sampling (field.hpp:82-93), LM step, damping / rejection, pyramid
    Volume3 ramp(d);
    for (int z = 0; z < d.nz; ++z)
        for (int y = 0; y < d.ny; ++y)
            for (int x = 0; x < d.nx; ++x) ramp.data[x + d.nx * (y + d.ny * z)] = x;
    const auto sg = wlm_warplm::sample_trilinear_grad(ramp, 3.25, 2.0, 1.5);  // value 3.25, grad (1, 0, 0)
    const auto sf = wlm_warplm::sample_field(v, 0.0, 0.0, 0.0);              // v at voxel 0
    DispField3 g1(Dims3{1, 1, 1});
    g1.data[0] = 1.0;
    const DispField3 st = wlm_warplm::lm_step_pointwise(2.0, g1, 1.0);       // (-1, 0, 0)
    wlm_lm_state ls{0.006, 0, 0.0, 0.0};
    const wlm_reg_config cfg = wlm_warplm::default_reg_config();
    wlm_warplm::update_damping(ls, 0.9, cfg.lm);                             // no history: lambda * mu+
    const bool rej = wlm_warplm::rejection_test(1.05, 0.9, 1.0, 1.0);        // reject
    const Volume3 half = wlm_warplm::downsample(ramp, 2);
    const DispField3 up = wlm_warplm::upsample_warp(v, Dims3{24, 20, 16}, 2.0);
    const bool ok2 = sg.value == 3.25 && sg.grad[0] == 1.0 && sf[0] == v.data[0] && st.data[0] == -1.0 &&
                     std::fabs(ls.lambda - 0.009) < 1e-15 && rej && half.dims.nx == 6 && half.dims.nz == 4 &&
                     up.data.size() == 3u * 24 * 20 * 16;
    std::printf("compose max err %.3g, eps %.6f, dim-mismatch throws %d, jac(0) %.1f, mse %.1f, demons %.3f\n",
                err, eps, (int)threw, jac, mse.r, dm.data[0]);
    std::printf("point sample %.4f grad %.1f, lm step %.1f, lambda %.4f, reject %d, downsample %dx%dx%d\n",
                sg.value, sg.grad[0], st.data[0], ls.lambda, (int)rej, half.dims.nx, half.dims.ny, half.dims.nz);
    return (err == 0.0 && threw && jac == 1.0 && mse.r == 1.0 && std::fabs(dm.data[0] - 0.4) < 1e-15 &&
            t1.data.size() == v.data.size() && ok2)
               ? 0
               : 1;
}
