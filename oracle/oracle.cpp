// oracle.cpp -- TEST INFRASTRUCTURE ONLY (see oracle.h header comment).
//
// fp64 restatement of the reference path.  Build variants (oracle/Makefile):
//   liboracle.so           : everything restated here (self-contained; travels
//                            to the GPU box, no /root/reference needed)
//   _ref/liboracle_ref.so  : compiled with -DORC_WITH_REF_FIELD and linked with
//                            the reference's own proj/src/field.cpp, so every
//                            field primitive (sampling, compose, normalize,
//                            Jacobian, Gaussian smoothing) is the reference's
//                            code; only the spec-only modules are restated.
//                            This is the "reference" CPU arm of bench.py.
#include "oracle.h"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <limits>
#include <vector>

#include <thread>

#ifdef ORC_WITH_REF_FIELD
#include "warplm/field.hpp"
#endif

namespace {

using Vec = std::vector<double>;
constexpr double kNaN = std::numeric_limits<double>::quiet_NaN();

int g_threads = 1;
// Storage-precision emulation: when set, every
// quantity the device stores in fp32 (window coefficients A and B, gradient
// g, smoothed step dU_s, warps, upsampled warps, Adam moments) is rounded to
// fp32 at the same point of the computation; all arithmetic stays fp64.
int g_fp32_storage = 0;  // 0 fp64, 1 fp32 storage points, 2 + device fp32 arithmetic
int g_dev_k3norm64 = 0;
int g_dev_flags = 3;  // mode 2: bit0 K3 step+smooth fp32, bit1 K4 smooth fp32, bit2 compose fp32
inline double r32(double v) { return g_fp32_storage ? (double)(float)v : v; }

// Static-partition parallel loop over [lo, hi) on g_threads std::threads.
// Each index is computed independently, so results do not depend on the
// thread count (reductions are done per index range, then combined in a
// fixed order by the caller).
template <class Fn>
void par_for(long long lo, long long hi, Fn fn) {
    const long long n = hi - lo;
    const int T = (int)std::min<long long>(g_threads, n);
    if (T <= 1) {
        for (long long i = lo; i < hi; ++i) fn(i);
        return;
    }
    std::vector<std::thread> th;
    th.reserve(T);
    for (int t = 0; t < T; ++t) {
        const long long a = lo + n * t / T, b = lo + n * (t + 1) / T;
        th.emplace_back([=] { for (long long i = a; i < b; ++i) fn(i); });
    }
    for (auto& x : th) x.join();
}

inline size_t nvox(orc_dims d) { return (size_t)d.nx * (size_t)d.ny * (size_t)d.nz; }
inline size_t lin(orc_dims d, int x, int y, int z) {
    return (size_t)x + (size_t)d.nx * ((size_t)y + (size_t)d.ny * (size_t)z);
}
inline bool same(orc_dims a, orc_dims b) { return a.nx == b.nx && a.ny == b.ny && a.nz == b.nz; }

// ---------------------------------------------------------------------------
// Axis resolution for clamp-to-edge trilinear sampling (field.cpp:19-39).
// n == 1: degenerate axis, both taps index 0, weight 0, flagged clamped.
// Positions strictly outside [0, n-1] are clamped and flagged; exactly on the
// border they are not flagged.  The cell is [floor(c), floor(c)+1] with the
// last cell reused at c == n-1 (so the gradient there is the backward one).
struct Tap { int lo, hi; double w; bool outside; };

inline Tap resolve(double p, int n) {
    Tap a{0, 0, 0.0, false};
    if (n == 1) { a.outside = true; return a; }
    const double top = (double)(n - 1);
    double c = p;
    if (c <= 0.0) { a.outside = c < 0.0; c = 0.0; }
    else if (c >= top) { a.outside = c > top; c = top; }
    int lo = (int)c;
    if (lo > n - 2) lo = n - 2;
    a.lo = lo; a.hi = lo + 1; a.w = c - (double)lo;
    return a;
}

// Value + analytic gradient of the trilinear interpolant (field.cpp:47-90).
// The x-differences are formed first and collapsed y then z, matching the
// reference's rounding order so the two agree bit-for-bit.
double sample_grad(const double* vol, orc_dims d, double px, double py, double pz,
                   double* grad) {
    if (!std::isfinite(px) || !std::isfinite(py) || !std::isfinite(pz)) {
        if (grad) grad[0] = grad[1] = grad[2] = 0.0;
        return kNaN;
    }
    const Tap X = resolve(px, d.nx), Y = resolve(py, d.ny), Z = resolve(pz, d.nz);
    auto at = [&](int x, int y, int z) { return vol[lin(d, x, y, z)]; };
    const double a = at(X.lo, Y.lo, Z.lo), b = at(X.hi, Y.lo, Z.lo);
    const double c = at(X.lo, Y.hi, Z.lo), e = at(X.hi, Y.hi, Z.lo);
    const double f = at(X.lo, Y.lo, Z.hi), h = at(X.hi, Y.lo, Z.hi);
    const double k = at(X.lo, Y.hi, Z.hi), l = at(X.hi, Y.hi, Z.hi);
    const double dx_00 = b - a, dx_10 = e - c, dx_01 = h - f, dx_11 = l - k;
    const double r00 = a + X.w * dx_00, r10 = c + X.w * dx_10;
    const double r01 = f + X.w * dx_01, r11 = k + X.w * dx_11;
    const double s0 = r00 + Y.w * (r10 - r00), s1 = r01 + Y.w * (r11 - r01);
    const double val = s0 + Z.w * (s1 - s0);
    if (grad) {
        const double gx0 = dx_00 + Y.w * (dx_10 - dx_00);
        const double gx1 = dx_01 + Y.w * (dx_11 - dx_01);
        grad[0] = X.outside ? 0.0 : gx0 + Z.w * (gx1 - gx0);
        const double gy0 = r10 - r00, gy1 = r11 - r01;
        grad[1] = Y.outside ? 0.0 : gy0 + Z.w * (gy1 - gy0);
        grad[2] = Z.outside ? 0.0 : s1 - s0;
    }
    return val;
}

// Three-component sample of an AoS field (field.cpp:92-121).
void sample3(const double* u, orc_dims d, double px, double py, double pz, double* out) {
    if (!std::isfinite(px) || !std::isfinite(py) || !std::isfinite(pz)) {
        out[0] = out[1] = out[2] = kNaN;
        return;
    }
    const Tap X = resolve(px, d.nx), Y = resolve(py, d.ny), Z = resolve(pz, d.nz);
    for (int ch = 0; ch < 3; ++ch) {
        auto at = [&](int x, int y, int z) { return u[3 * lin(d, x, y, z) + ch]; };
        const double a = at(X.lo, Y.lo, Z.lo), b = at(X.hi, Y.lo, Z.lo);
        const double c = at(X.lo, Y.hi, Z.lo), e = at(X.hi, Y.hi, Z.lo);
        const double f = at(X.lo, Y.lo, Z.hi), h = at(X.hi, Y.lo, Z.hi);
        const double k = at(X.lo, Y.hi, Z.hi), l = at(X.hi, Y.hi, Z.hi);
        const double r00 = a + X.w * (b - a), r10 = c + X.w * (e - c);
        const double r01 = f + X.w * (h - f), r11 = k + X.w * (l - k);
        const double s0 = r00 + Y.w * (r10 - r00), s1 = r01 + Y.w * (r11 - r01);
        out[ch] = s0 + Z.w * (s1 - s0);
    }
}

#ifdef ORC_WITH_REF_FIELD
// Adapters: move buffers into the reference's value types and back.
warplm::Dims3 rdims(orc_dims d) { warplm::Dims3 r; r.nx = d.nx; r.ny = d.ny; r.nz = d.nz; return r; }
warplm::DispField3 as_field(const double* p, orc_dims d) {
    warplm::DispField3 f(rdims(d));
    std::memcpy(f.data.data(), p, sizeof(double) * 3 * nvox(d));
    return f;
}
warplm::Volume3 as_vol(const double* p, orc_dims d) {
    warplm::Volume3 v(rdims(d));
    std::memcpy(v.data.data(), p, sizeof(double) * nvox(d));
    return v;
}
#endif

// Compositive update u'(x) = eps v(x) + u(x + eps v(x)) (field.cpp:123-142).
void compose(const double* u, const double* v, orc_dims d, double eps, double* out) {
#ifdef ORC_WITH_REF_FIELD
    const warplm::DispField3 r = warplm::compose_warp(as_field(u, d), as_field(v, d), eps);
    std::memcpy(out, r.data.data(), sizeof(double) * 3 * nvox(d));
#else
    par_for(0, d.nz, [&](long long zz) {
        const int z = (int)zz;
        for (int y = 0; y < d.ny; ++y)
            for (int x = 0; x < d.nx; ++x) {
                const size_t i = 3 * lin(d, x, y, z);
                const double sx = eps * v[i], sy = eps * v[i + 1], sz = eps * v[i + 2];
                double s[3];
                sample3(u, d, x + sx, y + sy, z + sz, s);
                out[i] = sx + s[0];
                out[i + 1] = sy + s[1];
                out[i + 2] = sz + s[2];
            }
    });
#endif
}

double max_abs(const double* v, size_t count) {
    double m = 0.0;
    for (size_t i = 0; i < count; ++i) m = std::max(m, std::fabs(v[i]));
    return m;
}

// det(I + grad u) minimum over the interior, central differences
// (field.cpp:157-201).  One-sided differences only where an axis has n == 2.
double jac_min(const double* u, orc_dims d) {
    if (d.nx < 2 || d.ny < 2 || d.nz < 2) return kNaN;
#ifdef ORC_WITH_REF_FIELD
    return warplm::jacobian_det_min(as_field(u, d));
#else
    const int n[3] = {d.nx, d.ny, d.nz};
    int lo[3], hi[3];
    for (int a = 0; a < 3; ++a) {
        lo[a] = n[a] >= 3 ? 1 : 0;
        hi[a] = n[a] >= 3 ? n[a] - 2 : n[a] - 1;
    }
    std::vector<double> plane_min(d.nz, std::numeric_limits<double>::infinity());
    par_for(lo[2], hi[2] + 1, [&](long long zz) {
        const int z = (int)zz;
        double best = std::numeric_limits<double>::infinity();
        for (int y = lo[1]; y <= hi[1]; ++y)
            for (int x = lo[0]; x <= hi[0]; ++x) {
                const int p[3] = {x, y, z};
                double J[3][3];
                for (int a = 0; a < 3; ++a) {
                    int q1[3] = {x, y, z}, q0[3] = {x, y, z};
                    double scale;
                    if (p[a] >= 1 && p[a] + 1 <= n[a] - 1) { q1[a] = p[a] + 1; q0[a] = p[a] - 1; scale = 0.5; }
                    else if (p[a] == 0) { q1[a] = 1; q0[a] = 0; scale = 1.0; }
                    else { q1[a] = p[a]; q0[a] = p[a] - 1; scale = 1.0; }
                    const size_t i1 = 3 * lin(d, q1[0], q1[1], q1[2]);
                    const size_t i0 = 3 * lin(d, q0[0], q0[1], q0[2]);
                    for (int c = 0; c < 3; ++c) {
                        const double diff = u[i1 + c] - u[i0 + c];
                        J[c][a] = scale == 0.5 ? 0.5 * diff : diff;
                    }
                }
                for (int c = 0; c < 3; ++c) J[c][c] += 1.0;
                const double det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
                                   J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
                                   J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
                best = std::min(best, det);
            }
        plane_min[z] = best;
    });
    double best = std::numeric_limits<double>::infinity();
    for (double v : plane_min) best = std::min(best, v);
    return best;
#endif
}

// Separable Gaussian, radius max(1, ceil(3 sigma)), per-output renormalisation
// over in-bounds taps, axes x, y, z in turn (field.cpp:205-269).
void smooth(double* data, orc_dims d, int nchan, double sigma) {
    if (!(sigma > 0.0)) return;
#ifdef ORC_WITH_REF_FIELD
    if (nchan == 1) {
        const warplm::Volume3 r = warplm::gaussian_smooth(as_vol(data, d), sigma);
        std::memcpy(data, r.data.data(), sizeof(double) * nvox(d));
    } else {
        const warplm::DispField3 r = warplm::gaussian_smooth(as_field(data, d), sigma);
        std::memcpy(data, r.data.data(), sizeof(double) * 3 * nvox(d));
    }
    return;
#else
    int R = (int)std::ceil(3.0 * sigma);
    if (R < 1) R = 1;
    std::vector<double> w(2 * R + 1);
    for (int i = -R; i <= R; ++i) w[i + R] = std::exp(-0.5 * (double)(i * i) / (sigma * sigma));
    const int n3[3] = {d.nx, d.ny, d.nz};
    for (int axis = 0; axis < 3; ++axis) {
        const int n = n3[axis];
        if (n == 1) continue;
        const int na = axis == 0 ? d.ny : d.nx;
        const int nb = axis == 2 ? d.ny : d.nz;
        const size_t stride = axis == 0 ? 1 : axis == 1 ? (size_t)d.nx : (size_t)d.nx * d.ny;
        par_for(0, (long long)nb * na, [&](long long ab) {
            std::vector<double> line(n);
            {
                const int b = (int)(ab / na), a = (int)(ab % na);
                {
                    size_t base;
                    if (axis == 0) base = lin(d, 0, a, b);
                    else if (axis == 1) base = lin(d, a, 0, b);
                    else base = lin(d, a, b, 0);
                    for (int c = 0; c < nchan; ++c) {
                        for (int p = 0; p < n; ++p) line[p] = data[(size_t)nchan * (base + p * stride) + c];
                        for (int p = 0; p < n; ++p) {
                            const int q0 = std::max(0, p - R), q1 = std::min(n - 1, p + R);
                            double num = 0.0, den = 0.0;
                            for (int q = q0; q <= q1; ++q) {
                                num += w[q - p + R] * line[q];
                                den += w[q - p + R];
                            }
                            data[(size_t)nchan * (base + p * stride) + c] = num / den;
                        }
                    }
                }
            }
        });
    }
#endif
}

// ---- device-arithmetic emulation (fp32-storage mode 2) ----
// The engine's K3/K4 step and Gaussian passes run in fp32 (DESIGN.md
// "Precision"); mode 2 reproduces their exact operation order so the
// fp32-storage bar stays a tight check of the device algorithm:
//   weights w[|d|] = (float)exp(-d^2 / 2 sigma^2), full = (float)(fp64 sum);
//   each pass s = fmaf(w[d], in[p - R + d], s) for d = 0..2R over a
//   zero-filled halo; out = s_z * ((1 / (Wx Wy)) * (1 / Wz)), W* the fp32
//   in-bounds weight sums (hot_kernels.cu k_step_smooth / k_compose_smooth).
struct DevKernel {
    int R = 0;
    float w[8] = {0};
    float wlo[8] = {0};  // w64 - w (exact-shape experiment)
    double w64[8] = {0};
    float full = 1.f;
};
int g_dev_hilo = 0;
DevKernel dev_kernel(double sigma) {
    DevKernel k;
    if (!(sigma > 0.0)) { k.w[0] = 1.f; return k; }
    k.R = std::max(1, (int)std::ceil(3.0 * sigma));
    double s = 0.0;
    for (int d = 0; d <= k.R; ++d) {
        const double v = std::exp(-0.5 * (double)(d * d) / (sigma * sigma));
        k.w[d] = (float)v;
        k.wlo[d] = (float)(v - (double)k.w[d]);
        k.w64[d] = v;
        s += d == 0 ? v : 2.0 * v;
    }
    k.full = (float)s;
    return k;
}
float dev_wsum(int p, int n, const DevKernel& k) {
    if (p >= k.R && p + k.R <= n - 1) return k.full;
    float s = 0.f;
    for (int d = -k.R; d <= k.R; ++d) {
        const int q = p + d;
        if (q >= 0 && q < n) s += k.w[d < 0 ? -d : d];
    }
    return s;
}
// Exact fp64 sum of the fp32 weights over the in-bounds taps.
double dev_wsum64(int p, int n, const DevKernel& k) {
    double s = 0.0;
    for (int d = -k.R; d <= k.R; ++d) {
        const int q = p + d;
        if (q >= 0 && q < n) s += g_dev_hilo ? k.w64[d < 0 ? -d : d] : (double)k.w[d < 0 ? -d : d];
    }
    return s;
}
// data: AoS 3-channel field (values already fp32), smoothed in place.
// norm64: normalise in fp64 by the exact weight sums (K4, where a scale bias
// would accumulate in the warp) instead of the fp32 reciprocal (K3, whose
// output is max-normalised anyway).
void dev_smooth32(double* data, orc_dims d, double sigma, bool norm64) {
    const DevKernel k = dev_kernel(sigma);
    const bool hilo = norm64 && g_dev_hilo;
    if (k.R == 0) return;
    const int R = k.R;
    const size_t N = nvox(d);
    std::vector<float> a(3 * N), b(3 * N);
    for (size_t i = 0; i < 3 * N; ++i) a[i] = (float)data[i];
    const int n3[3] = {d.nx, d.ny, d.nz};
    auto pass = [&](const std::vector<float>& in, std::vector<float>& out, int axis) {
        const long long stride = axis == 0 ? 1 : axis == 1 ? d.nx : (long long)d.nx * d.ny;
        const int n = n3[axis];
        par_for(0, d.nz, [&](long long zz) {
            const int z = (int)zz;
            for (int y = 0; y < d.ny; ++y)
                for (int x = 0; x < d.nx; ++x) {
                    const int pcoord = axis == 0 ? x : axis == 1 ? y : z;
                    const size_t i = lin(d, x, y, z);
                    for (int c = 0; c < 3; ++c) {
                        float s = 0.f;
                        for (int t = 0; t <= 2 * R; ++t) {
                            const int q = pcoord - R + t;
                            const float v = (q >= 0 && q < n) ? in[3 * (i + (long long)(q - pcoord) * stride) + c] : 0.f;
                            const int dd = t < R ? R - t : t - R;
                            s = std::fmaf(k.w[dd], v, s);
                            if (hilo) s = std::fmaf(k.wlo[dd], v, s);
                        }
                        out[3 * i + c] = s;
                    }
                }
        });
    };
    pass(a, b, 0);
    pass(b, a, 1);
    pass(a, b, 2);
    par_for(0, d.nz, [&](long long zz) {
        const int z = (int)zz;
        const float iz = 1.f / dev_wsum(z, d.nz, k);
        const double wz64 = dev_wsum64(z, d.nz, k);
        for (int y = 0; y < d.ny; ++y)
            for (int x = 0; x < d.nx; ++x) {
                const size_t i = lin(d, x, y, z);
                if (norm64) {
                    // exact sums of the fp32 weights, fp64 normalisation: no scale bias
                    const double inv = 1.0 / (dev_wsum64(x, d.nx, k) * dev_wsum64(y, d.ny, k) * wz64);
                    for (int c = 0; c < 3; ++c) data[3 * i + c] = (double)(float)((double)b[3 * i + c] * inv);
                } else {
                    const float ixy = 1.f / (dev_wsum(x, d.nx, k) * dev_wsum(y, d.ny, k));
                    const float inv = ixy * iz;
                    for (int c = 0; c < 3; ++c) data[3 * i + c] = (double)(b[3 * i + c] * inv);
                }
            }
    });
}
// Experimental fp32 compose (mode 2 with orc_set_dev_compose32): d rounded
// to fp32, split-form taps (exact), fp32 fused lerps, u' = d + u(x + d).
void dev_compose32(const double* u, const double* v, orc_dims d, double eps, double* out) {
    par_for(0, d.nz, [&](long long zz) {
        const int z = (int)zz;
        for (int y = 0; y < d.ny; ++y)
            for (int x = 0; x < d.nx; ++x) {
                const size_t i = 3 * lin(d, x, y, z);
                const float sx = (float)(eps * v[i]), sy = (float)(eps * v[i + 1]), sz = (float)(eps * v[i + 2]);
                const Tap X = resolve((double)x + sx, d.nx), Y = resolve((double)y + sy, d.ny),
                          Z = resolve((double)z + sz, d.nz);
                const float wx = (float)X.w, wy = (float)Y.w, wz = (float)Z.w;
                const float dd[3] = {sx, sy, sz};
                for (int ch = 0; ch < 3; ++ch) {
                    auto at = [&](int xx, int yy, int zq) { return (float)u[3 * lin(d, xx, yy, zq) + ch]; };
                    const float a = at(X.lo, Y.lo, Z.lo), b = at(X.hi, Y.lo, Z.lo);
                    const float c = at(X.lo, Y.hi, Z.lo), e = at(X.hi, Y.hi, Z.lo);
                    const float f = at(X.lo, Y.lo, Z.hi), h = at(X.hi, Y.lo, Z.hi);
                    const float k = at(X.lo, Y.hi, Z.hi), l = at(X.hi, Y.hi, Z.hi);
                    const float r00 = std::fmaf(wx, b - a, a), r10 = std::fmaf(wx, e - c, c);
                    const float r01 = std::fmaf(wx, h - f, f), r11 = std::fmaf(wx, l - k, k);
                    const float s0 = std::fmaf(wy, r10 - r00, r00), s1 = std::fmaf(wy, r11 - r01, r01);
                    out[i + ch] = (double)(dd[ch] + std::fmaf(wz, s1 - s0, s0));
                }
            }
    });
}
// K3's step in fp32: k = -(float)r * (1 / (|g|^2 + (float)lambda)) (LM),
// (float)(-lr) (GD), 1 (Adam: the Adam step is already in g).
void dev_step32(const double* g, size_t N, int opt, double r, double lambda, double lr, double* out) {
    const float rf = (float)r, lf = (float)lambda;
    for (size_t i = 0; i < N; ++i) {
        const float a = (float)g[3 * i], b = (float)g[3 * i + 1], c = (float)g[3 * i + 2];
        float k = opt == ORC_OPT_GD ? (float)-lr : 1.f;
        if (opt == ORC_OPT_LM) k = -rf * (1.f / (std::fmaf(a, a, std::fmaf(b, b, c * c)) + lf));
        out[3 * i] = (double)(k * a);
        out[3 * i + 1] = (double)(k * b);
        out[3 * i + 2] = (double)(k * c);
    }
}

// Warp of the moving image with the analytic interpolant gradient.
void warp(const double* M, const double* u, orc_dims d, double* Mw, double* gM) {
#ifdef ORC_WITH_REF_FIELD
    const warplm::Volume3 vol = as_vol(M, d);
#endif
    par_for(0, d.nz, [&](long long zz) {
        const int z = (int)zz;
        for (int y = 0; y < d.ny; ++y)
            for (int x = 0; x < d.nx; ++x) {
                const size_t i = lin(d, x, y, z);
                const double px = x + u[3 * i], py = y + u[3 * i + 1], pz = z + u[3 * i + 2];
#ifdef ORC_WITH_REF_FIELD
                const warplm::SampleGrad s = warplm::sample_trilinear_grad(vol, px, py, pz);
                Mw[i] = s.value;
                if (gM) { gM[3 * i] = s.grad[0]; gM[3 * i + 1] = s.grad[1]; gM[3 * i + 2] = s.grad[2]; }
#else
                double gr[3];
                Mw[i] = sample_grad(M, d, px, py, pz, gr);
                if (gM) { gM[3 * i] = gr[0]; gM[3 * i + 1] = gr[1]; gM[3 * i + 2] = gr[2]; }
#endif
            }
    });
}

// Truncated box sum of radius R along one axis, in place on `nch` planar
// channels (channel stride N).  Out-of-grid taps are absent (SPEC.md:138,
// DESIGN.md A2).
void box_axis(double* data, int nch, orc_dims d, int axis, int R) {
    const int n3[3] = {d.nx, d.ny, d.nz};
    const int n = n3[axis];
    const size_t N = nvox(d);
    const int na = axis == 0 ? d.ny : d.nx;
    const int nb = axis == 2 ? d.ny : d.nz;
    const size_t stride = axis == 0 ? 1 : axis == 1 ? (size_t)d.nx : (size_t)d.nx * d.ny;
    par_for(0, (long long)nb * na, [&](long long ab) {
        std::vector<double> line(n);
        {
            const int b = (int)(ab / na), a = (int)(ab % na);
            {
                size_t base;
                if (axis == 0) base = lin(d, 0, a, b);
                else if (axis == 1) base = lin(d, a, 0, b);
                else base = lin(d, a, b, 0);
                for (int c = 0; c < nch; ++c) {
                    double* ch = data + (size_t)c * N;
                    for (int p = 0; p < n; ++p) line[p] = ch[base + p * stride];
                    for (int p = 0; p < n; ++p) {
                        const int q0 = std::max(0, p - R), q1 = std::min(n - 1, p + R);
                        double s = 0.0;
                        for (int q = q0; q <= q1; ++q) s += line[q];
                        ch[base + p * stride] = s;
                    }
                }
            }
        }
    });
}

inline int axis_count(int p, int n, int R) { return std::min(n - 1, p + R) - std::max(0, p - R) + 1; }

// Degenerate-window rule (A3): a window is
// degenerate when either centred second moment is <= kDegRel times its raw
// second moment (or the raw moment is 0).
constexpr double kDegRel = 1e-9;

}  // namespace

// ===========================================================================
extern "C" {

void orc_set_threads(int n) { g_threads = n < 1 ? 1 : n; }
void orc_set_fp32_storage(int on) { g_fp32_storage = on == 2 ? 2 : on ? 1 : 0; }
void orc_set_dev_flags(int flags) { g_dev_flags = flags & 7; g_dev_hilo = (flags >> 3) & 1; g_dev_k3norm64 = (flags >> 4) & 1; }
void orc_dev_smooth32(double* data, orc_dims d, double sigma, int norm64) { dev_smooth32(data, d, sigma, norm64 != 0); }

void orc_default_reg_config(orc_reg_config* c) {
    std::memset(c, 0, sizeof(*c));
    c->lncc_radius = 2;
    c->optimizer = ORC_OPT_LM;
    c->lm.lambda0 = 0.006; c->lm.mu_plus = 1.5; c->lm.mu_minus = 0.975;
    c->lm.tile_size = 1; c->lm.rejection = 0; c->lm.tau = 1.0;
    c->lm.lambda_max = 1.0; c->lm.max_retries = 10;
    c->adam.beta1 = 0.9; c->adam.beta2 = 0.999; c->adam.eps_hat = 1e-8; c->adam.lr = 0.5;
    c->gd_lr = 1.0;
    c->nlevels = 3;
    c->factors[0] = 4; c->factors[1] = 2; c->factors[2] = 1;
    c->iters[0] = 100; c->iters[1] = 75; c->iters[2] = 50;
    c->target_max_disp = 0.4; c->step_floor = 1e-12;      // field.hpp:75-78
    c->sigma_update = 1.0; c->sigma_warp = 0.5;
    c->log_jacobian = 0;
    c->metric = ORC_METRIC_LNCC;
    c->demons_alpha = 1.0;
    c->mi_bins = 32; c->mi_sigma = 1.0;
}

double orc_sample_trilinear_grad(const double* vol, orc_dims d, double px, double py,
                                 double pz, double* grad3) {
    return sample_grad(vol, d, px, py, pz, grad3);
}
void orc_sample_field(const double* u, orc_dims d, double px, double py, double pz,
                      double* out3) {
    sample3(u, d, px, py, pz, out3);
}
void orc_warp_volume(const double* M, const double* u, orc_dims d, double* Mw, double* gradM) {
    warp(M, u, d, Mw, gradM);
}
void orc_compose_warp(const double* u, const double* v, orc_dims d, double eps, double* out) {
    compose(u, v, d, eps, out);
}
double orc_max_abs_component(const double* v, size_t count) { return max_abs(v, count); }
double orc_normalize_step(const double* v, size_t count, double target, double floor_) {
    if (!(target > 0.0 && target < 0.5)) return kNaN;  // field.cpp:151-153
    return target / std::max(max_abs(v, count), floor_);
}
double orc_jacobian_det_min(const double* u, orc_dims d) { return jac_min(u, d); }
void orc_gaussian_smooth(double* data, orc_dims d, int nchan, double sigma) {
    smooth(data, d, nchan, sigma);
}
int orc_all_finite(const double* data, size_t count) {
    for (size_t i = 0; i < count; ++i)
        if (!std::isfinite(data[i])) return 0;
    return 1;
}

// LNCC residual r = 1 - mean_y rho(y) and its gradient g = dr/du.
//   window W(y): cube of radius R truncated to the grid, n(y) voxels
//   rho(y) = c / sqrt(vf vm) (signed, A1), 0 when degenerate
//   d rho(y)/d m_x = A(y) f_x + B(y) m_x - E(y) for x in W(y), with
//   A = 1/(n sqrt(vf vm)), B = -rho/(n vm), E = A mu_f + B mu_m
//   dr/dMw(x) = -(1/N) sum_{y in W(x)} [A f_x + B m_x - E]
//   g(x) = dr/dMw(x) * gradM(x + u(x))
double orc_residual_lncc(const double* F, const double* M, const double* u, orc_dims d,
                         int R, double* g, double* lncc, double* internals) {
    if (R < 1 || d.nx <= 2 * R || d.ny <= 2 * R || d.nz <= 2 * R) return kNaN;
    const size_t N = nvox(d);
    Vec Mw(N), gM(3 * N);
    warp(M, u, d, Mw.data(), gM.data());
    Vec mom(5 * N);
    par_for(0, (long long)N, [&](long long i) {
        const double f = F[i], m = Mw[i];
        mom[i] = f; mom[N + i] = m; mom[2 * N + i] = f * f; mom[3 * N + i] = m * m;
        mom[4 * N + i] = f * m;
    });
    for (int a = 0; a < 3; ++a) box_axis(mom.data(), 5, d, a, R);
    Vec coef(3 * N), rho(N);
    par_for(0, d.nz, [&](long long zz) {
        const int z = (int)zz;
        for (int y = 0; y < d.ny; ++y)
            for (int x = 0; x < d.nx; ++x) {
                const size_t i = lin(d, x, y, z);
                const double n = (double)axis_count(x, d.nx, R) * axis_count(y, d.ny, R) *
                                 axis_count(z, d.nz, R);
                const double mf = mom[i] / n, mm = mom[N + i] / n;
                const double sff = mom[2 * N + i] / n, smm = mom[3 * N + i] / n;
                const double vf = sff - mf * mf, vm = smm - mm * mm;
                const double cv = mom[4 * N + i] / n - mf * mm;
                double r = 0.0, A = 0.0, B = 0.0, E = 0.0;
                // degenerate test written so that NaN moments are NOT degenerate:
                // a non-finite input propagates into the loss
                const bool degenerate = !(sff > 0.0 || std::isnan(sff)) || !(smm > 0.0 || std::isnan(smm)) ||
                                        vf <= kDegRel * sff || vm <= kDegRel * smm;
                if (!degenerate) {
                    const double alpha = 1.0 / std::sqrt(vf * vm);
                    r = cv * alpha;
                    A = r32(alpha / n);
                    B = r32(-r / (vm * n));
                    E = A * mf + B * mm;
                }
                rho[i] = r;
                coef[i] = A; coef[N + i] = B; coef[2 * N + i] = E;
            }
    });
    double total = 0.0;  // fixed serial order
    for (size_t i = 0; i < N; ++i) total += rho[i];
    const double L = total / (double)N;
    if (lncc) *lncc = L;
    if (internals) {
        std::memcpy(internals, Mw.data(), sizeof(double) * N);
        std::memcpy(internals + N, rho.data(), sizeof(double) * N);
        std::memcpy(internals + 2 * N, coef.data(), sizeof(double) * 3 * N);
    }
    if (g || internals) {
        Vec adj(coef);
        for (int a = 0; a < 3; ++a) box_axis(adj.data(), 3, d, a, R);
        const double invN = 1.0 / (double)N;
        par_for(0, (long long)N, [&](long long i) {
            const double dm = -invN * (F[i] * adj[i] + Mw[i] * adj[N + i] - adj[2 * N + i]);
            if (internals) internals[5 * N + i] = dm;
            if (g) {
                g[3 * i] = r32(dm * gM[3 * i]);
                g[3 * i + 1] = r32(dm * gM[3 * i + 1]);
                g[3 * i + 2] = r32(dm * gM[3 * i + 2]);
            }
        });
        if (internals) std::memcpy(internals + 6 * N, gM.data(), sizeof(double) * 3 * N);
    }
    return 1.0 - L;
}

double orc_residual_mse(const double* F, const double* M, const double* u, orc_dims d,
                        double* g) {
    const size_t N = nvox(d);
    Vec Mw(N), gM(3 * N);
    warp(M, u, d, Mw.data(), gM.data());
    double s = 0.0;  // fixed serial order
    for (size_t i = 0; i < N; ++i) { const double e = F[i] - Mw[i]; s += e * e; }
    if (g)
        for (size_t i = 0; i < N; ++i) {
            const double k = -2.0 * (F[i] - Mw[i]) / (double)N;
            for (int c = 0; c < 3; ++c) g[3 * i + c] = r32(k * gM[3 * i + c]);
        }
    return s / (double)N;
}

// Eq. (5): tiled LM.  Non-overlapping k^3 tiles (partial at
// the far faces); H = sum over the tile of g g^T, accumulated in z, y, x
// order; Delta u(x) = -r (H + lambda I)^{-1} g(x) with the explicit
// (adjugate / determinant) inverse of the symmetric 3x3.
void tile_step_matrix(const double H[6], double r, double lambda, double Mout[6]) {
    // H = [a b c; b d e; c e f] + lambda I
    const double a = H[0] + lambda, b = H[1], c = H[2], d = H[3] + lambda, e = H[4], f = H[5] + lambda;
    const double c00 = d * f - e * e, c01 = c * e - b * f, c02 = b * e - c * d;
    const double c11 = a * f - c * c, c12 = b * c - a * e, c22 = a * d - b * b;
    const double det = a * c00 + b * c01 + c * c02;
    const double s = -r / det;
    Mout[0] = s * c00; Mout[1] = s * c01; Mout[2] = s * c02;
    Mout[3] = s * c11; Mout[4] = s * c12; Mout[5] = s * c22;
}
void orc_lm_step_tiled(double r, const double* g, orc_dims d, double lambda, int k, double* out) {
    const int tx = (d.nx + k - 1) / k, ty = (d.ny + k - 1) / k, tz = (d.nz + k - 1) / k;
    par_for(0, (long long)tx * ty * tz, [&](long long t) {
        const int bx = (int)(t % tx), by = (int)((t / tx) % ty), bz = (int)(t / ((long long)tx * ty));
        const int x1 = std::min(d.nx, (bx + 1) * k), y1 = std::min(d.ny, (by + 1) * k),
                  z1 = std::min(d.nz, (bz + 1) * k);
        double H[6] = {0, 0, 0, 0, 0, 0};
        for (int z = bz * k; z < z1; ++z)
            for (int y = by * k; y < y1; ++y)
                for (int x = bx * k; x < x1; ++x) {
                    const double* gi = g + 3 * lin(d, x, y, z);
                    H[0] += gi[0] * gi[0]; H[1] += gi[0] * gi[1]; H[2] += gi[0] * gi[2];
                    H[3] += gi[1] * gi[1]; H[4] += gi[1] * gi[2]; H[5] += gi[2] * gi[2];
                }
        double Mt[6];
        tile_step_matrix(H, r, lambda, Mt);
        for (int z = bz * k; z < z1; ++z)
            for (int y = by * k; y < y1; ++y)
                for (int x = bx * k; x < x1; ++x) {
                    const size_t i = 3 * lin(d, x, y, z);
                    const double g0 = g[i], g1 = g[i + 1], g2 = g[i + 2];
                    out[i] = Mt[0] * g0 + Mt[1] * g1 + Mt[2] * g2;
                    out[i + 1] = Mt[1] * g0 + Mt[3] * g1 + Mt[4] * g2;
                    out[i + 2] = Mt[2] * g0 + Mt[4] * g1 + Mt[5] * g2;
                }
    });
}

// Eq. (9): Demons active forces r_x n_x / (|n_x|^2 +
// alpha^2 r_x^2); both terms zero -> 0.
void orc_demons_step_mse(const double* r, const double* n, size_t N, double alpha, double* out) {
    par_for(0, (long long)N, [&](long long i) {
        const double rx = r[i], a = n[3 * i], b = n[3 * i + 1], c = n[3 * i + 2];
        const double den = a * a + b * b + c * c + alpha * alpha * rx * rx;
        const double s = den > 0.0 ? rx / den : 0.0;
        out[3 * i] = s * a; out[3 * i + 1] = s * b; out[3 * i + 2] = s * c;
    });
}

// ---- Parzen-window mutual information ----
// Pinned choices (A13-A15): F and M min-max normalised over the
// whole (level) volume; Parzen coordinate t = v (B - 1), bins 0..B-1; kernel
// exp(-s^2 / 2 sigma^2) on |s| <= 4 sigma (sigma in bin widths), normalised
// per sample over the in-range bins, so p = (1/N) sum_x a(t_f) b(t_m)^T sums
// to 1; logs floored at 1e-12; MI in bits, r = log2 B - MI.
struct Parzen {
    int lo, n;        // first bin, bin count (<= 9 for sigma = 1)
    double w[64], dw[64];  // normalised weights and d/dt
};
Parzen parzen(double t, int B, double sigma) {
    Parzen P;
    const double reach = 4.0 * sigma;
    int lo = (int)std::ceil(t - reach), hi = (int)std::floor(t + reach);
    lo = std::max(lo, 0);
    hi = std::min(hi, B - 1);
    P.lo = lo;
    P.n = std::max(0, std::min(hi - lo + 1, 64));
    double S = 0.0, Sd = 0.0, raw[64], draw[64];
    for (int k = 0; k < P.n; ++k) {
        const double sft = t - (double)(lo + k);
        raw[k] = std::exp(-0.5 * sft * sft / (sigma * sigma));
        draw[k] = -sft / (sigma * sigma) * raw[k];
        S += raw[k];
        Sd += draw[k];
    }
    for (int k = 0; k < P.n; ++k) {
        P.w[k] = raw[k] / S;
        P.dw[k] = (draw[k] * S - raw[k] * Sd) / (S * S);
    }
    return P;
}
void minmax(const double* v, size_t N, double* lo, double* range) {
    double a = v[0], b = v[0];
    for (size_t i = 1; i < N; ++i) { a = std::min(a, v[i]); b = std::max(b, v[i]); }
    *lo = a;
    *range = b > a ? b - a : 1.0;
}

double orc_residual_mi(const double* F, const double* M, const double* u, orc_dims d, int B, double sigma,
                       double* g, double* mi_out) {
    if (B < 2 || !(sigma > 0.0)) return kNaN;
    const size_t N = nvox(d);
    Vec Mw(N), gM(3 * N);
    warp(M, u, d, Mw.data(), gM.data());
    double flo, frange, mlo, mrange;
    minmax(F, N, &flo, &frange);
    minmax(M, N, &mlo, &mrange);
    const double sf = (double)(B - 1) / frange, sm = (double)(B - 1) / mrange;
    std::vector<double> P((size_t)B * B, 0.0);
    // fixed serial order
    for (size_t i = 0; i < N; ++i) {
        const Parzen a = parzen((F[i] - flo) * sf, B, sigma), b = parzen((Mw[i] - mlo) * sm, B, sigma);
        for (int ii = 0; ii < a.n; ++ii)
            for (int jj = 0; jj < b.n; ++jj) P[(size_t)(a.lo + ii) * B + b.lo + jj] += a.w[ii] * b.w[jj];
    }
    const double invN = 1.0 / (double)N, eps = 1e-12, il2 = 1.0 / std::log(2.0);
    std::vector<double> pf(B, 0.0), pm(B, 0.0);
    for (int i = 0; i < B; ++i)
        for (int j = 0; j < B; ++j) {
            const double p = P[(size_t)i * B + j] * invN;
            P[(size_t)i * B + j] = p;
            pf[i] += p;
            pm[j] += p;
        }
    double mi = 0.0;
    for (int i = 0; i < B; ++i)
        for (int j = 0; j < B; ++j) {
            const double p = P[(size_t)i * B + j];
            mi += p * std::log2(std::max(p, eps));
        }
    for (int i = 0; i < B; ++i) mi -= pf[i] * std::log2(std::max(pf[i], eps));
    for (int j = 0; j < B; ++j) mi -= pm[j] * std::log2(std::max(pm[j], eps));
    if (mi_out) *mi_out = mi;
    if (g) {
        // dMI/dp_ij (joint minus moving-marginal part; the fixed marginal does
        // not depend on u)
        std::vector<double> T((size_t)B * B);
        for (int i = 0; i < B; ++i)
            for (int j = 0; j < B; ++j) {
                const double p = P[(size_t)i * B + j];
                const double lj = std::log2(std::max(p, eps)) + (p >= eps ? il2 : 0.0);
                const double lm = std::log2(std::max(pm[j], eps)) + (pm[j] >= eps ? il2 : 0.0);
                T[(size_t)i * B + j] = lj - lm;
            }
        par_for(0, (long long)N, [&](long long ix) {
            const size_t i = (size_t)ix;
            const Parzen a = parzen((F[i] - flo) * sf, B, sigma), b = parzen((Mw[i] - mlo) * sm, B, sigma);
            double s = 0.0;
            for (int ii = 0; ii < a.n; ++ii) {
                double t = 0.0;
                for (int jj = 0; jj < b.n; ++jj) t += b.dw[jj] * T[(size_t)(a.lo + ii) * B + b.lo + jj];
                s += a.w[ii] * t;
            }
            const double dr = -invN * sm * s;  // dr/dMw = -dMI/dMw
            g[3 * i] = r32(dr * gM[3 * i]);
            g[3 * i + 1] = r32(dr * gM[3 * i + 1]);
            g[3 * i + 2] = r32(dr * gM[3 * i + 2]);
        });
    }
    return std::log2((double)B) - mi;
}

// Eq. (4): dU = -r g / (|g|^2 + lambda); zero gradient -> exactly zero.
void orc_lm_step_pointwise(double r, const double* g, size_t n, double lambda, double* out) {
    par_for(0, (long long)n, [&](long long i) {
        const double gx = g[3 * i], gy = g[3 * i + 1], gz = g[3 * i + 2];
        const double s = -r / (gx * gx + gy * gy + gz * gz + lambda);
        out[3 * i] = s * gx; out[3 * i + 1] = s * gy; out[3 * i + 2] = s * gz;
    });
}

// Explicit damped 3x3 solve by Gaussian elimination with partial pivoting.
void orc_lm_step_dense3(double r, const double* g, double lambda, double* out) {
    double A[3][4];
    for (int i = 0; i < 3; ++i) {
        for (int j = 0; j < 3; ++j) A[i][j] = g[i] * g[j] + (i == j ? lambda : 0.0);
        A[i][3] = -r * g[i];
    }
    for (int c = 0; c < 3; ++c) {
        int p = c;
        for (int i = c + 1; i < 3; ++i) if (std::fabs(A[i][c]) > std::fabs(A[p][c])) p = i;
        if (p != c) for (int j = 0; j < 4; ++j) std::swap(A[c][j], A[p][j]);
        for (int i = c + 1; i < 3; ++i) {
            const double f = A[i][c] / A[c][c];
            for (int j = c; j < 4; ++j) A[i][j] -= f * A[c][j];
        }
    }
    for (int i = 2; i >= 0; --i) {
        double s = A[i][3];
        for (int j = i + 1; j < 3; ++j) s -= A[i][j] * out[j];
        out[i] = s / A[i][i];
    }
}

// Eq. (6) with the SPEC's tie rule (==: good), empty history ->
// bad (A4), cap and 1e-12 floor (:333).
void orc_update_damping(orc_lm_state* s, double loss_new, const orc_lm_config* c) {
    const bool bad = s->hist_n == 0 || loss_new > s->L1;
    double lam = bad ? c->mu_plus * s->lambda : c->mu_minus * s->lambda;
    if (c->lambda_max > 0.0 && std::isfinite(c->lambda_max)) lam = std::min(lam, c->lambda_max);
    s->lambda = std::max(lam, 1e-12);
    s->L2 = s->L1;
    s->L1 = loss_new;
    s->hist_n = std::min(s->hist_n + 1, 2);
}

// Eq. (10), multiplicative form: reject iff
// L_new - L1 > tau |L1 - L2|.
int orc_rejection_test(double loss_new, double L1, double L2, double tau) {
    return (loss_new - L1) > tau * std::fabs(L1 - L2) ? 1 : 0;
}

}  // extern "C"

namespace {
// Attempt decision inside lm_iterate: returns true when
// the attempt is rejected and another is due (lambda bumped, capped).
bool attempt_rejected(orc_lm_state& s, const orc_lm_config& c, double loss_new, int& retries) {
    if (!c.rejection || s.hist_n < 2 || retries >= c.max_retries) return false;
    if (!orc_rejection_test(loss_new, s.L1, s.L2, c.tau)) return false;
    double lam = c.mu_plus * s.lambda;
    if (c.lambda_max > 0.0 && std::isfinite(c.lambda_max)) lam = std::min(lam, c.lambda_max);
    s.lambda = lam;
    ++retries;
    return true;
}
}  // namespace

extern "C" {

int orc_lm_replay(const double* losses, int n, int iters, const orc_lm_config* c,
                  double* lambda_out, int* decision_out, orc_lm_state* st) {
    orc_lm_state s = *st;
    int k = 0;
    for (int it = 0; it < iters && k < n; ++it) {
        int retries = 0;
        for (;;) {
            if (k >= n) { *st = s; return k; }
            const double L = losses[k];
            const bool rej = attempt_rejected(s, *c, L, retries);
            if (!rej) orc_update_damping(&s, L, c);
            if (lambda_out) lambda_out[k] = s.lambda;
            if (decision_out) decision_out[k] = rej ? 1 : 0;
            ++k;
            if (!rej) break;
        }
    }
    *st = s;
    return k;
}

// Bias-corrected Adam; t is the 1-based step count.
void orc_adam_step(const double* g, double* m, double* v, size_t count, int t,
                   const orc_adam_config* c, double* out) {
    const double bc1 = 1.0 - std::pow(c->beta1, t), bc2 = 1.0 - std::pow(c->beta2, t);
    for (size_t i = 0; i < count; ++i) {
        m[i] = r32(c->beta1 * m[i] + (1.0 - c->beta1) * g[i]);
        v[i] = r32(c->beta2 * v[i] + (1.0 - c->beta2) * g[i] * g[i]);
        const double mh = m[i] / bc1, vh = v[i] / bc2;
        out[i] = r32(-c->lr * mh / (std::sqrt(vh) + c->eps_hat));
    }
}

orc_dims orc_level_dims(orc_dims d, int f) {
    orc_dims r{(d.nx + f - 1) / f, (d.ny + f - 1) / f, (d.nz + f - 1) / f};
    return r;
}

// Gaussian sigma = 0.5 f (same kernel rules as gaussian_smooth), then stride f
// with the coarse voxel i at fine voxel i*f (A9).
void orc_downsample(const double* vol, orc_dims d, int f, double* out) {
    const size_t N = nvox(d);
    if (f <= 1) { std::memcpy(out, vol, sizeof(double) * N); return; }
    Vec tmp(vol, vol + N);
    smooth(tmp.data(), d, 1, 0.5 * f);
    const orc_dims nd = orc_level_dims(d, f);
    for (int z = 0; z < nd.nz; ++z)
        for (int y = 0; y < nd.ny; ++y)
            for (int x = 0; x < nd.nx; ++x) out[lin(nd, x, y, z)] = tmp[lin(d, x * f, y * f, z * f)];
}

// Trilinear resample onto the new grid (x_old = x_new / scale) then multiply
// by scale.
void orc_upsample_warp(const double* u, orc_dims d, orc_dims nd, double scale, double* out) {
    par_for(0, nd.nz, [&](long long zz) {
        const int z = (int)zz;
        for (int y = 0; y < nd.ny; ++y)
            for (int x = 0; x < nd.nx; ++x) {
                double s[3];
                sample3(u, d, x / scale, y / scale, z / scale, s);
                const size_t i = 3 * lin(nd, x, y, z);
                out[i] = r32(scale * s[0]); out[i + 1] = r32(scale * s[1]); out[i + 2] = r32(scale * s[2]);
            }
    });
}

// lm_iterate x iters at one level.  Each iteration:
//   (r, g) at u  ->  attempts { dU = LM step; dU_s = smooth(dU, sigma_update);
//   eps = normalize_step(dU_s); u' = compose(u, dU_s, eps);
//   u' = smooth(u', sigma_warp); r' = residual(u'); reject? }  ->
//   update_damping(r'); u <- u'.
// Adam / GD share the smooth-normalize-compose path (A10).
// Wall time of every attempt (LM step .. residual at the trial warp) of the
// calling thread's orc_lm_run_level_timed call: the CPU baseline's
// per-iteration cost without the level's initial residual (bench.py).
static thread_local double* t_attempt_s = nullptr;
static thread_local int t_attempt_cap = 0, t_attempt_n = 0;

int orc_lm_run_level(const double* F, const double* M, orc_dims d, double* u,
                     const orc_reg_config* c, orc_lm_state* state, int level, int iters,
                     orc_step_log* trace, int* ntrace) {
    const size_t N = nvox(d);
    const int R = c->lncc_radius;
    Vec g(3 * N), step(3 * N), unew(3 * N), gnew(3 * N), am, av;
    if (c->optimizer == ORC_OPT_ADAM) { am.assign(3 * N, 0.0); av.assign(3 * N, 0.0); }
    // MetricConfig.kind: loss_raw is LNCC (r = 1 - LNCC) or the
    // MSE itself (r = MSE)
    auto residual = [&](const double* uu, double* gg, double* raw) {
        if (c->metric == ORC_METRIC_MSE) {
            const double m = orc_residual_mse(F, M, uu, d, gg);
            *raw = m;
            return m;
        }
        if (c->metric == ORC_METRIC_MI) return orc_residual_mi(F, M, uu, d, c->mi_bins, c->mi_sigma, gg, raw);
        return orc_residual_lncc(F, M, uu, d, R, gg, raw, nullptr);
    };
    double lncc = 0.0;
    double r = residual(u, g.data(), &lncc);
    if (!std::isfinite(r)) return ORC_NONFINITE;
    int nt = 0;
    for (int it = 0; it < iters; ++it) {
        int retries = 0;
        double rn = 0.0, ln = 0.0, eps = 0.0, jac = kNaN;
        bool forced = false;
        for (;;) {
            const auto t_att0 = std::chrono::steady_clock::now();
            const bool dev = g_fp32_storage == 2 && (g_dev_flags & 1);
            const bool dev4 = g_fp32_storage == 2 && (g_dev_flags & 2);
            if (c->optimizer == ORC_OPT_LM && c->lm.tile_size > 1) {
                orc_lm_step_tiled(r, g.data(), d, state->lambda, c->lm.tile_size, step.data());
            } else if (c->optimizer == ORC_OPT_LM) {
                if (dev) dev_step32(g.data(), N, ORC_OPT_LM, r, state->lambda, 0.0, step.data());
                else orc_lm_step_pointwise(r, g.data(), N, state->lambda, step.data());
            } else if (c->optimizer == ORC_OPT_ADAM) {
                orc_adam_step(g.data(), am.data(), av.data(), 3 * N, it + 1, &c->adam, step.data());
            } else if (c->optimizer == ORC_OPT_DEMONS) {
                // Eq. 9 from the MSE per-voxel residual at the accepted warp
                Vec Mw(N), gM(3 * N), rx(N);
                warp(M, u, d, Mw.data(), gM.data());
                for (size_t i = 0; i < N; ++i) rx[i] = F[i] - Mw[i];
                orc_demons_step_mse(rx.data(), gM.data(), N, c->demons_alpha, step.data());
                for (auto& v : step) v = r32(v);  // stored where the device keeps g
            } else if (dev) {
                dev_step32(g.data(), N, ORC_OPT_GD, 0.0, 0.0, c->gd_lr, step.data());
            } else {
                for (size_t i = 0; i < 3 * N; ++i) step[i] = -c->gd_lr * g[i];
            }
            if (dev) dev_smooth32(step.data(), d, c->sigma_update, g_dev_k3norm64 != 0);
            else smooth(step.data(), d, 3, c->sigma_update);
            if (g_fp32_storage)
                for (auto& v : step) v = (double)(float)v;
            eps = orc_normalize_step(step.data(), 3 * N, c->target_max_disp, c->step_floor);
            if (!std::isfinite(eps)) return ORC_INVALID_ARG;
            compose(u, step.data(), d, eps, unew.data());
            if (g_fp32_storage == 2 && (g_dev_flags & 4)) dev_compose32(u, step.data(), d, eps, unew.data());
            if (dev4) {
                for (auto& v : unew) v = (double)(float)v;
                dev_smooth32(unew.data(), d, c->sigma_warp, true);
            } else {
                smooth(unew.data(), d, 3, c->sigma_warp);
            }
            if (g_fp32_storage)
                for (auto& v : unew) v = (double)(float)v;
            if (c->log_jacobian) {
                Vec inc(3 * N);
                for (size_t i = 0; i < 3 * N; ++i) inc[i] = eps * step[i];
                jac = jac_min(inc.data(), d);
            }
            rn = residual(unew.data(), gnew.data(), &ln);
            if (t_attempt_s && t_attempt_n < t_attempt_cap)
                t_attempt_s[t_attempt_n++] =
                    std::chrono::duration<double>(std::chrono::steady_clock::now() - t_att0).count();
            if (!std::isfinite(rn)) {
                if (trace && ntrace) *ntrace = nt;
                return ORC_NONFINITE;
            }
            if (c->optimizer != ORC_OPT_LM) break;
            const int before = retries;
            if (!attempt_rejected(*state, c->lm, rn, retries)) {
                forced = c->lm.rejection && before == c->lm.max_retries && state->hist_n >= 2 &&
                         orc_rejection_test(rn, state->L1, state->L2, c->lm.tau);
                break;
            }
        }
        if (c->optimizer == ORC_OPT_LM) orc_update_damping(state, rn, &c->lm);
        std::swap(g, gnew);
        std::memcpy(u, unew.data(), sizeof(double) * 3 * N);
        r = rn;
        if (trace) {
            orc_step_log& L = trace[nt];
            L.level = level; L.iter = it; L.loss_raw = ln; L.r = rn;
            L.lambda = c->optimizer == ORC_OPT_LM ? state->lambda : 0.0;
            L.eps = eps; L.accepted = forced ? 0 : 1; L.retries = retries;
            L.jac_det_min = jac;
        }
        ++nt;
    }
    if (ntrace) *ntrace = nt;
    return ORC_OK;
}

int orc_lm_run_level_timed(const double* F, const double* M, orc_dims d, double* u,
                           const orc_reg_config* c, orc_lm_state* state, int level, int iters,
                           orc_step_log* trace, int* ntrace, double* attempt_s, int cap, int* nattempts) {
    t_attempt_s = attempt_s;
    t_attempt_cap = cap;
    t_attempt_n = 0;
    const int rc = orc_lm_run_level(F, M, d, u, c, state, level, iters, trace, ntrace);
    if (nattempts) *nattempts = t_attempt_n;
    t_attempt_s = nullptr;
    t_attempt_cap = t_attempt_n = 0;
    return rc;
}

// register(F, M, cfg): coarse -> fine, warp inherited with
// upsample_warp, lambda carried, loss history reset per level.
int orc_register(const float* Ff, const float* Mf, orc_dims d, const orc_reg_config* c,
                 double* warp_out, orc_step_log* trace, size_t cap, size_t* len,
                 double* jac_final) {
    if (c->nlevels < 1 || c->nlevels > ORC_MAX_LEVELS) return ORC_INVALID_ARG;
    if (c->factors[c->nlevels - 1] != 1) return ORC_INVALID_ARG;
    for (int l = 0; l < c->nlevels; ++l) {
        if (c->factors[l] < 1 || c->iters[l] < 0) return ORC_INVALID_ARG;
        if (l > 0 && c->factors[l] >= c->factors[l - 1]) return ORC_INVALID_ARG;
    }
    if (c->lm.tile_size < 1) return ORC_INVALID_ARG;
    const size_t N = nvox(d);
    Vec F(Ff, Ff + N), M(Mf, Mf + N);
    orc_lm_state st{c->lm.lambda0, 0, 0.0, 0.0};
    Vec u;
    orc_dims ud{0, 0, 0};
    size_t used = 0;
    for (int l = 0; l < c->nlevels; ++l) {
        const int f = c->factors[l];
        const orc_dims ld = orc_level_dims(d, f);
        const size_t LN = nvox(ld);
        Vec Fl(LN), Ml(LN);
        orc_downsample(F.data(), d, f, Fl.data());
        orc_downsample(M.data(), d, f, Ml.data());
        // level images are materialised in fp32, the precision of the VOL3
        // inputs (A11); the full-resolution level is already fp32
        for (size_t i = 0; i < LN; ++i) { Fl[i] = (float)Fl[i]; Ml[i] = (float)Ml[i]; }
        Vec ul(3 * LN, 0.0);
        if (l > 0) orc_upsample_warp(u.data(), ud, ld, (double)c->factors[l - 1] / f, ul.data());
        st.hist_n = 0;
        std::vector<orc_step_log> lt(c->iters[l]);
        int nt = 0;
        const int rc = orc_lm_run_level(Fl.data(), Ml.data(), ld, ul.data(), c, &st, l,
                                        c->iters[l], lt.data(), &nt);
        for (int i = 0; i < nt && used < cap; ++i) trace[used++] = lt[i];
        if (len) *len = used;
        if (rc != ORC_OK) return rc;
        u.swap(ul);
        ud = ld;
    }
    std::memcpy(warp_out, u.data(), sizeof(double) * 3 * N);
    if (jac_final) *jac_final = jac_min(u.data(), d);
    return ORC_OK;
}

uint64_t orc_splitmix64(uint64_t* s) {
    uint64_t z = (*s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

}  // extern "C"

namespace {
struct Rng {
    uint64_t s;
    bool have = false;
    double spare = 0.0;
    double uniform() { return (double)(orc_splitmix64(&s) >> 11) * 0x1.0p-53; }
    double normal() {  // Box-Muller, second variate cached
        if (have) { have = false; return spare; }
        const double u1 = 1.0 - uniform(), u2 = uniform();
        const double rad = std::sqrt(-2.0 * std::log(u1));
        spare = rad * std::sin(2.0 * M_PI * u2);
        have = true;
        return rad * std::cos(2.0 * M_PI * u2);
    }
};
}  // namespace

extern "C" {

// synth_pair: blob image in [0,1], smoothed random warp
// rescaled to warp_max with positive Jacobian (redrawn up to 10 times),
// moving = clean fixed through Id + u_true, independent N(0, noise^2) on both.
int orc_synth_pair(const orc_synth_spec* sp, float* Fo, float* Mo, float* Uo) {
    const orc_dims d = sp->dims;
    const size_t N = nvox(d);
    Rng rng{sp->seed};
    const int K = sp->num_blobs;
    const double mind = (double)std::min(d.nx, std::min(d.ny, d.nz));
    std::vector<double> ex((size_t)K * d.nx), ey((size_t)K * d.ny), ez((size_t)K * d.nz), amp(K);
    for (int k = 0; k < K; ++k) {
        const double cx = (0.2 + 0.6 * rng.uniform()) * d.nx;
        const double cy = (0.2 + 0.6 * rng.uniform()) * d.ny;
        const double cz = (0.2 + 0.6 * rng.uniform()) * d.nz;
        const double sg = (0.05 + 0.07 * rng.uniform()) * mind;
        amp[k] = 0.3 + 0.7 * rng.uniform();
        const double q = 1.0 / (2.0 * sg * sg);
        for (int x = 0; x < d.nx; ++x) ex[(size_t)k * d.nx + x] = std::exp(-(x - cx) * (x - cx) * q);
        for (int y = 0; y < d.ny; ++y) ey[(size_t)k * d.ny + y] = std::exp(-(y - cy) * (y - cy) * q);
        for (int z = 0; z < d.nz; ++z) ez[(size_t)k * d.nz + z] = std::exp(-(z - cz) * (z - cz) * q);
    }
    Vec F(N);
    par_for(0, d.nz, [&](long long zz) {
        const int z = (int)zz;
        for (int y = 0; y < d.ny; ++y)
            for (int x = 0; x < d.nx; ++x) {
                double s = 0.0;
                for (int k = 0; k < K; ++k)
                    s += amp[k] * ex[(size_t)k * d.nx + x] * ey[(size_t)k * d.ny + y] *
                         ez[(size_t)k * d.nz + z];
                F[lin(d, x, y, z)] = s;
            }
    });
    double lo = F[0], hi = F[0];
    for (size_t i = 0; i < N; ++i) { lo = std::min(lo, F[i]); hi = std::max(hi, F[i]); }
    const double span = hi > lo ? hi - lo : 1.0;
    for (size_t i = 0; i < N; ++i) F[i] = (F[i] - lo) / span;

    const double ws = sp->warp_sigma > 0.0 ? sp->warp_sigma : mind / 16.0;
    Vec u(3 * N, 0.0);
    bool ok = sp->warp_max <= 0.0;
    for (int attempt = 0; attempt < 10 && !ok; ++attempt) {
        for (size_t i = 0; i < 3 * N; ++i) u[i] = rng.normal();
        smooth(u.data(), d, 3, ws);
        const double m = max_abs(u.data(), 3 * N);
        const double sc = m > 0.0 ? sp->warp_max / m : 0.0;
        for (size_t i = 0; i < 3 * N; ++i) u[i] *= sc;
        ok = !(d.nx >= 2 && d.ny >= 2 && d.nz >= 2) || jac_min(u.data(), d) > 0.0;
    }
    if (!ok) return ORC_INVALID_ARG;
    if (sp->warp_max <= 0.0) std::fill(u.begin(), u.end(), 0.0);

    Vec Mv(N);
    warp(F.data(), u.data(), d, Mv.data(), nullptr);
    for (size_t i = 0; i < N; ++i) Fo[i] = (float)(F[i] + sp->noise_sigma * rng.normal());
    for (size_t i = 0; i < N; ++i) Mo[i] = (float)(Mv[i] + sp->noise_sigma * rng.normal());
    if (Uo)
        for (size_t i = 0; i < 3 * N; ++i) Uo[i] = (float)u[i];
    return ORC_OK;
}

}  // extern "C"
