// common.cuh -- shared device helpers for the sm_100a kernels.
//
// HBM layout: every scalar volume is one fp32
// plane stack [nz][ny][nx] (x fastest, reference Dims3::index,
// field.hpp:25-30); a displacement field is three such stacks, one per
// component (SoA), so every per-component access is a unit-stride coalesced
// row.  Batches of independent pairs are stacked outermost.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "wlm.h"

namespace wlm {

// In-volume offsets are 32-bit: one volume holds < 2^31 voxels (the
// reference caps files at 2^31, io.cpp:13; engines reject larger volumes).
// Batch/pair/channel bases are applied as 64-bit pointer offsets.
//
// z-slab decomposition (config 5): a rank owns planes
// [zs, ze) of the global volume; its per-voxel buffers (warps, coefficients,
// gradient, step) hold planes [zlo, zlo + nzl) = owned planes plus halo
// planes filled by the exchange.  F and M are replicated whole (nfull).
// Volume faces are always the global ones (z = 0, nz - 1).
struct Geo {
    int nx, ny, nz;   // global volume
    long long n;      // voxels of one local buffer plane-stack (nx * ny * nzl)
    int zs, ze;       // owned planes (global z)
    int zlo, nzl;     // local buffer planes [zlo, zlo + nzl)
    long long nfull;  // voxels of the whole volume (F, M)
    __host__ __device__ int at(int x, int y, int z) const { return x + nx * (y + ny * z); }
    __host__ __device__ int lat(int x, int y, int z) const { return x + nx * (y + ny * (z - zlo)); }
};

inline Geo make_geo(wlm_dims d) {
    Geo g;
    g.nx = d.nx; g.ny = d.ny; g.nz = d.nz;
    g.n = (long long)d.nx * d.ny * d.nz;
    g.zs = 0; g.ze = d.nz; g.zlo = 0; g.nzl = d.nz;
    g.nfull = g.n;
    return g;
}

// Slab geometry: owned [zs, ze), halo h planes each side (clipped to the volume).
inline Geo make_slab_geo(wlm_dims d, int zs, int ze, int h) {
    Geo g = make_geo(d);
    g.zs = zs; g.ze = ze;
    g.zlo = zs - h < 0 ? 0 : zs - h;
    const int zhi = ze + h > d.nz ? d.nz : ze + h;
    g.nzl = zhi - g.zlo;
    g.n = (long long)d.nx * d.ny * g.nzl;
    return g;
}

// ---------------------------------------------------------------------------
// Clamp-to-edge trilinear axis resolution for p = x + u, the reference's
// resolve_axis (field.cpp:19-39) evaluated in split form: the integer part
// of the displacement is added to the integer grid coordinate first, so the
// cell choice (and hence the one-sided gradient at knots)
// matches the fp64 reference even when fp32 x + u would round.
struct AxisTap {
    int i0, i1;
    float t;
    bool outside;
};

__device__ __forceinline__ AxisTap axis_tap(int x, float u, int n) {
    AxisTap a;
    if (n == 1) { a.i0 = a.i1 = 0; a.t = 0.f; a.outside = true; return a; }
    const float fl = floorf(u);
    const int i = x + (int)fl;
    const float t = u - fl;  // in [0, 1]; may round up to exactly 1
    if (i < 0) { a.i0 = 0; a.i1 = 1; a.t = 0.f; a.outside = true; return a; }
    if (i > n - 1 || (i == n - 1 && t > 0.f)) {
        a.i0 = n - 2; a.i1 = n - 1; a.t = 1.f; a.outside = true; return a;
    }
    if (i == n - 1) { a.i0 = n - 2; a.i1 = n - 1; a.t = 1.f; a.outside = false; return a; }
    a.i0 = i; a.i1 = i + 1; a.t = t; a.outside = false;
    return a;
}

// Value and analytic interpolant gradient of vol at (x,y,z) + (ux,uy,uz),
// same collapse order as field.cpp:47-90.  Non-finite displacement -> NaN
// value, zero gradient (field.cpp:49-52).
__device__ __forceinline__ float sample_grad(const float* __restrict__ vol, const Geo& g, int x,
                                             int y, int z, float ux, float uy, float uz,
                                             float& gx, float& gy, float& gz) {
    if (!(isfinite(ux) && isfinite(uy) && isfinite(uz))) {
        gx = gy = gz = 0.f;
        return __int_as_float(0x7fc00000);
    }
    const AxisTap X = axis_tap(x, ux, g.nx), Y = axis_tap(y, uy, g.ny), Z = axis_tap(z, uz, g.nz);
    const int r00 = g.nx * (Y.i0 + g.ny * Z.i0);
    const int r10 = g.nx * (Y.i1 + g.ny * Z.i0);
    const int r01 = g.nx * (Y.i0 + g.ny * Z.i1);
    const int r11 = g.nx * (Y.i1 + g.ny * Z.i1);
    const float a = __ldg(vol + r00 + X.i0), b = __ldg(vol + r00 + X.i1);
    const float c = __ldg(vol + r10 + X.i0), e = __ldg(vol + r10 + X.i1);
    const float f = __ldg(vol + r01 + X.i0), h = __ldg(vol + r01 + X.i1);
    const float k = __ldg(vol + r11 + X.i0), l = __ldg(vol + r11 + X.i1);
    const float d00 = b - a, d10 = e - c, d01 = h - f, d11 = l - k;
    const float v00 = fmaf(X.t, d00, a), v10 = fmaf(X.t, d10, c);
    const float v01 = fmaf(X.t, d01, f), v11 = fmaf(X.t, d11, k);
    const float s0 = fmaf(Y.t, v10 - v00, v00), s1 = fmaf(Y.t, v11 - v01, v01);
    const float gx0 = fmaf(Y.t, d10 - d00, d00), gx1 = fmaf(Y.t, d11 - d01, d01);
    gx = X.outside ? 0.f : fmaf(Z.t, gx1 - gx0, gx0);
    const float gy0 = v10 - v00, gy1 = v11 - v01;
    gy = Y.outside ? 0.f : fmaf(Z.t, gy1 - gy0, gy0);
    gz = Z.outside ? 0.f : s1 - s0;
    return fmaf(Z.t, s1 - s0, s0);
}

// Value only (field.cpp:43-45 / sample_field :92-121 per component).
struct Cell {
    int o000, o100, o010, o110, o001, o101, o011, o111;
    float tx, ty, tz;
    bool finite;
};

__device__ __forceinline__ Cell make_cell(const Geo& g, int x, int y, int z, float ux, float uy,
                                          float uz) {
    Cell c;
    c.finite = isfinite(ux) && isfinite(uy) && isfinite(uz);
    const AxisTap X = axis_tap(x, c.finite ? ux : 0.f, g.nx);
    const AxisTap Y = axis_tap(y, c.finite ? uy : 0.f, g.ny);
    const AxisTap Z = axis_tap(z, c.finite ? uz : 0.f, g.nz);
    const int r00 = g.nx * (Y.i0 + g.ny * Z.i0);
    const int r10 = g.nx * (Y.i1 + g.ny * Z.i0);
    const int r01 = g.nx * (Y.i0 + g.ny * Z.i1);
    const int r11 = g.nx * (Y.i1 + g.ny * Z.i1);
    c.o000 = r00 + X.i0; c.o100 = r00 + X.i1; c.o010 = r10 + X.i0; c.o110 = r10 + X.i1;
    c.o001 = r01 + X.i0; c.o101 = r01 + X.i1; c.o011 = r11 + X.i0; c.o111 = r11 + X.i1;
    c.tx = X.t; c.ty = Y.t; c.tz = Z.t;
    return c;
}

__device__ __forceinline__ float cell_sample(const float* __restrict__ v, const Cell& c) {
    if (!c.finite) return __int_as_float(0x7fc00000);
    const float a = __ldg(v + c.o000), b = __ldg(v + c.o100);
    const float cc = __ldg(v + c.o010), e = __ldg(v + c.o110);
    const float f = __ldg(v + c.o001), h = __ldg(v + c.o101);
    const float k = __ldg(v + c.o011), l = __ldg(v + c.o111);
    const float v00 = fmaf(c.tx, b - a, a), v10 = fmaf(c.tx, e - cc, cc);
    const float v01 = fmaf(c.tx, h - f, f), v11 = fmaf(c.tx, l - k, k);
    const float s0 = fmaf(c.ty, v10 - v00, v00), s1 = fmaf(c.ty, v11 - v01, v01);
    return fmaf(c.tz, s1 - s0, s0);
}

// fp64 variants for the LNCC path.  The interpolated intensities feed window
// variances of O(noise^2); an fp32 lerp error (~1e-7 absolute) is 1e-5 of a
// 0.01 deviation, so M(x + u) and its gradient are evaluated in fp64 from the
// fp32 samples.  With u fp32, t = u - floor(u) is exact in fp64, so this is
// the fp64 reference's sample for the same warp.
struct AxisTapD {
    int i0, i1;
    double t;
    bool outside;
};

__device__ __forceinline__ AxisTapD axis_tap_dd(int x, float u, int n) {
    AxisTapD a;
    if (n == 1) { a.i0 = a.i1 = 0; a.t = 0.0; a.outside = true; return a; }
    const double ud = (double)u;
    const double fl = floor(ud);
    const int i = x + (int)fl;
    const double t = ud - fl;  // exact
    if (i < 0) { a.i0 = 0; a.i1 = 1; a.t = 0.0; a.outside = true; return a; }
    if (i > n - 1 || (i == n - 1 && t > 0.0)) {
        a.i0 = n - 2; a.i1 = n - 1; a.t = 1.0; a.outside = true; return a;
    }
    if (i == n - 1) { a.i0 = n - 2; a.i1 = n - 1; a.t = 1.0; a.outside = false; return a; }
    a.i0 = i; a.i1 = i + 1; a.t = t; a.outside = false;
    return a;
}

// Value (and optionally the analytic gradient) of vol at (x,y,z) + u in fp64,
// collapse order of field.cpp:47-90.
template <bool GRAD>
__device__ __forceinline__ double sample_d(const float* __restrict__ vol, const Geo& g, int x, int y,
                                           int z, float ux, float uy, float uz, double* grad) {
    if (!(isfinite(ux) && isfinite(uy) && isfinite(uz))) {
        if (GRAD) grad[0] = grad[1] = grad[2] = 0.0;
        return __longlong_as_double(0x7ff8000000000000ll);
    }
    const AxisTapD X = axis_tap_dd(x, ux, g.nx), Y = axis_tap_dd(y, uy, g.ny), Z = axis_tap_dd(z, uz, g.nz);
    const int r00 = g.nx * (Y.i0 + g.ny * Z.i0);
    const int r10 = g.nx * (Y.i1 + g.ny * Z.i0);
    const int r01 = g.nx * (Y.i0 + g.ny * Z.i1);
    const int r11 = g.nx * (Y.i1 + g.ny * Z.i1);
    const double a = __ldg(vol + r00 + X.i0), b = __ldg(vol + r00 + X.i1);
    const double c = __ldg(vol + r10 + X.i0), e = __ldg(vol + r10 + X.i1);
    const double f = __ldg(vol + r01 + X.i0), h = __ldg(vol + r01 + X.i1);
    const double k = __ldg(vol + r11 + X.i0), l = __ldg(vol + r11 + X.i1);
    const double d00 = b - a, d10 = e - c, d01 = h - f, d11 = l - k;
    const double v00 = fma(X.t, d00, a), v10 = fma(X.t, d10, c);
    const double v01 = fma(X.t, d01, f), v11 = fma(X.t, d11, k);
    const double s0 = fma(Y.t, v10 - v00, v00), s1 = fma(Y.t, v11 - v01, v01);
    if (GRAD) {
        const double gx0 = fma(Y.t, d10 - d00, d00), gx1 = fma(Y.t, d11 - d01, d01);
        grad[0] = X.outside ? 0.0 : fma(Z.t, gx1 - gx0, gx0);
        const double gy0 = v10 - v00, gy1 = v11 - v01;
        grad[1] = Y.outside ? 0.0 : fma(Z.t, gy1 - gy0, gy0);
        grad[2] = Z.outside ? 0.0 : s1 - s0;
    }
    return fma(Z.t, s1 - s0, s0);
}

// fp64 three-component sample of an SoA field at (x,y,z) + d with d in fp64
// (sample_field, field.cpp:92-121), for the compositive resample.
__device__ __forceinline__ AxisTapD axis_tap_dd(int x, double u, int n) {
    AxisTapD a;
    if (n == 1) { a.i0 = a.i1 = 0; a.t = 0.0; a.outside = true; return a; }
    const double fl = floor(u);
    const int i = x + (int)fl;
    const double t = u - fl;
    if (i < 0) { a.i0 = 0; a.i1 = 1; a.t = 0.0; a.outside = true; return a; }
    if (i > n - 1 || (i == n - 1 && t > 0.0)) {
        a.i0 = n - 2; a.i1 = n - 1; a.t = 1.0; a.outside = true; return a;
    }
    if (i == n - 1) { a.i0 = n - 2; a.i1 = n - 1; a.t = 1.0; a.outside = false; return a; }
    a.i0 = i; a.i1 = i + 1; a.t = t; a.outside = false;
    return a;
}

__device__ __forceinline__ void sample3_d(const float* __restrict__ u, long long n, const Geo& g,
                                          int x, int y, int z, double dx, double dy, double dz,
                                          double* out) {
    if (!(isfinite(dx) && isfinite(dy) && isfinite(dz))) {
        out[0] = out[1] = out[2] = __longlong_as_double(0x7ff8000000000000ll);
        return;
    }
    const AxisTapD X = axis_tap_dd(x, dx, g.nx), Y = axis_tap_dd(y, dy, g.ny), Z = axis_tap_dd(z, dz, g.nz);
    const int r00 = g.nx * (Y.i0 + g.ny * Z.i0);
    const int r10 = g.nx * (Y.i1 + g.ny * Z.i0);
    const int r01 = g.nx * (Y.i0 + g.ny * Z.i1);
    const int r11 = g.nx * (Y.i1 + g.ny * Z.i1);
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
        const float* v = u + ch * n;
        const double a = __ldg(v + r00 + X.i0), b = __ldg(v + r00 + X.i1);
        const double c = __ldg(v + r10 + X.i0), e = __ldg(v + r10 + X.i1);
        const double f = __ldg(v + r01 + X.i0), h = __ldg(v + r01 + X.i1);
        const double k = __ldg(v + r11 + X.i0), l = __ldg(v + r11 + X.i1);
        const double v00 = fma(X.t, b - a, a), v10 = fma(X.t, e - c, c);
        const double v01 = fma(X.t, h - f, f), v11 = fma(X.t, l - k, k);
        const double s0 = fma(Y.t, v10 - v00, v00), s1 = fma(Y.t, v11 - v01, v01);
        out[ch] = fma(Z.t, s1 - s0, s0);
    }
}

// Non-negative float max via ordered unsigned bits (exact, order-free).
__device__ __forceinline__ void atomic_max_nonneg(unsigned* addr, float v) {
    atomicMax(addr, __float_as_uint(v));
}
// Signed float min via the order-preserving int mapping.
__device__ __forceinline__ int float_to_ordered(float f) {
    const int i = __float_as_int(f);
    return i >= 0 ? i : i ^ 0x7fffffff;
}
__host__ __device__ inline float ordered_to_float(int i) {
#ifdef __CUDA_ARCH__
    return __int_as_float(i >= 0 ? i : i ^ 0x7fffffff);
#else
    union { int i; float f; } u;
    u.i = i >= 0 ? i : i ^ 0x7fffffff;
    return u.f;
#endif
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Per-axis Gaussian weight normaliser for the truncated, renormalised kernel
// (field.cpp:236-244): sum of the taps that fall inside [0, n-1].
__device__ __forceinline__ float axis_wsum(int p, int n, int R, const float* w, float full) {
    if (p >= R && p + R <= n - 1) return full;
    float s = 0.f;
    for (int d = -R; d <= R; ++d) {
        const int q = p + d;
        if (q >= 0 && q < n) s += w[d < 0 ? -d : d];
    }
    return s;
}
// Box-window voxel count along one axis (truncated window, A2).
__device__ __forceinline__ int axis_count(int p, int n, int R) {
    return min(n - 1, p + R) - max(0, p - R) + 1;
}

}  // namespace wlm
