// field64.cu -- fp64 device versions of the reference `field` module
// (field.hpp:82-117) for the host-buffer mirror entry points, plus fp64
// pyramid helpers.
//
// Data stay fp64 and in the caller's layout (x-fastest, component-innermost
// AoS, field.hpp:57), and every kernel evaluates the reference's expressions
// in the reference's operation order with explicitly rounded operations
// (__dmul_rn / __dadd_rn / __ddiv_rn: no fused multiply-adds, IEEE division),
// so a mirror call returns the reference function's bits, not an fp32
// approximation of them:
//   resolve_axis / sample_trilinear_grad / sample_field   field.cpp:19-121
//   compose_warp                                          field.cpp:123-142
//   max_abs_component / normalize_step                    field.cpp:144-155
//   jacobian_det_min                                      field.cpp:157-201
//   gaussian_smooth (separable, per-output renormalised)  field.cpp:203-269
// The hot path does not use these (it computes on fp32 storage in fused
// kernels, hot_kernels.cu); the engine's generic-radius smoothing does.
#include <cmath>
#include <vector>

#include "internal.cuh"

namespace wlm {

namespace {

struct Axis64 {
    int i0, i1;
    double t;
    bool clamped;
};

// field.cpp:19-39
__device__ __forceinline__ Axis64 resolve_axis64(double p, int n) {
    Axis64 a{0, 0, 0.0, false};
    if (n == 1) {
        a.clamped = true;
        return a;
    }
    double c = p;
    if (c <= 0.0) {
        a.clamped = c < 0.0;
        c = 0.0;
    } else if (c >= (double)(n - 1)) {
        a.clamped = c > (double)(n - 1);
        c = (double)(n - 1);
    }
    int i0 = (int)c;
    if (i0 > n - 2) i0 = n - 2;
    a.i0 = i0;
    a.i1 = i0 + 1;
    a.t = __dsub_rn(c, (double)i0);
    return a;
}

__device__ __forceinline__ double lerp_ref(double a, double t, double d) { return __dadd_rn(a, __dmul_rn(t, d)); }

// field.cpp:47-90 on an fp64 volume (value + analytic interpolant gradient)
__device__ double sample_grad64(const double* __restrict__ v, int nx, int ny, int nz, double px, double py,
                                double pz, double* g) {
    if (!isfinite(px) || !isfinite(py) || !isfinite(pz)) {
        g[0] = g[1] = g[2] = 0.0;
        return __longlong_as_double(0x7ff8000000000000ll);
    }
    const Axis64 ax = resolve_axis64(px, nx), ay = resolve_axis64(py, ny), az = resolve_axis64(pz, nz);
    auto at = [&](int x, int y, int z) { return v[(long long)x + (long long)nx * ((long long)y + (long long)ny * z)]; };
    const double c000 = at(ax.i0, ay.i0, az.i0), c100 = at(ax.i1, ay.i0, az.i0);
    const double c010 = at(ax.i0, ay.i1, az.i0), c110 = at(ax.i1, ay.i1, az.i0);
    const double c001 = at(ax.i0, ay.i0, az.i1), c101 = at(ax.i1, ay.i0, az.i1);
    const double c011 = at(ax.i0, ay.i1, az.i1), c111 = at(ax.i1, ay.i1, az.i1);
    const double tx = ax.t, ty = ay.t, tz = az.t;
    const double d00 = __dsub_rn(c100, c000), d10 = __dsub_rn(c110, c010);
    const double d01 = __dsub_rn(c101, c001), d11 = __dsub_rn(c111, c011);
    const double v00 = lerp_ref(c000, tx, d00), v10 = lerp_ref(c010, tx, d10);
    const double v01 = lerp_ref(c001, tx, d01), v11 = lerp_ref(c011, tx, d11);
    const double v0 = lerp_ref(v00, ty, __dsub_rn(v10, v00));
    const double v1 = lerp_ref(v01, ty, __dsub_rn(v11, v01));
    const double value = lerp_ref(v0, tz, __dsub_rn(v1, v0));
    const double gx0 = lerp_ref(d00, ty, __dsub_rn(d10, d00));
    const double gx1 = lerp_ref(d01, ty, __dsub_rn(d11, d01));
    g[0] = ax.clamped ? 0.0 : lerp_ref(gx0, tz, __dsub_rn(gx1, gx0));
    const double gy0 = __dsub_rn(v10, v00), gy1 = __dsub_rn(v11, v01);
    g[1] = ay.clamped ? 0.0 : lerp_ref(gy0, tz, __dsub_rn(gy1, gy0));
    g[2] = az.clamped ? 0.0 : __dsub_rn(v1, v0);
    return value;
}

// field.cpp:92-121 on an fp64 AoS field
__device__ void sample_field64(const double* __restrict__ u, int nx, int ny, int nz, double px, double py,
                               double pz, double* out) {
    if (!isfinite(px) || !isfinite(py) || !isfinite(pz)) {
        out[0] = out[1] = out[2] = __longlong_as_double(0x7ff8000000000000ll);
        return;
    }
    const Axis64 ax = resolve_axis64(px, nx), ay = resolve_axis64(py, ny), az = resolve_axis64(pz, nz);
    const double tx = ax.t, ty = ay.t, tz = az.t;
    auto at = [&](int x, int y, int z, int c) {
        return u[3 * ((long long)x + (long long)nx * ((long long)y + (long long)ny * z)) + c];
    };
    for (int c = 0; c < 3; ++c) {
        const double c000 = at(ax.i0, ay.i0, az.i0, c), c100 = at(ax.i1, ay.i0, az.i0, c);
        const double c010 = at(ax.i0, ay.i1, az.i0, c), c110 = at(ax.i1, ay.i1, az.i0, c);
        const double c001 = at(ax.i0, ay.i0, az.i1, c), c101 = at(ax.i1, ay.i0, az.i1, c);
        const double c011 = at(ax.i0, ay.i1, az.i1, c), c111 = at(ax.i1, ay.i1, az.i1, c);
        const double v00 = lerp_ref(c000, tx, __dsub_rn(c100, c000));
        const double v10 = lerp_ref(c010, tx, __dsub_rn(c110, c010));
        const double v01 = lerp_ref(c001, tx, __dsub_rn(c101, c001));
        const double v11 = lerp_ref(c011, tx, __dsub_rn(c111, c011));
        const double v0 = lerp_ref(v00, ty, __dsub_rn(v10, v00));
        const double v1 = lerp_ref(v01, ty, __dsub_rn(v11, v01));
        out[c] = lerp_ref(v0, tz, __dsub_rn(v1, v0));
    }
}

inline int grid_1d(long long n) { return (int)std::min<long long>(148 * 32, std::max<long long>(1, (n + 255) / 256)); }

#define WLM_GRID_STRIDE(i, n) \
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < (n); i += (long long)gridDim.x * blockDim.x)

__global__ void k_warp_volume64(const double* __restrict__ M, const double* __restrict__ u, wlm_dims d,
                                double* __restrict__ Mw, double* __restrict__ gM) {
    const long long n = (long long)d.nx * d.ny * d.nz;
    WLM_GRID_STRIDE(i, n) {
        const int x = (int)(i % d.nx), y = (int)((i / d.nx) % d.ny), z = (int)(i / ((long long)d.nx * d.ny));
        double g[3];
        // ref_warp_volume: sample at (x + u_x, y + u_y, z + u_z)
        Mw[i] = sample_grad64(M, d.nx, d.ny, d.nz, __dadd_rn((double)x, u[3 * i]), __dadd_rn((double)y, u[3 * i + 1]),
                              __dadd_rn((double)z, u[3 * i + 2]), g);
        if (gM) {
            gM[3 * i] = g[0];
            gM[3 * i + 1] = g[1];
            gM[3 * i + 2] = g[2];
        }
    }
}

__global__ void k_compose64(const double* __restrict__ u, const double* __restrict__ v, double eps, wlm_dims d,
                            double* __restrict__ out) {
    const long long n = (long long)d.nx * d.ny * d.nz;
    WLM_GRID_STRIDE(i, n) {
        const int x = (int)(i % d.nx), y = (int)((i / d.nx) % d.ny), z = (int)(i / ((long long)d.nx * d.ny));
        const double sx = __dmul_rn(eps, v[3 * i]), sy = __dmul_rn(eps, v[3 * i + 1]), sz = __dmul_rn(eps, v[3 * i + 2]);
        double s[3];
        sample_field64(u, d.nx, d.ny, d.nz, __dadd_rn((double)x, sx), __dadd_rn((double)y, sy),
                       __dadd_rn((double)z, sz), s);
        out[3 * i] = __dadd_rn(sx, s[0]);
        out[3 * i + 1] = __dadd_rn(sy, s[1]);
        out[3 * i + 2] = __dadd_rn(sz, s[2]);
    }
}

__global__ void k_sample_points64(const double* __restrict__ u, wlm_dims d, const double* __restrict__ pts,
                                  long long npts, double* __restrict__ out) {
    WLM_GRID_STRIDE(i, npts) {
        sample_field64(u, d.nx, d.ny, d.nz, pts[3 * i], pts[3 * i + 1], pts[3 * i + 2], out + 3 * i);
    }
}

__global__ void k_sample_grad_points64(const double* __restrict__ v, wlm_dims d, const double* __restrict__ pts,
                                       long long npts, double* __restrict__ val, double* __restrict__ grad) {
    WLM_GRID_STRIDE(i, npts) {
        double g[3];
        val[i] = sample_grad64(v, d.nx, d.ny, d.nz, pts[3 * i], pts[3 * i + 1], pts[3 * i + 2], g);
        if (grad) {
            grad[3 * i] = g[0];
            grad[3 * i + 1] = g[1];
            grad[3 * i + 2] = g[2];
        }
    }
}

// Non-negative doubles order like their bit patterns: exact, order-free max.
__global__ void k_max_abs64(const double* __restrict__ v, long long count, unsigned long long* out) {
    double m = 0.0;
    WLM_GRID_STRIDE(i, count) m = fmax(m, fabs(v[i]));
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

// Ordered 64-bit key of a double (total order of finite values; NaN above +inf).
__device__ __forceinline__ unsigned long long dkey(double v) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(v);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__host__ __device__ inline double dkey_inv(unsigned long long k) {
    const unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
    double v;
    memcpy(&v, &b, 8);
    return v;
}

// field.cpp:157-201: det(I + grad u), central differences, min over the
// interior (the whole axis where n == 2).
// element (voxel i, component c) of an fp64 AoS field or of an fp32 SoA
// field (the engine's warp, widened exactly)
struct Aos64 {
    const double* u;
    __device__ double operator()(long long i, int c, long long) const { return u[3 * i + c]; }
};
struct Soa32 {
    const float* u;
    __device__ double operator()(long long i, int c, long long n) const { return (double)u[c * n + i]; }
};

template <class Acc>
__device__ __forceinline__ double axis_derivative64(const Acc& u, wlm_dims d, int x, int y, int z, int c, int axis) {
    const int n = axis == 0 ? d.nx : axis == 1 ? d.ny : d.nz;
    const int p = axis == 0 ? x : axis == 1 ? y : z;
    const long long nv = (long long)d.nx * d.ny * d.nz;
    auto value = [&](int q) {
        const int xx = axis == 0 ? q : x, yy = axis == 1 ? q : y, zz = axis == 2 ? q : z;
        return u((long long)xx + (long long)d.nx * ((long long)yy + (long long)d.ny * zz), c, nv);
    };
    if (p >= 1 && p + 1 <= n - 1) return __dmul_rn(0.5, __dsub_rn(value(p + 1), value(p - 1)));
    if (p == 0) return __dsub_rn(value(1), value(0));
    return __dsub_rn(value(p), value(p - 1));
}

template <class Acc>
__global__ void k_jacobian_min64(Acc u, wlm_dims d, unsigned long long* out) {
    const int x0 = d.nx >= 3 ? 1 : 0, x1 = d.nx >= 3 ? d.nx - 2 : d.nx - 1;
    const int y0 = d.ny >= 3 ? 1 : 0, y1 = d.ny >= 3 ? d.ny - 2 : d.ny - 1;
    const int z0 = d.nz >= 3 ? 1 : 0, z1 = d.nz >= 3 ? d.nz - 2 : d.nz - 1;
    const long long wx = x1 - x0 + 1, wy = y1 - y0 + 1, wz = z1 - z0 + 1;
    unsigned long long best = dkey(__longlong_as_double(0x7ff0000000000000ll));  // +inf
    WLM_GRID_STRIDE(i, wx * wy * wz) {
        const int x = x0 + (int)(i % wx), y = y0 + (int)((i / wx) % wy), z = z0 + (int)(i / (wx * wy));
        double J[3][3];
        for (int c = 0; c < 3; ++c) {
            for (int a = 0; a < 3; ++a) J[c][a] = axis_derivative64(u, d, x, y, z, c, a);
            J[c][c] = __dadd_rn(J[c][c], 1.0);
        }
        const double t0 = __dmul_rn(J[0][0], __dsub_rn(__dmul_rn(J[1][1], J[2][2]), __dmul_rn(J[1][2], J[2][1])));
        const double t1 = __dmul_rn(J[0][1], __dsub_rn(__dmul_rn(J[1][0], J[2][2]), __dmul_rn(J[1][2], J[2][0])));
        const double t2 = __dmul_rn(J[0][2], __dsub_rn(__dmul_rn(J[1][0], J[2][1]), __dmul_rn(J[1][1], J[2][0])));
        const double det = __dadd_rn(__dsub_rn(t0, t1), t2);
        const unsigned long long k = dkey(det);
        best = k < best ? k : best;
    }
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long other = __shfl_xor_sync(0xffffffffu, best, o);
        best = other < best ? other : best;
    }
    if ((threadIdx.x & 31) == 0) atomicMin(out, best);
}

// One separable pass of field.cpp:217-248 along `axis` of an nchan-channel
// field (element (p, c) at base + c * cstride + p * estride): the in-bounds
// taps accumulate acc += w * x and wsum += w in tap order, out = acc / wsum.
__global__ void k_smooth_axis64(const double* __restrict__ in, double* __restrict__ out, wlm_dims d, int nchan,
                                long long cstride, long long estride, int axis, const double* __restrict__ w, int R) {
    const long long n = (long long)d.nx * d.ny * d.nz;
    const int na = axis == 0 ? d.nx : axis == 1 ? d.ny : d.nz;
    const long long st = axis == 0 ? 1 : axis == 1 ? d.nx : (long long)d.nx * d.ny;
    WLM_GRID_STRIDE(j, n * nchan) {
        const int c = (int)(j / n);
        const long long i = j % n;
        const long long base = c * cstride;
        const int p = axis == 0 ? (int)(i % d.nx) : axis == 1 ? (int)((i / d.nx) % d.ny)
                                                            : (int)(i / ((long long)d.nx * d.ny));
        if (na == 1) {
            out[base + i * estride] = in[base + i * estride];
            continue;
        }
        const int lo = max(0, p - R), hi = min(na - 1, p + R);
        double acc = 0.0, wsum = 0.0;
        for (int q = lo; q <= hi; ++q) {
            const double wq = w[q - p + R];
            acc = __dadd_rn(acc, __dmul_rn(wq, in[base + (i + (long long)(q - p) * st) * estride]));
            wsum = __dadd_rn(wsum, wq);
        }
        out[base + i * estride] = __ddiv_rn(acc, wsum);
    }
}

// orc_lm_step_pointwise / SPEC.md:250: s = -r / (|g|^2 + lambda), out = s g
__global__ void k_lm_step64(double r, const double* __restrict__ g, long long n, double lambda,
                            double* __restrict__ out) {
    WLM_GRID_STRIDE(i, n) {
        const double gx = g[3 * i], gy = g[3 * i + 1], gz = g[3 * i + 2];
        const double nn = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(gx, gx), __dmul_rn(gy, gy)), __dmul_rn(gz, gz)),
                                    lambda);
        const double s = __ddiv_rn(-r, nn);
        out[3 * i] = __dmul_rn(s, gx);
        out[3 * i + 1] = __dmul_rn(s, gy);
        out[3 * i + 2] = __dmul_rn(s, gz);
    }
}

// downsample's stride: coarse i <- fine i * f
__global__ void k_stride64(const double* __restrict__ in, wlm_dims d, int f, double* __restrict__ out, wlm_dims nd) {
    const long long n = (long long)nd.nx * nd.ny * nd.nz;
    WLM_GRID_STRIDE(i, n) {
        const int x = (int)(i % nd.nx), y = (int)((i / nd.nx) % nd.ny), z = (int)(i / ((long long)nd.nx * nd.ny));
        out[i] = in[(long long)x * f + (long long)d.nx * ((long long)y * f + (long long)d.ny * ((long long)z * f))];
    }
}

// upsample_warp: sample at x / scale, times scale
__global__ void k_upsample64(const double* __restrict__ u, wlm_dims d, wlm_dims nd, double scale,
                             double* __restrict__ out) {
    const long long n = (long long)nd.nx * nd.ny * nd.nz;
    WLM_GRID_STRIDE(i, n) {
        const int x = (int)(i % nd.nx), y = (int)((i / nd.nx) % nd.ny), z = (int)(i / ((long long)nd.nx * nd.ny));
        double s[3];
        sample_field64(u, d.nx, d.ny, d.nz, __ddiv_rn((double)x, scale), __ddiv_rn((double)y, scale),
                       __ddiv_rn((double)z, scale), s);
        out[3 * i] = __dmul_rn(scale, s[0]);
        out[3 * i + 1] = __dmul_rn(scale, s[1]);
        out[3 * i + 2] = __dmul_rn(scale, s[2]);
    }
}

}  // namespace

// field.cpp:205-213: radius max(1, ceil(3 sigma)), w_i = exp(-i^2 / 2 sigma^2)
std::vector<double> gaussian_taps64(double sigma, int* R) {
    int r = (int)std::ceil(3.0 * sigma);
    if (r < 1) r = 1;
    std::vector<double> w(2 * r + 1);
    for (int i = -r; i <= r; ++i) w[i + r] = std::exp(-0.5 * (i * i) / (sigma * sigma));
    *R = r;
    return w;
}

void launch_warp_volume64(const double* M, const double* u, wlm_dims d, double* Mw, double* gM, cudaStream_t s) {
    k_warp_volume64<<<grid_1d((long long)nvox(d)), 256, 0, s>>>(M, u, d, Mw, gM);
    ++g_kernel_launches;
}

void launch_compose64(const double* u, const double* v, double eps, wlm_dims d, double* out, cudaStream_t s) {
    k_compose64<<<grid_1d((long long)nvox(d)), 256, 0, s>>>(u, v, eps, d, out);
    ++g_kernel_launches;
}

void launch_sample_points64(const double* u, wlm_dims d, const double* pts, long long npts, double* out,
                            cudaStream_t s) {
    k_sample_points64<<<grid_1d(npts), 256, 0, s>>>(u, d, pts, npts, out);
    ++g_kernel_launches;
}

void launch_sample_grad_points64(const double* v, wlm_dims d, const double* pts, long long npts, double* val,
                                 double* grad, cudaStream_t s) {
    k_sample_grad_points64<<<grid_1d(npts), 256, 0, s>>>(v, d, pts, npts, val, grad);
    ++g_kernel_launches;
}

void launch_max_abs64(const double* v, long long count, unsigned long long* out, cudaStream_t s) {
    k_max_abs64<<<grid_1d(count), 256, 0, s>>>(v, count, out);
    ++g_kernel_launches;
}

void launch_jacobian_min64(const double* u, wlm_dims d, unsigned long long* out, cudaStream_t s) {
    k_jacobian_min64<<<grid_1d((long long)nvox(d)), 256, 0, s>>>(Aos64{u}, d, out);
    ++g_kernel_launches;
}

void launch_jacobian_min64_soa32(const float* u, wlm_dims d, unsigned long long* out, cudaStream_t s) {
    k_jacobian_min64<<<grid_1d((long long)nvox(d)), 256, 0, s>>>(Soa32{u}, d, out);
    ++g_kernel_launches;
}

double jacobian_key_to_double(unsigned long long k) { return dkey_inv(k); }
unsigned long long jacobian_key_init() {
    return 0xfff0000000000000ull;  // dkey(+inf): +inf bits with the sign bit set
}

// x, y, z passes in turn between two buffers; the result ends in `data`.
void smooth64(double* data, double* tmp, const double* dw, int R, wlm_dims d, int nchan, long long cstride,
              long long estride, cudaStream_t s) {
    const long long n = (long long)nvox(d) * nchan;
    k_smooth_axis64<<<grid_1d(n), 256, 0, s>>>(data, tmp, d, nchan, cstride, estride, 0, dw, R);
    k_smooth_axis64<<<grid_1d(n), 256, 0, s>>>(tmp, data, d, nchan, cstride, estride, 1, dw, R);
    k_smooth_axis64<<<grid_1d(n), 256, 0, s>>>(data, tmp, d, nchan, cstride, estride, 2, dw, R);
    cudaMemcpyAsync(data, tmp, sizeof(double) * n, cudaMemcpyDeviceToDevice, s);
    g_kernel_launches += 3;
}

void launch_lm_step64(double r, const double* g, long long n, double lambda, double* out, cudaStream_t s) {
    k_lm_step64<<<grid_1d(n), 256, 0, s>>>(r, g, n, lambda, out);
    ++g_kernel_launches;
}

void launch_stride64(const double* in, wlm_dims d, int f, double* out, wlm_dims nd, cudaStream_t s) {
    k_stride64<<<grid_1d((long long)nvox(nd)), 256, 0, s>>>(in, d, f, out, nd);
    ++g_kernel_launches;
}

void launch_upsample64(const double* u, wlm_dims d, wlm_dims nd, double scale, double* out, cudaStream_t s) {
    k_upsample64<<<grid_1d((long long)nvox(nd)), 256, 0, s>>>(u, d, nd, scale, out);
    ++g_kernel_launches;
}

}  // namespace wlm
