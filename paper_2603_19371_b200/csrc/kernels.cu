// kernels.cu -- the per-iteration support kernels of the factored-LM
// iteration (Adam step, Jacobian diagnostic, level / iteration state, the
// intensity shifts, tiled-LM matrices, Demons), the pyramid kernels, the
// synth_pair helpers (fp32 smoothing, max, Jacobian) and the layout
// conversions.  The stencil kernels K1-K4 are in hot_kernels.cu, the fp64
// field mirrors in field64.cu, the generic-radius paths in generic.cu.
//
// All hot-path kernels share one z-marching separable-stencil schedule: a
// CTA owns a 32 x TY column of output voxels and a chunk of z planes; each
// input plane (with an R-voxel x/y halo) is produced once into shared memory,
// filtered along x then y from shared memory, and the filtered column enters a
// register ring of 2R+1 planes that is filtered along z.  Every global
// read/write is a unit-stride row of one SoA plane (coalesced), the halo
// overlap between neighbouring CTAs is served by L2, and there are no float
// atomics: sums are per-CTA fp64 partials reduced in a fixed order, one CTA
// per plane (deterministic), maxima use exact
// ordered-integer atomics.
#include <algorithm>
#include <cfloat>
#include <climits>
#include <cmath>

#include "kernels.cuh"

namespace wlm {

uint64_t g_kernel_launches = 0;

namespace {
constexpr int TX = 32;
constexpr int TY = 8;
constexpr int NT = TX * TY;
constexpr int kNumSMs = 148;

__host__ __device__ inline int cdiv(int a, int b) { return (a + b - 1) / b; }
}  // namespace

dim3 LaunchShape::grid() const { return dim3(tiles_x * tiles_y, chunks, 1); }

LaunchShape shape_for(const Geo& g, int pairs, int ty, int ctas_per_sm) {
    LaunchShape s;
    s.tiles_x = cdiv(g.nx, TX);
    s.tiles_y = cdiv(g.ny, ty);
    const long long tiles = (long long)s.tiles_x * s.tiles_y * pairs;
    // chunks of the owned planes: aim for ~4 CTAs per SM worth of work (a
    // pair group, whose tails the other group fills, aims for 1: every
    // chunk re-reads 2R halo planes); keep >= 8 planes a chunk
    const int nzo = g.ze - g.zs;
    const long long want = (long long)kNumSMs * (ctas_per_sm > 0 ? ctas_per_sm : 4);
    int chunks = (int)std::max<long long>(1, std::min<long long>(nzo, (want + tiles - 1) / tiles));
    int len = cdiv(nzo, chunks);
    len = std::max(len, std::min(nzo, 8));
    s.chunk_len = len;
    s.chunks = cdiv(nzo, len);
    return s;
}

// Block-wide fixed-order double sum (result valid in thread 0).
__device__ double block_sum(double v, double* red) {
    v = warp_sum(v);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) red[w] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0)
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i];
    __syncthreads();
    return s;
}

// Adam, pointwise; t = accepted iterations + 1 at this level.
// fp64 arithmetic with fp32 storage of m, v and the step, in the oracle's
// operation order (orc_adam_step: no fused multiply-adds, IEEE division and
// square root, bias corrections from the host's std::pow), so the stored
// values are the fp32-storage oracle's bit for bit.
__global__ void k_adam(Batch b, LmParams p) {
    const int pair = b.pair0 + blockIdx.y;
    const PairState* st = b.st + pair;
    if (st->done) return;
    const long long n = b.g.n, n3 = 3 * n;
    float* G = b.G + (long long)pair * n3;
    float* Mm = b.AM + (long long)pair * n3;
    float* Vv = b.AV + (long long)pair * n3;
    const int t = min(st->iter + 1, p.adam_bc_n);
    const double b1 = p.adam_b1, b2 = p.adam_b2;
    const double c1 = __dadd_rn(1.0, -b1), c2 = __dadd_rn(1.0, -b2);
    const double bc1 = p.adam_bc[t - 1], bc2 = p.adam_bc[p.adam_bc_n + t - 1];
    const double lr = p.adam_lr, ep = p.adam_eps;
    // owned planes of each component (slab halos are refreshed by exchange)
    const long long nxy = (long long)b.g.nx * b.g.ny;
    const long long lo = (b.g.zs - b.g.zlo) * nxy, cnt = (b.g.ze - b.g.zs) * nxy;
    for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < 3 * cnt;
         j += (long long)gridDim.x * blockDim.x) {
        const long long i = (j / cnt) * n + lo + j % cnt;
        const double gi = G[i];
        const float m = (float)__dadd_rn(__dmul_rn(b1, (double)Mm[i]), __dmul_rn(c1, gi));
        const float v = (float)__dadd_rn(__dmul_rn(b2, (double)Vv[i]), __dmul_rn(__dmul_rn(c2, gi), gi));
        Mm[i] = m;
        Vv[i] = v;
        const double mh = __ddiv_rn((double)m, bc1), vh = __ddiv_rn((double)v, bc2);
        G[i] = (float)__ddiv_rn(__dmul_rn(-lr, mh), __dadd_rn(__dsqrt_rn(vh), ep));
    }
}

// det(I + grad d) at (x,y,z) of an SoA field scaled by `scale`, central
// differences, one-sided only on 2-voxel axes (field.cpp:157-201).
__device__ float det_at(const float* U, const Geo& g, int x, int y, int z, float scale) {
    const int p[3] = {x, y, z};
    const int nn[3] = {g.nx, g.ny, g.nz};
    float J[3][3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        int q1[3] = {x, y, z}, q0[3] = {x, y, z};
        float k = 0.5f;
        if (p[a] >= 1 && p[a] + 1 <= nn[a] - 1) { q1[a] = p[a] + 1; q0[a] = p[a] - 1; }
        else if (p[a] == 0) { q1[a] = 1; q0[a] = 0; k = 1.f; }
        else { q1[a] = p[a]; q0[a] = p[a] - 1; k = 1.f; }
        const int i1 = g.lat(q1[0], q1[1], q1[2]), i0 = g.lat(q0[0], q0[1], q0[2]);
#pragma unroll
        for (int c = 0; c < 3; ++c) J[c][a] = k * scale * (__ldg(U + c * g.n + i1) - __ldg(U + c * g.n + i0));
    }
    J[0][0] += 1.f; J[1][1] += 1.f; J[2][2] += 1.f;
    return J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
           J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
           J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
}

__device__ __forceinline__ void interior(int n, int& lo, int& hi) {
    lo = n >= 3 ? 1 : 0;
    hi = n >= 3 ? n - 2 : n - 1;
}

__global__ void k_jacobian_diag(Batch b, LmParams p) {
    __shared__ float s_min[32];
    const int pair = b.pair0 + blockIdx.y;
    PairState* st = b.st + pair;
    if (st->done) return;
    const Geo g = b.g;
    const float* V = b.VS + (long long)pair * b.vs_ps;
    const double eps = p.target / fmax((double)__uint_as_float(st->max_bits), p.step_floor);
    int xl, xh, yl, yh, zl, zh;
    interior(g.nx, xl, xh); interior(g.ny, yl, yh); interior(g.nz, zl, zh);
    zl = max(zl, g.zs);       // owned planes only (slabs)
    zh = min(zh, g.ze - 1);
    const long long cx = xh - xl + 1, cy = yh - yl + 1, cz = max(zh - zl + 1, 0);
    const long long tot = cx * cy * cz;
    float mn = FLT_MAX;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < tot;
         i += (long long)gridDim.x * blockDim.x) {
        const int x = xl + (int)(i % cx), y = yl + (int)((i / cx) % cy), z = zl + (int)(i / (cx * cy));
        mn = fminf(mn, det_at(V, g, x, y, z, eps));
    }
    for (int o = 16; o > 0; o >>= 1) mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    if ((threadIdx.x & 31) == 0) s_min[threadIdx.x >> 5] = mn;
    __syncthreads();
    if (threadIdx.x == 0) {
        float m = FLT_MAX;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) m = fminf(m, s_min[i]);
        atomicMin(&st->jac_bits, float_to_ordered(m));
    }
}

__global__ void k_loop_cond(const PairState* st, int pairs, cudaGraphConditionalHandle h) {
    int any = 0;
    for (int i = 0; i < pairs; ++i) any |= !st[i].done;
    cudaGraphSetConditional(h, any ? 1u : 0u);
}

__global__ void k_begin_level(PairState* st, int pairs, int level, int reset_lambda, double lambda0) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= pairs) return;
    PairState& s = st[i];
    if (reset_lambda) s.lambda = lambda0;
    s.hist_n = 0; s.L1 = 0.0; s.L2 = 0.0;
    s.iter = 0; s.retries = 0; s.done = 0; s.status = 0; s.trace_len = 0; s.attempt = 0;
    s.last_rejected = 0; s.iters_target = INT_MAX; s.level = level;
    s.max_bits = 0u; s.jac_bits = 0x7f800000;
}

__global__ void k_set_targets(PairState* st, int pairs, int iters) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= pairs) return;
    if (st[i].status != 0) return;
    st[i].iters_target = st[i].iter + iters;
    st[i].done = iters <= 0;
}

// Deterministic per-pair means: fixed chunking into kShiftBlocks CTAs, then a
// fixed-order final sum (independent of scheduling).
constexpr int kShiftBlocks = 256;

// part: [pair][2][kShiftBlocks] sums, then [pair][2][kShiftBlocks][2] (min,
// max) at offset pairs * 2 * kShiftBlocks (the MI normalisation range).
__global__ void k_shift_partials(Batch b, double* part) {
    __shared__ double red[32];
    __shared__ float rmin[32], rmax[32];
    const int pair = blockIdx.y, which = blockIdx.z;
    const long long n = b.g.nfull;  // F, M are whole-volume (replicated across slabs)
    const float* v = (which == 0 ? b.F : b.M) + (long long)pair * n;
    const long long per = (n + kShiftBlocks - 1) / kShiftBlocks;
    const long long lo = blockIdx.x * per, hi = min(n, lo + per);
    double s = 0.0;
    float mn = INFINITY, mx = -INFINITY;
    for (long long i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        const float x = v[i];
        s += (double)x;
        mn = fminf(mn, x);
        mx = fmaxf(mx, x);
    }
    for (int o = 16; o > 0; o >>= 1) {
        mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if ((threadIdx.x & 31) == 0) { rmin[threadIdx.x >> 5] = mn; rmax[threadIdx.x >> 5] = mx; }
    const double t = block_sum(s, red);  // contains __syncthreads
    if (threadIdx.x == 0) {
        part[((long long)pair * 2 + which) * kShiftBlocks + blockIdx.x] = t;
        float a = rmin[0], c = rmax[0];
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) { a = fminf(a, rmin[w]); c = fmaxf(c, rmax[w]); }
        double* mm = part + (long long)b.pairs * 2 * kShiftBlocks;
        mm[(((long long)pair * 2 + which) * kShiftBlocks + blockIdx.x) * 2] = a;
        mm[(((long long)pair * 2 + which) * kShiftBlocks + blockIdx.x) * 2 + 1] = c;
    }
}

__global__ void k_shift_final(Batch b, const double* part) {
    __shared__ double red[32];
    const int pair = blockIdx.x, which = blockIdx.y;
    const double v = threadIdx.x < kShiftBlocks ? part[((long long)pair * 2 + which) * kShiftBlocks + threadIdx.x] : 0.0;
    const double t = block_sum(v, red);
    if (threadIdx.x == 0) {
        const float mean = (float)(t / (double)b.g.nfull);
        const double* mm = part + (long long)b.pairs * 2 * kShiftBlocks + ((long long)pair * 2 + which) * kShiftBlocks * 2;
        double a = mm[0], c = mm[1];
        for (int i = 1; i < kShiftBlocks; ++i) { a = fmin(a, mm[2 * i]); c = fmax(c, mm[2 * i + 1]); }
        PairState& st = b.st[pair];
        if (which == 0) { st.shift_f = mean; st.lo_f = a; st.hi_f = c; }
        else { st.shift_m = mean; st.lo_m = a; st.hi_m = c; }
    }
}

// ---------------------------------------------------------------------------
// launch wrappers
void launch_adam(const Batch& b, const LmParams& p, cudaStream_t s) {
    dim3 grid(kNumSMs * 4, b.pairs);
    k_adam<<<grid, 256, 0, s>>>(b, p);
    ++g_kernel_launches;
}

void launch_jacobian_diag(const Batch& b, const LmParams& p, cudaStream_t s) {
    dim3 grid(kNumSMs * 2, b.pairs);
    k_jacobian_diag<<<grid, 256, 0, s>>>(b, p);
    ++g_kernel_launches;
}

void launch_loop_cond(const Batch& b, cudaGraphConditionalHandle h, cudaStream_t s) {
    k_loop_cond<<<1, 1, 0, s>>>(b.st + b.pair0, b.pairs, h);
    ++g_kernel_launches;
}

void launch_begin_level(const Batch& b, const LmParams&, int level, int reset_lambda, double lambda0,
                        cudaStream_t s) {
    k_begin_level<<<cdiv(b.pairs, 128), 128, 0, s>>>(b.st, b.pairs, level, reset_lambda, lambda0);
    ++g_kernel_launches;
}

void launch_set_targets(const Batch& b, int iters, cudaStream_t s) {
    k_set_targets<<<cdiv(b.pairs, 128), 128, 0, s>>>(b.st, b.pairs, iters);
    ++g_kernel_launches;
}

void launch_shifts(const Batch& b, cudaStream_t s) {
    k_shift_partials<<<dim3(kShiftBlocks, b.pairs, 2), 256, 0, s>>>(b, b.shift_part);
    k_shift_final<<<dim3(b.pairs, 2), kShiftBlocks, 0, s>>>(b, b.shift_part);
    g_kernel_launches += 2;
}

// ===========================================================================
// Standalone field operations (reference field.hpp mirror).

namespace {
__device__ __forceinline__ AxisTap axis_tap_d(double p, int n) {
    const double fl = floor(p);
    const int i = (int)fmax(fmin(fl, 2147483000.0), -2147483000.0);
    AxisTap a;
    if (n == 1) { a.i0 = a.i1 = 0; a.t = 0.f; a.outside = true; return a; }
    const float t = (float)(p - fl);
    if (i < 0) { a.i0 = 0; a.i1 = 1; a.t = 0.f; a.outside = true; return a; }
    if (i > n - 1 || (i == n - 1 && t > 0.f)) { a.i0 = n - 2; a.i1 = n - 1; a.t = 1.f; a.outside = true; return a; }
    if (i == n - 1) { a.i0 = n - 2; a.i1 = n - 1; a.t = 1.f; a.outside = false; return a; }
    a.i0 = i; a.i1 = i + 1; a.t = t; a.outside = false;
    return a;
}

__device__ Cell cell_at_point(const Geo& g, double px, double py, double pz) {
    Cell c;
    c.finite = isfinite(px) && isfinite(py) && isfinite(pz);
    const AxisTap X = axis_tap_d(c.finite ? px : 0.0, g.nx), Y = axis_tap_d(c.finite ? py : 0.0, g.ny),
                  Z = axis_tap_d(c.finite ? pz : 0.0, g.nz);
    const int r00 = g.nx * (Y.i0 + g.ny * Z.i0);
    const int r10 = g.nx * (Y.i1 + g.ny * Z.i0);
    const int r01 = g.nx * (Y.i0 + g.ny * Z.i1);
    const int r11 = g.nx * (Y.i1 + g.ny * Z.i1);
    c.o000 = r00 + X.i0; c.o100 = r00 + X.i1; c.o010 = r10 + X.i0; c.o110 = r10 + X.i1;
    c.o001 = r01 + X.i0; c.o101 = r01 + X.i1; c.o011 = r11 + X.i0; c.o111 = r11 + X.i1;
    c.tx = X.t; c.ty = Y.t; c.tz = Z.t;
    return c;
}

inline int grid_for(long long n, int threads) {
    long long b = (n + threads - 1) / threads;
    return (int)std::min<long long>(std::max<long long>(b, 1), kNumSMs * 32);
}
}  // namespace

// One separable Gaussian pass along `axis` for all channels (generic radius,
// truncated at max(1, ceil(3 sigma)) and renormalised, field.cpp:205-269).
struct Taps {
    int R;
    float w[2 * 64 + 1];
};

__global__ void k_smooth_axis(const float* __restrict__ in, float* __restrict__ out, int nchan,
                              Geo g, int axis, Taps t) {
    const long long tot = g.n * nchan;
    const int n = axis == 0 ? g.nx : axis == 1 ? g.ny : g.nz;
    const long long stride = axis == 0 ? 1 : axis == 1 ? g.nx : (long long)g.nx * g.ny;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < tot;
         i += (long long)gridDim.x * blockDim.x) {
        const long long v = i % g.n;
        const int p = axis == 0 ? (int)(v % g.nx) : axis == 1 ? (int)((v / g.nx) % g.ny)
                                                              : (int)(v / ((long long)g.nx * g.ny));
        if (n == 1) { out[i] = in[i]; continue; }
        const int q0 = max(0, p - t.R), q1 = min(n - 1, p + t.R);
        float num = 0.f, den = 0.f;
        for (int q = q0; q <= q1; ++q) {
            const float wq = t.w[q - p + t.R];
            num = fmaf(wq, in[i + (q - p) * stride], num);
            den += wq;
        }
        out[i] = num / den;
    }
}

void launch_smooth_generic(const float* in, float* out, float* tmp, int nchan, const Geo& g,
                           double sigma, cudaStream_t s) {
    if (!(sigma > 0.0)) {
        cudaMemcpyAsync(out, in, sizeof(float) * nchan * g.n, cudaMemcpyDeviceToDevice, s);
        return;
    }
    Taps t;
    t.R = std::max(1, (int)std::ceil(3.0 * sigma));
    if (t.R > 64) t.R = 64;  // callers reject sigma > 21 (WLM_UNSUPPORTED)
    for (int i = -t.R; i <= t.R; ++i) t.w[i + t.R] = (float)std::exp(-0.5 * (double)(i * i) / (sigma * sigma));
    const int blocks = grid_for(g.n * nchan, 256);
    // x: in -> out, y: out -> tmp, z: tmp -> out
    k_smooth_axis<<<blocks, 256, 0, s>>>(in, out, nchan, g, 0, t);
    k_smooth_axis<<<blocks, 256, 0, s>>>(out, tmp, nchan, g, 1, t);
    k_smooth_axis<<<blocks, 256, 0, s>>>(tmp, out, nchan, g, 2, t);
    g_kernel_launches += 3;
}

__global__ void k_max_abs(const float* __restrict__ v, long long count, unsigned* out) {
    __shared__ float sm[32];
    float m = 0.f;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
         i += (long long)gridDim.x * blockDim.x)
        m = fmaxf(m, fabsf(v[i]));
    m = warp_max(m);
    if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        float t = 0.f;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t = fmaxf(t, sm[i]);
        atomic_max_nonneg(out, t);
    }
}

void launch_max_abs(const float* v, long long count, unsigned* out_bits, cudaStream_t s) {
    k_max_abs<<<grid_for(count, 256), 256, 0, s>>>(v, count, out_bits);
    ++g_kernel_launches;
}

__global__ void k_jacdet(const float* __restrict__ u, Geo g, int* out) {
    __shared__ float s_min[32];
    int xl, xh, yl, yh, zl, zh;
    interior(g.nx, xl, xh); interior(g.ny, yl, yh); interior(g.nz, zl, zh);
    const long long cx = xh - xl + 1, cy = yh - yl + 1, cz = zh - zl + 1;
    float mn = FLT_MAX;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < cx * cy * cz;
         i += (long long)gridDim.x * blockDim.x) {
        const int x = xl + (int)(i % cx), y = yl + (int)((i / cx) % cy), z = zl + (int)(i / (cx * cy));
        mn = fminf(mn, det_at(u, g, x, y, z, 1.f));
    }
    for (int o = 16; o > 0; o >>= 1) mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    if ((threadIdx.x & 31) == 0) s_min[threadIdx.x >> 5] = mn;
    __syncthreads();
    if (threadIdx.x == 0) {
        float m = FLT_MAX;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) m = fminf(m, s_min[i]);
        atomicMin(out, float_to_ordered(m));
    }
}

void launch_jacdet(const float* u, const Geo& g, int* out_ordered, cudaStream_t s) {
    k_jacdet<<<grid_for(g.n, 256), 256, 0, s>>>(u, g, out_ordered);
    ++g_kernel_launches;
}


// -r (H + lambda I)^{-1} by the adjugate, rounding steps as the oracle's
// tile_step_matrix (no contraction).
__device__ __forceinline__ void tile_matrix(const double H[6], double r, double lambda, double* Mo) {
    const double a = __dadd_rn(H[0], lambda), b = H[1], c = H[2], d = __dadd_rn(H[3], lambda), e = H[4],
                 f = __dadd_rn(H[5], lambda);
    const double c00 = __dsub_rn(__dmul_rn(d, f), __dmul_rn(e, e));
    const double c01 = __dsub_rn(__dmul_rn(c, e), __dmul_rn(b, f));
    const double c02 = __dsub_rn(__dmul_rn(b, e), __dmul_rn(c, d));
    const double c11 = __dsub_rn(__dmul_rn(a, f), __dmul_rn(c, c));
    const double c12 = __dsub_rn(__dmul_rn(b, c), __dmul_rn(a, e));
    const double c22 = __dsub_rn(__dmul_rn(a, d), __dmul_rn(b, b));
    const double det = __dadd_rn(__dadd_rn(__dmul_rn(a, c00), __dmul_rn(b, c01)), __dmul_rn(c, c02));
    const double s = __ddiv_rn(-r, det);
    Mo[0] = __dmul_rn(s, c00); Mo[1] = __dmul_rn(s, c01); Mo[2] = __dmul_rn(s, c02);
    Mo[3] = __dmul_rn(s, c11); Mo[4] = __dmul_rn(s, c12); Mo[5] = __dmul_rn(s, c22);
}
__device__ __forceinline__ void add_outer(double H[6], double g0, double g1, double g2) {
    H[0] = __dadd_rn(H[0], __dmul_rn(g0, g0)); H[1] = __dadd_rn(H[1], __dmul_rn(g0, g1));
    H[2] = __dadd_rn(H[2], __dmul_rn(g0, g2)); H[3] = __dadd_rn(H[3], __dmul_rn(g1, g1));
    H[4] = __dadd_rn(H[4], __dmul_rn(g1, g2)); H[5] = __dadd_rn(H[5], __dmul_rn(g2, g2));
}

// Engine: one thread per (pair, tile); g is the stored fp32 gradient (SoA).
__global__ void k_tile_matrix(Batch b, LmParams p) {
    const long long ntiles = (long long)b.tkx * b.tky * b.tkz;
    const int pair = b.pair0 + blockIdx.y;
    const PairState* st = b.st + pair;
    if (st->done) return;
    const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (t >= ntiles) return;
    const Geo g = b.g;
    const int k = p.tile_k;
    const int bx = (int)(t % b.tkx), by = (int)((t / b.tkx) % b.tky), bz = (int)(t / ((long long)b.tkx * b.tky));
    if (bz * k < g.zs || bz * k >= g.ze) return;  // slabs: tiles of the owned (tile-aligned) planes
    const int x1 = min(g.nx, (bx + 1) * k), y1 = min(g.ny, (by + 1) * k), z1 = min(g.nz, (bz + 1) * k);
    const float* G = b.G + (long long)pair * 3 * g.n;
    double H[6] = {0, 0, 0, 0, 0, 0};
    for (int z = bz * k; z < z1; ++z)
        for (int y = by * k; y < y1; ++y)
            for (int x = bx * k; x < x1; ++x) {
                const int o = g.lat(x, y, z);
                add_outer(H, G[o], G[g.n + o], G[2 * g.n + o]);
            }
    tile_matrix(H, st->r_cur, st->lambda, b.TM + ((long long)pair * ntiles + t) * 6);
}

void launch_tile_matrix(const Batch& b, const LmParams& p, cudaStream_t s) {
    const long long ntiles = (long long)b.tkx * b.tky * b.tkz;
    k_tile_matrix<<<dim3((unsigned)((ntiles + 127) / 128), b.pairs), 128, 0, s>>>(b, p);
    ++g_kernel_launches;
}

// Mirror op (fp64 AoS, one thread per tile): bitwise the oracle's
// orc_lm_step_tiled.
__global__ void k_lm_tiled_fp64(double r, const double* __restrict__ g, Geo geo, double lambda, int k, int tkx,
                                int tky, int tkz, double* __restrict__ out) {
    const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (t >= (long long)tkx * tky * tkz) return;
    const int bx = (int)(t % tkx), by = (int)((t / tkx) % tky), bz = (int)(t / ((long long)tkx * tky));
    const int x1 = min(geo.nx, (bx + 1) * k), y1 = min(geo.ny, (by + 1) * k), z1 = min(geo.nz, (bz + 1) * k);
    double H[6] = {0, 0, 0, 0, 0, 0};
    for (int z = bz * k; z < z1; ++z)
        for (int y = by * k; y < y1; ++y)
            for (int x = bx * k; x < x1; ++x) {
                const double* gi = g + 3 * (long long)geo.at(x, y, z);
                add_outer(H, gi[0], gi[1], gi[2]);
            }
    double M[6];
    tile_matrix(H, r, lambda, M);
    for (int z = bz * k; z < z1; ++z)
        for (int y = by * k; y < y1; ++y)
            for (int x = bx * k; x < x1; ++x) {
                const long long i = 3 * (long long)geo.at(x, y, z);
                const double g0 = g[i], g1 = g[i + 1], g2 = g[i + 2];
                out[i] = __dadd_rn(__dadd_rn(__dmul_rn(M[0], g0), __dmul_rn(M[1], g1)), __dmul_rn(M[2], g2));
                out[i + 1] = __dadd_rn(__dadd_rn(__dmul_rn(M[1], g0), __dmul_rn(M[3], g1)), __dmul_rn(M[4], g2));
                out[i + 2] = __dadd_rn(__dadd_rn(__dmul_rn(M[2], g0), __dmul_rn(M[4], g1)), __dmul_rn(M[5], g2));
            }
}

void launch_lm_tiled_fp64(double r, const double* g, const Geo& geo, double lambda, int k, double* tm,
                          double* out, cudaStream_t s) {
    (void)tm;
    const int tkx = cdiv(geo.nx, k), tky = cdiv(geo.ny, k), tkz = cdiv(geo.nz, k);
    const long long nt = (long long)tkx * tky * tkz;
    k_lm_tiled_fp64<<<(unsigned)((nt + 127) / 128), 128, 0, s>>>(r, g, geo, lambda, k, tkx, tky, tkz, out);
    ++g_kernel_launches;
}

__global__ void k_demons_pointwise(const double* __restrict__ r, const double* __restrict__ n, long long N,
                                   double alpha, double* __restrict__ out) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N;
         i += (long long)gridDim.x * blockDim.x)
        demons_step(r[i], n[3 * i], n[3 * i + 1], n[3 * i + 2], alpha, out + 3 * i);
}

void launch_demons_pointwise(const double* r, const double* n, long long N, double alpha, double* out,
                             cudaStream_t s) {
    k_demons_pointwise<<<grid_for(N, 256), 256, 0, s>>>(r, n, N, alpha, out);
    ++g_kernel_launches;
}

__global__ void k_nonfinite(const float* __restrict__ v, long long count, int* flag) {
    int bad = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
         i += (long long)gridDim.x * blockDim.x)
        bad |= !isfinite(v[i]);
    bad = __syncthreads_or(bad);
    if (threadIdx.x == 0 && bad) atomicOr(flag, 1);
}

void launch_nonfinite(const float* v, long long count, int* flag, cudaStream_t s) {
    k_nonfinite<<<grid_for(count, 256), 256, 0, s>>>(v, count, flag);
    ++g_kernel_launches;
}

// downsample: separable Gaussian (sigma = 0.5 f, radius
// max(1, ceil(3 sigma)), per-axis renormalised) evaluated directly at the
// strided output voxels in fp64 -- the product of the per-axis normalised
// passes of field.cpp:253-260 -- then rounded to fp32 once (A11).
struct TapsD {
    int R;
    double w[2 * 64 + 1];
};

__global__ void k_downsample_gauss(const float* __restrict__ in, Geo g, int f, TapsD t, float* out, Geo gd) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < gd.n;
         i += (long long)gridDim.x * blockDim.x) {
        const int x = (int)(i % gd.nx), y = (int)((i / gd.nx) % gd.ny), z = (int)(i / ((long long)gd.nx * gd.ny));
        const int cx = x * f, cy = y * f, cz = z * f;
        const int x0 = max(0, cx - t.R), x1 = min(g.nx - 1, cx + t.R);
        const int y0 = max(0, cy - t.R), y1 = min(g.ny - 1, cy + t.R);
        const int z0 = max(0, cz - t.R), z1 = min(g.nz - 1, cz + t.R);
        double wx = 0.0, wy = 0.0, wz = 0.0;
        for (int q = x0; q <= x1; ++q) wx += t.w[q - cx + t.R];
        for (int q = y0; q <= y1; ++q) wy += t.w[q - cy + t.R];
        for (int q = z0; q <= z1; ++q) wz += t.w[q - cz + t.R];
        if (g.nx == 1) wx = 1.0;
        if (g.ny == 1) wy = 1.0;
        if (g.nz == 1) wz = 1.0;
        double acc = 0.0;
        for (int qz = z0; qz <= z1; ++qz) {
            const double w3 = g.nz == 1 ? 1.0 : t.w[qz - cz + t.R];
            double sy = 0.0;
            for (int qy = y0; qy <= y1; ++qy) {
                const double w2 = g.ny == 1 ? 1.0 : t.w[qy - cy + t.R];
                const float* row = in + g.at(0, qy, qz);
                double sx = 0.0;
                for (int qx = x0; qx <= x1; ++qx) sx = fma(g.nx == 1 ? 1.0 : t.w[qx - cx + t.R], (double)__ldg(row + qx), sx);
                sy = fma(w2, sx, sy);
            }
            acc = fma(w3, sy, acc);
        }
        out[i] = (float)(acc / (wx * wy * wz));
    }
}

void launch_downsample_gauss(const float* in, const Geo& g, int f, float* out, const Geo& gd, cudaStream_t s) {
    const double sigma = 0.5 * f;
    TapsD t;
    t.R = std::min(64, std::max(1, (int)std::ceil(3.0 * sigma)));
    for (int i = -t.R; i <= t.R; ++i) t.w[i + t.R] = std::exp(-0.5 * (double)(i * i) / (sigma * sigma));
    k_downsample_gauss<<<grid_for(gd.n, 128), 128, 0, s>>>(in, g, f, t, out, gd);
    ++g_kernel_launches;
}

// upsample_warp in fp64: trilinear at x / scale, * scale.
__global__ void k_upsample(const float* __restrict__ u, Geo g, Geo gd, double scale, float* out) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < gd.n;
         i += (long long)gridDim.x * blockDim.x) {
        const int x = (int)(i % gd.nx), y = (int)((i / gd.nx) % gd.ny), z = (int)(i / ((long long)gd.nx * gd.ny));
        double s[3];
        sample3_d(u, g.n, g, 0, 0, 0, x / scale, y / scale, z / scale, s);
        out[i] = (float)(scale * s[0]);
        out[gd.n + i] = (float)(scale * s[1]);
        out[2 * gd.n + i] = (float)(scale * s[2]);
    }
}

void launch_upsample(const float* u, const Geo& g, const Geo& gd, float scale, float* out, cudaStream_t s) {
    k_upsample<<<grid_for(gd.n, 256), 256, 0, s>>>(u, g, gd, (double)scale, out);
    ++g_kernel_launches;
}


__global__ void k_aos_to_soa(const double* __restrict__ in, float* __restrict__ out, long long n, int nchan) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n * nchan;
         i += (long long)gridDim.x * blockDim.x) {
        const long long v = i / nchan;
        const int c = (int)(i % nchan);
        out[(long long)c * n + v] = (float)in[i];
    }
}

__global__ void k_soa_to_aos(const float* __restrict__ in, double* __restrict__ out, long long n, int nchan) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n * nchan;
         i += (long long)gridDim.x * blockDim.x) {
        const long long v = i / nchan;
        const int c = (int)(i % nchan);
        out[i] = (double)in[(long long)c * n + v];
    }
}

void launch_aos_to_soa(const double* in, float* out, long long n, int nchan, cudaStream_t s) {
    k_aos_to_soa<<<grid_for(n * nchan, 256), 256, 0, s>>>(in, out, n, nchan);
    ++g_kernel_launches;
}

void launch_soa_to_aos(const float* in, double* out, long long n, int nchan, cudaStream_t s) {
    k_soa_to_aos<<<grid_for(n * nchan, 256), 256, 0, s>>>(in, out, n, nchan);
    ++g_kernel_launches;
}

}  // namespace wlm
