// generic.cu -- device paths of the LM attempt for the parameters the fused
// hot kernels are not instantiated for: LNCC radius != 2 (SPEC.md:122-123,
// lncc_radius >= 1) and smoothing radii > 6 (sigma_update / sigma_warp > 2;
// the reference's gaussian_smooth takes any sigma > 0, field.cpp:205-213).
//
// Same algorithm and storage points as the fused kernels (DESIGN.md §4:
// fp64 arithmetic, A and B fp32 + E fp64, g / dU_s / u' fp32), written as
// flat passes over fp64 scratch planes in HBM (Batch::X64, [pair][10][n]):
//   K1b': moments (f', m', f'^2, m'^2, f'm') -> box passes x, y, z ->
//         rho, A, B, E; sum(rho) partials in K1b's (plane, tile, warp)
//         layout, so k_plane_sums / K5 and every decision are unchanged
//   K2':  A, B, E -> box passes -> dr/dMw -> g = dr/dMw grad M(x+u)
//   K3':  LM / GD / Adam / tiled step -> Gaussian passes -> dU_s, max |dU_s|
//   K4':  compositive resample -> Gaussian passes -> u'
// The Gaussian passes are the reference's own (field.cpp:217-248, per-pass
// renormalisation over in-bounds taps, fp64 weights from std::exp).  These
// paths run on single-domain engines (slab groups refuse them) and trade
// speed for generality: ~10 full-volume passes instead of one fused one.
// There is no CPU fallback.
#include <cmath>
#include <vector>

#include "internal.cuh"

namespace wlm {

namespace {

constexpr int kScratchCh = 10;  // fp64 scratch planes per pair

inline int gblocks(long long n) { return (int)std::min<long long>(148 * 8, std::max<long long>(1, (n + 255) / 256)); }

#define GEN_LOOP(i, n) \
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < (n); i += (long long)gridDim.x * blockDim.x)

__device__ __forceinline__ double* scratch(const Batch& b, int pair, int ch) {
    return b.X64 + ((long long)pair * kScratchCh + ch) * b.g.n;
}

// One separable pass along `axis` over channels [c0, c0 + nch) of the
// scratch, in -> out (channel offsets): box (unnormalised truncated window
// sum, LNCC) or Gaussian (field.cpp:217-248).
__global__ void k_gen_pass(Batch b, int c_in, int c_out, int nch, int axis, const double* __restrict__ w, int R,
                           int box, int skip_rejected) {
    const int pair = b.pair0 + blockIdx.y;
    const PairState* st = b.st + pair;
    if (st->done || (skip_rejected && st->last_rejected)) return;
    const Geo g = b.g;
    const int na = axis == 0 ? g.nx : axis == 1 ? g.ny : g.nz;
    const long long stp = axis == 0 ? 1 : axis == 1 ? g.nx : (long long)g.nx * g.ny;
    GEN_LOOP(j, g.n * nch) {
        const int c = (int)(j / g.n);
        const long long i = j % g.n;
        const double* in = scratch(b, pair, c_in + c);
        double* out = scratch(b, pair, c_out + c);
        const int p = axis == 0 ? (int)(i % g.nx) : axis == 1 ? (int)((i / g.nx) % g.ny)
                                                            : (int)(i / ((long long)g.nx * g.ny));
        const int lo = max(0, p - R), hi = min(na - 1, p + R);
        if (box) {
            double acc = 0.0;
            for (int q = lo; q <= hi; ++q) acc += in[i + (long long)(q - p) * stp];
            out[i] = acc;
        } else {
            if (na == 1) { out[i] = in[i]; continue; }
            double acc = 0.0, wsum = 0.0;
            for (int q = lo; q <= hi; ++q) {
                const double wq = w[q - p + R];
                acc = __dadd_rn(acc, __dmul_rn(wq, in[i + (long long)(q - p) * stp]));
                wsum = __dadd_rn(wsum, wq);
            }
            out[i] = __ddiv_rn(acc, wsum);
        }
    }
}

// ---- LNCC (any radius) ----
__global__ void k_gen_moments(Batch b) {
    const int pair = b.pair0 + blockIdx.y;
    const PairState* st = b.st + pair;
    if (st->done) return;
    const double shf = st->shift_f, shm = st->shift_m;
    const float* F = b.F + (long long)pair * b.g.nfull;
    const double* MW = b.MW + (long long)pair * b.g.n;
    GEN_LOOP(i, b.g.n) {
        const double f = (double)F[i] - shf, m = MW[i] - shm;
        scratch(b, pair, 0)[i] = f;
        scratch(b, pair, 1)[i] = m;
        scratch(b, pair, 2)[i] = f * f;
        scratch(b, pair, 3)[i] = m * m;
        scratch(b, pair, 4)[i] = f * m;
    }
}

// rho, A, B, E from the window sums in channels 5..9 (K1b's arithmetic);
// rho -> channel 0
__global__ void k_gen_coeffs(Batch b, int R) {
    const int pair = b.pair0 + blockIdx.y;
    const PairState* st = b.st + pair;
    if (st->done) return;
    const Geo g = b.g;
    const double shf = st->shift_f, shm = st->shift_m;
    float* Aout = b.ABE + (long long)pair * 4 * g.n;
    float* Bout = Aout + g.n;
    double* Eout = reinterpret_cast<double*>(Aout + 2 * g.n);
    GEN_LOOP(i, g.n) {
        const int x = (int)(i % g.nx), y = (int)((i / g.nx) % g.ny), z = (int)(i / ((long long)g.nx * g.ny));
        double Sm[5];
        for (int c = 0; c < 5; ++c) Sm[c] = scratch(b, pair, 5 + c)[i];
        const int cnt = axis_count(x, g.nx, R) * axis_count(y, g.ny, R) * axis_count(z, g.nz, R);
        const double inv = 1.0 / (double)cnt;
        const double mf = Sm[0] * inv, mm = Sm[1] * inv;
        const double vf = fma(-mf, mf, Sm[2] * inv);
        const double vm = fma(-mm, mm, Sm[3] * inv);
        const double cv = fma(-mf, mm, Sm[4] * inv);
        const double af = mf + shf, am = mm + shm;
        const double msf = fma(af, af, vf), msm = fma(am, am, vm);
        double rho = 0.0, Ee = 0.0;
        float Aa = 0.f, Bb = 0.f;
        const bool degenerate = msf <= 0.0 || msm <= 0.0 || vf <= 1e-9 * msf || vm <= 1e-9 * msm;
        if (!degenerate) {
            const double alpha = rsqrt(vf * vm);
            rho = cv * alpha;
            Aa = (float)(alpha * inv);
            Bb = (float)(-rho * alpha * alpha * vf * inv);
            Ee = fma((double)Aa, mf, (double)Bb * mm);
        }
        Aout[i] = Aa;
        Bout[i] = Bb;
        Eout[i] = Ee;
        scratch(b, pair, 0)[i] = rho;
    }
}

// sum(rho) partials in K1b's layout: one per (plane, 32 x 8 tile, row)
__global__ void k_gen_rho_partials(Batch b) {
    const int pair = b.pair0 + blockIdx.z;
    const PairState* st = b.st + pair;
    if (st->done) return;
    const Geo g = b.g;
    const int tiles_x = (g.nx + 31) / 32, tiles = tiles_x * ((g.ny + 7) / 8);
    const int z = blockIdx.y;
    const int x = (blockIdx.x % tiles_x) * 32 + (threadIdx.x & 31);
    const int y = (blockIdx.x / tiles_x) * 8 + (threadIdx.x >> 5);
    double rho = 0.0;
    if (x < g.nx && y < g.ny) rho = scratch(b, pair, 0)[x + (long long)g.nx * (y + (long long)g.ny * z)];
    rho = warp_sum(rho);
    if ((threadIdx.x & 31) == 0)
        b.partials[(((long long)pair * g.nz + z) * tiles + blockIdx.x) * 8 + (threadIdx.x >> 5)] = rho;
}

__global__ void k_gen_abe64(Batch b) {
    const int pair = b.pair0 + blockIdx.y;
    const PairState* st = b.st + pair;
    if (st->done || st->last_rejected) return;
    const float* A = b.ABE + (long long)pair * 4 * b.g.n;
    const double* E = reinterpret_cast<const double*>(A + 2 * b.g.n);
    GEN_LOOP(i, b.g.n) {
        scratch(b, pair, 0)[i] = (double)A[i];
        scratch(b, pair, 1)[i] = (double)A[b.g.n + i];
        scratch(b, pair, 2)[i] = E[i];
    }
}

// K2's output arithmetic from the window sums in channels 5..7
__global__ void k_gen_grad(Batch b) {
    const int pair = b.pair0 + blockIdx.y;
    const PairState* st = b.st + pair;
    if (st->done || st->last_rejected) return;
    const Geo g = b.g;
    const double shf = st->shift_f, shm = st->shift_m;
    const double invN = 1.0 / (double)g.nfull;
    const float* F = b.F + (long long)pair * g.nfull;
    const double* MW = b.MW + (long long)pair * g.n;
    const double* GM = b.GM + (long long)pair * 3 * g.n;
    float* G = b.G + (long long)pair * 3 * g.n;
    GEN_LOOP(i, g.n) {
        const double f = (double)F[i] - shf;
        const double S0 = scratch(b, pair, 5)[i], S1 = scratch(b, pair, 6)[i], S2 = scratch(b, pair, 7)[i];
        const double dm = -invN * (fma(f, S0, (MW[i] - shm) * S1) - S2);
        G[i] = (float)(dm * GM[i]);
        G[g.n + i] = (float)(dm * GM[g.n + i]);
        G[2 * g.n + i] = (float)(dm * GM[2 * g.n + i]);
    }
}

// ---- K3' / K4' ----
__device__ __forceinline__ double rcp_newton(double x) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    double e = fma(-x, y, 1.0);
    y = fma(y, e, y);
    e = fma(-x, y, 1.0);
    return fma(y, e, y);
}

__global__ void k_gen_step(Batch b, LmParams p) {
    const int pair = b.pair0 + blockIdx.y;
    const PairState* st = b.st + pair;
    if (st->done) return;
    const Geo g = b.g;
    const float* Gin = b.G + (long long)pair * 3 * g.n;
    const double r = st->r_cur, lam = st->lambda;
    const bool tiled = p.optimizer == WLM_OPT_LM && p.tile_k > 1;
    const double* TM = tiled ? b.TM + (long long)pair * 6 * b.tkx * b.tky * b.tkz : nullptr;
    GEN_LOOP(i, g.n) {
        const double a = Gin[i], bb = Gin[g.n + i], c = Gin[2 * g.n + i];
        double o0, o1, o2;
        if (tiled) {
            const int x = (int)(i % g.nx), y = (int)((i / g.nx) % g.ny), z = (int)(i / ((long long)g.nx * g.ny));
            const int k = p.tile_k;
            const double* M6 = TM + ((long long)(z / k) * b.tkx * b.tky + (y / k) * b.tkx + x / k) * 6;
            o0 = M6[0] * a + M6[1] * bb + M6[2] * c;
            o1 = M6[1] * a + M6[3] * bb + M6[4] * c;
            o2 = M6[2] * a + M6[4] * bb + M6[5] * c;
        } else {
            double k = p.optimizer == WLM_OPT_GD ? -p.gd_lr : 1.0;
            if (p.optimizer == WLM_OPT_LM) k = -r * rcp_newton(fma(a, a, fma(bb, bb, c * c)) + lam);
            o0 = k * a; o1 = k * bb; o2 = k * c;
        }
        scratch(b, pair, 0)[i] = o0;
        scratch(b, pair, 1)[i] = o1;
        scratch(b, pair, 2)[i] = o2;
    }
}

__global__ void k_gen_store_vs(Batch b, int c0) {
    __shared__ float s_max[32];
    const int pair = b.pair0 + blockIdx.y;
    PairState* st = b.st + pair;
    if (st->done) return;
    const long long n = b.g.n;
    float* V = b.VS + (long long)pair * b.vs_ps;
    float mx = 0.f;
    GEN_LOOP(j, 3 * n) {
        const float v = (float)scratch(b, pair, c0 + (int)(j / n))[j % n];
        V[j] = v;
        mx = fmaxf(mx, fabsf(v));
    }
    mx = warp_max(mx);
    if ((threadIdx.x & 31) == 0) s_max[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        float m = 0.f;
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) m = fmaxf(m, s_max[k]);
        atomic_max_nonneg(&st->max_bits, m);
    }
}

__device__ __forceinline__ void clamp_cell(int& i, double& t, int n) {
    if (n == 1) { i = 0; t = 0.0; return; }
    if (i < 0) { i = 0; t = 0.0; }
    else if (i > n - 2) { i = n - 2; t = 1.0; }
}

// K4's compositive resample, u' = d + u(x + d), d = eps dU_s (fp64)
__global__ void k_gen_compose(Batch b, LmParams p) {
    const int pair = b.pair0 + blockIdx.y;
    const PairState* st = b.st + pair;
    if (st->done) return;
    const Geo g = b.g;
    const long long n = g.n;
    const float* V = b.VS + (long long)pair * b.vs_ps;
    const float* U = b.U + ((long long)pair * 2 + st->cur) * 3 * n;
    const double eps = p.target / fmax((double)__uint_as_float(st->max_bits), p.step_floor);
    GEN_LOOP(i, n) {
        const int x = (int)(i % g.nx), y = (int)((i / g.nx) % g.ny), z = (int)(i / ((long long)g.nx * g.ny));
        const double dx = eps * V[i], dy = eps * V[n + i], dz = eps * V[2 * n + i];
        double o3[3];
        if (isfinite(dx + dy + dz)) {
            const double fx = floor(dx), fy = floor(dy), fz = floor(dz);
            double tx = dx - fx, ty = dy - fy, tz = dz - fz;
            int ix = x + (int)fx, iy = y + (int)fy, iz = z + (int)fz;
            clamp_cell(ix, tx, g.nx);
            clamp_cell(iy, ty, g.ny);
            clamp_cell(iz, tz, g.nz);
            const int sx = g.nx > 1 ? 1 : 0, sy = g.ny > 1 ? g.nx : 0;
            const long long sz = g.nz > 1 ? (long long)g.nx * g.ny : 0;
            for (int ch = 0; ch < 3; ++ch) {
                const float* q = U + ch * n + ix + (long long)g.nx * (iy + (long long)g.ny * iz);
                const double c000 = q[0], c100 = q[sx], c010 = q[sy], c110 = q[sy + sx];
                const double c001 = q[sz], c101 = q[sz + sx], c011 = q[sz + sy], c111 = q[sz + sy + sx];
                const double v00 = fma(tx, c100 - c000, c000), v10 = fma(tx, c110 - c010, c010);
                const double v01 = fma(tx, c101 - c001, c001), v11 = fma(tx, c111 - c011, c011);
                const double s0 = fma(ty, v10 - v00, v00), s1 = fma(ty, v11 - v01, v01);
                o3[ch] = fma(tz, s1 - s0, s0);
            }
            o3[0] += dx;
            o3[1] += dy;
            o3[2] += dz;
        } else {
            o3[0] = o3[1] = o3[2] = __longlong_as_double(0x7ff8000000000000ll);
        }
        scratch(b, pair, 0)[i] = o3[0];
        scratch(b, pair, 1)[i] = o3[1];
        scratch(b, pair, 2)[i] = o3[2];
    }
}

__global__ void k_gen_store_u(Batch b, int c0) {
    const int pair = b.pair0 + blockIdx.y;
    const PairState* st = b.st + pair;
    if (st->done) return;
    const long long n = b.g.n;
    float* Un = b.U + ((long long)pair * 2 + (1 - st->cur)) * 3 * n;
    GEN_LOOP(j, 3 * n) Un[j] = (float)scratch(b, pair, c0 + (int)(j / n))[j % n];
}

// x, y, z passes: channels [c, c + nch) -> (via c + 5) -> back in place
void passes(const Batch& b, int c, int nch, const double* w, int R, int box, int skip_rej, cudaStream_t s) {
    const dim3 grid(gblocks(b.g.n * nch), b.pairs);
    k_gen_pass<<<grid, 256, 0, s>>>(b, c, c + 5, nch, 0, w, R, box, skip_rej);
    k_gen_pass<<<grid, 256, 0, s>>>(b, c + 5, c, nch, 1, w, R, box, skip_rej);
    k_gen_pass<<<grid, 256, 0, s>>>(b, c, c + 5, nch, 2, w, R, box, skip_rej);
    g_kernel_launches += 3;
}

}  // namespace

size_t generic_scratch_doubles(const Geo& g) { return (size_t)kScratchCh * (size_t)g.n; }

// K1b' (the window sums end in channels 5..9)
void launch_lncc_fwd_generic(const Batch& b, const LmParams& p, int mode, cudaStream_t s) {
    const int R = p.radius;
    launch_warp_moving_grad(b, mode, 0, b.g.nz, s);
    const dim3 grid(gblocks(b.g.n), b.pairs);
    k_gen_moments<<<grid, 256, 0, s>>>(b);
    ++g_kernel_launches;
    passes(b, 0, 5, nullptr, R, 1, 0, s);
    k_gen_coeffs<<<grid, 256, 0, s>>>(b, R);
    const int tiles = ((b.g.nx + 31) / 32) * ((b.g.ny + 7) / 8);
    k_gen_rho_partials<<<dim3(tiles, b.g.nz, b.pairs), 256, 0, s>>>(b);
    g_kernel_launches += 2;
    launch_plane_sums(b, s);
}

// K2'
void launch_lncc_bwd_generic(const Batch& b, const LmParams& p, cudaStream_t s) {
    const dim3 grid(gblocks(b.g.n), b.pairs);
    k_gen_abe64<<<grid, 256, 0, s>>>(b);
    ++g_kernel_launches;
    passes(b, 0, 3, nullptr, p.radius, 1, 1, s);
    k_gen_grad<<<grid, 256, 0, s>>>(b);
    ++g_kernel_launches;
}

// K3' (weights: device fp64 taps w[0 .. 2R])
void launch_step_smooth_generic(const Batch& b, const LmParams& p, const double* w, int R, cudaStream_t s) {
    const dim3 grid(gblocks(b.g.n), b.pairs);
    k_gen_step<<<grid, 256, 0, s>>>(b, p);
    ++g_kernel_launches;
    if (R > 0) passes(b, 0, 3, w, R, 0, 0, s);  // result in channels 5..7
    k_gen_store_vs<<<dim3(gblocks(3 * b.g.n), b.pairs), 256, 0, s>>>(b, R > 0 ? 5 : 0);
    ++g_kernel_launches;
}

// K4'
void launch_compose_smooth_generic(const Batch& b, const LmParams& p, const double* w, int R, cudaStream_t s) {
    const dim3 grid(gblocks(b.g.n), b.pairs);
    k_gen_compose<<<grid, 256, 0, s>>>(b, p);
    ++g_kernel_launches;
    if (R > 0) passes(b, 0, 3, w, R, 0, 0, s);  // result in channels 5..7
    k_gen_store_u<<<dim3(gblocks(3 * b.g.n), b.pairs), 256, 0, s>>>(b, R > 0 ? 5 : 0);
    ++g_kernel_launches;
}

}  // namespace wlm
