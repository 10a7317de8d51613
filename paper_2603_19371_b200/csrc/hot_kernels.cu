// hot_kernels.cu -- the kernels of one LM attempt.
//
//   K1a k_warp_moving    Mw = M(x + u) and grad M(x + u) in fp64 (flat gather kernel)
//   K1b k_lncc_fwd       LNCC window moments -> rho, A, B, E; sum(rho) per (plane, tile, warp)
//       k_plane_sums     per-plane sum(rho), one CTA per plane, fixed order
//   K5  k_finalize       sum(rho) in z order -> r; loss/damping/rejection state
//   K2  k_lncc_bwd       adjoint window sums -> g (F, Mw, grad M staged by cp.async)
//   K3  k_step_smooth    LM step + Gaussian(sigma_update) + max|.| (column y-pass)
//   K4  k_compose_smooth compositive resample (TMA-staged warp ring) + Gaussian(sigma_warp)
//   MSE / MI: k_mse_fwd, k_mse_grad, k_mi_hist, k_mi_finalize, k_mi_grad
//
// The engine launches these per pair group (internal.cuh): a Batch view with
// pair0 / pairs, one stream of attempt graphs per group.
//
// Schedule of the stencil kernels (hot.cuh): a CTA owns a 32 x 8 column of
// output voxels and a chunk of the rank's owned z planes.  Per input plane it
//   * produces an fp64 halo tile in shared memory from inputs prefetched into
//     registers one or two planes ahead,
//   * filters it along x (shared memory), y (shared memory -> registers) and
//     z through a statically indexed register ring (the z loop is unrolled by
//     the ring length; z sums are taken directly over the ring, so every
//     voxel's arithmetic is independent of chunking and of the slab split).
// Every global access is a unit-stride row of one SoA plane.  Sums are fp64
// (DESIGN.md "Precision"); sum(rho) is reduced per plane in a fixed order and
// then over planes in z order, so results are bit-identical for any batch
// size, chunking or number of z slabs.
//
// Slabs (Geo in common.cuh): per-voxel buffers are local ([zlo, zlo+nzl),
// indexed with Geo::lat), F and M are whole-volume (Geo::at), faces are the
// global ones.
#include <atomic>
#include <cstring>
#include <cfloat>
#include <climits>

#include <cuda_pipeline.h>

#include "hot.cuh"
#include "kernels.cuh"

// K4's Gaussian taps as constant-bank DFMA operands instead of registers
// (WLM_CW_K4: K4 11.60 -> 11.43 ms; the same in K3 costs 7.45 -> 7.78, so K3
// keeps its taps in registers)
#ifndef WLM_CW_K4
#define WLM_CW_K4 1
#endif
namespace wlm {

using hot::NT;
using hot::TX;
using hot::TY;

namespace {
__host__ __device__ inline int cdiv(int a, int b) { return (a + b - 1) / b; }
}  // namespace

__constant__ double c_inv_count[126];  // 1/n for truncated window counts n <= 125

// Constant memory and function attributes are per device: one bit per
// device ordinal (a process may drive several devices through several
// contexts).
static std::atomic<unsigned long long> g_const_ready{0ull};
static unsigned long long device_bit() {
    int dev = 0;
    cudaGetDevice(&dev);
    return 1ull << (dev & 63);
}

void init_constants() {
    const unsigned long long bit = device_bit();
    if (g_const_ready.load() & bit) return;
    double inv[126];
    inv[0] = 0.0;
    for (int i = 1; i < 126; ++i) inv[i] = 1.0 / (double)i;
    cudaMemcpyToSymbol(c_inv_count, inv, sizeof(inv));
    g_const_ready.fetch_or(bit);
}

// ---------------------------------------------------------------------------
// Loss / damping / rejection state machine.  Identical fp64
// arithmetic to the oracle (oracle.cpp orc_update_damping /
// attempt_rejected), so the lambda trajectory is bit-identical whenever the
// accept/reject decisions agree.
__device__ void update_damping_dev(PairState* st, const LmParams& p, double r) {
    const bool bad = st->hist_n == 0 || r > st->L1;
    double lam = bad ? p.mu_plus * st->lambda : p.mu_minus * st->lambda;
    if (p.lambda_max > 0.0 && isfinite(p.lambda_max)) lam = fmin(lam, p.lambda_max);
    st->lambda = fmax(lam, 1e-12);
    st->L2 = st->L1;
    st->L1 = r;
    st->hist_n = min(st->hist_n + 1, 2);
}

__device__ bool rejection_fires(const PairState* st, const LmParams& p, double r) {
    return p.rejection && st->hist_n >= 2 && (r - st->L1) > p.tau * fabs(st->L1 - st->L2);
}

// val: mean rho (LNCC: loss_raw = LNCC, r = 1 - LNCC) or the MSE (loss_raw =
// r = MSE).  PairState's lncc_* fields hold loss_raw.
__device__ void finalize_pair(PairState* st, const LmParams& p, int mode, double val, int pair) {
    // loss_raw -> r: LNCC 1 - LNCC, MSE itself, MI log2 B - MI
    const double top = p.metric == WLM_METRIC_MI ? log2((double)p.mi_bins) : 1.0;
    const bool mse = p.metric == WLM_METRIC_MSE;
    double lncc = val;
    double r = mse ? val : top - val;
    if (mode == 0) {
        st->r_cur = r;
        st->lncc_cur = lncc;
        if (!isfinite(r)) { st->status = WLM_NONFINITE; st->done = 1; }
        st->max_bits = 0u;
        st->jac_bits = 0x7f800000;  // +inf
        return;
    }
    if (p.script && p.script_n > 0) {
        r = p.script[(long long)pair * p.script_n + min(st->attempt, p.script_n - 1)];
        lncc = mse ? r : top - r;
    }
    st->attempt += 1;
    st->r_try = r;
    st->lncc_try = lncc;
    const double maxv = (double)__uint_as_float(st->max_bits);
    const double eps = p.target / fmax(maxv, p.step_floor);
    if (!isfinite(r)) {  // abort
        st->status = WLM_NONFINITE;
        st->done = 1;
        return;
    }
    bool rej = false;
    if (p.optimizer == WLM_OPT_LM && st->retries < p.max_retries && rejection_fires(st, p, r)) {
        double lam = p.mu_plus * st->lambda;
        if (p.lambda_max > 0.0 && isfinite(p.lambda_max)) lam = fmin(lam, p.lambda_max);
        st->lambda = lam;
        st->retries += 1;
        rej = true;
    }
    if (rej) {
        st->last_rejected = 1;
    } else {
        const bool forced = p.optimizer == WLM_OPT_LM && st->retries >= p.max_retries &&
                            rejection_fires(st, p, r);
        if (p.optimizer == WLM_OPT_LM) update_damping_dev(st, p, r);
        st->cur ^= 1;
        st->r_cur = r;
        st->lncc_cur = lncc;
        st->last_rejected = 0;
        if (p.trace && st->trace_len < p.trace_cap) {
            wlm_step_log* row = p.trace + (long long)pair * p.trace_cap + st->trace_len;
            row->level = st->level;
            row->iter = st->iter;
            row->loss_raw = lncc;
            row->r = r;
            row->lambda = p.optimizer == WLM_OPT_LM ? st->lambda : 0.0;
            row->eps = eps;
            row->accepted = forced ? 0 : 1;
            row->retries = st->retries;
            row->jac_det_min = p.log_jacobian ? (double)ordered_to_float(st->jac_bits)
                                              : __longlong_as_double(0x7ff8000000000000ll);
            st->trace_len += 1;
        }
        st->iter += 1;
        st->retries = 0;
        if (st->iter >= st->iters_target) st->done = 1;
    }
    st->max_bits = 0u;
    st->jac_bits = 0x7f800000;
}

// Item of slot s of this thread when NI halo items are dealt over NT
// threads in SL = ceil(NI / NT) slots: full slots in thread order, the
// partial last slot on the highest threads (the x-passes run on the lowest
// threads), -1 for none.  Constant arguments fold at compile time.
__device__ __forceinline__ int halo_item(int s, int SL, int NI, int NT) {
    if (s < SL - 1) return (int)threadIdx.x + s * NT;
    const int rem = NI - (SL - 1) * NT;
    return (int)threadIdx.x >= NT - rem ? (SL - 1) * NT + (int)threadIdx.x - (NT - rem) : -1;
}

// Block-wide fixed-order double sum (result valid in thread 0).
static __device__ double block_sum(double v, double* red) {
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

// Geometry shared by the stencil kernels: this CTA's 32 x 8 column and its
// chunk of owned planes.
struct Tile {
    int x0, y0, zb, ze;
    int ox, oy, x, y;
    bool own;
    int nxy;
    __device__ __forceinline__ void init(const Geo& g, int chunk_len) {
        const int tiles_x = cdiv(g.nx, TX);
        x0 = (blockIdx.x % tiles_x) * TX;
        y0 = (blockIdx.x / tiles_x) * TY;
        zb = g.zs + blockIdx.y * chunk_len;
        ze = min(zb + chunk_len, g.ze);
        ox = threadIdx.x & 31;
        oy = threadIdx.x >> 5;
        x = x0 + ox;
        y = y0 + oy;
        own = x < g.nx && y < g.ny;
        nxy = g.nx * g.ny;
    }
    // offset of plane z in a local (slab) buffer / in a whole-volume buffer
    __device__ __forceinline__ int lp(const Geo& g, int z) const { return (z - g.zlo) * nxy; }
    __device__ __forceinline__ int gp(int z) const { return z * nxy; }
};

// One axis of the split-form cell (field.cpp:19-39): integer corner index,
// exact fp64 weight, "outside" flag (gradient 0).  Interior samples take the
// first branch; the clamp rules only run near the volume faces.
struct Tap {
    int i0, step;
    double t;
    bool outside;
};

__device__ __forceinline__ Tap axis_split(int x, float u, int n) {
    Tap a;
    const float fl = floorf(u);
    const int i = x + (int)fl;
    const double tt = (double)u - (double)fl;  // exact, in [0, 1)
    if (i >= 0 && i <= n - 2) { a.i0 = i; a.step = 1; a.t = tt; a.outside = false; return a; }
    if (n == 1) { a.i0 = 0; a.step = 0; a.t = 0.0; a.outside = true; return a; }
    if (i < 0) { a.i0 = 0; a.step = 1; a.t = 0.0; a.outside = true; return a; }
    a.i0 = n - 2; a.step = 1; a.t = 1.0;
    a.outside = i > n - 1 || tt > 0.0;  // exactly on the last voxel: not outside
    return a;
}

// Sample (and analytic gradient) of a whole-volume fp32 image at voxel
// (x,y,z) + u, fp64, collapse order of field.cpp:47-90.  Non-finite u ->
// NaN value, zero gradient (field.cpp:49-52).
template <bool GRAD>
__device__ __forceinline__ double sample_vol(const float* __restrict__ M, const Geo& g, int x, int y, int z,
                                             float ux, float uy, float uz, double* grad) {
    if (!(isfinite(ux) && isfinite(uy) && isfinite(uz))) {
        if (GRAD) grad[0] = grad[1] = grad[2] = 0.0;
        return __longlong_as_double(0x7ff8000000000000ll);
    }
    const Tap X = axis_split(x, ux, g.nx), Y = axis_split(y, uy, g.ny), Z = axis_split(z, uz, g.nz);
    const float* p = M + X.i0 + g.nx * (Y.i0 + g.ny * Z.i0);
    const int sx = X.step, dy = Y.step * g.nx, dz = Z.step * g.nx * g.ny;
    const double a = __ldg(p), b = __ldg(p + sx);
    const double c = __ldg(p + dy), e = __ldg(p + dy + sx);
    const double f = __ldg(p + dz), h = __ldg(p + dz + sx);
    const double k = __ldg(p + dz + dy), l = __ldg(p + dz + dy + sx);
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

constexpr double kNaN64 = __builtin_nan("");

// ---------------------------------------------------------------------------
// Fused halo stores (Batch::peer): plane z of kind k goes to neighbour side sd
// when it lies in that side's send range; the remote voxel index follows the
// neighbour's buffer origin.
__device__ __forceinline__ bool peer_sends(const Batch& b, int sd, int k, int z) {
    return sd == 0 ? z < b.peer.lo_end[k] : z >= b.peer.hi_begin[k];
}
__device__ __forceinline__ long long peer_index(const Batch& b, int sd, int z, int nxy, int ooff) {
    return (long long)(z - b.peer.zlo[sd]) * nxy + ooff;
}

// ---------------------------------------------------------------------------
// K1a: warp of the moving image, Mw(x) = M(x + u(x)) in fp64, for the owned
// planes plus the 2 halo planes the window pass reads.  Block (32 x 8) = a
// 32 x 8 (x, y) tile of one plane; one voxel per thread, few registers (high
// occupancy hides the gather latency).
// Each thread warps kZP planes of one (x, y) column: all displacement loads
// are issued first, then all 8 kZP corner gathers, so a thread keeps kZP
// independent load chains in flight (the kernel is gather-latency bound).
// With GRAD (LNCC) it also stores the analytic interpolant gradient: the
// evaluated warp becomes the accepted one exactly when K2 runs next (K2 is
// skipped after a rejection), so K2 reads Mw and grad M instead of
// re-gathering M at the same points.
#ifndef WLM_K1A_ZP
#define WLM_K1A_ZP 4
#endif
constexpr int kZP = WLM_K1A_ZP;
template <bool GRAD>
__global__ void __launch_bounds__(256) k_warp_moving(Batch b, int mode, int z_first, int z_last) {
    const int pair = b.pair0 + blockIdx.z;
    const PairState* st = b.st + pair;
    if (st->done) return;
    const Geo g = b.g;
    const int tiles_x = cdiv(g.nx, 32);
    const int x = (blockIdx.x % tiles_x) * 32 + (threadIdx.x & 31);
    const int y = (blockIdx.x / tiles_x) * 8 + (threadIdx.x >> 5);
    if (x >= g.nx || y >= g.ny) return;
    const int zf = z_first + blockIdx.y * kZP;
    const int buf = mode == 0 ? st->cur : 1 - st->cur;
    const float* __restrict__ M = b.M + (long long)pair * g.nfull;
    const float* __restrict__ U = b.U + ((long long)pair * 2 + buf) * 3 * g.n;
    double* __restrict__ MW = b.MW + (long long)pair * g.n;
    float u[kZP][3];
#pragma unroll
    for (int k = 0; k < kZP; ++k) {
        const int z = min(zf + k, z_last - 1);
        const int o = g.lat(x, y, z);
        u[k][0] = __ldg(U + o); u[k][1] = __ldg(U + g.n + o); u[k][2] = __ldg(U + 2 * g.n + o);
    }
#pragma unroll
    for (int k = 0; k < kZP; ++k) {
        const int z = zf + k;
        if (z >= z_last) continue;
        const int o = g.lat(x, y, z);
        if (GRAD) {
            double gr[3];
            MW[o] = sample_vol<true>(M, g, x, y, z, u[k][0], u[k][1], u[k][2], gr);
            double* GMp = b.GM + (long long)pair * 3 * g.n;
            GMp[o] = gr[0];
            GMp[g.n + o] = gr[1];
            GMp[2 * g.n + o] = gr[2];
        } else {
            MW[o] = sample_vol<false>(M, g, x, y, z, u[k][0], u[k][1], u[k][2], nullptr);
        }
    }
}

// Per-plane sum(rho) (or sum e^2) from the (plane, tile, warp) partials: one
// CTA per (plane, pair), strided coalesced loads, then a fixed tree, so the
// sum depends on neither the chunking nor the slab split (and not on which
// CTA finished last).  Planes outside [zs, ze) are zeroed for the NCCL
// all-reduce of a distributed slab group.
__global__ void __launch_bounds__(256) k_plane_sums(Batch b) {
    __shared__ double red[32];
    const int z = blockIdx.x;
    const int pair = b.pair0 + blockIdx.y;
    const PairState* st = b.st + pair;
    if (st->done) return;
    const Geo g = b.g;
    double* __restrict__ psum = b.plane_sum + (long long)pair * g.nz;
    if (z < g.zs || z >= g.ze) {
        if (b.zero_foreign_planes && threadIdx.x == 0) psum[z] = 0.0;
        return;
    }
    const long long m = (long long)cdiv(g.nx, 32) * cdiv(g.ny, 8) * 8;
    const double* __restrict__ pz = b.partials + ((long long)pair * g.nz + z) * m;
    double s = 0.0;
    for (long long i = threadIdx.x; i < m; i += blockDim.x) s += __ldcg(pz + i);
    s = block_sum(s, red);
    if (threadIdx.x == 0) psum[z] = s;
}

void launch_plane_sums(const Batch& b, cudaStream_t s) {
    k_plane_sums<<<dim3(b.g.nz, b.pairs), 256, 0, s>>>(b);
    ++g_kernel_launches;
}

// MSE forward: one fp64 partial of sum (f - Mw)^2 per
// (plane, tile, warp) in the K1b layout, then the same fixed-order plane
// reduction; K5 turns it into r = loss_raw = MSE.
__global__ void __launch_bounds__(256) k_mse_fwd(Batch b, int chunk_len) {
    const int pair = b.pair0 + blockIdx.z;
    const PairState* st = b.st + pair;
    if (st->done) return;
    const Geo g = b.g;
    const int nxy = g.nx * g.ny;
    const int tiles_x = cdiv(g.nx, 32);
    const int tiles = tiles_x * cdiv(g.ny, 8);
    const int ox = threadIdx.x & 31, oy = threadIdx.x >> 5;
    const int x = (blockIdx.x % tiles_x) * 32 + ox, y = (blockIdx.x / tiles_x) * 8 + oy;
    const bool own = x < g.nx && y < g.ny;
    const int zb = g.zs + blockIdx.y * chunk_len, ze = min(zb + chunk_len, g.ze);
    const float* __restrict__ F = b.F + (long long)pair * g.nfull;
    const double* __restrict__ MW = b.MW + (long long)pair * g.n;
    double* __restrict__ part = b.partials + (long long)pair * g.nz * tiles * 8;
    const int ooff = x + g.nx * y;
    for (int z = zb; z < ze; ++z) {
        double e2 = 0.0;
        if (own) {
            const double e = (double)__ldg(F + z * nxy + ooff) - __ldg(MW + (z - g.zlo) * nxy + ooff);
            e2 = e * e;
        }
        e2 = warp_sum(e2);
        if (ox == 0) part[((long long)z * tiles + blockIdx.x) * 8 + oy] = e2;
    }
}

// MSE gradient: g = -2 (f - Mw) / N * grad M(x+u) at the accepted warp
// (the oracle's orc_residual_mse arithmetic); skipped after a rejection, like
// K2, because the gradient is unchanged.  With the Demons optimizer the same
// per-voxel residual r_x = f - Mw and n_x = grad M(x+u) give the Eq. 9 step
// instead, which K3 then smooths like an Adam step.
__global__ void __launch_bounds__(256) k_mse_grad(Batch b, int demons, double alpha) {
    const int pair = b.pair0 + blockIdx.z;
    const PairState* st = b.st + pair;
    if (st->done || st->last_rejected) return;
    const Geo g = b.g;
    const int tiles_x = cdiv(g.nx, 32);
    const int x = (blockIdx.x % tiles_x) * 32 + (threadIdx.x & 31);
    const int y = (blockIdx.x / tiles_x) * 8 + (threadIdx.x >> 5);
    if (x >= g.nx || y >= g.ny) return;
    const int z = g.zs + blockIdx.y;
    const long long n = g.n;
    const float* __restrict__ M = b.M + (long long)pair * g.nfull;
    const float* __restrict__ F = b.F + (long long)pair * g.nfull;
    const float* __restrict__ U = b.U + ((long long)pair * 2 + st->cur) * 3 * n;
    float* __restrict__ G = b.G + (long long)pair * 3 * n;
    const int o = g.lat(x, y, z);
    double grad[3];
    const double mw = sample_vol<true>(M, g, x, y, z, __ldg(U + o), __ldg(U + n + o), __ldg(U + 2 * n + o), grad);
    const double e = (double)__ldg(F + g.at(x, y, z)) - mw;
    if (demons) {
        double st3[3];
        demons_step(e, grad[0], grad[1], grad[2], alpha, st3);
        G[o] = (float)st3[0];
        G[n + o] = (float)st3[1];
        G[2 * n + o] = (float)st3[2];
        return;
    }
    const double k = -2.0 * e / (double)g.nfull;
    G[o] = (float)(k * grad[0]);
    G[n + o] = (float)(k * grad[1]);
    G[2 * n + o] = (float)(k * grad[2]);
}

// ---- MI (A13-A15, the oracle's orc_residual_mi) ----
constexpr int kParzenMax = 17;  // bins reached by |t - k| <= 4 sigma, sigma <= 2
struct ParzenD {
    int lo, n;
    double w[kParzenMax], dw[kParzenMax];
};
__device__ __forceinline__ void parzen_d(double t, int B, double sigma, ParzenD& P, bool deriv) {
    const double reach = 4.0 * sigma;
    const int lo = max((int)ceil(t - reach), 0), hi = min((int)floor(t + reach), B - 1);
    P.lo = lo;
    P.n = max(0, min(hi - lo + 1, kParzenMax));
    double S = 0.0, Sd = 0.0;
    for (int k = 0; k < P.n; ++k) {
        const double sft = t - (double)(lo + k);
        const double raw = exp(-0.5 * sft * sft / (sigma * sigma));
        P.w[k] = raw;
        P.dw[k] = -sft / (sigma * sigma) * raw;
        S += raw;
        Sd += P.dw[k];
    }
    for (int k = 0; k < P.n; ++k) {
        if (deriv) P.dw[k] = (P.dw[k] * S - P.w[k] * Sd) / (S * S);
        P.w[k] = P.w[k] / S;
    }
}
__device__ __forceinline__ double mi_scale(double lo, double hi, int B) {
    return (double)(B - 1) / (hi > lo ? hi - lo : 1.0);
}

// Joint histogram of the owned voxels: per-CTA fixed-point (2^-32) shared
// histogram, integer atomics (exact, so the sum is independent of order,
// chunking and slab split), merged into HIST.
__global__ void __launch_bounds__(256) k_mi_hist(Batch b, LmParams p, int chunk_len) {
    extern __shared__ unsigned long long sh_hist[];
    const int pair = b.pair0 + blockIdx.z;
    const PairState* st = b.st + pair;
    if (st->done) return;
    const Geo g = b.g;
    const int B = p.mi_bins;
    for (int i = threadIdx.x; i < B * B; i += blockDim.x) sh_hist[i] = 0ull;
    __syncthreads();
    const int nxy = g.nx * g.ny;
    const int tiles_x = cdiv(g.nx, 32);
    const int x = (blockIdx.x % tiles_x) * 32 + (threadIdx.x & 31), y = (blockIdx.x / tiles_x) * 8 + (threadIdx.x >> 5);
    const int zb = g.zs + blockIdx.y * chunk_len, ze = min(zb + chunk_len, g.ze);
    const double sf = mi_scale(st->lo_f, st->hi_f, B), sm = mi_scale(st->lo_m, st->hi_m, B);
    const float* __restrict__ F = b.F + (long long)pair * g.nfull;
    const double* __restrict__ MW = b.MW + (long long)pair * g.n;
    if (x < g.nx && y < g.ny) {
        for (int z = zb; z < ze; ++z) {
            ParzenD a, c;
            parzen_d(((double)__ldg(F + z * nxy + x + g.nx * y) - st->lo_f) * sf, B, p.mi_sigma, a, false);
            parzen_d((__ldg(MW + (z - g.zlo) * nxy + x + g.nx * y) - st->lo_m) * sm, B, p.mi_sigma, c, false);
            for (int i = 0; i < a.n; ++i)
                for (int j = 0; j < c.n; ++j)
                    atomicAdd(&sh_hist[(a.lo + i) * B + c.lo + j],
                              (unsigned long long)llrint(a.w[i] * c.w[j] * 4294967296.0));
        }
    }
    __syncthreads();
    unsigned long long* H = b.HIST + (long long)pair * B * B;
    for (int i = threadIdx.x; i < B * B; i += blockDim.x)
        if (sh_hist[i]) atomicAdd(&H[i], sh_hist[i]);
}

// MI from the histogram (fixed-order reductions), the gradient table, then
// the loss / damping / rejection state machine; clears the histogram.
__global__ void k_mi_finalize(Batch b, LmParams p, int mode) {
    __shared__ double red[32];
    __shared__ double s_pm[64];
    const int pair = b.pair0 + blockIdx.x;
    PairState* st = b.st + pair;
    if (st->done) return;
    const int B = p.mi_bins;
    unsigned long long* H = b.HIST + (long long)pair * B * B;
    double* T = b.MIT + (long long)pair * B * B;
    const double invN = 1.0 / (double)b.g.nfull, unit = 1.0 / 4294967296.0, eps = 1e-12;
    const double il2 = 1.0 / log(2.0);
    // marginals: thread j sums column j (moving), thread B + i row i (fixed)
    double part = 0.0;
    if (threadIdx.x < B) {
        double s = 0.0;
        for (int i = 0; i < B; ++i) s += (double)H[i * B + threadIdx.x] * unit * invN;
        s_pm[threadIdx.x] = s;
    }
    __syncthreads();
    if (threadIdx.x < B) {  // - p_m log p_m
        const double pm = s_pm[threadIdx.x];
        part -= pm * log2(fmax(pm, eps));
    } else if (threadIdx.x < 2 * B) {  // - p_f log p_f
        const int i = threadIdx.x - B;
        double pf = 0.0;
        for (int j = 0; j < B; ++j) pf += (double)H[i * B + j] * unit * invN;
        part -= pf * log2(fmax(pf, eps));
    }
    for (int k = threadIdx.x; k < B * B; k += blockDim.x) {  // + p log p, gradient table
        const double pij = (double)H[k] * unit * invN;
        const double pm = s_pm[k % B];
        part += pij * log2(fmax(pij, eps));
        T[k] = (log2(fmax(pij, eps)) + (pij >= eps ? il2 : 0.0)) - (log2(fmax(pm, eps)) + (pm >= eps ? il2 : 0.0));
    }
    const double mi = block_sum(part, red);
    for (int k = threadIdx.x; k < B * B; k += blockDim.x) H[k] = 0ull;
    if (threadIdx.x == 0) finalize_pair(st, p, mode, mi, pair);
}

// g = dr/dMw grad M(x+u), dr/dMw = -(1/N) s_m sum_i a_i(t_f) sum_j b'_j(t_m) T_ij
// at the accepted warp; skipped after a rejection (gradient unchanged).
__global__ void __launch_bounds__(256) k_mi_grad(Batch b, LmParams p) {
    const int pair = b.pair0 + blockIdx.z;
    const PairState* st = b.st + pair;
    if (st->done || st->last_rejected) return;
    const Geo g = b.g;
    const int tiles_x = cdiv(g.nx, 32);
    const int x = (blockIdx.x % tiles_x) * 32 + (threadIdx.x & 31);
    const int y = (blockIdx.x / tiles_x) * 8 + (threadIdx.x >> 5);
    if (x >= g.nx || y >= g.ny) return;
    const int z = g.zs + blockIdx.y;
    const int B = p.mi_bins;
    const long long n = g.n;
    const float* __restrict__ M = b.M + (long long)pair * g.nfull;
    const float* __restrict__ F = b.F + (long long)pair * g.nfull;
    const float* __restrict__ U = b.U + ((long long)pair * 2 + st->cur) * 3 * n;
    const double* __restrict__ T = b.MIT + (long long)pair * B * B;
    float* __restrict__ G = b.G + (long long)pair * 3 * n;
    const int o = g.lat(x, y, z);
    double grad[3];
    const double mw = sample_vol<true>(M, g, x, y, z, __ldg(U + o), __ldg(U + n + o), __ldg(U + 2 * n + o), grad);
    const double sf = mi_scale(st->lo_f, st->hi_f, B), sm = mi_scale(st->lo_m, st->hi_m, B);
    ParzenD a, c;
    parzen_d(((double)__ldg(F + g.at(x, y, z)) - st->lo_f) * sf, B, p.mi_sigma, a, false);
    parzen_d((mw - st->lo_m) * sm, B, p.mi_sigma, c, true);
    double s = 0.0;
    for (int i = 0; i < a.n; ++i) {
        double t = 0.0;
        for (int j = 0; j < c.n; ++j) t += c.dw[j] * __ldg(T + (a.lo + i) * B + c.lo + j);
        s += a.w[i] * t;
    }
    const double dr = -(1.0 / (double)g.nfull) * sm * s;
    G[o] = (float)(dr * grad[0]);
    G[n + o] = (float)(dr * grad[1]);
    G[2 * n + o] = (float)(dr * grad[2]);
}

// K1b: LNCC forward window pass.
//   halo tile (H = R): f' = F - shift_f, m' = Mw - shift_m              (fp64)
//   box sums S_f, S_m, S_ff, S_mm, S_fm over the truncated window      (fp64)
//   rho = c / sqrt(vf vm); A = 1/(n sqrt(vf vm)); B = -rho/(n vm)  -> fp32
//   E = A' mu_f' + B' mu_m'  (fp64, from the rounded A', B', so K2's
//   f' S_A + m' S_B - S_E cancels exactly).
//   sum(rho): one partial per (plane, tile, warp); k_plane_sums (one CTA per
//   plane) reduces them in a fixed order into plane_sum[z].
// Schedule (as K3): one barrier per plane; phase p runs the y-pass of plane p
// (z ring, plane p - R out), the x-pass of plane p+1 (two outputs per thread
// from 16-byte shared loads), the halo tile of plane p+2 and the loads of
// plane p+3.
namespace k1 {
constexpr int TX = 32, TY = 8, NT = 256;
template <int R>
struct Shape {
    static constexpr int IWP = TX + 2 * R, IH = TY + 2 * R, NI = IWP * IH;
    static constexpr int SL = (NI + NT - 1) / NT;
    static constexpr int NV = (2 + 2 * R + 1) / 2;
};
}  // namespace k1

template <int R, bool PEER = false>
__global__ void __launch_bounds__(k1::NT, 2) k_lncc_fwd(Batch b, int chunk_len) {
    using S = k1::Shape<R>;
    constexpr int TX = k1::TX, NT = k1::NT, W = 2 * R + 1;
    constexpr int IWP = S::IWP, IH = S::IH, NI = S::NI, SL = S::SL, NV = S::NV;
    __shared__ __align__(16) double s_in[2][2][NI];  // [buffer][f', m'][tile]
    __shared__ __align__(16) double s_x[2][5][IH * TX];

    const int pair = b.pair0 + blockIdx.z;
    PairState* st = b.st + pair;
    if (st->done) return;
    const Geo g = b.g;
    const int nxy = g.nx * g.ny;
    const int tiles_x = cdiv(g.nx, TX);
    const int x0 = (blockIdx.x % tiles_x) * TX, y0 = (blockIdx.x / tiles_x) * k1::TY;
    const int zb = g.zs + blockIdx.y * chunk_len, ze = min(zb + chunk_len, g.ze);
    const float* __restrict__ F = b.F + (long long)pair * g.nfull;
    const double* __restrict__ MW = b.MW + (long long)pair * g.n;
    float* __restrict__ Aout = b.ABE + (long long)pair * 4 * g.n;
    float* __restrict__ Bout = Aout + g.n;
    double* __restrict__ Eout = reinterpret_cast<double*>(Aout + 2 * g.n);
    const double shf = st->shift_f, shm = st->shift_m;
    const int tiles = cdiv(g.nx, TX) * cdiv(g.ny, k1::TY);
    double* __restrict__ part = b.partials + (long long)pair * g.nz * tiles * (NT / 32);
    double* __restrict__ part_cta = part + blockIdx.x * (NT / 32) + (threadIdx.x >> 5);  // + plane * part_plane
    const int part_plane = tiles * (NT / 32);

    int hoff[SL];
#pragma unroll
    for (int s = 0; s < SL; ++s) {
        const int idx = threadIdx.x + s * NT;
        const int gx = x0 - R + idx % IWP, gy = y0 - R + idx / IWP;
        hoff[s] = (idx < NI && gx >= 0 && gx < g.nx && gy >= 0 && gy < g.ny) ? gx + g.nx * gy : -1;
    }
    float df[SL];
    double dm[SL];
    auto load_dense = [&](int z) {
        const bool zin = z >= 0 && z < g.nz && z < ze + R;
#pragma unroll
        for (int s = 0; s < SL; ++s) {
            if (zin && hoff[s] >= 0) {
                df[s] = __ldg(F + z * nxy + hoff[s]);
                dm[s] = __ldg(MW + (z - g.zlo) * nxy + hoff[s]);
            } else {
                df[s] = 0.f;
                dm[s] = 0.0;
            }
        }
    };
    // absent (out-of-volume) items contribute 0 to every sum (truncated
    // windows, A2); present items may carry NaN, which propagates
    auto complete = [&](int z, double* dst) {
        const bool zin = z >= 0 && z < g.nz;
#pragma unroll
        for (int s = 0; s < SL; ++s) {
            const int idx = threadIdx.x + s * NT;
            if (idx >= NI) continue;
            const bool present = zin && hoff[s] >= 0;
            dst[idx] = present ? (double)df[s] - shf : 0.0;
            dst[NI + idx] = present ? dm[s] - shm : 0.0;
        }
    };
    // x pass: 5-tap box of (f, m, ff, mm, fm), two adjacent outputs
    const int xr = threadIdx.x >> 4, xj = threadIdx.x & 15;
    auto x_pass = [&](const double* in, double* out) {
        if (xr >= IH) return;
        double f[2 * NV], m[2 * NV];
        const double2* sf = reinterpret_cast<const double2*>(in + xr * IWP + 2 * xj);
        const double2* sm = reinterpret_cast<const double2*>(in + NI + xr * IWP + 2 * xj);
#pragma unroll
        for (int q = 0; q < NV; ++q) {
            const double2 a = sf[q], c = sm[q];
            f[2 * q] = a.x; f[2 * q + 1] = a.y;
            m[2 * q] = c.x; m[2 * q + 1] = c.y;
        }
        double a[2][5];
        // the two windows share taps 1..W-1: sum them once, then add the
        // outer tap of each side (a fixed order per output: chunk- and
        // slab-invariant like the direct sums)
        {
            double c0 = f[1], c1 = m[1], c2 = f[1] * f[1], c3 = m[1] * m[1], c4 = f[1] * m[1];
#pragma unroll
            for (int d = 2; d < W; ++d) {
                const double fv = f[d], mv = m[d];
                c0 += fv;
                c1 += mv;
                c2 = fma(fv, fv, c2);
                c3 = fma(mv, mv, c3);
                c4 = fma(fv, mv, c4);
            }
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const double fv = f[j * W], mv = m[j * W];
                a[j][0] = c0 + fv;
                a[j][1] = c1 + mv;
                a[j][2] = fma(fv, fv, c2);
                a[j][3] = fma(mv, mv, c3);
                a[j][4] = fma(fv, mv, c4);
            }
        }
        // the two outputs of a moment are adjacent: one 16-byte store each
#pragma unroll
        for (int c = 0; c < 5; ++c)
            *reinterpret_cast<double2*>(out + c * IH * TX + xr * TX + 2 * xj) = make_double2(a[0][c], a[1][c]);
    };

    const int ox = threadIdx.x & 31, oy = threadIdx.x >> 5;
    const int x = x0 + ox, y = y0 + oy;
    const bool own = x < g.nx && y < g.ny;
    const int cxy = own ? axis_count(x, g.nx, R) * axis_count(y, g.ny, R) : 1;
    const int ooff = x + g.nx * y;
    double ring[W][5];
#pragma unroll
    for (int d = 0; d < W; ++d)
#pragma unroll
        for (int c = 0; c < 5; ++c) ring[d][c] = 0.0;

    const int z0 = zb - R, z1 = ze + R;  // input planes [z0, z1)
    double* in_a = &s_in[0][0][0];
    double* in_b = &s_in[1][0][0];
    double* x_a = &s_x[0][0][0];
    double* x_b = &s_x[1][0][0];
    load_dense(z0);
    complete(z0, in_a);
    load_dense(z0 + 1);
    complete(z0 + 1, in_b);
    __syncthreads();
    x_pass(in_a, x_a);
    load_dense(z0 + 2);
    __syncthreads();
    for (int zbase = z0; zbase < z1; zbase += W) {
#pragma unroll
        for (int rs = 0; rs < W; ++rs) {
            const int zi = zbase + rs;
            if (zi < z1) {
                // y pass into the static ring; z sum taken directly over the ring
#pragma unroll
                for (int c = 0; c < 5; ++c) {
                    double s = x_a[c * IH * TX + oy * TX + ox];
#pragma unroll
                    for (int d = 1; d < W; ++d) s += x_a[c * IH * TX + (oy + d) * TX + ox];
                    ring[rs][c] = s;
                }
                const int zo = zi - R;
                if (zo >= zb) {
                    double rho = 0.0;
                    if (own) {
                        double Sm[5];
#pragma unroll
                        for (int c = 0; c < 5; ++c) {
                            double s = ring[(rs + 1) % W][c];
#pragma unroll
                            for (int d = 1; d < W; ++d) s += ring[(rs + 1 + d) % W][c];
                            Sm[c] = s;
                        }
                        const double inv = c_inv_count[cxy * axis_count(zo, g.nz, R)];
                        const double mf = Sm[0] * inv, mm = Sm[1] * inv;
                        const double vf = fma(-mf, mf, Sm[2] * inv);
                        const double vm = fma(-mm, mm, Sm[3] * inv);
                        const double cv = fma(-mf, mm, Sm[4] * inv);
                        const double af = mf + shf, am = mm + shm;
                        const double msf = fma(af, af, vf), msm = fma(am, am, vm);
                        double Ee = 0.0;
                        float Aa = 0.f, Bb = 0.f;
                        // NaN moments are not degenerate: non-finite inputs reach the loss
                        const bool degenerate = msf <= 0.0 || msm <= 0.0 || vf <= 1e-9 * msf || vm <= 1e-9 * msm;
                        if (!degenerate) {
                            const double alpha = hot::rsqrt_d(vf * vm);
                            rho = cv * alpha;
                            Aa = (float)(alpha * inv);
                            Bb = (float)(-rho * alpha * alpha * vf * inv);  // -rho / (n vm)
                            Ee = fma((double)Aa, mf, (double)Bb * mm);
                        }
                        const int o = (zo - g.zlo) * nxy + ooff;
                        Aout[o] = Aa;
                        Bout[o] = Bb;
                        Eout[o] = Ee;
                        if (PEER) {
#pragma unroll
                            for (int sd = 0; sd < 2; ++sd)
                                if (peer_sends(b, sd, 3, zo)) {
                                    float* Rm = b.peer.abe[sd];
                                    const long long rn = b.peer.n[sd], ri = peer_index(b, sd, zo, nxy, ooff);
                                    Rm[ri] = Aa;
                                    Rm[rn + ri] = Bb;
                                    reinterpret_cast<double*>(Rm + 2 * rn)[ri] = Ee;
                                    __threadfence_system();  // visible to the peer GPU before the token
                                }
                        }
                    }
                    rho = warp_sum(rho);
                    if (ox == 0) part_cta[(long long)zo * part_plane] = rho;
                }
                x_pass(in_b, x_b);
                complete(zi + 2, in_a);
                load_dense(zi + 3);
                double* t = in_a; in_a = in_b; in_b = t;
                t = x_a; x_a = x_b; x_b = t;
                __syncthreads();
            }
        }
    }

}

// K5: r from the per-plane sums in z order (identical on every rank for any
// slab split), then the loss / damping / rejection state machine.
__global__ void k_finalize(Batch b, LmParams p, int mode) {
    __shared__ double red[32];
    const int pair = b.pair0 + blockIdx.x;
    PairState* st = b.st + pair;
    if (st->done) return;
    const double* psum = b.plane_sum + (long long)pair * b.g.nz;
    double s = 0.0;
    // fixed partition of z (thread t: z = t, t+NT, ...), then a fixed tree
    for (int z = threadIdx.x; z < b.g.nz; z += blockDim.x) s += psum[z];
    const double tot = block_sum(s, red);
    if (threadIdx.x == 0) finalize_pair(st, p, mode, tot / (double)b.g.nfull, pair);
}

// ---------------------------------------------------------------------------
// K2: LNCC backward.  Adjoint box sums of (A, B, E) over the same windows in
// fp64; dr/dMw(x) = -(1/N)(f'_x S_A + m'_x S_B - S_E); g = dr/dMw grad M(x+u).
// Schedule (as K1b): one barrier per plane; phase p runs the y-pass of plane p
// (z ring, output plane p - R), the x-pass of plane p+1 (two outputs per
// thread from 16-byte shared loads), the halo tile of plane p+2 and the loads
// of plane p+3.  F, Mw and grad M(x+u) of the output voxels (K1a's
// evaluation of this warp, no gathers here) are copied one plane ahead by
// cp.async into shared memory, which keeps them out of the register file:
// K2 0.99 -> 0.90 ms against register staging three planes ahead.  The
// tunables below were measured with tools/ab_bench.sh.
namespace k2 {
constexpr int TX = 32, TY = 8, NT = 256;
template <int R>
struct Shape {
    static constexpr int IWP = TX + 2 * R, IH = TY + 2 * R, NI = IWP * IH;
    static constexpr int SL = (NI + NT - 1) / NT;
    static constexpr int NV = (2 + 2 * R + 1) / 2;
};
// per-voxel inputs of the output planes (F, Mw, grad M from K1a), staged by
// cp.async into a ring of OWN_SLOTS planes in dynamic shared memory; each
// thread copies and later reads only its own voxel, so no barrier guards it
#ifndef WLM_K2_OWN_SLOTS
#define WLM_K2_OWN_SLOTS 2
#endif
#ifndef WLM_K2_HALO_DEPTH
#define WLM_K2_HALO_DEPTH 1
#endif
constexpr int HALO_DEPTH = WLM_K2_HALO_DEPTH;  // halo planes in flight in registers
constexpr int OWN_SLOTS = WLM_K2_OWN_SLOTS;  // power of two
constexpr int OWN_AHEAD = OWN_SLOTS - 1;
struct OwnSlot {
    double mw[NT];
    double gm[3][NT];
    float f[NT];
};
// low-memory layout: the accepted warp of the output voxel instead of K1a's
// Mw and grad M; K2 gathers M(x + u) itself (sample_vol, K1a's arithmetic)
struct OwnSlotLean {
    float u[3][NT];
    float f[NT];
};
constexpr size_t OWN_BYTES = sizeof(OwnSlot) * OWN_SLOTS;
constexpr size_t OWN_BYTES_LEAN = sizeof(OwnSlotLean) * OWN_SLOTS;
}  // namespace k2

template <int R, bool LEAN, bool PEER = false>
#ifndef WLM_K2_MIN_BLOCKS
#define WLM_K2_MIN_BLOCKS 2
#endif
__global__ void __launch_bounds__(k2::NT, WLM_K2_MIN_BLOCKS) k_lncc_bwd(Batch b, LmParams p, int chunk_len) {
    using S = k2::Shape<R>;
    constexpr int TX = k2::TX, NT = k2::NT, W = 2 * R + 1;
    constexpr int IWP = S::IWP, IH = S::IH, NI = S::NI, SL = S::SL, NV = S::NV;
    __shared__ __align__(16) double s_in[2][3][NI];
    __shared__ __align__(16) double s_x[2][3][IH * TX];
    extern __shared__ __align__(16) unsigned char k2_smem[];
    k2::OwnSlot* const s_own = reinterpret_cast<k2::OwnSlot*>(k2_smem);
    k2::OwnSlotLean* const s_lean = reinterpret_cast<k2::OwnSlotLean*>(k2_smem);
    (void)p;

    const int pair = b.pair0 + blockIdx.z;
    const PairState* st = b.st + pair;
    if (st->done || st->last_rejected) return;
    const Geo g = b.g;
    const long long n = g.n;
    const int nxy = g.nx * g.ny;
    const int tiles_x = cdiv(g.nx, TX);
    const int x0 = (blockIdx.x % tiles_x) * TX, y0 = (blockIdx.x / tiles_x) * k2::TY;
    const int zb = g.zs + blockIdx.y * chunk_len, ze = min(zb + chunk_len, g.ze);
    const float* __restrict__ F = b.F + (long long)pair * g.nfull;
    const float* __restrict__ A = b.ABE + (long long)pair * 4 * n;
    const float* __restrict__ Bc = A + n;
    const double* __restrict__ E = reinterpret_cast<const double*>(A + 2 * n);
    float* __restrict__ G = b.G + (long long)pair * 3 * n;
    const double shf = st->shift_f, shm = st->shift_m;
    const double invN = 1.0 / (double)g.nfull;

    int hoff[SL];
#pragma unroll
    for (int s = 0; s < SL; ++s) {
        const int idx = halo_item(s, SL, NI, NT);
        const int gx = x0 - R + idx % IWP, gy = y0 - R + idx / IWP;
        hoff[s] = (idx >= 0 && gx >= 0 && gx < g.nx && gy >= 0 && gy < g.ny) ? gx + g.nx * gy : -1;
    }
    // halo registers, HALO_DEPTH planes in flight: h[0] is stored this
    // phase, the rest were loaded in earlier phases and move down after it
    constexpr int HD = k2::HALO_DEPTH;
    float ha[HD][SL], hb[HD][SL];
    double he[HD][SL];
    auto load_halo = [&](int z, int j) {
        const bool zin = z >= 0 && z < g.nz && z < ze + R;
        const int base = (z - g.zlo) * nxy;
#pragma unroll
        for (int s = 0; s < SL; ++s) {
            if (zin && hoff[s] >= 0) {
                ha[j][s] = __ldg(A + base + hoff[s]);
                hb[j][s] = __ldg(Bc + base + hoff[s]);
                he[j][s] = __ldg(E + base + hoff[s]);
            } else {
                ha[j][s] = hb[j][s] = 0.f;
                he[j][s] = 0.0;
            }
        }
    };
    auto store_halo = [&](double* dst) {
#pragma unroll
        for (int s = 0; s < SL; ++s) {
            const int idx = halo_item(s, SL, NI, NT);
            if (idx < 0) continue;
            dst[idx] = (double)ha[0][s];
            dst[NI + idx] = (double)hb[0][s];
            dst[2 * NI + idx] = he[0][s];
        }
    };
    auto shift_halo = [&] {
#pragma unroll
        for (int j = 0; j + 1 < HD; ++j)
#pragma unroll
            for (int s = 0; s < SL; ++s) {
                ha[j][s] = ha[j + 1][s];
                hb[j][s] = hb[j + 1][s];
                he[j][s] = he[j + 1][s];
            }
    };
    const int xr = threadIdx.x >> 4, xj = threadIdx.x & 15;
    auto x_pass = [&](const double* in, double* out) {
        if (xr >= IH) return;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            double v[2 * NV];
            const double2* src = reinterpret_cast<const double2*>(in + c * NI + xr * IWP + 2 * xj);
#pragma unroll
            for (int q = 0; q < NV; ++q) {
                const double2 t = src[q];
                v[2 * q] = t.x; v[2 * q + 1] = t.y;
            }
            // taps 1..W-1 are shared by the two windows (as K1b)
            double core = v[1];
#pragma unroll
            for (int d = 2; d < W; ++d) core += v[d];
            *reinterpret_cast<double2*>(out + c * IH * TX + xr * TX + 2 * xj) = make_double2(v[0] + core, core + v[W]);
        }
    };

    const int ox = threadIdx.x & 31, oy = threadIdx.x >> 5;
    const int x = x0 + ox, y = y0 + oy;
    const bool own = x < g.nx && y < g.ny;
    const int ooff = x + g.nx * y;
    // output pipeline: F, Mw and grad M of the accepted warp (K1a), copied
    // asynchronously OWN_AHEAD planes ahead, one commit group per plane
    const double* __restrict__ MWp = b.MW + (long long)pair * n;
    const double* __restrict__ GMp = b.GM + (long long)pair * 3 * n;
    const int t = threadIdx.x;
    const float* __restrict__ Uacc = b.U + ((long long)pair * 2 + st->cur) * 3 * n;
    auto issue_own = [&](int zo) {
        if (LEAN) {
            if (own && zo >= zb && zo < ze) {
                k2::OwnSlotLean& sl = s_lean[zo & (k2::OWN_SLOTS - 1)];
                const int o = (zo - g.zlo) * nxy + ooff;
                __pipeline_memcpy_async(&sl.f[t], F + zo * nxy + ooff, sizeof(float));
                __pipeline_memcpy_async(&sl.u[0][t], Uacc + o, sizeof(float));
                __pipeline_memcpy_async(&sl.u[1][t], Uacc + n + o, sizeof(float));
                __pipeline_memcpy_async(&sl.u[2][t], Uacc + 2 * n + o, sizeof(float));
            }
            __pipeline_commit();
            return;
        }
        if (own && zo >= zb && zo < ze) {
            k2::OwnSlot& sl = s_own[zo & (k2::OWN_SLOTS - 1)];
            const int o = (zo - g.zlo) * nxy + ooff;
            __pipeline_memcpy_async(&sl.f[t], F + zo * nxy + ooff, sizeof(float));
            __pipeline_memcpy_async(&sl.mw[t], MWp + o, sizeof(double));
            __pipeline_memcpy_async(&sl.gm[0][t], GMp + o, sizeof(double));
            __pipeline_memcpy_async(&sl.gm[1][t], GMp + n + o, sizeof(double));
            __pipeline_memcpy_async(&sl.gm[2][t], GMp + 2 * n + o, sizeof(double));
        }
        __pipeline_commit();
    };

    double ring[W][3];
#pragma unroll
    for (int d = 0; d < W; ++d)
#pragma unroll
        for (int c = 0; c < 3; ++c) ring[d][c] = 0.0;

    const int z0 = zb - R, z1 = ze + R;
    double* in_a = &s_in[0][0][0];
    double* in_b = &s_in[1][0][0];
    double* x_a = &s_x[0][0][0];
    double* x_b = &s_x[1][0][0];
    for (int q = 0; q < k2::OWN_AHEAD; ++q) issue_own(zb + q);
    load_halo(z0, 0);
    store_halo(in_a);
    load_halo(z0 + 1, 0);
    store_halo(in_b);
    __syncthreads();
    x_pass(in_a, x_a);
#pragma unroll
    for (int j = 0; j < HD; ++j) load_halo(z0 + 2 + j, j);
    __syncthreads();
    for (int zbase = z0; zbase < z1; zbase += W) {
#pragma unroll
        for (int rs = 0; rs < W; ++rs) {
            const int zi = zbase + rs;
            if (zi < z1) {
                const int zo = zi - R;
                const bool emit = zo >= zb;
                if (emit) issue_own(zo + k2::OWN_AHEAD);
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    double s = x_a[c * IH * TX + oy * TX + ox];
#pragma unroll
                    for (int d = 1; d < W; ++d) s += x_a[c * IH * TX + (oy + d) * TX + ox];
                    ring[rs][c] = s;
                }
                if (emit) __pipeline_wait_prior(k2::OWN_AHEAD);  // plane zo has landed
                if (emit && own) {
                    double Sm[3];
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        double s = ring[(rs + 1) % W][c];
#pragma unroll
                        for (int d = 1; d < W; ++d) s += ring[(rs + 1 + d) % W][c];
                        Sm[c] = s;
                    }
                    double mw, gm[3], fv;
                    if (LEAN) {
                        const k2::OwnSlotLean& sl = s_lean[zo & (k2::OWN_SLOTS - 1)];
                        mw = sample_vol<true>(b.M + (long long)pair * g.nfull, g, x, y, zo, sl.u[0][t], sl.u[1][t],
                                              sl.u[2][t], gm);
                        fv = sl.f[t];
                    } else {
                        const k2::OwnSlot& sl = s_own[zo & (k2::OWN_SLOTS - 1)];
                        mw = sl.mw[t];
                        gm[0] = sl.gm[0][t]; gm[1] = sl.gm[1][t]; gm[2] = sl.gm[2][t];
                        fv = sl.f[t];
                    }
                    const double f = fv - shf;
                    const double dm = -invN * (fma(f, Sm[0], (mw - shm) * Sm[1]) - Sm[2]);
                    const int o = (zo - g.zlo) * nxy + ooff;
                    G[o] = (float)(dm * gm[0]);
                    G[n + o] = (float)(dm * gm[1]);
                    G[2 * n + o] = (float)(dm * gm[2]);
                    if (PEER) {
#pragma unroll
                        for (int sd = 0; sd < 2; ++sd)
                            if (peer_sends(b, sd, 0, zo)) {
                                float* Rm = b.peer.g[sd] + peer_index(b, sd, zo, nxy, ooff);
                                const long long rn = b.peer.n[sd];
                                Rm[0] = (float)(dm * gm[0]);
                                Rm[rn] = (float)(dm * gm[1]);
                                Rm[2 * rn] = (float)(dm * gm[2]);
                                __threadfence_system();
                            }
                    }
                }
                x_pass(in_b, x_b);
                store_halo(in_a);
                shift_halo();
                load_halo(zi + 2 + HD, HD - 1);
                double* t = in_a; in_a = in_b; in_b = t;
                t = x_a; x_a = x_b; x_b = t;
                __syncthreads();
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Gaussian weights w[|d|] are truncated at R and renormalised per axis over
// in-bounds taps (field.cpp:236-244): zero-filled halos and a final divide by
// Wx(x) Wy(y) Wz(z).
template <class T>
__device__ __forceinline__ T axis_wsum_t(int p, int n, int R, const T* w, T full) {
    if (p >= R && p + R <= n - 1) return full;
    T s = 0;
    for (int d = -R; d <= R; ++d) {
        const int q = p + d;
        if (q >= 0 && q < n) s += w[d < 0 ? -d : d];
    }
    return s;
}

// K3: dU = -r g / (|g|^2 + lambda) (Eq. 4) | -lr g (GD) | Adam step (in G);
// Gaussian(sigma_update) in fp64; dU_s stored fp32; max |dU_s| (of the
// stored values) -> PairState.max_bits.
//
// fp64 arithmetic, fp32 storage (fp32 passes bias the
// trajectory, tools/precision_modes.py).  Tile 32 x 8; per plane a single
// barrier-separated phase does four independent things: the y-pass of plane
// p (s_x column -> z register ring -> plane p - R out), the x-pass of plane
// p+1 (two adjacent outputs per thread from 16-byte shared loads), the step
// of plane p+2 into the halo tile, and the global loads of plane p+3.
// fp64 reciprocal: hardware estimate + two Newton steps (x > 0 normal; within
// an ulp of the correctly rounded quotient, a fifth of __drcp_rn's cost).
__device__ __forceinline__ double rcp_d(double x) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    double e = fma(-x, y, 1.0);
    y = fma(y, e, y);
    e = fma(-x, y, 1.0);
    return fma(y, e, y);
}

// 1 / (in-bounds weight sum) of the 2R border planes of an axis of length n:
// t[k] for p = k, t[R + k] for p = n - 1 - k (k < R); filled once per CTA.
__device__ __forceinline__ void fill_border_inv(double* t, int n, int R, const double* w, double full) {
    const int k = threadIdx.x;
    if (k < 2 * R) {
        const int pp = k < R ? k : n - 1 - (k - R);
        t[k] = (pp >= 0 && pp < n) ? 1.0 / axis_wsum_t<double>(pp, n, R, w, full) : 0.0;
    }
}
__device__ __forceinline__ double border_inv(const double* t, int p, int n, int R) {
    return p < R ? t[p] : t[R + (n - 1 - p)];
}

#ifndef WLM_K3_COLUMN_Y
#define WLM_K3_COLUMN_Y 1
#endif
#ifndef WLM_K3_TY
#define WLM_K3_TY 16
#endif
namespace k3 {
// 32 x TY tiles of 32 TY threads; TY = 16 (one CTA of 512 per SM) halves
// the halo share of the LM-step producer against 32 x 8 (2.08 -> 1.63 halo
// items and 1.75 -> 1.375 x-pass rows per output)
constexpr int TX = 32, TY = WLM_K3_TY, NT = 32 * TY;
constexpr int MINB = NT <= 256 ? 2 : 1;
constexpr bool COLY = WLM_K3_COLUMN_Y;
constexpr int NQ = TY / 4;  // column y-pass: 4 outputs per thread, NQ per column
template <int R>
struct Shape {
    static constexpr int IWP = TX + 2 * R;  // halo row (even: 16-byte aligned rows of doubles)
    static constexpr int IH = TY + 2 * R;
    static constexpr int NI = IWP * IH;
    static constexpr int SLOTS = (NI + NT - 1) / NT;
    static constexpr int NV = (2 + 2 * R + 1) / 2;  // 16-byte loads per x pair
    // dynamic shared memory (doubles): s_in[2][3][NI], s_x[2][3][IH*TX],
    // s_y[2][3][TY*TX] (column y-pass only)
    static constexpr int IN_D = 2 * 3 * NI, X_D = 2 * 3 * IH * TX, Y_D = COLY ? 2 * 3 * TY * TX : 0;
    static constexpr size_t BYTES = sizeof(double) * (IN_D + X_D + Y_D);
};
}  // namespace k3

template <int R, bool TILED, bool PEER = false>
__global__ void __launch_bounds__(k3::NT, k3::MINB) k_step_smooth(Batch b, LmParams p, int chunk_len) {
    using S = k3::Shape<R>;
    constexpr int TX = k3::TX, NT = k3::NT, W = 2 * R + 1;
    constexpr int IWP = S::IWP, IH = S::IH, NI = S::NI, SL = S::SLOTS, NV = S::NV;
    extern __shared__ __align__(16) double k3_smem[];
    double* const s_in0 = k3_smem;                 // [buffer][channel][NI]
    double* const s_x0 = k3_smem + S::IN_D;        // [buffer][channel][IH][TX]
    double* const s_y0 = s_x0 + S::X_D;            // [buffer][channel][TY][TX]
    __shared__ float s_max[NT / 32];
    __shared__ double s_binv[2 * (R > 0 ? R : 1)];

    const int pair = b.pair0 + blockIdx.z;
    PairState* st = b.st + pair;
    if (st->done) return;
    const Geo g = b.g;
    const long long n = g.n;
    const int nxy = g.nx * g.ny;
    const int tiles_x = cdiv(g.nx, TX);
    const int x0 = (blockIdx.x % tiles_x) * TX, y0 = (blockIdx.x / tiles_x) * k3::TY;
    fill_border_inv(s_binv, g.nz, R, p.wud, p.wud_full);
    const int zb = g.zs + blockIdx.y * chunk_len, ze = min(zb + chunk_len, g.ze);
    const float* __restrict__ Gin = b.G + (long long)pair * 3 * n;
    float* __restrict__ V = b.VS + (long long)pair * b.vs_ps;
    const int opt = p.optimizer;
    const double r = st->r_cur, lam = st->lambda;
    const double kc = opt == WLM_OPT_GD ? -p.gd_lr : 1.0;

    int hoff[SL];
#pragma unroll
    for (int s = 0; s < SL; ++s) {
        const int idx = halo_item(s, SL, NI, NT);
        const int ix = idx % IWP, iy = idx / IWP;
        const int gx = x0 - R + ix, gy = y0 - R + iy;
        hoff[s] = (idx >= 0 && gx >= 0 && gx < g.nx && gy >= 0 && gy < g.ny) ? gx + g.nx * gy : -1;
    }
    float hg[SL][3];
    auto load_halo = [&](int z) {
        const bool zin = z >= 0 && z < g.nz && z < ze + R;
        const int base = (z - g.zlo) * nxy;
#pragma unroll
        for (int s = 0; s < SL; ++s) {
            if (zin && hoff[s] >= 0) {
                const int o = base + hoff[s];
                hg[s][0] = __ldg(Gin + o); hg[s][1] = __ldg(Gin + n + o); hg[s][2] = __ldg(Gin + 2 * n + o);
            } else {
                hg[s][0] = hg[s][1] = hg[s][2] = 0.f;
            }
        }
    };
    // tiled LM (Eq. 5): the item's k^3 tile matrix -r (H + lambda I)^{-1}
    const int tk = p.tile_k;
    constexpr bool tiled = TILED;  // launched only for LM with tile_size > 1
    const double* __restrict__ TM = tiled ? b.TM + (long long)pair * 6 * b.tkx * b.tky * b.tkz : nullptr;
    int htile[SL];  // (y tile) * tkx + x tile of each halo item
#pragma unroll
    for (int s = 0; s < SL; ++s) {
        const int idx = halo_item(s, SL, NI, NT);
        const int gx = x0 - R + idx % IWP, gy = y0 - R + idx / IWP;
        htile[s] = (tiled && hoff[s] >= 0) ? (gy / tk) * b.tkx + gx / tk : 0;
    }
    int hz = 0;  // z tile of the plane being stored
    auto store_halo = [&](double* dst) {
#pragma unroll
        for (int s = 0; s < SL; ++s) {
            const int idx = halo_item(s, SL, NI, NT);
            if (idx < 0) continue;
            const double a = hg[s][0], bb = hg[s][1], c = hg[s][2];
            if (tiled) {
                const double* M6 = TM + ((long long)hz * b.tkx * b.tky + htile[s]) * 6;
                dst[idx] = M6[0] * a + M6[1] * bb + M6[2] * c;
                dst[NI + idx] = M6[1] * a + M6[3] * bb + M6[4] * c;
                dst[2 * NI + idx] = M6[2] * a + M6[4] * bb + M6[5] * c;
                continue;
            }
            double k = kc;
            if (opt == WLM_OPT_LM) k = -r * rcp_d(fma(a, a, fma(bb, bb, c * c)) + lam);
            dst[idx] = k * a;
            dst[NI + idx] = k * bb;
            dst[2 * NI + idx] = k * c;
        }
    };
    double w_[W];
#pragma unroll
    for (int d = 0; d < W; ++d) w_[d] = p.wud[d < R ? R - d : d - R];
#define w(d) w_[d]

    // x-pass item: row xr, pair xj (outputs x = 2xj, 2xj + 1); NT / 16 rows
    // per sweep, so radii with IH > 16 rows (R > 4) take a second sweep
    const int xr0 = threadIdx.x >> 4, xj = threadIdx.x & 15;
    auto x_row = [&](const double* in, double* out, int xr) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            double v[2 * NV];
            const double2* src = reinterpret_cast<const double2*>(in + c * NI + xr * IWP + 2 * xj);
#pragma unroll
            for (int q = 0; q < NV; ++q) {
                const double2 t = src[q];
                v[2 * q] = t.x; v[2 * q + 1] = t.y;
            }
            double o0 = 0.0, o1 = 0.0;
#pragma unroll
            for (int d = 0; d < W; ++d) {
                o0 = fma(w(d), v[d], o0);
                o1 = fma(w(d), v[d + 1], o1);
            }
            *reinterpret_cast<double2*>(out + c * IH * TX + xr * TX + 2 * xj) = make_double2(o0, o1);
        }
    };
    auto x_pass = [&](const double* in, double* out) {
        if (IH <= NT / 16) {
            if (xr0 < IH) x_row(in, out, xr0);
        } else {
            for (int xr = xr0; xr < IH; xr += NT / 16) x_row(in, out, xr);
        }
    };

    const int ox = threadIdx.x & 31, oy = threadIdx.x >> 5;
    const int x = x0 + ox, y = y0 + oy;
    const bool own = x < g.nx && y < g.ny;
    const double inv_xy = own ? 1.0 / (axis_wsum_t<double>(x, g.nx, R, p.wud, p.wud_full) *
                                       axis_wsum_t<double>(y, g.ny, R, p.wud, p.wud_full))
                              : 0.0;
    const double inv_full = inv_xy / p.wud_full;
    const int ooff = x + g.nx * y;

    double ring[W][3];
#pragma unroll
    for (int d = 0; d < W; ++d)
#pragma unroll
        for (int c = 0; c < 3; ++c) ring[d][c] = 0.0;
    float mx = 0.f;

    const int z0 = zb - R, z1 = ze + R;
    double* in_a = s_in0;              // halo tile of plane p + 2 (written)
    double* in_b = s_in0 + 3 * NI;     // halo tile of plane p + 1 (x-passed)
    double* x_a = s_x0;                // x-passed plane p (y-passed)
    double* x_b = s_x0 + 3 * IH * TX;
    double* y_a = s_y0;                // column pass: y-passed plane p (read by the ring)
    double* y_b = s_y0 + 3 * k3::TY * TX;
    // column y-pass: thread (channel yc, column ox, quarter yh) of the last
    // 3 NQ warps forms 4 outputs from its column's 4 + 2R x-sums held in
    // registers, in the same fma order as the per-output 7-tap sum
    constexpr int YH = 4, NQ = k3::NQ;
    // the column pass runs on the highest warps and the x-pass on the
    // lowest, so fewer warps carry both (K3 0.970 -> 0.966 ms at TY = 8)
    const int yt = (int)threadIdx.x - (NT - 3 * NQ * 32);
    const int yc = yt >= 0 ? yt / (NQ * 32) : 3, yh = (yt >> 5) % NQ;
    auto y_pass = [&](const double* in, double* out) {
        if (yc >= 3) return;
        double v[YH + 2 * R];
#pragma unroll
        for (int r = 0; r < YH + 2 * R; ++r) v[r] = in[yc * IH * TX + (yh * YH + r) * TX + ox];
#pragma unroll
        for (int o = 0; o < YH; ++o) {
            double acc = 0.0;
#pragma unroll
            for (int d = 0; d < W; ++d) acc = fma(w(d), v[o + d], acc);
            out[yc * k3::TY * TX + (yh * YH + o) * TX + ox] = acc;
        }
    };
    auto ztile = [&](int z) { return tiled && z >= 0 && z < g.nz ? z / tk : 0; };
    load_halo(z0);
    hz = ztile(z0);
    store_halo(in_a);
    load_halo(z0 + 1);
    hz = ztile(z0 + 1);
    store_halo(in_b);
    __syncthreads();
    x_pass(in_a, x_a);
    if (k3::COLY) {
        // deeper prologue: y_a = plane z0, x_b = plane z0+1, in_a = plane z0+2
        x_pass(in_b, x_b);
        load_halo(z0 + 2);
        __syncthreads();
        y_pass(x_a, y_a);
        hz = ztile(z0 + 2);
        store_halo(in_a);
        load_halo(z0 + 3);
        __syncthreads();
    } else {
        load_halo(z0 + 2);
        __syncthreads();
    }
    for (int zbase = z0; zbase < z1; zbase += W) {
#pragma unroll
        for (int rs = 0; rs < W; ++rs) {
            const int zi = zbase + rs;
            if (zi < z1) {
                if (k3::COLY) {
#pragma unroll
                    for (int c = 0; c < 3; ++c) ring[rs][c] = y_a[c * k3::TY * TX + oy * TX + ox];
                } else {
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        double s = 0.0;
#pragma unroll
                        for (int d = 0; d < W; ++d) s = fma(w(d), x_a[c * IH * TX + (oy + d) * TX + ox], s);
                        ring[rs][c] = s;
                    }
                }
                const int zo = zi - R;
                if (zo >= zb && own) {
                    double inv = inv_full;
                    if (zo < R || zo + R > g.nz - 1) inv = inv_xy * border_inv(s_binv, zo, g.nz, R);
                    const int o = (zo - g.zlo) * nxy + ooff;
                    float vv[3];
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        double s = 0.0;
#pragma unroll
                        for (int d = 0; d < W; ++d) s = fma(w(d), ring[(rs + 1 + d) % W][c], s);
                        const float v = (float)(s * inv);
                        V[c * n + o] = v;
                        vv[c] = v;
                        mx = fmaxf(mx, fabsf(v));
                    }
                    if (PEER) {
#pragma unroll
                        for (int sd = 0; sd < 2; ++sd)
                            if (peer_sends(b, sd, 1, zo)) {
                                float* Rm = b.peer.v[sd] + peer_index(b, sd, zo, nxy, ooff);
                                const long long rn = b.peer.n[sd];
                                Rm[0] = vv[0];
                                Rm[rn] = vv[1];
                                Rm[2 * rn] = vv[2];
                                __threadfence_system();
                            }
                    }
                }
                if (k3::COLY) {
                    y_pass(x_b, y_b);
                    x_pass(in_a, x_a);
                    hz = ztile(zi + 3);
                    store_halo(in_b);
                    load_halo(zi + 4);
                    double* t = y_a; y_a = y_b; y_b = t;
                } else {
                    x_pass(in_b, x_b);
                    hz = ztile(zi + 2);
                    store_halo(in_a);
                    load_halo(zi + 3);
                }
                double* t = in_a; in_a = in_b; in_b = t;
                t = x_a; x_a = x_b; x_b = t;
                __syncthreads();
            }
        }
    }
    mx = warp_max(mx);
    if ((threadIdx.x & 31) == 0) s_max[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        float m = 0.f;
        for (int i = 0; i < NT / 32; ++i) m = fmaxf(m, s_max[i]);
        atomic_max_nonneg(&st->max_bits, m);
    }
}

#undef w

// K4: u'(x) = d(x) + u(x + d(x)), d = eps dU_s, eps = target / max(max|dU_s|,
// floor) (Eq. 2, field.cpp:123-155), then Gaussian(sigma_warp); fp64
// arithmetic, fp32 storage.  The normalised step bounds |d| <= target < 0.5
// voxel, so every resample corner lies in the 3x3x3 neighbourhood of its
// voxel: the accepted warp (fp32 in HBM) is staged exactly in a 4-plane
// fp32 shared-memory ring (halo R + 1) and the compose "gathers" are
// shared-memory reads widened to fp64 (F2F runs on its own pipe; fp64 staging
// would double the shared-memory traffic of the gathers, the limiter).
// Reads the accepted buffer, writes the other one.
//
// Tile 32 x 8, one barrier per plane.  Phase p: y-pass of plane p (z ring,
// plane p - R out); x-pass of plane p+1; compose of plane p+2 into the halo
// tile (warp planes p+1..p+3 from the ring, its step from registers); warp
// plane p+4 into the ring; global loads of warp plane p+5 and step p+3.
#ifndef WLM_K4_FAST
#define WLM_K4_FAST 1
#endif
#ifndef WLM_K4_ROWS
#define WLM_K4_ROWS 1
#endif
#ifndef WLM_K4_FLOATTEST
#define WLM_K4_FLOATTEST 1
#endif
#ifndef WLM_K4_UW32
#define WLM_K4_UW32 0
#endif
namespace k4 {
constexpr int TX = 32, TY = 16, NT = 512;
template <int R>
struct Shape {
    // composed tile: IW = TX + 2R items a row, stored with the warp tile's row
    // stride so a warp's corner reads are consecutive (bank-conflict free)
    static constexpr int IW = TX + 2 * R, IH = TY + 2 * R;
    // warp tile: x origin x0 - XO (a 16-byte aligned TMA box start), rows
    // padded to 16 bytes (the box's inner extent), covering x0 - R - 1 ..
    // x0 + TX + R
    static constexpr int XO = 4;
    // WLM_K4_UW32 pads the rows to a multiple of 32 floats: the resample
    // reads of a warp come from two ring rows wherever the sign of d_y
    // changes along it, and a 40-float row stride (8 banks) makes lanes 24
    // apart collide (ncu: ~50% excess wavefronts on the corner reads).  The
    // 64-float rows remove that but cost more (TMA box and tile 60% wider):
    // K4 1.522 -> 1.600 ms, so the default keeps 40.
    static constexpr int UW0 = (TX + R + 1 + XO + 3) / 4 * 4;
    static constexpr int UW = WLM_K4_UW32 && R == 2 ? (UW0 + 31) / 32 * 32 : UW0;
    static constexpr int UH = TY + 2 * R + 2, UN = UW * UH;
    static constexpr int IWP = UW, NI = IWP * IH;
    // composed items enumerated compactly (IW per row); the last, partial
    // slot goes to the highest threads, away from the x-pass threads (the
    // lowest 16 * IH), so few warps carry both
    static constexpr int NIV = IW * IH;
    static constexpr int SL = (NIV + NT - 1) / NT, USL = (UN + NT - 1) / NT;
    static constexpr int NV = (2 + 2 * R + 1) / 2;
    // ring slot: [3][UH][UW] fp32 (one TMA box), 128-byte aligned
    static constexpr int SLOT = (3 * UN + 31) / 32 * 32;
    static constexpr uint32_t BOX_BYTES = 3u * UN * 4u;
    // dynamic shared memory layout (doubles)
    static constexpr int OFF_U = 0, OFF_IN = 4 * SLOT / 2, OFF_X = OFF_IN + 2 * 3 * NI;  // s_u fp32
    static constexpr int TOTAL = OFF_X + 2 * 3 * IH * TX;
    static constexpr int OFF_BAR = TOTAL + 8;  // 4 mbarriers (after s_binv)
    static constexpr size_t BYTES = sizeof(double) * (OFF_BAR + 4) + 128;  // + base alignment slack
};
}  // namespace k4

// ---- TMA (cp.async.bulk.tensor) + mbarrier helpers ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
// Bounded wait: a lost transfer traps (kernel error) instead of hanging.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    for (long long spins = 0; !done; ++spins) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
        if (spins > (1ll << 28)) __trap();
    }
}
__device__ __forceinline__ void tma_load_5d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                            int c4, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
        "%5, %6}], [%7];" ::"r"(smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(bar))
        : "memory");
}

// TMA: the accepted warp's plane z (all three components, the (UW x UH)
// box at the tile origin, zero-filled outside the volume like the register
// path) arrives in its ring slot by one bulk tensor copy issued by thread 0;
// consumers wait on the slot's mbarrier.  Used when the U rows are 16-byte
// multiples (nx % 4 == 0), else the register-staged path.
template <int R, bool TMA, bool PEER = false>
__global__ void __launch_bounds__(k4::NT, 1) k_compose_smooth(Batch b, LmParams p, int chunk_len,
                                                              const __grid_constant__ CUtensorMap tmap_u) {
    using S = k4::Shape<R>;
    constexpr int TX = k4::TX, NT = k4::NT, W = 2 * R + 1;
    constexpr int IWP = S::IWP, IH = S::IH, NI = S::NI, UW = S::UW, UN = S::UN, SL = S::SL, USL = S::USL,
                  NV = S::NV;
    extern __shared__ __align__(16) double k4_smem_raw[];
    // TMA writes need 128-byte aligned destinations: align the whole layout
    double* k4_smem = reinterpret_cast<double*>(
        reinterpret_cast<char*>(k4_smem_raw) + ((128 - (smem_u32(k4_smem_raw) & 127)) & 127));
    float* s_u = reinterpret_cast<float*>(k4_smem + S::OFF_U);  // [4 slots][3][UN] fp32
    double* s_in = k4_smem + S::OFF_IN;  // [2][3][NI]
    double* s_x = k4_smem + S::OFF_X;    // [2][3][IH * TX]
    double* s_binv = k4_smem + S::TOTAL; // [2R]
    uint64_t* s_bar = reinterpret_cast<uint64_t*>(k4_smem + S::OFF_BAR);  // [4] TMA ring slots

    const int pair = b.pair0 + blockIdx.z;
    const PairState* st = b.st + pair;
    if (st->done) return;
    const Geo g = b.g;
    const long long n = g.n;
    const int nxy = g.nx * g.ny;
    const int tiles_x = cdiv(g.nx, TX);
    const int x0 = (blockIdx.x % tiles_x) * TX, y0 = (blockIdx.x / tiles_x) * k4::TY;
    const int zb = g.zs + blockIdx.y * chunk_len, ze = min(zb + chunk_len, g.ze);
    const int cur = st->cur;
    const float* __restrict__ Vin = b.VS + (long long)pair * b.vs_ps;
    const float* __restrict__ U = b.U + ((long long)pair * 2 + cur) * 3 * n;
    float* __restrict__ UN_ = b.U + ((long long)pair * 2 + (1 - cur)) * 3 * n;
    const double eps = p.target / fmax((double)__uint_as_float(st->max_bits), p.step_floor);
    fill_border_inv(s_binv, g.nz, R, p.wwd, p.wwd_full);

    // warp staging items (tile origin x0 - XO, y0 - R - 1)
    int uoff[USL];
#pragma unroll
    for (int s = 0; s < USL; ++s) {
        const int idx = threadIdx.x + s * NT;
        const int gx = x0 - S::XO + idx % UW, gy = y0 - R - 1 + idx / UW;
        uoff[s] = (idx < UN && gx >= 0 && gx < g.nx && gy >= 0 && gy < g.ny) ? gx + g.nx * gy : -1;
    }
    // composed items (tile origin x0 - R, y0 - R): slot s of this thread is
    // item j (row j / IW, column j % IW) at tile index iidx[s] (-1: none)
    int voff[SL], vx[SL], vy[SL], iidx[SL];
#pragma unroll
    for (int s = 0; s < SL; ++s) {
        constexpr int REM = S::NIV - (SL - 1) * NT;  // items of the last slot
        int j = s < SL - 1 ? threadIdx.x + s * NT
                           : ((int)threadIdx.x >= NT - REM ? (SL - 1) * NT + (int)threadIdx.x - (NT - REM) : -1);
        if (WLM_K4_ROWS && R == 2 && SL == 2) {
            // Row-aligned dealing: a warp composes 32 consecutive columns of
            // one row (x0 .. x0 + 31), so its resample reads of a corner are
            // 32 consecutive floats of one ring row (conflict-free when the
            // lanes share the sign of d; the compact dealing straddled two
            // rows, 56% excess wavefronts).  Slot 0: warp w -> row w; slot 1:
            // the highest 4 warps -> rows 16..19, the 3 below them -> the
            // 2R-wide row ends (80 items), away from the x-pass warps.
            const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
            constexpr int NW = NT / 32, IHr = S::IH;
            constexpr int EXTRA = IHr - NW;         // rows left for slot 1 (4)
            constexpr int EDGE = IHr * 2 * R;        // row-end items (80)
            constexpr int EW = (EDGE + 31) / 32;     // warps for them (3)
            int row = -1, col = 0;
            if (s == 0) {
                row = w; col = R + lane;
            } else if (w >= NW - EXTRA) {
                row = NW + (w - (NW - EXTRA)); col = R + lane;
            } else if (w >= NW - EXTRA - EW) {
                const int e = (w - (NW - EXTRA - EW)) * 32 + lane;
                constexpr int R2 = 2 * R > 0 ? 2 * R : 1;  // (the branch runs for R == 2 only)
                if (e < EDGE) { row = e / R2; const int k = e % R2; col = k < R ? k : TX + k; }
            }
            j = row >= 0 ? row * S::IW + col : -1;
        }
        const int row = j / S::IW, col = j % S::IW;
        iidx[s] = j >= 0 ? row * IWP + col : -1;
        vx[s] = x0 - R + col;
        vy[s] = y0 - R + row;
        voff[s] = (j >= 0 && vx[s] >= 0 && vx[s] < g.nx && vy[s] >= 0 && vy[s] < g.ny) ? vx[s] + g.nx * vy[s] : -1;
    }
    float pu[USL][3], pv[SL][3];
    auto load_u = [&](int z) {
        const bool zin = z >= 0 && z < g.nz && z <= ze + R;
        const int base = (z - g.zlo) * nxy;
#pragma unroll
        for (int s = 0; s < USL; ++s) {
            if (zin && uoff[s] >= 0) {
                const int o = base + uoff[s];
                pu[s][0] = __ldg(U + o); pu[s][1] = __ldg(U + n + o); pu[s][2] = __ldg(U + 2 * n + o);
            } else {
                pu[s][0] = pu[s][1] = pu[s][2] = 0.f;
            }
        }
    };
    auto store_u = [&](int z) {
        float* dst = s_u + ((z + 4) & 3) * S::SLOT;
#pragma unroll
        for (int s = 0; s < USL; ++s) {
            const int idx = threadIdx.x + s * NT;
            if (idx >= UN) continue;
            dst[idx] = pu[s][0];
            dst[UN + idx] = pu[s][1];
            dst[2 * UN + idx] = pu[s][2];
        }
    };
    auto load_v = [&](int z) {
        const bool zin = z >= 0 && z < g.nz && z < ze + R;
        const int base = (z - g.zlo) * nxy;
#pragma unroll
        for (int s = 0; s < SL; ++s) {
            if (zin && voff[s] >= 0) {
                const int o = base + voff[s];
                pv[s][0] = __ldg(Vin + o); pv[s][1] = __ldg(Vin + n + o); pv[s][2] = __ldg(Vin + 2 * n + o);
            } else {
                pv[s][0] = pv[s][1] = pv[s][2] = 0.f;
            }
        }
    };
    // Every item in one branch-free path: |d| <= target < 1, so the cell
    // origin is x + floor(d) with floor(d) in {-1, 0}; the clamp rules of
    // field.cpp:19-39 (origin < 0 -> 0 with t = 0; origin > n-2 -> n-2 with
    // t = 1, which also covers a sample exactly on the last voxel) are two
    // selects per axis; n == 1 axes sample index 0 with t = 0.
    auto clamp_axis = [](int& i, double& t, int n) {
        if (n == 1) { i = 0; t = 0.0; return; }
        if (i < 0) { i = 0; t = 0.0; }
        else if (i > n - 2) { i = n - 2; t = 1.0; }
    };
    // Tiles whose composed items and resample cells all lie inside the
    // volume (x0 - R - 1 >= 0 ... x0 + TX + R <= nx - 2, likewise y; plane z
    // in [1, nz - 2]) take a path without the clamp rules and bounds tests:
    // every cell origin x + floor(d) is then in [0, n - 2] and no item is
    // absent, so both paths give the same bits (8% of K4's instructions were
    // the clamp tests).
    const bool tile_inner = WLM_K4_FAST && x0 - R - 1 >= 0 && x0 + TX + R <= g.nx - 2 && y0 - R - 1 >= 0 &&
                            y0 + k4::TY + R <= g.ny - 2;
    auto compose_inner = [&](int z, double* dst) {
#pragma unroll
        for (int s = 0; s < SL; ++s) {
            const int idx = iidx[s];
            if (idx < 0) continue;
            double o3[3];
            const double dx = eps * pv[s][0], dy = eps * pv[s][1], dz = eps * pv[s][2];
            // d = eps dU_s is finite iff the stored fp32 step is (eps <= target
            // / max |dU_s| keeps |d| <= target), and its sign is the step's
#if WLM_K4_FLOATTEST
            if (fmaxf(fabsf(pv[s][0]), fmaxf(fabsf(pv[s][1]), fabsf(pv[s][2]))) <= FLT_MAX) {
                const int fx = pv[s][0] < 0.f ? -1 : 0, fy = pv[s][1] < 0.f ? -1 : 0, fz = pv[s][2] < 0.f ? -1 : 0;
#else
            if (isfinite(dx + dy + dz)) {
                const int fx = dx < 0.0 ? -1 : 0, fy = dy < 0.0 ? -1 : 0, fz = dz < 0.0 ? -1 : 0;
#endif
                const double tx = dx - (double)fx, ty = dy - (double)fy, tz = dz - (double)fz;
                const int a = (vy[s] + fy - (y0 - R - 1)) * UW + vx[s] + fx - (x0 - S::XO);
                const float* p0 = s_u + ((z + fz + 4) & 3) * S::SLOT + a;
                const float* p1 = s_u + ((z + fz + 5) & 3) * S::SLOT + a;
#pragma unroll
                for (int ch = 0; ch < 3; ++ch) {
                    const double c000 = p0[ch * UN], c100 = p0[ch * UN + 1];
                    const double c010 = p0[ch * UN + UW], c110 = p0[ch * UN + UW + 1];
                    const double c001 = p1[ch * UN], c101 = p1[ch * UN + 1];
                    const double c011 = p1[ch * UN + UW], c111 = p1[ch * UN + UW + 1];
                    const double v00 = fma(tx, c100 - c000, c000), v10 = fma(tx, c110 - c010, c010);
                    const double v01 = fma(tx, c101 - c001, c001), v11 = fma(tx, c111 - c011, c011);
                    const double s0 = fma(ty, v10 - v00, v00), s1 = fma(ty, v11 - v01, v01);
                    o3[ch] = fma(tz, s1 - s0, s0);
                }
                o3[0] += dx;
                o3[1] += dy;
                o3[2] += dz;
            } else {
                o3[0] = o3[1] = o3[2] = kNaN64;
            }
            dst[idx] = o3[0];
            dst[NI + idx] = o3[1];
            dst[2 * NI + idx] = o3[2];
        }
    };
    // composed value of the items of plane z (step in pv) -> dst
    auto compose = [&](int z, double* dst) {
        if (tile_inner && z >= 1 && z <= g.nz - 2) {
            compose_inner(z, dst);
            return;
        }
        const bool zin = z >= 0 && z < g.nz;
#pragma unroll
        for (int s = 0; s < SL; ++s) {
            const int idx = iidx[s];
            if (idx < 0) continue;
            double o3[3] = {0.0, 0.0, 0.0};
            if (zin && voff[s] >= 0) {
                const double dx = eps * pv[s][0], dy = eps * pv[s][1], dz = eps * pv[s][2];
                if (isfinite(dx + dy + dz)) {
                    const int fx = dx < 0.0 ? -1 : 0, fy = dy < 0.0 ? -1 : 0, fz = dz < 0.0 ? -1 : 0;
                    double tx = dx - (double)fx, ty = dy - (double)fy, tz = dz - (double)fz;
                    int ix = vx[s] + fx, iy = vy[s] + fy, iz = z + fz;
                    clamp_axis(ix, tx, g.nx);
                    clamp_axis(iy, ty, g.ny);
                    clamp_axis(iz, tz, g.nz);
                    const int a = (iy - (y0 - R - 1)) * UW + ix - (x0 - S::XO);
                    const float* p0 = s_u + ((iz + 4) & 3) * S::SLOT + a;
                    const float* p1 = s_u + ((iz + 5) & 3) * S::SLOT + a;
#pragma unroll
                    for (int ch = 0; ch < 3; ++ch) {
                        const double c000 = p0[ch * UN], c100 = p0[ch * UN + 1];
                        const double c010 = p0[ch * UN + UW], c110 = p0[ch * UN + UW + 1];
                        const double c001 = p1[ch * UN], c101 = p1[ch * UN + 1];
                        const double c011 = p1[ch * UN + UW], c111 = p1[ch * UN + UW + 1];
                        const double v00 = fma(tx, c100 - c000, c000), v10 = fma(tx, c110 - c010, c010);
                        const double v01 = fma(tx, c101 - c001, c001), v11 = fma(tx, c111 - c011, c011);
                        const double s0 = fma(ty, v10 - v00, v00), s1 = fma(ty, v11 - v01, v01);
                        o3[ch] = fma(tz, s1 - s0, s0);
                    }
                    o3[0] += dx;
                    o3[1] += dy;
                    o3[2] += dz;
                } else {
                    o3[0] = o3[1] = o3[2] = kNaN64;
                }
            }
            dst[idx] = o3[0];
            dst[NI + idx] = o3[1];
            dst[2 * NI + idx] = o3[2];
        }
    };
    // TMA ring: plane q lands in slot (q + 4) & 3; its n-th use of the slot
    // (n = (q - first) / 4 with first = z0 - 1) completes mbarrier phase n & 1
    const int zfirst = zb - R - 1;
    auto tma_issue = [&](int z) {
        if (!TMA || threadIdx.x != 0) return;
        const int slot = (z + 4) & 3;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // prior generic reads of the slot
        mbar_expect_tx(&s_bar[slot], S::BOX_BYTES);
        tma_load_5d(s_u + slot * S::SLOT, &tmap_u, x0 - S::XO, y0 - R - 1, z - g.zlo, cur * 3, pair, &s_bar[slot]);
    };
    auto tma_wait = [&](int z) {
        if (TMA) mbar_wait(&s_bar[(z + 4) & 3], (uint32_t)(((z - zfirst) >> 2) & 1));
    };
#if WLM_CW_K4
#define wk(d) p.wwd[(d) < R ? R - (d) : (d) - R]
#else
    double wk_[W];
#pragma unroll
    for (int d = 0; d < W; ++d) wk_[d] = p.wwd[d < R ? R - d : d - R];
#define wk(d) wk_[d]
#endif
    const int xr = threadIdx.x >> 4, xj = threadIdx.x & 15;
    auto x_pass = [&](const double* in, double* out) {
        if (xr >= IH) return;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            double v[2 * NV];
            const double2* src = reinterpret_cast<const double2*>(in + c * NI + xr * IWP + 2 * xj);
#pragma unroll
            for (int q = 0; q < NV; ++q) {
                const double2 t = src[q];
                v[2 * q] = t.x; v[2 * q + 1] = t.y;
            }
            double o0 = 0.0, o1 = 0.0;
#pragma unroll
            for (int d = 0; d < W; ++d) {
                o0 = fma(wk(d), v[d], o0);
                o1 = fma(wk(d), v[d + 1], o1);
            }
            *reinterpret_cast<double2*>(out + c * IH * TX + xr * TX + 2 * xj) = make_double2(o0, o1);
        }
    };

    const int ox = threadIdx.x & 31, oy = threadIdx.x >> 5;
    const int x = x0 + ox, y = y0 + oy;
    const bool own = x < g.nx && y < g.ny;
    const double inv_xy = own ? 1.0 / (axis_wsum_t<double>(x, g.nx, R, p.wwd, p.wwd_full) *
                                       axis_wsum_t<double>(y, g.ny, R, p.wwd, p.wwd_full))
                              : 0.0;
    const double inv_full = inv_xy / p.wwd_full;
    const int ooff = x + g.nx * y;
    double ring[W][3];
#pragma unroll
    for (int d = 0; d < W; ++d)
#pragma unroll
        for (int c = 0; c < 3; ++c) ring[d][c] = 0.0;

    const int z0 = zb - R, z1 = ze + R;
    // prologue: warp planes z0-1 .. z0+2 staged; composed z0, z0+1; x-pass z0
    if (TMA) {
        if (threadIdx.x == 0) {
            for (int i = 0; i < 4; ++i) mbar_init(&s_bar[i], 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
        tma_issue(z0 - 1);
        tma_issue(z0);
        tma_issue(z0 + 1);
        tma_issue(z0 + 2);
    } else {
        load_u(z0 - 1); store_u(z0 - 1);
        load_u(z0);     store_u(z0);
        load_u(z0 + 1); store_u(z0 + 1);
        load_u(z0 + 2); store_u(z0 + 2);
    }
    load_v(z0);
    // double buffers as swapped pointers: halo tiles (composed) and x-passed
    double* in_a = s_in;           // composed plane p + 2 is written here
    double* in_b = s_in + 3 * NI;  // composed plane p + 1 is read here
    double* x_a = s_x;             // x-passed plane p is read here
    double* x_b = s_x + 3 * IH * TX;
    __syncthreads();
    tma_wait(z0 - 1);
    tma_wait(z0);
    tma_wait(z0 + 1);
    compose(z0, in_a);
    load_v(z0 + 1);
    if (!TMA) load_u(z0 + 3);
    __syncthreads();
    tma_issue(z0 + 3);  // slot of plane z0 - 1 (last read by compose(z0))
    x_pass(in_a, x_a);
    tma_wait(z0 + 2);
    compose(z0 + 1, in_b);
    if (!TMA) {
        store_u(z0 + 3);  // slot of plane z0 - 1 (not read by compose(z0 + 1))
        load_u(z0 + 4);
    }
    load_v(z0 + 2);
    __syncthreads();
    for (int zbase = z0; zbase < z1; zbase += W) {
#pragma unroll
        for (int rs = 0; rs < W; ++rs) {
            const int zi = zbase + rs;
            if (zi < z1) {
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    double s = 0.0;
#pragma unroll
                    for (int d = 0; d < W; ++d) s = fma(wk(d), x_a[c * IH * TX + (oy + d) * TX + ox], s);
                    ring[rs][c] = s;
                }
                const int zo = zi - R;
                if (zo >= zb && own) {
                    double inv = inv_full;
                    if (zo < R || zo + R > g.nz - 1) inv = inv_xy * border_inv(s_binv, zo, g.nz, R);
                    const int o = (zo - g.zlo) * nxy + ooff;
                    float uu[3];
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        double s = 0.0;
#pragma unroll
                        for (int d = 0; d < W; ++d) s = fma(wk(d), ring[(rs + 1 + d) % W][c], s);
                        uu[c] = (float)(s * inv);
                        UN_[c * n + o] = uu[c];
                    }
                    if (PEER) {
#pragma unroll
                        for (int sd = 0; sd < 2; ++sd)
                            if (peer_sends(b, sd, 2, zo)) {
                                const long long rn = b.peer.n[sd];
                                float* Rm = b.peer.u[sd] + (1 - cur) * 3 * rn + peer_index(b, sd, zo, nxy, ooff);
                                Rm[0] = uu[0];
                                Rm[rn] = uu[1];
                                Rm[2 * rn] = uu[2];
                                __threadfence_system();
                            }
                    }
                }
                // plane zi was last read by compose(zi + 1) before the barrier
                if (TMA && zi + 4 <= z1 + 2) tma_issue(zi + 4);
                x_pass(in_b, x_b);
                tma_wait(zi + 3);
                compose(zi + 2, in_a);
                if (!TMA) {
                    store_u(zi + 4);
                    load_u(zi + 5);
                }
                load_v(zi + 3);
                double* t = in_a; in_a = in_b; in_b = t;
                t = x_a; x_a = x_b; x_b = t;
                __syncthreads();
            }
        }
    }
}

// ---------------------------------------------------------------------------
#undef wk
#define WLM_DISPATCH_R(R_, CALL)                       \
    switch (R_) {                                      \
        case 0: { constexpr int RR = 0; CALL; } break; \
        case 1: { constexpr int RR = 1; CALL; } break; \
        case 2: { constexpr int RR = 2; CALL; } break; \
        case 3: { constexpr int RR = 3; CALL; } break; \
        case 4: { constexpr int RR = 4; CALL; } break; \
        case 5: { constexpr int RR = 5; CALL; } break; \
        case 6: { constexpr int RR = 6; CALL; } break; \
        default: break;                                \
    }

int plane_tiles(const Geo& g) { return cdiv(g.nx, TX) * cdiv(g.ny, TY); }

void launch_mse_fwd(const Batch& b, const LmParams& p, int mode, cudaStream_t s) {
    (void)p;
    const dim3 wgrid(cdiv(b.g.nx, 32) * cdiv(b.g.ny, 8), cdiv(b.g.ze - b.g.zs, kZP), b.pairs);
    k_warp_moving<false><<<wgrid, 256, 0, s>>>(b, mode, b.g.zs, b.g.ze);
    const LaunchShape sh = shape_for(b.g, b.pairs, 8, b.ctas_per_sm);
    dim3 grid = sh.grid();
    grid.z = b.pairs;
    k_mse_fwd<<<grid, 256, 0, s>>>(b, sh.chunk_len);
    g_kernel_launches += 2;
    launch_plane_sums(b, s);
}

void launch_mi_fwd(const Batch& b, const LmParams& p, int mode, cudaStream_t s) {
    const dim3 wgrid(cdiv(b.g.nx, 32) * cdiv(b.g.ny, 8), cdiv(b.g.ze - b.g.zs, kZP), b.pairs);
    k_warp_moving<false><<<wgrid, 256, 0, s>>>(b, mode, b.g.zs, b.g.ze);
    const LaunchShape sh = shape_for(b.g, b.pairs, 8, b.ctas_per_sm);
    dim3 grid = sh.grid();
    grid.z = b.pairs;
    k_mi_hist<<<grid, 256, sizeof(unsigned long long) * p.mi_bins * p.mi_bins, s>>>(b, p, sh.chunk_len);
    g_kernel_launches += 2;
}

void launch_mi_finalize(const Batch& b, const LmParams& p, int mode, cudaStream_t s) {
    k_mi_finalize<<<b.pairs, 256, 0, s>>>(b, p, mode);
    ++g_kernel_launches;
}

void launch_mi_grad(const Batch& b, const LmParams& p, cudaStream_t s) {
    const dim3 grid(cdiv(b.g.nx, 32) * cdiv(b.g.ny, 8), b.g.ze - b.g.zs, b.pairs);
    k_mi_grad<<<grid, 256, 0, s>>>(b, p);
    ++g_kernel_launches;
}

void launch_mse_grad(const Batch& b, const LmParams& p, cudaStream_t s) {
    const dim3 grid(cdiv(b.g.nx, 32) * cdiv(b.g.ny, 8), b.g.ze - b.g.zs, b.pairs);
    k_mse_grad<<<grid, 256, 0, s>>>(b, p.optimizer == WLM_OPT_DEMONS, p.demons_alpha);
    ++g_kernel_launches;
}

void launch_warp_moving_grad(const Batch& b, int mode, int zf, int zl, cudaStream_t s) {
    const dim3 wgrid(cdiv(b.g.nx, 32) * cdiv(b.g.ny, 8), cdiv(zl - zf, kZP), b.pairs);
    k_warp_moving<true><<<wgrid, 256, 0, s>>>(b, mode, zf, zl);
    ++g_kernel_launches;
}

// K1a over the owned planes plus the window pass's 2-plane halo
void launch_lncc_warp(const Batch& b, const LmParams& p, int mode, cudaStream_t s) {
    const int zf = std::max(0, b.g.zs - 2), zl = std::min(b.g.nz, b.g.ze + 2);
    const dim3 wgrid(cdiv(b.g.nx, 32) * cdiv(b.g.ny, 8), cdiv(zl - zf, kZP), b.pairs);
    if (p.lean)
        k_warp_moving<false><<<wgrid, 256, 0, s>>>(b, mode, zf, zl);  // K2 gathers grad M itself
    else
        k_warp_moving<true><<<wgrid, 256, 0, s>>>(b, mode, zf, zl);
    ++g_kernel_launches;
}

// K1b over the owned planes [b.g.zs, b.g.ze) (a slab's boundary or interior
// view: every voxel's arithmetic is independent of the range)
void launch_lncc_window(const Batch& b, cudaStream_t s) {
    const LaunchShape sh = shape_for(b.g, b.pairs, k1::TY, b.ctas_per_sm);
    dim3 grid = sh.grid();
    grid.z = b.pairs;
    if (b.peer_on)
        k_lncc_fwd<2, true><<<grid, k1::NT, 0, s>>>(b, sh.chunk_len);
    else
        k_lncc_fwd<2><<<grid, k1::NT, 0, s>>>(b, sh.chunk_len);
    ++g_kernel_launches;
}

void launch_lncc_fwd(const Batch& b, const LmParams& p, int mode, cudaStream_t s) {
    if (p.radius != 2) {
        launch_lncc_fwd_generic(b, p, mode, s);
        return;
    }
    launch_lncc_warp(b, p, mode, s);
    launch_lncc_window(b, s);
    launch_plane_sums(b, s);
}

void launch_finalize(const Batch& b, const LmParams& p, int mode, cudaStream_t s) {
    k_finalize<<<b.pairs, 256, 0, s>>>(b, p, mode);
    ++g_kernel_launches;
}

void launch_lncc_bwd(const Batch& b, const LmParams& p, cudaStream_t s) {
    if (p.radius != 2) {
        launch_lncc_bwd_generic(b, p, s);
        return;
    }
    const LaunchShape sh = shape_for(b.g, b.pairs, k2::TY, b.ctas_per_sm);
    dim3 grid = sh.grid();
    grid.z = b.pairs;
    static std::atomic<unsigned long long> attr{0ull};  // per device
    const unsigned long long bit = device_bit();
    if (!(attr.load() & bit)) {
        cudaFuncSetAttribute(k_lncc_bwd<2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k2::OWN_BYTES);
        cudaFuncSetAttribute(k_lncc_bwd<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)k2::OWN_BYTES_LEAN);
        cudaFuncSetAttribute(k_lncc_bwd<2, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)k2::OWN_BYTES);
        cudaFuncSetAttribute(k_lncc_bwd<2, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)k2::OWN_BYTES_LEAN);
        attr.fetch_or(bit);
    }
    if (p.lean && b.peer_on)
        k_lncc_bwd<2, true, true><<<grid, k2::NT, k2::OWN_BYTES_LEAN, s>>>(b, p, sh.chunk_len);
    else if (p.lean)
        k_lncc_bwd<2, true><<<grid, k2::NT, k2::OWN_BYTES_LEAN, s>>>(b, p, sh.chunk_len);
    else if (b.peer_on)
        k_lncc_bwd<2, false, true><<<grid, k2::NT, k2::OWN_BYTES, s>>>(b, p, sh.chunk_len);
    else
        k_lncc_bwd<2, false><<<grid, k2::NT, k2::OWN_BYTES, s>>>(b, p, sh.chunk_len);
    ++g_kernel_launches;
}

void launch_step_smooth(const Batch& b, const LmParams& p, cudaStream_t s) {
    if (p.Ru > 6) {
        launch_step_smooth_generic(b, p, p.taps_u, p.Ru, s);
        return;
    }
    const LaunchShape sh = shape_for(b.g, b.pairs, k3::TY, b.ctas_per_sm);
    dim3 grid = sh.grid();
    grid.z = b.pairs;
    WLM_DISPATCH_R(p.Ru, ({
        static std::atomic<unsigned long long> attr{0ull};  // per device
        const unsigned long long bit = device_bit();
        if (!(attr.load() & bit)) {
            cudaFuncSetAttribute(k_step_smooth<RR, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)k3::Shape<RR>::BYTES);
            cudaFuncSetAttribute(k_step_smooth<RR, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)k3::Shape<RR>::BYTES);
            cudaFuncSetAttribute(k_step_smooth<RR, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)k3::Shape<RR>::BYTES);
            attr.fetch_or(bit);
        }
        if (p.optimizer == WLM_OPT_LM && p.tile_k > 1) {
            k_step_smooth<RR, true><<<grid, k3::NT, k3::Shape<RR>::BYTES, s>>>(b, p, sh.chunk_len);
        } else if (b.peer_on) {  // fused halo stores (slab groups; never tiled)
            k_step_smooth<RR, false, true><<<grid, k3::NT, k3::Shape<RR>::BYTES, s>>>(b, p, sh.chunk_len);
        } else {
            k_step_smooth<RR, false><<<grid, k3::NT, k3::Shape<RR>::BYTES, s>>>(b, p, sh.chunk_len);
        }
    }));
    ++g_kernel_launches;
}

void make_tma_u(Batch& b, int Rw) {
    b.tma_u_ok = 0;
    std::memset(&b.tma_u, 0, sizeof(b.tma_u));
    const Geo& g = b.g;
    if (g.nx % 4 != 0 || Rw > 3) return;
    typedef CUresult (*Encode)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                               const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                               CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static Encode encode = nullptr;
    if (!encode) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !fn)
            return;
        encode = reinterpret_cast<Encode>(fn);
    }
    int uw = 0, uh = 0;
    WLM_DISPATCH_R(Rw, (uw = k4::Shape<RR>::UW, uh = k4::Shape<RR>::UH));
    const cuuint64_t dims[5] = {(cuuint64_t)g.nx, (cuuint64_t)g.ny, (cuuint64_t)g.nzl, 6, (cuuint64_t)b.pairs};
    const cuuint64_t strides[4] = {(cuuint64_t)g.nx * 4, (cuuint64_t)g.nx * g.ny * 4, (cuuint64_t)g.n * 4,
                                   (cuuint64_t)g.n * 6 * 4};
    const cuuint32_t box[5] = {(cuuint32_t)uw, (cuuint32_t)uh, 1, 3, 1};
    const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    const CUresult r = encode(&b.tma_u, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, b.U, dims, strides, box, estr,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    b.tma_u_ok = r == CUDA_SUCCESS ? 1 : 0;
}

void launch_compose_smooth(const Batch& b, const LmParams& p, cudaStream_t s) {
    if (p.Rw > 6) {
        launch_compose_smooth_generic(b, p, p.taps_w, p.Rw, s);
        return;
    }
    const LaunchShape sh = shape_for(b.g, b.pairs, k4::TY, b.ctas_per_sm);
    dim3 grid = sh.grid();
    grid.z = b.pairs;
    WLM_DISPATCH_R(p.Rw, ({
        static std::atomic<unsigned long long> attr{0ull};  // per device
        const unsigned long long bit = device_bit();
        if (!(attr.load() & bit)) {
            cudaFuncSetAttribute(k_compose_smooth<RR, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)k4::Shape<RR>::BYTES);
            cudaFuncSetAttribute(k_compose_smooth<RR, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)k4::Shape<RR>::BYTES);
            cudaFuncSetAttribute(k_compose_smooth<RR, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)k4::Shape<RR>::BYTES);
            cudaFuncSetAttribute(k_compose_smooth<RR, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)k4::Shape<RR>::BYTES);
            attr.fetch_or(bit);
        }
        if (b.peer_on && b.tma_u_ok)
            k_compose_smooth<RR, true, true><<<grid, k4::NT, k4::Shape<RR>::BYTES, s>>>(b, p, sh.chunk_len, b.tma_u);
        else if (b.peer_on)
            k_compose_smooth<RR, false, true><<<grid, k4::NT, k4::Shape<RR>::BYTES, s>>>(b, p, sh.chunk_len, b.tma_u);
        else if (b.tma_u_ok)
            k_compose_smooth<RR, true><<<grid, k4::NT, k4::Shape<RR>::BYTES, s>>>(b, p, sh.chunk_len, b.tma_u);
        else
            k_compose_smooth<RR, false><<<grid, k4::NT, k4::Shape<RR>::BYTES, s>>>(b, p, sh.chunk_len, b.tma_u);
    }));
    ++g_kernel_launches;
}

}  // namespace wlm
