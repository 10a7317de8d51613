// kernels.cuh -- device state and launch wrappers of the LM hot path.
#pragma once

#include <cuda.h>  // CUtensorMap (types only; the encoder is fetched at run time)
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "wlm.h"

namespace wlm {

// Per-pair device-resident optimizer state.  Mutated only by the finalize
// kernel (one CTA per pair, one writer), read by the other kernels, so an
// iteration needs no host round trip.
struct PairState {
    double lambda, L1, L2;   // LmState
    double r_cur, lncc_cur;  // residual at the accepted warp
    double r_try, lncc_try;  // residual at the latest attempt
    int hist_n;              // accepted losses held (0..2)
    int cur;                 // which warp buffer holds the accepted warp
    int last_rejected;       // latest attempt rejected -> gradient kept
    int iter;                // accepted iterations at this level
    int retries;             // rejections in the current iteration
    int done;                // reached iters_target (or aborted)
    int status;              // wlm_status of the pair
    int trace_len;
    int attempt;             // attempts at this level (scripted-loss index)
    int iters_target;
    int level;
    unsigned max_bits;       // max |dU_s| as ordered bits (K3 -> K4)
    int jac_bits;            // min det(I + grad eps dU_s), ordered int
    // per-pair intensity shifts; 8-byte aligned so the stencil kernels read
    // both with one 64-bit load (measured: K1b 1.34 -> 1.17 ms against an
    // offset that split them, through different code generation)
    alignas(8) float shift_f;
    float shift_m;
    double lo_f, hi_f, lo_m, hi_m;  // min / max of F and M (MI normalisation)
};

// Launch-invariant parameters of one engine (passed by value).
struct LmParams {
    double mu_plus, mu_minus, lambda_max, tau;
    double target, step_floor;
    double adam_b1, adam_b2, adam_eps, adam_lr, gd_lr;
    // Adam bias corrections 1 - beta^t for t = 1 .. adam_bc_n (host
    // std::pow, the oracle's own values): [0][t-1] beta1, [1][t-1] beta2
    const double* adam_bc;
    int adam_bc_n;
    // fp64 Gaussian taps w[0 .. 2R] of sigma_update / sigma_warp for the
    // generic smoothing paths (radius > 6), device pointers or null
    const double* taps_u;
    const double* taps_w;
    int rejection, max_retries, optimizer, log_jacobian;
    int trace_cap;
    int script_n;
    wlm_step_log* trace;   // [pair][trace_cap]
    const double* script;  // [pair][script_n] or null
    int Ru, Rw;            // smoothing radii (update, warp); 0 = identity
    float wu[8], ww[8];    // half-kernels w[|d|]
    float wu_full, ww_full;
    double wud[8], wud_full;  // fp64 copies of the kernels (K3/K4 sum in fp64)
    double wwd[8], wwd_full;
    int radius;            // LNCC window radius (2: fused K1b/K2; others: generic.cu)
    int metric;            // WLM_METRIC_LNCC | WLM_METRIC_MSE
    double demons_alpha;   // DemonsConfig.alpha (optimizer DEMONS)
    int tile_k;            // LmConfig.tile_size (Eq. 5); 1 = pointwise Eq. 4
    int lean;              // LNCC low-memory layout: no grad M buffer, K2 gathers (wlm_reg_config.low_memory)
    int mi_bins;           // MI: B x B Parzen grid
    double mi_sigma;       // MI: Parzen sigma in bin widths
};

// Buffers of a batch of `pairs` registrations of identical geometry.
// Fused halo stores of a slab group (slab.cu): an output plane
// that a neighbouring slab keeps as halo is stored by the producing kernel
// straight into that slab's buffer as well -- peer memory (CUDA IPC over
// NVLink) with one process per GPU, the same device in-process -- so no
// separate exchange moves it.  Buffer kinds: 0 g (K2), 1 dU_s (K3), 2 the
// attempt warp (K4), 3 A, B, E (K1b).  Side 0 is the lower neighbour, 1 the
// upper; slab engines hold one pair.
struct HaloPeer {
    float* g[2];
    float* v[2];
    float* u[2];      // the neighbour's U (both ping-pong buffers)
    float* abe[2];
    long long n[2];   // the neighbour's channel stride (voxels incl. its halo)
    int zlo[2];       // the neighbour's first buffer plane
    int lo_end[4];    // planes [g.zs, lo_end[k]) of kind k go to the lower neighbour
    int hi_begin[4];  // planes [hi_begin[k], g.ze) go to the upper one
};

struct Batch {
    Geo g;
    int pairs;        // pairs in this launch: pair0 .. pair0 + pairs - 1
    int pair0;        // first pair (a pair group of the engine's batch; 0 otherwise)
    const float* F;   // [pair][n]
    const float* M;   // [pair][n]
    float* U;         // [pair][2][3][n] ping-pong warps
    float* ABE;       // [pair][4][n]  LNCC window coefficients: A, B (fp32), E (fp64)
    double* MW;       // [pair][n]     warped moving image M(x + u) (fp64, K1a -> K1b, K2)
    double* GM;       // [pair][3][n]  grad M(x + u) of the evaluated warp (LNCC: K1a -> K2), or null
    float* G;         // [pair][3][n]  gradient g, Adam step in place
    float* VS;        // [pair][3][n]  smoothed step dU_s, pair stride vs_ps: it lives in the
                      // ABE buffer (A, B, E are dead from K2 to the next K1b, while dU_s lives)
    long long vs_ps;  // VS pair stride in floats (4 n)
    float* AM;        // [pair][3][n]  Adam first moment (or null)
    float* AV;        // [pair][3][n]  Adam second moment (or null)
    PairState* st;    // [pair]
    double* shift_part; // [pair][2][256] scratch for the intensity shifts
    double* partials; // [pair][nz][tiles][8] per-(plane, tile, warp) sum(rho)
    double* plane_sum;  // [pair][nz] per-plane sum(rho) (global z; shared by slabs)
    int zero_foreign_planes;  // NCCL slabs: zero non-owned planes before the all-reduce
    double* TM;       // [pair][tiles][6] tiled LM: -r (H + lambda I)^{-1} (symmetric), or null
    unsigned long long* HIST;  // [pair][B*B] MI joint histogram, fixed point 2^-32 (exact sums)
    double* MIT;      // [pair][B*B] MI gradient table dMI/dp_ij - dMI/dp_m(j)
    double* X64;      // [pair][10][n] fp64 scratch of the generic paths (generic.cu), or null
    int tkx, tky, tkz;  // tile counts (tile_k > 1)
    int tma_u_ok;       // K4 stages the accepted warp by TMA (tma_u valid)
    CUtensorMap tma_u;  // 5D map over U: (x, y, local z, buffer*3 + component, pair)
    int max_blocks;
    int ctas_per_sm;    // z-chunking target of this launch (0 -> 4; pair groups use 1)
    int peer_on;        // fused halo stores (peer valid)
    HaloPeer peer;
};

struct LaunchShape {
    int tiles_x, tiles_y, chunks, chunk_len;
    dim3 grid() const;
};
// z-chunking of a stencil launch: enough chunks that the launch has about
// ctas_per_sm x SMs CTAs (0 -> 4), each chunk >= 8 planes.
LaunchShape shape_for(const Geo& g, int pairs, int ty, int ctas_per_sm = 0);

// MSE: K1a warp + per-plane sum (f - Mw)^2; gradient
// g = -2 (f - Mw)/N grad M(x+u) (pointwise, analytic interpolant gradient).
void launch_mse_fwd(const Batch& b, const LmParams& p, int mode, cudaStream_t s);
// MI: K1a + fixed-point Parzen joint histogram; finalize
// (MI, gradient table, state machine); pointwise gradient.
void launch_mi_fwd(const Batch& b, const LmParams& p, int mode, cudaStream_t s);
void launch_mi_finalize(const Batch& b, const LmParams& p, int mode, cudaStream_t s);
void launch_mi_grad(const Batch& b, const LmParams& p, cudaStream_t s);
void launch_mse_grad(const Batch& b, const LmParams& p, cudaStream_t s);
// K4's TMA descriptor for the engine's U buffer (box = one warp-ring slot);
// leaves tma_u_ok = 0 when the layout does not allow it (nx % 4 != 0).
void make_tma_u(Batch& b, int R_warp);
// K1: warp + LNCC window moments + coefficients + per-plane sum(rho) (K1a,
// K1b, k_plane_sums); K5 then runs the loss/damping/rejection state machine.
// mode 0 evaluates the accepted warp (level start), mode 1 the attempt in
// the other buffer.
void launch_lncc_fwd(const Batch& b, const LmParams& p, int mode, cudaStream_t s);
// K5: r = 1 - mean(rho) from the per-plane sums (z order), then the state
// machine.  Runs after the plane sums of every slab are in place.
void launch_finalize(const Batch& b, const LmParams& p, int mode, cudaStream_t s);
// 32 x 8 tiles per plane (size of the per-plane partial arrays).
int plane_tiles(const Geo& g);
// K2: adjoint window sums -> dr/dMw -> g = dr/dMw * gradM(x + u).
void launch_lncc_bwd(const Batch& b, const LmParams& p, cudaStream_t s);
// Adam moment update (pointwise), writes the Adam step into G.
void launch_adam(const Batch& b, const LmParams& p, cudaStream_t s);
// K3: LM step (or GD / pass-through) + Gaussian(sigma_update) + max|.|.
void launch_step_smooth(const Batch& b, const LmParams& p, cudaStream_t s);
// K4: compositive resample with eps from the max + Gaussian(sigma_warp).
void launch_compose_smooth(const Batch& b, const LmParams& p, cudaStream_t s);
// Optional diagnostic: min det(I + grad(eps dU_s)) over the interior.
void launch_jacobian_diag(const Batch& b, const LmParams& p, cudaStream_t s);
// WHILE-loop condition: any pair not done.
void launch_loop_cond(const Batch& b, cudaGraphConditionalHandle h, cudaStream_t s);
// Per-pair state reset at level start.
void launch_begin_level(const Batch& b, const LmParams& p, int level, int reset_lambda,
                        double lambda0, cudaStream_t s);
void launch_set_targets(const Batch& b, int iters, cudaStream_t s);
// Intensity shifts (means of F and M per pair), deterministic.
void launch_shifts(const Batch& b, cudaStream_t s);
// Device constants (window-count reciprocals); idempotent.
void init_constants();

// ---- generator helpers (synth_pair; fp32 SoA device buffers) ----

void launch_smooth_generic(const float* in, float* out, float* tmp, int nchan, const Geo& g,
                           double sigma, cudaStream_t s);

void launch_max_abs(const float* v, long long count, unsigned* out_bits, cudaStream_t s);
void launch_jacdet(const float* u, const Geo& g, int* out_ordered, cudaStream_t s);
// Tiled LM (Eq. 5): per-tile -r (H + lambda I)^{-1}, H = sum g g^T.
void launch_tile_matrix(const Batch& b, const LmParams& p, cudaStream_t s);
// Mirror op: the same in fp64 on AoS buffers, operation order of the oracle.
void launch_lm_tiled_fp64(double r, const double* g, const Geo& geo, double lambda, int k, double* tm,
                          double* out, cudaStream_t s);
// Eq. 9 in fp64 with the oracle's operation order (no contraction): bitwise
// equal to orc_demons_step_mse.  r: [N], n, out: AoS [N][3].
__device__ __forceinline__ void demons_step(double rx, double a, double b, double c, double alpha, double* o) {
    const double den = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(a, a), __dmul_rn(b, b)), __dmul_rn(c, c)),
                                 __dmul_rn(__dmul_rn(__dmul_rn(alpha, alpha), rx), rx));
    const double s = den > 0.0 ? __ddiv_rn(rx, den) : 0.0;
    o[0] = __dmul_rn(s, a); o[1] = __dmul_rn(s, b); o[2] = __dmul_rn(s, c);
}
void launch_demons_pointwise(const double* r, const double* n, long long N, double alpha, double* out,
                             cudaStream_t s);

void launch_nonfinite(const float* v, long long count, int* flag, cudaStream_t s);
// K1a alone over planes [zf, zl) (the generic LNCC path's warp + gradient).
void launch_warp_moving_grad(const Batch& b, int mode, int zf, int zl, cudaStream_t s);
void launch_plane_sums(const Batch& b, cudaStream_t s);
// K1's pieces (the fused radius-2 path): K1a, K1b (range = b.g.zs .. b.g.ze)
void launch_lncc_warp(const Batch& b, const LmParams& p, int mode, cudaStream_t s);
void launch_lncc_window(const Batch& b, cudaStream_t s);
// generic.cu: LNCC radius != 2, smoothing radius > 6
size_t generic_scratch_doubles(const Geo& g);
void launch_lncc_fwd_generic(const Batch& b, const LmParams& p, int mode, cudaStream_t s);
void launch_lncc_bwd_generic(const Batch& b, const LmParams& p, cudaStream_t s);
void launch_step_smooth_generic(const Batch& b, const LmParams& p, const double* w, int R, cudaStream_t s);
void launch_compose_smooth_generic(const Batch& b, const LmParams& p, const double* w, int R, cudaStream_t s);
// Gaussian(sigma = 0.5 f) + stride f in one fp64 pass (pyramid levels).
void launch_downsample_gauss(const float* in, const Geo& g, int f, float* out, const Geo& gd,
                             cudaStream_t s);
void launch_upsample(const float* u, const Geo& g, const Geo& gd, float scale, float* out,
                     cudaStream_t s);

// AoS fp64 <-> SoA fp32 conversions.
void launch_aos_to_soa(const double* in, float* out, long long n, int nchan, cudaStream_t s);
void launch_soa_to_aos(const float* in, double* out, long long n, int nchan, cudaStream_t s);

extern uint64_t g_kernel_launches;  // per-process count (ctx keeps its own)

}  // namespace wlm
