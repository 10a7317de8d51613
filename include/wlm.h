/*
 * wlm.h -- C-ABI of the B200-native factored-LM registration hot path.
 *
 * This is the drop-in boundary.  It replaces, for the per-iteration path of
 * the reference `warplm` library (/root/reference, C++20, namespace warplm):
 *
 *   reference interface (file:line)                      replaced by
 *   --------------------------------------------------   ------------------------------
 *   field.hpp:82   sample_trilinear                      wlm_sample_trilinear_grad_points,
 *                                                        wlm_warp_volume (whole volume)
 *   field.hpp:90   sample_trilinear_grad                 wlm_sample_trilinear_grad_points,
 *                                                        wlm_warp_volume (+ gradient)
 *   field.hpp:93   sample_field                          wlm_sample_field_points
 *   field.hpp:96   compose_warp                          wlm_compose_warp
 *   field.hpp:99   max_abs_component                     wlm_max_abs_component
 *   field.hpp:104  normalize_step                        wlm_normalize_step
 *   field.hpp:108  jacobian_det_min                      wlm_jacobian_det_min
 *   field.hpp:113  gaussian_smooth(Volume3)              wlm_gaussian_smooth_vol
 *   field.hpp:114  gaussian_smooth(DispField3)           wlm_gaussian_smooth_field
 *   field.hpp:116-117 all_finite                         wlm_all_finite
 *   SPEC.md:127    residual_mse -> ResidualReport        wlm_residual_mse
 *   SPEC.md:145    residual_mi -> ResidualReport         wlm_residual_mi
 *   SPEC.md:136    residual_lncc -> ResidualReport       wlm_residual_lncc
 *   SPEC.md:247    lm_step_pointwise                     wlm_lm_step_pointwise
 *   SPEC.md:256    lm_step_tiled                         wlm_lm_step_tiled
 *   SPEC.md:301    demons_step_mse                       wlm_demons_step_mse
 *   SPEC.md:265    update_damping                        wlm_update_damping
 *   SPEC.md:274    rejection_test                        wlm_rejection_test
 *   SPEC.md:283    lm_iterate                            wlm_engine_* (device-resident)
 *   SPEC.md:292    adam_step                             wlm_engine_* (optimizer = ADAM)
 *   SPEC.md:188    downsample                            wlm_downsample
 *   SPEC.md:197    upsample_warp                         wlm_upsample_warp
 *   SPEC.md:362    register -> RegResult                 wlm_register
 *   SPEC.md:310    state_bytes                           wlm_state_bytes
 *   io.hpp:18-21   read/write_vol3, read/write_dsp3      wlm_read_vol3 ... wlm_write_dsp3
 *   SPEC.md:427    CSV trace                             wlm_write_trace_csv
 *
 * Host-buffer entry points take the reference's own layout: fp64, x-fastest
 * (field.hpp:25-30), displacement fields component-innermost AoS
 * (field.hpp:50-58).  They upload, run on the GPU and download, like a
 * by-value reference call; the field-module mirrors keep the data fp64 and
 * evaluate the reference's expressions in its operation order, so they
 * return the reference function's bits.  Device entry points (wlm_dev_*) take fp32
 * structure-of-arrays device pointers (one plane per component) and run on
 * the context's stream with no host synchronisation.
 *
 * Errors never cross the ABI as exceptions: every call returns wlm_status
 * and wlm_last_error(ctx) describes the last failure.  The reference's
 * std::invalid_argument maps to WLM_INVALID_ARG / WLM_DIM_MISMATCH, its
 * non-finite abort to WLM_NONFINITE.  There is no CPU
 * fallback: a missing device is WLM_CUDA.
 *
 * Threading: a context owns one CUDA stream and its
 * scratch; do not share a context between host threads without locking.
 * Distinct contexts run concurrently.
 */
#ifndef WLM_H
#define WLM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    WLM_OK = 0,
    WLM_INVALID_ARG = 1,
    WLM_DIM_MISMATCH = 2,
    WLM_NONFINITE = 3,
    WLM_OOM = 4,
    WLM_CUDA = 5,
    WLM_UNSUPPORTED = 6
} wlm_status;

typedef struct { int nx, ny, nz; } wlm_dims;

/* LmConfig. lambda_max <= 0 or inf: uncapped. */
typedef struct {
    double lambda0, mu_plus, mu_minus;
    int tile_size;   /* k of Eq. 5 (1 = pointwise Eq. 4) */
    int rejection;
    double tau, lambda_max;
    int max_retries;
} wlm_lm_config;

/* LmState. */
typedef struct {
    double lambda;
    int hist_n;
    double L1, L2;
} wlm_lm_state;

typedef struct { double beta1, beta2, eps_hat, lr; } wlm_adam_config;

/* DEMONS: Eq. 9 active forces from the MSE per-voxel residual;
 * requires metric = MSE. */
enum { WLM_OPT_LM = 0, WLM_OPT_ADAM = 1, WLM_OPT_GD = 2, WLM_OPT_DEMONS = 3 };
/* MetricConfig.kind. */
enum { WLM_METRIC_LNCC = 0, WLM_METRIC_MSE = 1, WLM_METRIC_MI = 2 };
#define WLM_MAX_LEVELS 8

/* RegConfig + MetricConfig + StepScale. */
typedef struct {
    int lncc_radius;
    int optimizer;
    wlm_lm_config lm;
    wlm_adam_config adam;
    double gd_lr;
    int nlevels;
    int factors[WLM_MAX_LEVELS];
    int iters[WLM_MAX_LEVELS];
    double target_max_disp, step_floor;
    double sigma_update, sigma_warp;
    int log_jacobian;
    int metric; /* WLM_METRIC_* (SPEC.md:121), default LNCC */
    double demons_alpha; /* DemonsConfig.alpha, default 1 */
    int mi_bins;         /* MetricConfig.mi_bins B, 2..64 (default 32) */
    double mi_sigma;     /* MetricConfig.mi_parzen_sigma in bin widths, (0, 2] (default 1) */
    /* Device layout (not a reference parameter): 0 = speed (K1a hands the
     * fp64 grad M(x+u) to K2, 92 B/voxel for LNCC); 1 = memory (K2
     * re-gathers M at x+u itself, 68 B/voxel).  Results are identical. */
    int low_memory;
} wlm_reg_config;

/* RegResult.loss_trace row (CSV columns SPEC.md:427). */
typedef struct {
    int level, iter;
    double loss_raw, r, lambda, eps;
    int accepted, retries;
    double jac_det_min;
} wlm_step_log;

typedef struct wlm_ctx wlm_ctx;
typedef struct wlm_engine wlm_engine;

/* ---- context ---- */
wlm_status wlm_ctx_create(int device, wlm_ctx** out);
void wlm_ctx_destroy(wlm_ctx* ctx);
const char* wlm_last_error(const wlm_ctx* ctx);
/* The context's stream (cudaStream_t as void*); device calls run on it. */
void* wlm_ctx_stream(wlm_ctx* ctx);
/* Use an external stream (e.g. torch's current stream) instead. */
wlm_status wlm_ctx_set_stream(wlm_ctx* ctx, void* stream);
wlm_status wlm_ctx_synchronize(wlm_ctx* ctx);
/* Number of this library's kernels launched on ctx since creation. */
uint64_t wlm_ctx_launch_count(const wlm_ctx* ctx);
void wlm_default_reg_config(wlm_reg_config* cfg);
/* Library build id string (arch, version). */
const char* wlm_version(void);
/* First 16 hex digits of sha256 over the library's sources (Makefile
 * SRC_HASH); the Python layer refuses a library built from other sources. */
const char* wlm_source_hash(void);

/* ---- host-buffer mirror of the reference field module (fp64, AoS) ---- */
wlm_status wlm_warp_volume(wlm_ctx* ctx, const double* M, const double* u, wlm_dims d,
                           double* Mw, double* gradM /* nullable */);
/* sample_trilinear(_grad) at npts points p = pts[3i..3i+2] (x, y, z): value
 * and analytic gradient (field.cpp:43-90, NaN value for a non-finite p). */
wlm_status wlm_sample_trilinear_grad_points(wlm_ctx* ctx, const double* vol, wlm_dims d,
                                            const double* pts /* 3*npts */, size_t npts,
                                            double* val /* npts */, double* grad /* 3*npts, nullable */);
wlm_status wlm_sample_field_points(wlm_ctx* ctx, const double* u, wlm_dims d,
                                   const double* pts /* 3*npts */, size_t npts,
                                   double* out /* 3*npts */);
wlm_status wlm_compose_warp(wlm_ctx* ctx, const double* u, wlm_dims du, const double* v,
                            wlm_dims dv, double eps, double* out);
wlm_status wlm_max_abs_component(wlm_ctx* ctx, const double* v, wlm_dims d, double* out);
wlm_status wlm_normalize_step(wlm_ctx* ctx, const double* v, wlm_dims d, double target,
                              double floor_, double* eps);
wlm_status wlm_jacobian_det_min(wlm_ctx* ctx, const double* u, wlm_dims d, double* out);
wlm_status wlm_gaussian_smooth_vol(wlm_ctx* ctx, const double* in, wlm_dims d, double sigma,
                                   double* out);
wlm_status wlm_gaussian_smooth_field(wlm_ctx* ctx, const double* in, wlm_dims d,
                                     double sigma, double* out);
wlm_status wlm_all_finite(wlm_ctx* ctx, const double* data, size_t count, int* out);

/* ---- host-buffer mirror of similarity / lmopt / pyramid (SPEC) ---- */
wlm_status wlm_residual_lncc(wlm_ctx* ctx, const double* F, const double* M,
                             const double* u, wlm_dims d, int radius, double* r,
                             double* lncc, double* g /* nullable, AoS */);
/* residual_mi: Parzen-window MI in bits on a B x B grid
 * (A13-A15); r = log2 B - MI; g nullable, AoS. */
wlm_status wlm_residual_mi(wlm_ctx* ctx, const double* F, const double* M, const double* u,
                           wlm_dims d, int bins, double sigma, double* r, double* mi, double* g);
/* residual_mse: r = mean (f - m(x+u))^2, g = grad_u r with
 * the analytic interpolant gradient; g nullable, AoS. */
wlm_status wlm_residual_mse(wlm_ctx* ctx, const double* F, const double* M, const double* u,
                            wlm_dims d, double* r, double* g);
wlm_status wlm_lm_step_pointwise(wlm_ctx* ctx, double r, const double* g, wlm_dims d,
                                 double lambda, double* out);
/* lm_step_tiled (Eq. 5): non-overlapping k^3 tiles (partial
 * at the far faces), H = sum g g^T per tile, Delta u = -r (H + lambda I)^{-1} g
 * with the explicit 3x3 inverse; fp64, bitwise the oracle's. */
wlm_status wlm_lm_step_tiled(wlm_ctx* ctx, double r, const double* g, wlm_dims d, double lambda,
                             int k, double* out);
/* demons_step_mse (Eq. 9): out = r_x n_x / (|n_x|^2 + alpha^2
 * r_x^2), 0 where the denominator is 0.  r: per-voxel residual f - m(x+u)
 * (N), n: moving-image gradient at x + u (AoS). */
wlm_status wlm_demons_step_mse(wlm_ctx* ctx, const double* r, const double* n, wlm_dims d,
                               double alpha, double* out);
void wlm_update_damping(wlm_lm_state* s, double loss_new, const wlm_lm_config* c);
int wlm_rejection_test(double loss_new, double loss_prev, double loss_prev2, double tau);
wlm_status wlm_downsample(wlm_ctx* ctx, const double* vol, wlm_dims d, int factor,
                          double* out, wlm_dims* out_dims);
wlm_status wlm_upsample_warp(wlm_ctx* ctx, const double* u, wlm_dims d, wlm_dims nd,
                             double scale, double* out);
/* state_bytes: persistent optimizer state, elem_bytes 4. */
size_t wlm_state_bytes(int optimizer, wlm_dims d, int elem_bytes);

/* ---- register: whole pyramid on the device ---- */
/* F, M host fp32 (the VOL3 payload type), warp_out host fp64 AoS. */
wlm_status wlm_register(wlm_ctx* ctx, const float* F, const float* M, wlm_dims d,
                        const wlm_reg_config* cfg, double* warp_out,
                        wlm_step_log* trace, size_t cap, size_t* len, double* jac_final);
/* Peak device bytes held by the last wlm_register / engine on ctx. */
size_t wlm_ctx_peak_bytes(const wlm_ctx* ctx);

/* ---- device-resident batched LM engine (the hot loop) ----
 * A batch of `pairs` independent registrations of identical dims; each pair
 * has its own lambda, loss history, accept/reject state and trace.
 * Device volumes are fp32 planes [pair][nz][ny][nx]; warps fp32
 * [pair][3][nz][ny][nx].                                                    */
wlm_status wlm_engine_create(wlm_ctx* ctx, wlm_dims d, int pairs, const wlm_reg_config* cfg,
                             wlm_engine** out);
void wlm_engine_destroy(wlm_engine* e);
/* Copy volumes in (device or host pointers; is_host selects). */
wlm_status wlm_engine_load(wlm_engine* e, const float* F, const float* M, int is_host);
/* Set the current warps (fp32 SoA, device or host); NULL -> zero warps. */
wlm_status wlm_engine_set_warp(wlm_engine* e, const float* u, int is_host);
wlm_status wlm_engine_get_warp(wlm_engine* e, float* u, int is_host);
/* New registrations on the loaded pairs: lambda back to lambda0, loss
 * history and counters cleared (begin_level keeps lambda, which is the
 * SPEC.md:389 carry between pyramid levels of one registration). */
wlm_status wlm_engine_reset(wlm_engine* e);
/* Start a level: reset loss history, evaluate r(u) (lambda kept). */
wlm_status wlm_engine_begin_level(wlm_engine* e, int level);
/* Launch `iters` lm_iterate steps for every active pair (asynchronous; with
 * rejection enabled the retries run inside a device-side WHILE graph). */
wlm_status wlm_engine_iterate(wlm_engine* e, int iters);
/* Launch exactly one attempt (K2..K4 + evaluation) per pair (rejection must
 * be disabled). */
wlm_status wlm_engine_step(wlm_engine* e);
/* Pair groups (1..4, default 2): with pairs > 1, iterate
 * runs the batch as that many independent streams of attempt graphs (with
 * rejection on: of device-side WHILE graphs, one per group)
 * (contiguous pair ranges) that join only when the call's iterations are
 * done, so the groups' kernels overlap.  Results are identical for any
 * grouping (each pair's arithmetic does not depend on it).  The environment
 * variable WLM_PAIR_GROUPS sets the default. */
wlm_status wlm_engine_set_pair_groups(wlm_engine* e, int groups);
/* Copy out per-pair state / trace rows written since begin_level (syncs). */
wlm_status wlm_engine_state(wlm_engine* e, int pair, wlm_lm_state* st, double* r,
                            double* lncc, int* iters_done);
wlm_status wlm_engine_trace(wlm_engine* e, int pair, wlm_step_log* rows, size_t cap,
                            size_t* len);
/* Device pointers of the engine's buffers (for tests / zero-copy callers). */
wlm_status wlm_engine_buffers(wlm_engine* e, const float** F, const float** M,
                              float** u_cur, float** g, float** vs, float** abe);
/* Host copy of one pair's buffer: which = 0 F, 1 M, 2 accepted warp,
 * 3 gradient g, 4 smoothed step dU_s, 5 LNCC coefficients (A, B, E planes);
 * count floats (syncs). */
wlm_status wlm_engine_read_buffer(wlm_engine* e, int which, int pair, float* host, size_t count);
/* Scripted-residual harness: when n > 0, the evaluation
 * kernels take attempt losses from `losses` (per pair: losses[pair*n + k])
 * instead of the LNCC sum; n == 0 restores the real residual. */
wlm_status wlm_engine_script_losses(wlm_engine* e, const double* losses, int n);

/* Launch one stage of the attempt on every active pair (profiling hook):
 * 0 = K1 evaluation of the attempt (warp + LNCC + state machine),
 * 1 = K2 LNCC gradient, 2 = K3 LM step + smoothing + max,
 * 3 = K4 compose + smoothing, 4 = K1 evaluation of the accepted warp. */
wlm_status wlm_engine_stage(wlm_engine* e, int stage);

/* ---- z-slab group: one registration split along z ----
 * nslabs slabs of >= 4 planes each; each slab computes its owned planes and
 * exchanges halo planes after every producer stage; sum(rho) is reduced per
 * plane in z order, so losses, decisions and warps are bit-identical for
 * every nslabs (and to wlm_engine with pairs = 1).  Warps are whole-volume
 * fp32 SoA [3][nz][ny][nx].  wlm_slab_group_create runs every slab on the
 * context's device; wlm_slab_group_create_nccl holds slab `rank` of
 * `nranks` in this process (one process per GPU) and exchanges halos with
 * NCCL send/recv and reduces with NCCL all-reduce (replaces the proposed
 * wlm_ctx_attach_comm).  Both execute the same halo plan.
 * Every loss (LNCC, MSE, MI) and step (pointwise or tiled LM, Adam, GD,
 * Demons) runs sharded.                                                      */
typedef struct wlm_slab_group wlm_slab_group;
/* One halo transfer of slab `slab`: buffer 0 = g, 1 = dU_s, 2 = warp,
 * 3 = LNCC coefficients A/B/E, 4 = tiled-LM step matrices (whole k^3
 * tile-planes); planes [z0, z1) received from (send == 0) or sent to
 * (send == 1) slab `peer`.  With lm.tile_size = k > 1 the slab boundaries
 * are rounded down to multiples of k. */
typedef struct {
    int buffer, peer, send, z0, z1;
} wlm_halo_xfer;
/* Owned planes [zs, ze) of slab `slab` (host only; INVALID_ARG if a slab
 * would be thinner than the 4-plane halo). */
wlm_status wlm_slab_partition(int nz, int nslabs, int slab, int* zs, int* ze);
/* The exchange plan of one slab (host only; rows may be NULL to query len). */
wlm_status wlm_slab_halo_plan(wlm_dims d, int nslabs, int slab, const wlm_reg_config* cfg,
                              wlm_halo_xfer* rows, size_t cap, size_t* len);
wlm_status wlm_slab_group_create(wlm_ctx* ctx, wlm_dims d, int nslabs,
                                 const wlm_reg_config* cfg, wlm_slab_group** out);
/* NCCL unique id (rank 0 creates, the caller broadcasts the 128 bytes).
 * nccl_lib: path of libnccl.so.2 to dlopen (NULL -> the loaded one). */
wlm_status wlm_nccl_unique_id(const char* nccl_lib, unsigned char id[128]);
wlm_status wlm_slab_group_create_nccl(wlm_ctx* ctx, wlm_dims d, int rank, int nranks,
                                      const unsigned char id[128], const char* nccl_lib,
                                      const wlm_reg_config* cfg, wlm_slab_group** out);
/* Planes [zs, ze) owned by this group's slabs (get_warp fills only these). */
wlm_status wlm_slab_group_owned(const wlm_slab_group* g, int* zs, int* ze);
/* Which halo exchanges the producing kernels fuse (bit k: buffer kind k of
 * wlm_halo_xfer -- 0 g, 1 dU_s, 2 warp, 3 A/B/E): the kernel stores the
 * neighbour's halo planes into its buffer itself (peer memory through CUDA
 * IPC across processes) and the exchange only orders.  0 with one slab or
 * WLM_SLAB_FUSED=0 (every exchange copies). */
wlm_status wlm_slab_group_fused_halos(const wlm_slab_group* g, int* mask);
void wlm_slab_group_destroy(wlm_slab_group* g);
wlm_status wlm_slab_group_load(wlm_slab_group* g, const float* F, const float* M, int is_host);
wlm_status wlm_slab_group_set_warp(wlm_slab_group* g, const float* u, int is_host);
wlm_status wlm_slab_group_get_warp(wlm_slab_group* g, float* u, int is_host);
/* New registration (lambda back to lambda0, as wlm_engine_reset). */
wlm_status wlm_slab_group_reset(wlm_slab_group* g);
wlm_status wlm_slab_group_begin_level(wlm_slab_group* g, int level);
wlm_status wlm_slab_group_iterate(wlm_slab_group* g, int iters);
/* Trace of the registration; fails if the slabs' state machines disagree. */
wlm_status wlm_slab_group_trace(wlm_slab_group* g, wlm_step_log* rows, size_t cap, size_t* len);
wlm_status wlm_slab_group_state(wlm_slab_group* g, wlm_lm_state* st, double* r, double* lncc,
                                int* iters_done);

/* ---- data formats either side of the path (io.hpp:15-21) ----
 * VOL3 / DSP3 exactly as the reference reads and writes them (same checks,
 * same messages, WLM_INVALID_ARG for every io_error).  dst / src are host
 * (on_device = 0; no CUDA call, ctx may be NULL) or device pointers; device
 * reads stream through double-buffered pinned staging; DSP3 is AoS on disk,
 * SoA fp32 [3][nz][ny][nx] in memory (transposed on the device). */
wlm_status wlm_io_dims(const char* path, int is_field, wlm_dims* d);
wlm_status wlm_read_vol3(wlm_ctx* ctx, const char* path, float* dst, size_t cap, int on_device, wlm_dims* d);
wlm_status wlm_read_dsp3(wlm_ctx* ctx, const char* path, float* dst_soa, size_t cap, int on_device,
                         wlm_dims* d);
wlm_status wlm_write_vol3(wlm_ctx* ctx, const char* path, const float* src, int on_device, wlm_dims d);
wlm_status wlm_write_dsp3(wlm_ctx* ctx, const char* path, const float* src_soa, int on_device, wlm_dims d);
/* RegResult.loss_trace as CSV: "# warplm-csv v1" + the SPEC.md:427 columns. */
wlm_status wlm_write_trace_csv(const char* path, const wlm_step_log* rows, size_t n);

/* ---- harness: synthetic pair on the GPU ----
 * u_true is SoA fp32 [3][nz][ny][nx] (nullable); on_device selects whether
 * F, M, u_true are device (1) or host (0) pointers. */
typedef struct {
    wlm_dims dims;
    int num_blobs;
    double warp_sigma; /* <= 0 -> min(dims)/16 */
    double warp_max;
    double noise_sigma;
    uint64_t seed;
} wlm_synth_spec;
wlm_status wlm_synth_pair(wlm_ctx* ctx, const wlm_synth_spec* spec, float* F, float* M,
                          float* u_true, int on_device);

#ifdef __cplusplus
}
#endif
#endif
