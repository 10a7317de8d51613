/*
 * oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * fp64 CPU restatement of the reference's factored-LM registration path, used
 * as the parity checker for the sm_100a product in paper_2603_19371_b200/.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  The product never links it.
 *
 * Sources restated (all paths relative to the reference root):
 *   field   : proj/src/field.cpp (code exists; restated and cross-checked
 *             bit-for-bit against the compiled reference, oracle/_ref)
 *   similarity / lmopt / pyramid / driver / synth : SPEC.md only (the
 *             reference ships no code for them -- SURVEY.md F1).  Every
 *             ambiguity is pinned in DESIGN.md "Oracle contract".
 *
 * Layout conventions follow the reference: Dims3::index is x-fastest
 * (field.hpp:25-30); displacement fields are component-innermost AoS
 * (field.hpp:50-58).  All arithmetic is fp64.
 */
#ifndef WLM_ORACLE_H
#define WLM_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct { int nx, ny, nz; } orc_dims;

/* LmConfig, SPEC.md:229-232 (defaults in orc_default_reg_config). */
typedef struct {
    double lambda0, mu_plus, mu_minus;
    int tile_size;          /* only 1 is supported (k>1 is SURVEY §8(f) next #2) */
    int rejection;          /* rejection_enabled */
    double tau, lambda_max; /* lambda_max <= 0 or +inf means uncapped */
    int max_retries;
} orc_lm_config;

/* LmState. hist_n = number of accepted losses held (0..2). */
typedef struct {
    double lambda;
    int hist_n;
    double L1, L2; /* L^{t-1}, L^{t-2} */
} orc_lm_state;

/* AdamConfig. */
typedef struct { double beta1, beta2, eps_hat, lr; } orc_adam_config;

enum { ORC_OPT_LM = 0, ORC_OPT_ADAM = 1, ORC_OPT_GD = 2, ORC_OPT_DEMONS = 3 };
enum { ORC_METRIC_LNCC = 0, ORC_METRIC_MSE = 1, ORC_METRIC_MI = 2 };

#define ORC_MAX_LEVELS 8
/* RegConfig, SPEC.md:352-355 plus MetricConfig and
 * StepScale (field.hpp:75-78). */
typedef struct {
    int lncc_radius;
    int optimizer;
    orc_lm_config lm;
    orc_adam_config adam;
    double gd_lr;
    int nlevels;
    int factors[ORC_MAX_LEVELS];
    int iters[ORC_MAX_LEVELS];
    double target_max_disp, step_floor;
    double sigma_update, sigma_warp;
    int log_jacobian; /* compute jacobian_det_min(eps*dU_s) per accepted step */
    int metric;       /* ORC_METRIC_* (MetricConfig.kind) */
    double demons_alpha; /* DemonsConfig.alpha */
    int mi_bins;         /* MetricConfig.mi_bins B */
    double mi_sigma;     /* MetricConfig.mi_parzen_sigma, bin widths */
} orc_reg_config;

/* One RegResult.loss_trace row + CSV extras. */
typedef struct {
    int level, iter;
    double loss_raw, r, lambda, eps;
    int accepted, retries;
    double jac_det_min;
} orc_step_log;

/* Status codes (shared meaning with wlm_status in include/wlm.h). */
enum {
    ORC_OK = 0, ORC_INVALID_ARG = 1, ORC_DIM_MISMATCH = 2, ORC_NONFINITE = 3,
    ORC_OOM = 4, ORC_UNSUPPORTED = 6
};

void orc_set_threads(int n);
/* 1: round every quantity the device stores in fp32 at the same point
 * (A, B, g, dU_s, warps, Adam moments); 0 (default): pure fp64 reference. */
/* 0: fp64; 1: round at the device's fp32 storage points; 2: 1 + the
 * device's fp32 arithmetic in the K3 step and both Gaussian smoothings. */
void orc_set_fp32_storage(int on);
/* Mode 2 detail: bit0 K3 step + smoothing in fp32, bit1 K4 smoothing in
 * fp32, bit2 compose in fp32 (default 3). */
void orc_set_dev_flags(int flags);
/* The mode-2 fp32 Gaussian of a 3-channel AoS field, in place. */
void orc_dev_smooth32(double* data, orc_dims d, double sigma, int norm64);
void orc_default_reg_config(orc_reg_config* c);

/* ---- field (reference field.cpp restated) ---- */
double orc_sample_trilinear_grad(const double* vol, orc_dims d, double px, double py,
                                 double pz, double* grad3 /* nullable */);
void orc_sample_field(const double* u, orc_dims d, double px, double py, double pz,
                      double* out3);
/* Mw(x) = M(x+u(x)), gradM(x) = grad of the interpolant there (AoS). */
void orc_warp_volume(const double* M, const double* u, orc_dims d, double* Mw,
                     double* gradM /* nullable */);
void orc_compose_warp(const double* u, const double* v, orc_dims d, double eps,
                      double* out);
double orc_max_abs_component(const double* v, size_t count);
/* returns eps, or NaN when target is outside (0, 0.5) (field.cpp:151-153) */
double orc_normalize_step(const double* v, size_t count, double target, double floor_);
/* returns NaN when a dim < 2 (field.cpp:174-176) */
double orc_jacobian_det_min(const double* u, orc_dims d);
void orc_gaussian_smooth(double* data, orc_dims d, int nchan, double sigma);
int orc_all_finite(const double* data, size_t count);

/* ---- similarity: LNCC ---- */
/* Returns r = 1 - LNCC (NaN on invalid dims).  g (3N AoS) and lncc nullable.
 * When internals is non-null it receives 9N doubles:
 *   [0,N) Mw, [N,2N) rho, [2N,3N) A, [3N,4N) B, [4N,5N) E, [5N,6N) dR/dMw,
 *   [6N,9N) gradM (AoS)                                                    */
double orc_residual_lncc(const double* F, const double* M, const double* u, orc_dims d,
                         int radius, double* g, double* lncc, double* internals);
/* demons_step_mse (Eq. 9); r: N per-voxel residuals
 * f - m(x+u), n: AoS moving gradient at x + u. */
void orc_demons_step_mse(const double* r, const double* n, size_t N, double alpha, double* out);
/* MI: r = log2 B - MI (bits), g nullable; *mi = MI. */
double orc_residual_mi(const double* F, const double* M, const double* u, orc_dims d, int B, double sigma,
                       double* g, double* mi);
/* MSE; g nullable */
double orc_residual_mse(const double* F, const double* M, const double* u, orc_dims d,
                        double* g);

/* ---- lmopt ---- */
void orc_lm_step_pointwise(double r, const double* g, size_t nvox, double lambda,
                           double* out);
/* Explicit 3x3 damped solve (g g^T + lambda I) d = -r g (Appendix A oracle). */
void orc_lm_step_dense3(double r, const double* g3, double lambda, double* out3);
/* lm_step_tiled (Eq. 5): k^3 tiles, explicit 3x3 inverse. */
void orc_lm_step_tiled(double r, const double* g, orc_dims d, double lambda, int k, double* out);
void orc_update_damping(orc_lm_state* s, double loss_new, const orc_lm_config* c);
int orc_rejection_test(double loss_new, double loss_prev, double loss_prev2, double tau);
/* Scripted-residual harness: replays `losses` (one per attempt)
 * through the same attempt/retry/damping state machine lm_iterate uses.
 * Writes per-attempt lambda-after and decision (0 accept, 1 retry) and returns
 * the number of attempts consumed (<= n) for `iters` iterations. */
int orc_lm_replay(const double* losses, int n, int iters, const orc_lm_config* c,
                  double* lambda_out, int* decision_out, orc_lm_state* final_state);
void orc_adam_step(const double* g, double* m, double* v, size_t count, int t,
                   const orc_adam_config* c, double* out);

/* ---- pyramid ---- */
orc_dims orc_level_dims(orc_dims d, int factor);
void orc_downsample(const double* vol, orc_dims d, int factor, double* out);
void orc_upsample_warp(const double* u, orc_dims d, orc_dims nd, double scale,
                       double* out);

/* ---- driver ---- */
/* Runs `iters` lm_iterate steps at one level (F, M already at level dims).
 * u is updated in place.  state carries lambda/history.  trace may be null. */
int orc_lm_run_level(const double* F, const double* M, orc_dims d, double* u,
                     const orc_reg_config* c, orc_lm_state* state, int level, int iters,
                     orc_step_log* trace, int* ntrace);
// orc_lm_run_level plus the wall time of each attempt (step -> residual at
// the trial warp) in attempt_s[0 .. *nattempts), at most cap entries.
int orc_lm_run_level_timed(const double* F, const double* M, orc_dims d, double* u,
                           const orc_reg_config* c, orc_lm_state* state, int level, int iters,
                           orc_step_log* trace, int* ntrace, double* attempt_s, int cap, int* nattempts);
int orc_register(const float* F, const float* M, orc_dims d, const orc_reg_config* c,
                 double* warp_out, orc_step_log* trace, size_t cap, size_t* len,
                 double* jac_final);

/* ---- harness synth_pair ---- */
typedef struct {
    orc_dims dims;
    int num_blobs;
    double warp_sigma; /* <= 0 -> min(dims)/16 */
    double warp_max;
    double noise_sigma;
    uint64_t seed;
} orc_synth_spec;
/* Returns 0 or ORC_INVALID_ARG (non-positive Jacobian after 10 draws). */
int orc_synth_pair(const orc_synth_spec* s, float* F, float* M, float* u_true);

/* Splitmix64 helpers exposed for determinism tests. */
uint64_t orc_splitmix64(uint64_t* state);

#ifdef __cplusplus
}
#endif
#endif
