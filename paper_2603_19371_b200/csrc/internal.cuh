// internal.cuh -- host-side plumbing shared by engine.cu and ops.cu:
// context, error mapping, tracked device allocations.
#pragma once

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "kernels.cuh"
#include "wlm.h"

struct wlm_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;   // launches
    cudaStream_t capture = nullptr;  // private stream for graph capture
    bool own_stream = true;
    std::string err;
    uint64_t launches = 0;
    size_t cur_bytes = 0, peak_bytes = 0;
};

namespace wlm {

struct Fail {
    wlm_status st;
};

inline void set_err(wlm_ctx* c, const std::string& m) {
    if (c) c->err = m;
}

#define CK(call)                                                                          \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess) {                                                          \
            set_err(ctx, std::string(#call) + ": " + cudaGetErrorString(e_));             \
            throw Fail{e_ == cudaErrorMemoryAllocation ? WLM_OOM : WLM_CUDA};             \
        }                                                                                 \
    } while (0)

template <class T>
struct DevBuf {
    wlm_ctx* ctx = nullptr;
    T* p = nullptr;
    size_t count = 0;
    DevBuf() = default;
    DevBuf(wlm_ctx* c, size_t n) : ctx(c), count(n) {
        if (n == 0) return;
        cudaError_t e = cudaMalloc(&p, sizeof(T) * n);
        if (e != cudaSuccess) {
            p = nullptr;
            set_err(c, std::string("cudaMalloc: ") + cudaGetErrorString(e));
            throw Fail{WLM_OOM};
        }
        c->cur_bytes += sizeof(T) * n;
        c->peak_bytes = std::max(c->peak_bytes, c->cur_bytes);
    }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept { *this = std::move(o); }
    DevBuf& operator=(DevBuf&& o) noexcept {
        release();
        ctx = o.ctx; p = o.p; count = o.count;
        o.p = nullptr; o.count = 0;
        return *this;
    }
    ~DevBuf() { release(); }
    void release() {
        if (p) {
            cudaFree(p);
            ctx->cur_bytes -= sizeof(T) * count;
            p = nullptr;
            count = 0;
        }
    }
};

inline bool valid_dims(wlm_dims d) { return d.nx > 0 && d.ny > 0 && d.nz > 0; }
inline bool same_dims(wlm_dims a, wlm_dims b) { return a.nx == b.nx && a.ny == b.ny && a.nz == b.nz; }
inline size_t nvox(wlm_dims d) { return (size_t)d.nx * d.ny * d.nz; }

inline int smooth_radius(double sigma) {
    if (!(sigma > 0.0)) return 0;
    return std::max(1, (int)std::ceil(3.0 * sigma));
}

template <class T>
inline void fill_half_kernel(double sigma, int R, T* w, T* full) {
    if (R == 0) { w[0] = T(1); *full = T(1); return; }
    double s = 0.0;
    for (int d = 0; d <= R; ++d) {
        const double v = std::exp(-0.5 * (double)(d * d) / (sigma * sigma));
        w[d] = (T)v;
        s += d == 0 ? v : 2.0 * v;
    }
    *full = (T)s;
}

inline wlm_status guard(wlm_ctx* ctx) {
    if (!ctx) return WLM_INVALID_ARG;
    cudaError_t e = cudaSetDevice(ctx->device);
    if (e != cudaSuccess) {
        set_err(ctx, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
        return WLM_CUDA;
    }
    return WLM_OK;
}

// Runs fn with CUDA errors mapped to wlm_status.  Kernel launches are
// credited to the outermost call only (entry points may nest).
inline int& run_depth() {
    static thread_local int d = 0;
    return d;
}

template <class Fn>
wlm_status run(wlm_ctx* ctx, Fn fn) {
    wlm_status s = guard(ctx);
    if (s != WLM_OK) return s;
    const uint64_t before = g_kernel_launches;
    ++run_depth();
    try {
        fn();
    } catch (const Fail& f) {
        if (--run_depth() == 0) ctx->launches += g_kernel_launches - before;
        return f.st;
    }
    if (--run_depth() == 0) ctx->launches += g_kernel_launches - before;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_err(ctx, std::string("kernel launch: ") + cudaGetErrorString(e));
        return WLM_CUDA;
    }
    return WLM_OK;
}

}  // namespace wlm


// ===========================================================================
// Engine
using namespace wlm;
struct wlm_engine {
    wlm_ctx* ctx = nullptr;
    Geo g{};
    wlm_dims dims{};
    int pairs = 0;
    wlm_reg_config cfg{};
    LmParams P{};
    DevBuf<float> F, M, U, ABE, G, AM, AV;  // dU_s lives inside ABE (Batch::VS)
    DevBuf<double> MW, GM;
    DevBuf<PairState> st;
    DevBuf<double> partials, script, shift_part, plane_sum, TM, MIT, ABC, X64, TAPU, TAPW;
    DevBuf<unsigned long long> HIST;
    DevBuf<wlm_step_log> trace;
    Batch B{};
    cudaGraphExec_t step_exec = nullptr, loop_exec = nullptr;
    cudaGraph_t step_graph = nullptr, loop_graph = nullptr;
    int body_kernels = 0;   // kernels per attempt graph (whole batch)
    int group_kernels = 0;  // kernels per attempt of both pair-group graphs
    // Pair groups: without rejection, iterate() runs the batch as two
    // independent streams of attempt graphs (pairs [0, h) and [h, pairs))
    // that only join at the end, so the two groups drift to different
    // stages and their kernels overlap (a bandwidth-bound stage of one group
    // beside a compute-bound stage of the other, and each other's tails).
    static constexpr int kMaxGroups = 4;
    int pair_groups = 1;
    cudaStream_t side[kMaxGroups] = {};  // side[0] unused (group 0 runs on the ctx stream)
    cudaEvent_t fork_ev = nullptr, join_ev[kMaxGroups] = {};
    cudaGraphExec_t group_exec[kMaxGroups] = {}, group_loop_exec[kMaxGroups] = {};
    cudaGraph_t group_graph[kMaxGroups] = {}, group_loop_graph[kMaxGroups] = {};
    bool shared_fm = false;         // F, M owned by a slab group (Batch set by the group)
    bool shared_plane_sum = false;  // per-plane sum(rho) owned by a slab group

    ~wlm_engine() {
        for (int i = 0; i < kMaxGroups; ++i) {
            if (group_exec[i]) cudaGraphExecDestroy(group_exec[i]);
            if (group_graph[i]) cudaGraphDestroy(group_graph[i]);
            if (group_loop_exec[i]) cudaGraphExecDestroy(group_loop_exec[i]);
            if (group_loop_graph[i]) cudaGraphDestroy(group_loop_graph[i]);
            if (side[i]) cudaStreamDestroy(side[i]);
            if (join_ev[i]) cudaEventDestroy(join_ev[i]);
        }
        if (fork_ev) cudaEventDestroy(fork_ev);
        if (step_exec) cudaGraphExecDestroy(step_exec);
        if (loop_exec) cudaGraphExecDestroy(loop_exec);
        if (step_graph) cudaGraphDestroy(step_graph);
        if (loop_graph) cudaGraphDestroy(loop_graph);
    }

    // Stages of one attempt (a slab group interleaves them with exchanges),
    // on the whole batch or on one pair group b.
    void stage_grad(const Batch& b, cudaStream_t s) {
        if (P.metric == WLM_METRIC_MSE) launch_mse_grad(b, P, s);
        else if (P.metric == WLM_METRIC_MI) launch_mi_grad(b, P, s);
        else launch_lncc_bwd(b, P, s);
        if (P.optimizer == WLM_OPT_ADAM) launch_adam(b, P, s);
    }
    void stage_step(const Batch& b, cudaStream_t s) {
        if (P.optimizer == WLM_OPT_LM && P.tile_k > 1) launch_tile_matrix(b, P, s);
        launch_step_smooth(b, P, s);
    }
    void stage_compose(const Batch& b, cudaStream_t s) {
        launch_compose_smooth(b, P, s);
        if (P.log_jacobian) launch_jacobian_diag(b, P, s);
    }
    void stage_eval(const Batch& b, int mode, cudaStream_t s) {
        if (P.metric == WLM_METRIC_MSE) launch_mse_fwd(b, P, mode, s);
        else if (P.metric == WLM_METRIC_MI) launch_mi_fwd(b, P, mode, s);
        else launch_lncc_fwd(b, P, mode, s);
    }
    void stage_finalize(const Batch& b, int mode, cudaStream_t s) {
        if (P.metric == WLM_METRIC_MI) launch_mi_finalize(b, P, mode, s);
        else launch_finalize(b, P, mode, s);
    }
    void stage_grad(cudaStream_t s) { stage_grad(B, s); }
    void stage_step(cudaStream_t s) { stage_step(B, s); }
    void stage_compose(cudaStream_t s) { stage_compose(B, s); }
    void stage_eval(int mode, cudaStream_t s) { stage_eval(B, mode, s); }
    void stage_finalize(int mode, cudaStream_t s) { stage_finalize(B, mode, s); }

    void attempt(const Batch& b, cudaStream_t s) {
        stage_grad(b, s);
        stage_step(b, s);
        stage_compose(b, s);
        stage_eval(b, 1, s);
        stage_finalize(b, 1, s);
    }

    // One attempt for every pair.
    void body(cudaStream_t s) { attempt(B, s); }

    // Pair groups: contiguous, sizes differing by at most one.
    int ngroups() const { return std::min(pair_groups, pairs); }
    Batch group(int gi) const {
        Batch b = B;
        const int G = ngroups(), q = pairs / G, r = pairs % G;
        b.pair0 = gi * q + std::min(gi, r);
        b.pairs = q + (gi < r ? 1 : 0);
        b.ctas_per_sm = 1;  // measured: 10.90 -> 11.28 Gvoxel/s at 8 x 192^3 against 4
        return b;
    }
    bool grouped() const { return ngroups() > 1; }

    void build_group_graphs() {
        if (group_exec[0]) return;
        const int G = ngroups();
        if (!fork_ev) CK(cudaEventCreateWithFlags(&fork_ev, cudaEventDisableTiming));
        for (int gi = 1; gi < G; ++gi) {
            if (!side[gi]) CK(cudaStreamCreateWithFlags(&side[gi], cudaStreamNonBlocking));
            if (!join_ev[gi]) CK(cudaEventCreateWithFlags(&join_ev[gi], cudaEventDisableTiming));
        }
        const uint64_t saved = g_kernel_launches;
        for (int gi = 0; gi < G; ++gi) {
            CK(cudaStreamBeginCapture(ctx->capture, cudaStreamCaptureModeThreadLocal));
            attempt(group(gi), ctx->capture);
            CK(cudaStreamEndCapture(ctx->capture, &group_graph[gi]));
            CK(cudaGraphInstantiate(&group_exec[gi], group_graph[gi], 0));
        }
        group_kernels = (int)(g_kernel_launches - saved);
        g_kernel_launches = saved;
    }

    // iters attempts of every pair as independent graph streams, one per
    // group, joined at the end (rejection off: an attempt is an iteration).
    void launch_grouped(int iters, cudaStream_t s) {
        build_group_graphs();
        const int G = ngroups();
        CK(cudaEventRecord(fork_ev, s));
        for (int gi = 1; gi < G; ++gi) CK(cudaStreamWaitEvent(side[gi], fork_ev, 0));
        for (int i = 0; i < iters; ++i)
            for (int gi = 0; gi < G; ++gi) CK(cudaGraphLaunch(group_exec[gi], gi == 0 ? s : side[gi]));
        for (int gi = 1; gi < G; ++gi) {
            CK(cudaEventRecord(join_ev[gi], side[gi]));
            CK(cudaStreamWaitEvent(s, join_ev[gi], 0));
        }
    }

    void invalidate_graphs() {
        for (int i = 0; i < kMaxGroups; ++i) {
            if (group_exec[i]) { cudaGraphExecDestroy(group_exec[i]); group_exec[i] = nullptr; }
            if (group_graph[i]) { cudaGraphDestroy(group_graph[i]); group_graph[i] = nullptr; }
            if (group_loop_exec[i]) { cudaGraphExecDestroy(group_loop_exec[i]); group_loop_exec[i] = nullptr; }
            if (group_loop_graph[i]) { cudaGraphDestroy(group_loop_graph[i]); group_loop_graph[i] = nullptr; }
        }
        if (step_exec) { cudaGraphExecDestroy(step_exec); step_exec = nullptr; }
        if (loop_exec) { cudaGraphExecDestroy(loop_exec); loop_exec = nullptr; }
        if (step_graph) { cudaGraphDestroy(step_graph); step_graph = nullptr; }
        if (loop_graph) { cudaGraphDestroy(loop_graph); loop_graph = nullptr; }
    }

    void build_step_graph() {
        if (step_exec) return;
        const uint64_t saved = g_kernel_launches;
        CK(cudaStreamBeginCapture(ctx->capture, cudaStreamCaptureModeThreadLocal));
        body(ctx->capture);
        CK(cudaStreamEndCapture(ctx->capture, &step_graph));
        body_kernels = (int)(g_kernel_launches - saved);
        g_kernel_launches = saved;
        CK(cudaGraphInstantiate(&step_exec, step_graph, 0));
    }

    // WHILE(any pair not done) { body; cond } -- rejection retries and the
    // iteration count live entirely on the device.
    // WHILE(any pair of b not done) { attempt(b); cond } -- rejection retries
    // and the iteration count live entirely on the device.
    void make_loop_graph(const Batch& b, cudaGraph_t& graph, cudaGraphExec_t& exec, int* kernels) {
        CK(cudaGraphCreate(&graph, 0));
        cudaGraphConditionalHandle h;
        CK(cudaGraphConditionalHandleCreate(&h, graph, 1, cudaGraphCondAssignDefault));
        alignas(cudaGraphNodeParams) unsigned char raw[sizeof(cudaGraphNodeParams)] = {};
        cudaGraphNodeParams& cp = *reinterpret_cast<cudaGraphNodeParams*>(raw);
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = h;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        cudaGraphNode_t node;
        CK(cudaGraphAddNode(&node, graph, nullptr, 0, &cp));
        cudaGraph_t bodyg = cp.conditional.phGraph_out[0];
        const uint64_t saved = g_kernel_launches;
        CK(cudaStreamBeginCaptureToGraph(ctx->capture, bodyg, nullptr, nullptr, 0,
                                         cudaStreamCaptureModeThreadLocal));
        attempt(b, ctx->capture);
        *kernels = (int)(g_kernel_launches - saved);
        launch_loop_cond(b, h, ctx->capture);
        cudaGraph_t out = nullptr;
        CK(cudaStreamEndCapture(ctx->capture, &out));
        g_kernel_launches = saved;
        CK(cudaGraphInstantiate(&exec, graph, 0));
    }
    void build_loop_graph() {
        if (loop_exec) return;
        make_loop_graph(B, loop_graph, loop_exec, &body_kernels);
    }
    // With rejection on, each pair group loops in its own WHILE graph on its
    // own stream; the groups join when all their pairs are done.
    void launch_grouped_loop(cudaStream_t s) {
        const int G = ngroups();
        if (!group_loop_exec[0]) {
            if (!fork_ev) CK(cudaEventCreateWithFlags(&fork_ev, cudaEventDisableTiming));
            for (int gi = 1; gi < G; ++gi) {
                if (!side[gi]) CK(cudaStreamCreateWithFlags(&side[gi], cudaStreamNonBlocking));
                if (!join_ev[gi]) CK(cudaEventCreateWithFlags(&join_ev[gi], cudaEventDisableTiming));
            }
            int k = 0, total = 0;
            for (int gi = 0; gi < G; ++gi) {
                make_loop_graph(group(gi), group_loop_graph[gi], group_loop_exec[gi], &k);
                total += k;
            }
            group_kernels = total;
        }
        CK(cudaEventRecord(fork_ev, s));
        for (int gi = 1; gi < G; ++gi) CK(cudaStreamWaitEvent(side[gi], fork_ev, 0));
        for (int gi = 0; gi < G; ++gi) CK(cudaGraphLaunch(group_loop_exec[gi], gi == 0 ? s : side[gi]));
        for (int gi = 1; gi < G; ++gi) {
            CK(cudaEventRecord(join_ev[gi], side[gi]));
            CK(cudaStreamWaitEvent(s, join_ev[gi], 0));
        }
    }
};


namespace wlm {
wlm_status engine_init(wlm_engine* e, wlm_ctx* ctx, wlm_dims d, int pairs, const wlm_reg_config* c);
void engine_alloc(wlm_engine* e);
void clear_adam_moments(wlm_engine* e, cudaStream_t s);
// fp64 reference-order field kernels (field64.cu)
std::vector<double> gaussian_taps64(double sigma, int* R);
void launch_warp_volume64(const double* M, const double* u, wlm_dims d, double* Mw, double* gM, cudaStream_t s);
void launch_compose64(const double* u, const double* v, double eps, wlm_dims d, double* out, cudaStream_t s);
void launch_sample_points64(const double* u, wlm_dims d, const double* pts, long long npts, double* out,
                            cudaStream_t s);
void launch_sample_grad_points64(const double* v, wlm_dims d, const double* pts, long long npts, double* val,
                                 double* grad, cudaStream_t s);
void launch_max_abs64(const double* v, long long count, unsigned long long* out, cudaStream_t s);
void launch_jacobian_min64(const double* u, wlm_dims d, unsigned long long* out, cudaStream_t s);
void launch_jacobian_min64_soa32(const float* u, wlm_dims d, unsigned long long* out, cudaStream_t s);
double jacobian_key_to_double(unsigned long long k);
unsigned long long jacobian_key_init();
void smooth64(double* data, double* tmp, const double* dw, int R, wlm_dims d, int nchan, long long cstride,
              long long estride, cudaStream_t s);
void launch_lm_step64(double r, const double* g, long long n, double lambda, double* out, cudaStream_t s);
void launch_stride64(const double* in, wlm_dims d, int f, double* out, wlm_dims nd, cudaStream_t s);
void launch_upsample64(const double* u, wlm_dims d, wlm_dims nd, double scale, double* out, cudaStream_t s);
std::vector<PairState> read_states(wlm_engine* e);
void copy_warps_in(wlm_engine* e, const float* u, int is_host);
}  // namespace wlm
