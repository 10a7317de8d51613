// synth.cu -- GPU synth_pair.
//
// Same recipe as the harness spec: a sum of Gaussian blobs normalised to
// [0, 1]; a Gaussian-smoothed random displacement rescaled to warp_max with a
// positive Jacobian (redrawn up to 10 times); moving = clean fixed through
// Id + u_true; independent N(0, noise^2) on both.  Random numbers come from a
// counter-based SplitMix64 hash of (seed, stream, voxel), so the output is
// seed-deterministic and independent of the launch shape.  (The fp64 oracle
// has its own serial-RNG synth for the parity tests; benchmark inputs are
// produced here so the product never depends on test infrastructure.)
#include <cmath>
#include <vector>

#include "internal.cuh"

using namespace wlm;

namespace {

__host__ __device__ inline uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ inline double uni(uint64_t seed, uint64_t stream, uint64_t i) {
    return (double)(mix64(seed ^ mix64(stream * 0x632BE59BD9B4E019ull + i)) >> 11) * 0x1.0p-53;
}

__device__ inline float normal(uint64_t seed, uint64_t stream, uint64_t i) {
    const double u1 = 1.0 - uni(seed, stream, 2 * i), u2 = uni(seed, stream, 2 * i + 1);
    return (float)(sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2));
}

struct Blob {
    float cx, cy, cz, q, amp;
};

__global__ void k_blobs(float* F, Geo g, const Blob* b, int K) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < g.n;
         i += (long long)gridDim.x * blockDim.x) {
        const float x = (float)(i % g.nx), y = (float)((i / g.nx) % g.ny), z = (float)(i / ((long long)g.nx * g.ny));
        float s = 0.f;
        for (int k = 0; k < K; ++k) {
            const float dx = x - b[k].cx, dy = y - b[k].cy, dz = z - b[k].cz;
            s += b[k].amp * __expf(-(dx * dx + dy * dy + dz * dz) * b[k].q);
        }
        F[i] = s;
    }
}

__global__ void k_minmax(const float* v, long long n, int* lo_hi) {
    float lo = INFINITY, hi = -INFINITY;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        lo = fminf(lo, v[i]);
        hi = fmaxf(hi, v[i]);
    }
    for (int o = 16; o > 0; o >>= 1) {
        lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(lo_hi, float_to_ordered(lo));
        atomicMax(lo_hi + 1, float_to_ordered(hi));
    }
}

__global__ void k_normalise(float* F, long long n, const int* lo_hi) {
    const float lo = ordered_to_float(lo_hi[0]), hi = ordered_to_float(lo_hi[1]);
    const float inv = hi > lo ? 1.f / (hi - lo) : 1.f;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        F[i] = (F[i] - lo) * inv;
}

__global__ void k_noise_field(float* u, long long n3, uint64_t seed, uint64_t stream) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n3;
         i += (long long)gridDim.x * blockDim.x)
        u[i] = normal(seed, stream, (uint64_t)i);
}

__global__ void k_scale(float* u, long long n3, const unsigned* maxbits, float target) {
    const float m = __uint_as_float(*maxbits);
    const float s = m > 0.f ? target / m : 0.f;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n3;
         i += (long long)gridDim.x * blockDim.x)
        u[i] *= s;
}

// fp64 lerps of the fp32 image, rounded once: at a knot (t = 0 or 1) the
// sample is exactly the voxel value, so warp_max = 0 gives moving == fixed
// even on the last index, where the cell has t = 1.
__device__ __forceinline__ float cell_sample_exact(const float* __restrict__ v, const Cell& c) {
    if (!c.finite) return __int_as_float(0x7fc00000);
    const double tx = c.tx, ty = c.ty, tz = c.tz;
    const double a = v[c.o000], b = v[c.o100], cc = v[c.o010], e = v[c.o110];
    const double f = v[c.o001], h = v[c.o101], k = v[c.o011], l = v[c.o111];
    const double v00 = fma(tx, b - a, a), v10 = fma(tx, e - cc, cc);
    const double v01 = fma(tx, h - f, f), v11 = fma(tx, l - k, k);
    const double s0 = fma(ty, v10 - v00, v00), s1 = fma(ty, v11 - v01, v01);
    return (float)fma(tz, s1 - s0, s0);
}

__global__ void k_moving(const float* F, const float* u, float* Fo, float* Mo, Geo g, float noise,
                         uint64_t seed) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < g.n;
         i += (long long)gridDim.x * blockDim.x) {
        const int x = (int)(i % g.nx), y = (int)((i / g.nx) % g.ny), z = (int)(i / ((long long)g.nx * g.ny));
        const Cell c = make_cell(g, x, y, z, u[i], u[g.n + i], u[2 * g.n + i]);
        const float m = cell_sample_exact(F, c);
        Fo[i] = F[i] + noise * normal(seed, 101, (uint64_t)i);
        Mo[i] = m + noise * normal(seed, 102, (uint64_t)i);
    }
}

inline int blocks_for(long long n) {
    return (int)std::min<long long>(148 * 32, std::max<long long>(1, (n + 255) / 256));
}

}  // namespace

extern "C" wlm_status wlm_synth_pair(wlm_ctx* ctx, const wlm_synth_spec* sp, float* F, float* M,
                                     float* u_true, int on_device) {
    if (!ctx || !sp || !F || !M || !valid_dims(sp->dims) || sp->num_blobs < 1 || sp->warp_max < 0)
        return WLM_INVALID_ARG;
    wlm_status result = WLM_OK;
    wlm_status s = run(ctx, [&] {
        const wlm_dims d = sp->dims;
        const Geo g = make_geo(d);
        const long long n = g.n;
        cudaStream_t st = ctx->stream;
        // blob parameters: serial SplitMix64 stream from the seed (host, K values)
        uint64_t state = sp->seed;
        auto u01 = [&] {
            const uint64_t r = mix64(state++);
            return (double)(r >> 11) * 0x1.0p-53;
        };
        const double mind = (double)std::min(d.nx, std::min(d.ny, d.nz));
        std::vector<Blob> hb(sp->num_blobs);
        for (auto& b : hb) {
            b.cx = (float)((0.2 + 0.6 * u01()) * d.nx);
            b.cy = (float)((0.2 + 0.6 * u01()) * d.ny);
            b.cz = (float)((0.2 + 0.6 * u01()) * d.nz);
            const double sg = (0.05 + 0.07 * u01()) * mind;
            b.q = (float)(1.0 / (2.0 * sg * sg));
            b.amp = (float)(0.3 + 0.7 * u01());
        }
        DevBuf<Blob> db(ctx, hb.size());
        CK(cudaMemcpyAsync(db.p, hb.data(), sizeof(Blob) * hb.size(), cudaMemcpyHostToDevice, st));
        DevBuf<float> Fc(ctx, n), U(ctx, 3 * n), T(ctx, 3 * n), S(ctx, 3 * n);
        DevBuf<int> mm(ctx, 2);
        const int init[2] = {0x7f800000, (int)0x807fffff};  // ordered(+inf), ordered(-inf)
        CK(cudaMemcpyAsync(mm.p, init, sizeof(init), cudaMemcpyHostToDevice, st));
        k_blobs<<<blocks_for(n), 256, 0, st>>>(Fc.p, g, db.p, sp->num_blobs);
        k_minmax<<<blocks_for(n), 256, 0, st>>>(Fc.p, n, mm.p);
        k_normalise<<<blocks_for(n), 256, 0, st>>>(Fc.p, n, mm.p);
        g_kernel_launches += 3;
        const double ws = sp->warp_sigma > 0.0 ? sp->warp_sigma : mind / 16.0;
        DevBuf<unsigned> mx(ctx, 1);
        DevBuf<int> jac(ctx, 1);
        bool ok = sp->warp_max == 0.0;
        if (ok) CK(cudaMemsetAsync(S.p, 0, sizeof(float) * 3 * n, st));
        for (int attempt = 0; attempt < 10 && !ok; ++attempt) {
            k_noise_field<<<blocks_for(3 * n), 256, 0, st>>>(U.p, 3 * n, sp->seed, 7 + attempt);
            ++g_kernel_launches;
            launch_smooth_generic(U.p, S.p, T.p, 3, g, std::min(ws, 21.0), st);
            CK(cudaMemsetAsync(mx.p, 0, sizeof(unsigned), st));
            launch_max_abs(S.p, 3 * n, mx.p, st);
            k_scale<<<blocks_for(3 * n), 256, 0, st>>>(S.p, 3 * n, mx.p, (float)sp->warp_max);
            ++g_kernel_launches;
            if (d.nx < 2 || d.ny < 2 || d.nz < 2) { ok = true; break; }
            const int inf_bits = 0x7f800000;
            CK(cudaMemcpyAsync(jac.p, &inf_bits, sizeof(int), cudaMemcpyHostToDevice, st));
            launch_jacdet(S.p, g, jac.p, st);
            int h = 0;
            CK(cudaMemcpyAsync(&h, jac.p, sizeof(int), cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            ok = ordered_to_float(h) > 0.f;
        }
        if (!ok) {
            set_err(ctx, "synth_pair: no positive-Jacobian warp after 10 draws");
            result = WLM_INVALID_ARG;
            return;
        }
        DevBuf<float> Fo(ctx, on_device ? 0 : n), Mo(ctx, on_device ? 0 : n);
        float* fo = on_device ? F : Fo.p;
        float* mo = on_device ? M : Mo.p;
        k_moving<<<blocks_for(n), 256, 0, st>>>(Fc.p, S.p, fo, mo, g, (float)sp->noise_sigma, sp->seed);
        ++g_kernel_launches;
        const cudaMemcpyKind k = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
        if (!on_device) {
            CK(cudaMemcpyAsync(F, Fo.p, sizeof(float) * n, k, st));
            CK(cudaMemcpyAsync(M, Mo.p, sizeof(float) * n, k, st));
        }
        if (u_true) CK(cudaMemcpyAsync(u_true, S.p, sizeof(float) * 3 * n, k, st));
        CK(cudaStreamSynchronize(st));
    });
    return s != WLM_OK ? s : result;
}
