// io.cu -- VOL3 / DSP3 streaming and the CSV trace (the data formats either
// side of the path; reference io.hpp:15-21, io.cpp:34-109).
//
//   VOL3: "VOL3", nx ny nz (u32 LE), nx*ny*nz float32 LE, x fastest
//   DSP3: "DSP3", same header, 3*n float32, component innermost (AoS)
//
// The device side is SoA fp32 planes, so reads stream the payload through two
// pinned staging buffers (file read of chunk i+1 overlaps the host->device
// copy of chunk i) and DSP3 is transposed AoS <-> SoA on the device.  Every
// reference io_error has the same condition and message here ("bad magic",
// "truncated header/payload", "non-positive dims", "dims too large",
// "non-finite value in payload"), returned as WLM_INVALID_ARG.  With
// on_device == 0 the calls touch no CUDA API (ctx may be NULL), so the host
// path runs anywhere.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "internal.cuh"

using namespace wlm;

namespace {

constexpr size_t kMaxVoxels = size_t{1} << 31;  // io.cpp:13
constexpr size_t kChunk = size_t{16} << 20;     // floats per staging buffer (64 MB)

struct IoFail {
    std::string msg;
};

struct File {
    FILE* f = nullptr;
    ~File() {
        if (f) std::fclose(f);
    }
};

uint32_t le32(const unsigned char* b) {
    return (uint32_t)b[0] | ((uint32_t)b[1] << 8) | ((uint32_t)b[2] << 16) | ((uint32_t)b[3] << 24);
}

wlm_dims read_header(FILE* f, const char* magic, const std::string& path) {
    unsigned char h[16];
    if (std::fread(h, 1, 4, f) != 4 || std::memcmp(h, magic, 4) != 0)
        throw IoFail{path + ": bad magic (expected " + magic + ")"};
    if (std::fread(h + 4, 1, 12, f) != 12) throw IoFail{path + ": truncated header"};
    wlm_dims d{(int)le32(h + 4), (int)le32(h + 8), (int)le32(h + 12)};
    if (d.nx <= 0 || d.ny <= 0 || d.nz <= 0) throw IoFail{path + ": non-positive dims"};
    if ((size_t)d.nx * d.ny * d.nz > kMaxVoxels) throw IoFail{path + ": dims too large"};
    return d;
}

void check_finite(const float* v, size_t n, const std::string& path) {
    for (size_t i = 0; i < n; ++i)
        if (!std::isfinite(v[i])) throw IoFail{path + ": non-finite value in payload"};
}

__global__ void k_aos3_to_soa(const float* __restrict__ in, float* __restrict__ out, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        for (int c = 0; c < 3; ++c) out[(long long)c * n + i] = in[3 * i + c];
}
__global__ void k_soa_to_aos3(const float* __restrict__ in, float* __restrict__ out, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        for (int c = 0; c < 3; ++c) out[3 * i + c] = in[(long long)c * n + i];
}
int blocks_for(long long n) { return (int)std::min<long long>(148 * 8, (n + 255) / 256); }

// Stream `count` floats of payload into dst (host, or device through pinned
// staging with the copy of one chunk overlapping the read of the next).
void stream_in(wlm_ctx* ctx, FILE* f, float* dst, size_t count, int on_device, const std::string& path) {
    if (!on_device) {
        if (std::fread(dst, 4, count, f) != count) throw IoFail{path + ": truncated payload"};
        check_finite(dst, count, path);
        return;
    }
    float* stage[2] = {nullptr, nullptr};
    cudaEvent_t done[2] = {nullptr, nullptr};
    const size_t chunk = std::min(kChunk, count);
    try {
        for (int i = 0; i < 2; ++i) {
            CK(cudaMallocHost(&stage[i], sizeof(float) * chunk));
            CK(cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming));
        }
        size_t off = 0;
        for (int k = 0; off < count; ++k) {
            const int s = k & 1;
            CK(cudaEventSynchronize(done[s]));  // staging buffer s is free again
            const size_t m = std::min(chunk, count - off);
            if (std::fread(stage[s], 4, m, f) != m) throw IoFail{path + ": truncated payload"};
            check_finite(stage[s], m, path);
            CK(cudaMemcpyAsync(dst + off, stage[s], sizeof(float) * m, cudaMemcpyHostToDevice, ctx->stream));
            CK(cudaEventRecord(done[s], ctx->stream));
            off += m;
        }
        CK(cudaStreamSynchronize(ctx->stream));
    } catch (...) {
        cudaStreamSynchronize(ctx->stream);
        for (int i = 0; i < 2; ++i) {
            if (stage[i]) cudaFreeHost(stage[i]);
            if (done[i]) cudaEventDestroy(done[i]);
        }
        throw;
    }
    for (int i = 0; i < 2; ++i) {
        cudaFreeHost(stage[i]);
        cudaEventDestroy(done[i]);
    }
}

void write_header(FILE* f, const char* magic, wlm_dims d, const std::string& path) {
    unsigned char h[16];
    std::memcpy(h, magic, 4);
    const uint32_t v[3] = {(uint32_t)d.nx, (uint32_t)d.ny, (uint32_t)d.nz};
    for (int i = 0; i < 3; ++i)
        for (int b = 0; b < 4; ++b) h[4 + 4 * i + b] = (unsigned char)((v[i] >> (8 * b)) & 0xff);
    if (std::fwrite(h, 1, 16, f) != 16) throw IoFail{path + ": write failed"};
}

// Write `count` floats from src (host, or device via chunked D2H copies).
void stream_out(wlm_ctx* ctx, FILE* f, const float* src, size_t count, int on_device, const std::string& path) {
    if (!on_device) {
        if (std::fwrite(src, 4, count, f) != count) throw IoFail{path + ": write failed"};
        return;
    }
    const size_t chunk = std::min(kChunk, count);
    std::vector<float> host(chunk);
    for (size_t off = 0; off < count; off += chunk) {
        const size_t m = std::min(chunk, count - off);
        CK(cudaMemcpy(host.data(), src + off, sizeof(float) * m, cudaMemcpyDeviceToHost));
        if (std::fwrite(host.data(), 4, m, f) != m) throw IoFail{path + ": write failed"};
    }
}

template <class Fn>
wlm_status io_run(wlm_ctx* ctx, int on_device, Fn fn) {
    try {
        if (on_device) {
            if (!ctx) return WLM_INVALID_ARG;
            return run(ctx, fn);
        }
        fn();
        return WLM_OK;
    } catch (const IoFail& e) {
        if (ctx) set_err(ctx, e.msg);
        else std::fprintf(stderr, "%s\n", e.msg.c_str());
        return WLM_INVALID_ARG;
    }
}

}  // namespace

extern "C" {

wlm_status wlm_io_dims(const char* path, int is_field, wlm_dims* d) {
    if (!path || !d) return WLM_INVALID_ARG;
    return io_run(nullptr, 0, [&] {
        File fh;
        fh.f = std::fopen(path, "rb");
        if (!fh.f) throw IoFail{std::string(path) + ": cannot open"};
        *d = read_header(fh.f, is_field ? "DSP3" : "VOL3", path);
    });
}

wlm_status wlm_read_vol3(wlm_ctx* ctx, const char* path, float* dst, size_t cap, int on_device, wlm_dims* d) {
    if (!path || !dst || !d) return WLM_INVALID_ARG;
    return io_run(ctx, on_device, [&] {
        File fh;
        fh.f = std::fopen(path, "rb");
        if (!fh.f) throw IoFail{std::string(path) + ": cannot open"};
        *d = read_header(fh.f, "VOL3", path);
        const size_t n = nvox(*d);
        if (n > cap) throw IoFail{std::string(path) + ": destination too small"};
        stream_in(ctx, fh.f, dst, n, on_device, path);
    });
}

wlm_status wlm_read_dsp3(wlm_ctx* ctx, const char* path, float* dst_soa, size_t cap, int on_device, wlm_dims* d) {
    if (!path || !dst_soa || !d) return WLM_INVALID_ARG;
    return io_run(ctx, on_device, [&] {
        File fh;
        fh.f = std::fopen(path, "rb");
        if (!fh.f) throw IoFail{std::string(path) + ": cannot open"};
        *d = read_header(fh.f, "DSP3", path);
        const size_t n = nvox(*d);
        if (3 * n > cap) throw IoFail{std::string(path) + ": destination too small"};
        if (!on_device) {
            std::vector<float> aos(3 * n);
            stream_in(ctx, fh.f, aos.data(), 3 * n, 0, path);
            for (size_t i = 0; i < n; ++i)
                for (int c = 0; c < 3; ++c) dst_soa[(size_t)c * n + i] = aos[3 * i + c];
            return;
        }
        DevBuf<float> aos(ctx, 3 * n);
        stream_in(ctx, fh.f, aos.p, 3 * n, 1, path);
        k_aos3_to_soa<<<blocks_for((long long)n), 256, 0, ctx->stream>>>(aos.p, dst_soa, (long long)n);
        ++g_kernel_launches;
        CK(cudaStreamSynchronize(ctx->stream));
    });
}

wlm_status wlm_write_vol3(wlm_ctx* ctx, const char* path, const float* src, int on_device, wlm_dims d) {
    if (!path || !src || !valid_dims(d)) return WLM_INVALID_ARG;
    return io_run(ctx, on_device, [&] {
        File fh;
        fh.f = std::fopen(path, "wb");
        if (!fh.f) throw IoFail{std::string(path) + ": cannot open for writing"};
        write_header(fh.f, "VOL3", d, path);
        stream_out(ctx, fh.f, src, nvox(d), on_device, path);
    });
}

wlm_status wlm_write_dsp3(wlm_ctx* ctx, const char* path, const float* src_soa, int on_device, wlm_dims d) {
    if (!path || !src_soa || !valid_dims(d)) return WLM_INVALID_ARG;
    return io_run(ctx, on_device, [&] {
        File fh;
        fh.f = std::fopen(path, "wb");
        if (!fh.f) throw IoFail{std::string(path) + ": cannot open for writing"};
        write_header(fh.f, "DSP3", d, path);
        const size_t n = nvox(d);
        if (!on_device) {
            std::vector<float> aos(3 * n);
            for (size_t i = 0; i < n; ++i)
                for (int c = 0; c < 3; ++c) aos[3 * i + c] = src_soa[(size_t)c * n + i];
            stream_out(ctx, fh.f, aos.data(), 3 * n, 0, path);
            return;
        }
        DevBuf<float> aos(ctx, 3 * n);
        k_soa_to_aos3<<<blocks_for((long long)n), 256, 0, ctx->stream>>>(src_soa, aos.p, (long long)n);
        ++g_kernel_launches;
        CK(cudaStreamSynchronize(ctx->stream));
        stream_out(ctx, fh.f, aos.p, 3 * n, 1, path);
    });
}

// CSV trace, SPEC.md:427 columns, versioned header line.
wlm_status wlm_write_trace_csv(const char* path, const wlm_step_log* rows, size_t n) {
    if (!path || (!rows && n)) return WLM_INVALID_ARG;
    FILE* f = std::fopen(path, "w");
    if (!f) return WLM_INVALID_ARG;
    std::fprintf(f, "# warplm-csv v1\nlevel,iter,loss_raw,r,lambda,eps,accepted,retries,jac_det_min\n");
    for (size_t i = 0; i < n; ++i) {
        const wlm_step_log& t = rows[i];
        std::fprintf(f, "%d,%d,%.17g,%.17g,%.17g,%.17g,%d,%d,%.17g\n", t.level, t.iter, t.loss_raw, t.r, t.lambda,
                     t.eps, t.accepted, t.retries, t.jac_det_min);
    }
    const bool ok = std::fclose(f) == 0;
    return ok ? WLM_OK : WLM_INVALID_ARG;
}

}  // extern "C"
