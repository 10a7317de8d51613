// Probe of the K4 TMA path: 5D tensor map over a U-like buffer, one box
// (40 x 22 x 1 x 3 x 1) into shared memory, mbarrier completion, compare.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstring>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k(const __grid_constant__ CUtensorMap map, float* out, int c0, int c1, int c2, int c3, int c4,
                  int* status) {
    extern __shared__ __align__(128) float sm[];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(40 * 22 * 3 * 4)
                     : "memory");
        asm volatile(
            "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
            "%4, %5, %6}], [%7];" ::"r"(smem_u32(sm)),
            "l"(&map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(&bar))
            : "memory");
    }
    uint32_t done = 0;
    long long spins = 0;
    while (!done) {
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                     : "=r"(done)
                     : "r"(smem_u32(&bar)), "r"(0)
                     : "memory");
        if (++spins > (1ll << 26)) { if (threadIdx.x == 0) *status = 2; return; }
    }
    for (int i = threadIdx.x; i < 40 * 22 * 3; i += blockDim.x) out[i] = sm[i];
    if (threadIdx.x == 0) *status = 1;
}

int main() {
    const int nx = 24, ny = 24, nz = 24, pairs = 1;
    const size_t n = (size_t)nx * ny * nz;
    std::vector<float> h(6 * n * pairs);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (float)i;
    float* d;
    cudaMalloc(&d, h.size() * 4);
    cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    typedef CUresult (*Encode)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                               const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                               CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    Encode encode = (Encode)fn;
    CUtensorMap map;
    const cuuint64_t dims[5] = {nx, ny, nz, 6, pairs};
    const cuuint64_t strides[4] = {nx * 4, (cuuint64_t)nx * ny * 4, n * 4, n * 6 * 4};
    const cuuint32_t box[5] = {40, 22, 1, 3, 1};
    const cuuint32_t es[5] = {1, 1, 1, 1, 1};
    CUresult r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, d, dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode r=%d\n", (int)r);
    float* out;
    int* st;
    cudaMalloc(&out, 40 * 22 * 3 * 4);
    cudaMalloc(&st, 4);
    const int C[6][2] = {{0, 0}, {1, 0}, {4, 0}, {0, -3}, {-4, 0}, {-3, 0}};
    for (int trial = 0; trial < 6; ++trial) {
        const int c0 = C[trial][0], c1 = C[trial][1], c2 = 5, c3 = 3, c4 = 0;
        cudaMemset(st, 0, 4);
        k<<<1, 256, 40 * 22 * 3 * 4 + 256>>>(map, out, c0, c1, c2, c3, c4, st);
        cudaError_t e = cudaDeviceSynchronize();
        int hs = 0;
        cudaMemcpy(&hs, st, 4, cudaMemcpyDeviceToHost);
        std::vector<float> ho(40 * 22 * 3);
        cudaMemcpy(ho.data(), out, ho.size() * 4, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int ch = 0; ch < 3; ++ch)
            for (int y = 0; y < 22; ++y)
                for (int x = 0; x < 40; ++x) {
                    const int gx = c0 + x, gy = c1 + y;
                    float want = 0.f;
                    if (gx >= 0 && gx < nx && gy >= 0 && gy < ny) want = h[(size_t)(c3 + ch) * n + (size_t)c2 * nx * ny + gy * nx + gx];
                    if (ho[(ch * 22 + y) * 40 + x] != want) ++bad;
                }
        printf("trial %d (x %d, y %d): err=%s status=%d mismatches=%d\n", trial, c0, c1, cudaGetErrorString(e), hs, bad);
        if (e != cudaSuccess) break;
    }
    return 0;
}
