// Throughput probes on this GPU (inform the precision / staging design):
// fp32 vs fp64 FMA rate, fp32 -> fp64 conversion rate, shared-memory
// double loads.
#include <cstdio>
template <class T>
__global__ void k(T* out, int iters) {
    T a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    const T b = (T)1.0000001, c = (T)0.0000001;
    for (int i = 0; i < iters; ++i) {
        a0 = a0 * b + c; a1 = a1 * b + c; a2 = a2 * b + c; a3 = a3 * b + c;
        a4 = a4 * b + c; a5 = a5 * b + c; a6 = a6 * b + c; a7 = a7 * b + c;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
// 8 independent fp32 -> fp64 conversions per iteration (plus one fp32 add
// each to defeat hoisting and one DADD to consume the result)
__global__ void kcvt(double* out, int iters) {
    float f[8];
    double acc[8];
    for (int j = 0; j < 8; ++j) { f[j] = threadIdx.x + j; acc[j] = 0.0; }
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            acc[j] += (double)f[j];
            f[j] += 1.0f;
        }
    }
    double s = 0.0;
    for (int j = 0; j < 8; ++j) s += acc[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <class T>
void run(const char* name) {
    T* d; const int blocks = 148 * 8, threads = 256, iters = 4096;
    cudaMalloc(&d, sizeof(T) * blocks * threads);
    k<T><<<blocks, threads>>>(d, 16);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<T><<<blocks, threads>>>(d, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * iters * (double)blocks * threads;
    printf("%s: %.1f TFLOP/s (FMA=2)\n", name, flops / ms / 1e9);
    cudaFree(d);
}
void run_cvt() {
    double* d; const int blocks = 148 * 8, threads = 256, iters = 4096;
    cudaMalloc(&d, sizeof(double) * blocks * threads);
    kcvt<<<blocks, threads>>>(d, 16);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    kcvt<<<blocks, threads>>>(d, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double n = 8.0 * iters * (double)blocks * threads;
    printf("F2F.F64.F32 (+DADD +FADD each): %.2f G/s = %.1f per clk per SM at 1.965 GHz\n", n / ms / 1e6,
           n / (ms * 1e-3) / 148 / 1.965e9);
    cudaFree(d);
}
int main() {
    run<float>("fp32");
    run<double>("fp64");
    run_cvt();
    return 0;
}
