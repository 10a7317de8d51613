// Throughput probe: fp64 vs fp32 FMA rate on this GPU (informs the LNCC precision design).
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
int main() { run<float>("fp32"); run<double>("fp64"); return 0; }
