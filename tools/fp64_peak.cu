// fp64 FMA throughput microbenchmark (roofline denominator for the sweep kernels):
// each thread runs CH independent DFMA chains; sweep warps per SM and chains per thread.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak tools/fp64_peak.cu && ./fp64_peak
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
    double x[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 1e-3 + c;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) x[c] = fma(x[c], a, b);
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += x[c];
    if (s == 12345.678) out[threadIdx.x] = s;
}

template <int CH>
void run(int warps_per_sm, double* d) {
    const int threads = 32 * warps_per_sm;
    const int iters = 4096;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    dfma_kernel<CH><<<148, threads>>>(d, iters, 0.999999, 1e-7);
    cudaEventRecord(e0);
    dfma_kernel<CH><<<148, threads>>>(d, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fma = 148.0 * threads * (double)iters * CH;
    printf("chains %2d warps/SM %2d : %.2f TFMA/s = %.2f TFLOP/s\n", CH, warps_per_sm, fma / ms / 1e9, 2 * fma / ms / 1e9);
}

int main() {
    double* d;
    cudaMalloc(&d, 1 << 20);
    for (int w : {4, 8, 16, 32}) run<8>(w, d);
    for (int w : {4, 8, 16, 32}) run<32>(w, d);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("clock %d kHz\n", clk);
    return 0;
}
