// FP64 microbenchmarks for the roofline denominator (not in MEASURED_PEAKS.json):
//   1. DFMA peak: independent FMA chains, all SMs, CUDA-event timed.
//   2. rsqrt.approx.ftz.f64 seed accuracy over a log-uniform sweep, and the
//      error after the one-step Newton correction used by the quadrature kernels.
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>

__global__ void dfma_peak(double* out, int iters, double a, double b) {
    double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
            x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__device__ __forceinline__ double seed(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    return y;
}

__global__ void rsqrt_err(double* err, long n) {
    long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
    double e0 = 0, e1 = 0;
    for (; i < n; i += (long)gridDim.x * blockDim.x) {
        double x = exp2(-60.0 + 120.0 * (double)i / (double)n) * (1.0 + 0.37 * ((i * 2654435761L) % 1000) / 1000.0);
        double t = seed(x);
        double exact = 1.0 / sqrt(x);
        e0 = fmax(e0, fabs(t - exact) / exact);
        double s = t * t;
        double c = fma(-x, s, 3.0);
        double y1 = 0.5 * t * c;
        e1 = fmax(e1, fabs(y1 - exact) / exact);
    }
    atomicMax((unsigned long long*)&err[0], __double_as_longlong(e0));
    atomicMax((unsigned long long*)&err[1], __double_as_longlong(e1));
}

int main() {
    int dev = 0, sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    double* out;
    cudaMalloc(&out, sizeof(double) * sms * 8 * 256);
    const int iters = 4096;
    dfma_peak<<<sms * 8, 256>>>(out, 64, 1.0000001, 1e-9);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    double best = 0;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(a);
        dfma_peak<<<sms * 8, 256>>>(out, iters, 1.0000001, 1e-9);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        double flops = 2.0 * 8 * 16 * (double)iters * sms * 8 * 256;
        best = fmax(best, flops / (ms * 1e-3) / 1e12);
    }
    double* err;
    cudaMalloc(&err, 2 * sizeof(double));
    cudaMemset(err, 0, 2 * sizeof(double));
    rsqrt_err<<<sms * 4, 256>>>(err, 1L << 26);
    double h[2];
    cudaMemcpy(h, err, sizeof(h), cudaMemcpyDeviceToHost);
    printf("{\"fp64_dfma_tflops\": %.3f, \"sms\": %d, \"rsqrt_seed_max_rel_err\": %.3e, \"rsqrt_newton1_max_rel_err\": %.3e}\n",
           best, sms, h[0], h[1]);
    return 0;
}
