// Micro-probe: per-SM throughput (ops / clock) of rsqrt.approx.ftz.f64
// (MUFU.RSQ64H), rsqrt.approx.ftz.f32 (MUFU.RSQ), cvt.rn.f32.f64 and DFMA, with
// 8 independent chains per thread and full occupancy.
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void k(double* out, int iters, long long* cyc) {
    double d[8];
    float f[8];
    for (int i = 0; i < 8; ++i) { d[i] = 1.0 + 1e-3 * (threadIdx.x + i); f[i] = (float)d[i]; }
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (OP == 0) { double y; asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d[i])); d[i] = y; }
            if (OP == 1) { float y; asm volatile("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(f[i])); f[i] = y; }
            if (OP == 2) { float y; asm volatile("cvt.rn.f32.f64 %0, %1;" : "=f"(y) : "d"(d[i])); d[i] = (double)y + 1.0; }
            if (OP == 3) d[i] = fma(d[i], 1.0000001, 1e-9);
        }
    }
    long long t1 = clock64();
    double s = 0;
    for (int i = 0; i < 8; ++i) s += d[i] + f[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

int main() {
    double* out; long long* cyc;
    cudaMalloc(&out, 148 * 8 * 1024 * 8); cudaMalloc(&cyc, 8);
    const int iters = 4096, blocks = 148 * 4, threads = 512;
    const char* names[] = {"rsqrt.f64 (MUFU.RSQ64H)", "rsqrt.f32 (MUFU.RSQ)", "cvt f64->f32 (+DADD)", "DFMA"};
    for (int op = 0; op < 4; ++op) {
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        auto launch = [&]() {
            if (op == 0) k<0><<<blocks, threads>>>(out, iters, cyc);
            if (op == 1) k<1><<<blocks, threads>>>(out, iters, cyc);
            if (op == 2) k<2><<<blocks, threads>>>(out, iters, cyc);
            if (op == 3) k<3><<<blocks, threads>>>(out, iters, cyc);
        };
        launch(); cudaDeviceSynchronize();
        cudaEventRecord(a); launch(); cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        const double ops = (double)blocks * threads * iters * 8;
        int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
        printf("%-26s %8.3f ms  %7.1f Gop/s  %5.2f ops/clk/SM (at %d MHz)\n", names[op], ms, ops / ms / 1e6,
               ops / (ms * 1e-3) / 148 / (clk * 1e3), clk / 1000);
    }
    return 0;
}
