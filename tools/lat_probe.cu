// Micro-probe: dependent-chain latencies (cycles) of DFMA, LDS.64, SHFL (f64)
// and DFMA issue throughput per warp, on one SM.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, int n) {
    __shared__ double sm[1024];
    __shared__ int idx[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) { sm[i] = 1.0 + i * 1e-9; idx[i] = (i + 33) & 1023; }
    __syncthreads();
    double a = out[0], b = 1.0000001, c = 1e-9;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) a = fma(a, b, c);
    long long t1 = clock64();
    int j = threadIdx.x;
    for (int i = 0; i < n; ++i) j = idx[j];
    long long t2 = clock64();
    double s = sm[j];
    for (int i = 0; i < n; ++i) s = __shfl_xor_sync(0xffffffffu, s, 1) + 1.0;
    long long t3 = clock64();
    double x0 = a, x1 = a + 1, x2 = a + 2, x3 = a + 3, x4 = a + 4, x5 = a + 5, x6 = a + 6, x7 = a + 7;
    for (int i = 0; i < n; ++i) {
        x0 = fma(x0, b, c); x1 = fma(x1, b, c); x2 = fma(x2, b, c); x3 = fma(x3, b, c);
        x4 = fma(x4, b, c); x5 = fma(x5, b, c); x6 = fma(x6, b, c); x7 = fma(x7, b, c);
    }
    long long t4 = clock64();
    double q = 0;
    for (int i = 0; i < n; ++i) q += sm[(threadIdx.x + i * 32) & 1023];
    long long t5 = clock64();
    if (threadIdx.x == 0) {
        cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4;
    }
    out[1 + threadIdx.x] = a + j + s + x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7 + q;
}
int main() {
    double* out; long long* cyc; cudaMalloc(&out, 8 * 2048); cudaMalloc(&cyc, 64);
    cudaMemset(out, 0, 8 * 2048);
    const int n = 4096;
    for (int warps = 1; warps <= 16; warps *= 4) {
        k<<<1, 32 * warps>>>(out, cyc, n);
        cudaDeviceSynchronize();
        long long h[5]; cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
        printf("warps/CTA %2d: DFMA dep %.1f  LDS dep %.1f  SHFL+DADD dep %.1f  8xDFMA/iter %.1f  LDS+DADD %.1f cycles\n",
               warps, h[0] / (double)n, h[1] / (double)n, h[2] / (double)n, h[3] / (double)n, h[4] / (double)n);
    }
    return 0;
}
