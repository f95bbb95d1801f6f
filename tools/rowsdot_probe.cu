// Micro-probe: cycles of the matvec band product (16-row register blocking,
// 128-thread group) with operands in shared memory, one CTA per SM, no other
// traffic.  Usage: rowsdot_probe rows cols
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <cstdint>

constexpr int kGT = 128, kGW = 4; // probe CTA = one 128-thread group (launch with 128)
__device__ __forceinline__ void gsync() { asm volatile("bar.sync 1, %0;" :: "r"((int)blockDim.x) : "memory"); }

__device__ __forceinline__ double warp_sum16(double (&a)[16], int lane) {
#pragma unroll
    for (int h = 8, o = 16; h >= 1; h >>= 1, o >>= 1) {
        const bool up = lane & o;
#pragma unroll
        for (int i = 0; i < h; ++i) {
            const double send = up ? a[i] : a[i + h], keep = up ? a[i + h] : a[i];
            a[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
    }
    return a[0] + __shfl_xor_sync(0xffffffffu, a[0], 1);
}


__device__ __forceinline__ double lds(uint32_t a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}

template <int N>
__device__ __forceinline__ double warp_sumN(double (&a)[N], int lane) {
    int o = 16;
#pragma unroll
    for (int h = N / 2; h >= 1; h >>= 1, o >>= 1) {
        const bool up = lane & o;
#pragma unroll
        for (int i = 0; i < h; ++i) {
            const double send = up ? a[i] : a[i + h], keep = up ? a[i + h] : a[i];
            a[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
    }
    double v = a[0];
    for (; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

template <int N>
__device__ __forceinline__ void chunkN(uint32_t M, int ld, int r0, int nr, int cols, uint32_t v, double* red,
                                       double* out) {
    const int t = threadIdx.x & 127, warp = t >> 5, lane = t & 31;
    uint32_t a[N];
#pragma unroll
    for (int i = 0; i < N; ++i) a[i] = M + 8u * (uint32_t)((r0 + min(i, nr - 1)) * ld + t);
    uint32_t av = v + 8u * t;
    double acc[N];
#pragma unroll
    for (int i = 0; i < N; ++i) acc[i] = 0.0;
    for (int c = t; c < cols; c += 128) {
        const double vc = lds(av);
        double m[N];
#pragma unroll
        for (int i = 0; i < N; ++i) m[i] = lds(a[i]);
#pragma unroll
        for (int i = 0; i < N; ++i) acc[i] = fma(m[i], vc, acc[i]);
        av += 1024u;
#pragma unroll
        for (int i = 0; i < N; ++i) a[i] += 1024u;
    }
    const double sum = warp_sumN<N>(acc, lane);
    constexpr int sh = N == 16 ? 1 : N == 8 ? 2 : N == 4 ? 3 : N == 2 ? 4 : 5;
    if ((lane & ((1 << sh) - 1)) == 0) red[warp * 16 + (lane >> sh)] = sum;
}

__device__ void rows_dot16(const double* M, int ld, int rows, int cols, const double* v, double* red, double* out) {
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    const int ri = ((lane >> 1) & 8) | ((lane >> 1) & 4) | ((lane >> 1) & 2) | ((lane >> 1) & 1);
    for (int r0 = 0; r0 < rows; r0 += 16) {
        const int nr = min(16, rows - r0);
        double acc[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i] = 0.0;
        const double* m0 = M + (long)r0 * ld;
        for (int c = t; c < cols; c += kGT) {
            const double vc = v[c];
#pragma unroll
            for (int i = 0; i < 16; ++i)
                if (i < nr) acc[i] = fma(m0[(long)i * ld + c], vc, acc[i]);
        }
        const double sum = warp_sum16(acc, lane);
        if ((lane & 1) == 0) red[warp * 16 + ri] = sum;
        gsync();
        if (t < nr) {
            double s = 0.0;
            for (int w = 0; w < kGW; ++w) s += red[w * 16 + t];
            out[r0 + t] = s;
        }
        gsync();
    }
}

__device__ void rows_dot_warp(const double* M, int ld, int rows, int cols, const double* v, double* out) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int r = warp; r < rows; r += kGW) {
        const double* row = M + (long)r * ld;
        double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
        int c = lane;
        for (; c + 96 < cols; c += 128) {
            a0 = fma(row[c], v[c], a0); a1 = fma(row[c + 32], v[c + 32], a1);
            a2 = fma(row[c + 64], v[c + 64], a2); a3 = fma(row[c + 96], v[c + 96], a3);
        }
        for (; c < cols; c += 32) a0 = fma(row[c], v[c], a0);
        double s = (a0 + a1) + (a2 + a3);
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) out[r] = s;
    }
    gsync();
}


__device__ void rows_dotS(const double* Mp, int ld, int rows, int cols, const double* vp, double* red, double* out) {
    const uint32_t M = (uint32_t)__cvta_generic_to_shared(Mp), v = (uint32_t)__cvta_generic_to_shared(vp);
    const int t = threadIdx.x & 127;
    for (int r0 = 0; r0 < rows; r0 += 16) {
        const int nr = min(16, rows - r0);
        if (nr > 8) chunkN<16>(M, ld, r0, nr, cols, v, red, out);
        else if (nr > 4) chunkN<8>(M, ld, r0, nr, cols, v, red, out);
        else if (nr > 2) chunkN<4>(M, ld, r0, nr, cols, v, red, out);
        else chunkN<2>(M, ld, r0, nr, cols, v, red, out);
        gsync();
        if (t < nr) {
            double s = 0.0;
            for (int w = 0; w < kGW; ++w) s += red[w * 16 + t];
            out[r0 + t] = s;
        }
        gsync();
    }
}


// warp per row, 16-byte shared loads (double2), 4 independent accumulators
__device__ void rows_dot_warp2(const double* M, int ld, int rows, int cols, const double* v, double* out) {
    const int warp = (threadIdx.x & 127) >> 5, lane = threadIdx.x & 31;
    const double2* v2 = reinterpret_cast<const double2*>(v);
    const int c2 = cols >> 1;  // cols even
    for (int r = warp; r < rows; r += kGW) {
        const double2* row = reinterpret_cast<const double2*>(M + (long)r * ld);
        double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
        int c = lane;
        for (; c + 32 < c2; c += 64) {
            const double2 m0 = row[c], m1 = row[c + 32], x0 = v2[c], x1 = v2[c + 32];
            a0 = fma(m0.x, x0.x, a0); a1 = fma(m0.y, x0.y, a1);
            a2 = fma(m1.x, x1.x, a2); a3 = fma(m1.y, x1.y, a3);
        }
        if (c < c2) {
            const double2 m0 = row[c], x0 = v2[c];
            a0 = fma(m0.x, x0.x, a0); a1 = fma(m0.y, x0.y, a1);
        }
        double s = (a0 + a1) + (a2 + a3);
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) out[r] = s;
    }
    gsync();
}

__global__ void k(int rows, int cols, int reps, int mode, long long* cyc, double* sink) {
    extern __shared__ double sm[];
    double* M = sm;
    double* v = M + rows * cols;
    double* red = v + cols;
    double* out = red + 128;
    for (int i = threadIdx.x; i < rows * cols; i += blockDim.x) M[i] = 1.0 / (i + 1);
    for (int i = threadIdx.x; i < cols; i += blockDim.x) v[i] = 1.0 + i;
    gsync();
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        if (mode == 0) rows_dot16(M, cols, rows, cols, v, red, out);
        else if (mode == 1) rows_dot_warp(M, cols, rows, cols, v, out);
        else if (mode == 2) rows_dotS(M, cols, rows, cols, v, red, out);
        else rows_dot_warp2(M, cols, rows, cols, v, out);
        if (threadIdx.x == 0) v[0] += out[0] * 1e-30;
        gsync();
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { cyc[blockIdx.x] = t1 - t0; sink[blockIdx.x] = out[0]; }
}

int main(int argc, char** argv) {
    int rows = argc > 1 ? atoi(argv[1]) : 9, cols = argc > 2 ? atoi(argv[2]) : 420;
    const int reps = 200;
    const int nthr = argc > 3 ? atoi(argv[3]) : 128;
    long long* cyc; double* sink;
    cudaMalloc(&cyc, 148 * 8); cudaMalloc(&sink, 148 * 8);
    size_t smem = 8 * (rows * cols + cols + 128 + rows + 16);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int mode = 0; mode < 4; ++mode) {
        k<<<148, nthr, smem>>>(rows, cols, reps, mode, cyc, sink);
        cudaError_t e = cudaDeviceSynchronize();
        long long h[148]; cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
        printf("rows %d cols %d mode %s: %.0f cycles per band (%s)\n", rows, cols, mode == 3 ? "warp-row2" : mode == 2 ? "lds-chunk" : mode ? "warp-row" : "16-row",
               (double)h[0] / reps, cudaGetErrorString(e));
    }
    return 0;
}
