// Micro-probe: __nanosleep granularity and the inter-CTA round trip of the
// matvec's LL hand-off (st.relaxed.gpu / ld.relaxed.gpu polling), CTA 0 <-> CTA 1
// (on different SMs), 1000 ping-pongs.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void st_rel(uint64_t* p, uint64_t v) {
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_rel(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__global__ void k_sleep(long long* out, int ns) {
    long long t0 = clock64();
    for (int i = 0; i < 1000; ++i) __nanosleep(ns);
    long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = (t1 - t0) / 1000;
}

__global__ void k_pingpong(uint64_t* flags, long long* out, int iters, int sleep_ns) {
    if (threadIdx.x != 0) return;
    uint64_t* mine = flags + 32 * blockIdx.x;
    uint64_t* other = flags + 32 * (1 - blockIdx.x);
    long long t0 = clock64();
    for (int i = 1; i <= iters; ++i) {
        if (blockIdx.x == 0) {
            st_rel(mine, i);
            while (ld_rel(other) != (uint64_t)i)
                if (sleep_ns) __nanosleep(sleep_ns);
        } else {
            while (ld_rel(other) != (uint64_t)i)
                if (sleep_ns) __nanosleep(sleep_ns);
            st_rel(mine, i);
        }
    }
    long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = (t1 - t0) / iters;
}

int main2();
int main() {
    main2();
    long long* out;
    uint64_t* flags;
    cudaMalloc(&out, 64);
    cudaMalloc(&flags, 4096);
    for (int ns : {0, 20, 32, 100, 500}) {
        k_sleep<<<1, 32>>>(out, ns);
        cudaDeviceSynchronize();
        long long h;
        cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
        printf("nanosleep(%d): %lld cycles\n", ns, h);
    }
    for (int ns : {0, 32, 100}) {
        cudaMemset(flags, 0, 4096);
        k_pingpong<<<2, 32>>>(flags, out, 1000, ns);
        cudaError_t e = cudaDeviceSynchronize();
        long long h;
        cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
        printf("LL ping-pong round trip (sleep %d): %lld cycles (%s)\n", ns, h, cudaGetErrorString(e));
    }
    return 0;
}
// (appended) globaltimer resolution
__global__ void k_gt(unsigned long long* out) {
    unsigned long long prev, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(prev));
    int n = 0;
    long long c0 = clock64();
    while (n < 8) {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t != prev) { out[n++] = t - prev; prev = t; }
    }
    out[8] = clock64() - c0;
}
int main2() {
    unsigned long long* d; cudaMalloc(&d, 16 * 8);
    k_gt<<<1, 1>>>(d); cudaDeviceSynchronize();
    unsigned long long h[9]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("globaltimer deltas (ns):"); for (int i = 0; i < 8; ++i) printf(" %llu", h[i]); printf("  (%llu cycles for 8 ticks)\n", h[8]);
    return 0;
}
