// Fused vector kernels of the Jacobi-preconditioned CG solve
// (solver.cg, reference src/solver.py:22-59), fp64, sm_100a.
//
// Each call is one pass over the vectors with a deterministic reduction: a
// fixed grid of CTAs writes per-CTA partial sums in a fixed order and the
// last CTA to finish adds them up in index order, so results do not depend on
// scheduling.  Scalars stay on the device: the host reads back only the
// residual for the stopping test.  With row-sharded vectors the host
// all-reduces the 1-2 scalars each call produces between calls.
#include "device_common.cuh"

namespace h2b {
namespace {

constexpr int kCgThreads = 256;
constexpr int kCgBlocks = 2 * 148;

template <int N>
__device__ void finish(double (&v)[N], double* partial, unsigned int* ticket, double* out) {
    __shared__ double red[N][kCgThreads / 32];
    __shared__ bool last;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int i = 0; i < N; ++i) {
        double s = v[i];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
        if (lane == 0) red[i][warp] = s;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll
        for (int i = 0; i < N; ++i) {
            double s = 0.0;
            for (int w = 0; w < kCgThreads / 32; ++w) s += red[i][w];
            partial[(int64_t)blockIdx.x * N + i] = s;
        }
        __threadfence();
        last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
        __threadfence();
#pragma unroll
        for (int i = 0; i < N; ++i) {
            double s = 0.0;
            for (unsigned b = 0; b < gridDim.x; ++b) s += __ldcg(partial + (int64_t)b * N + i);
            out[i] = s;
        }
        *ticket = 0u;  // ready for the next call
    }
}

__global__ void __launch_bounds__(kCgThreads) k_dot(const double* __restrict__ a, const double* __restrict__ b,
                                                    int64_t n, double* partial, unsigned int* ticket, double* out) {
    double v[1] = {0.0};
    for (int64_t i = (int64_t)blockIdx.x * kCgThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kCgThreads)
        v[0] = fma(a[i], b[i], v[0]);
    finish<1>(v, partial, ticket, out);
}

// alpha = rz / pAp; x += alpha p; r -= alpha Ap; z = D^-1 r; out = (r.z, r.r)
__global__ void __launch_bounds__(kCgThreads) k_step(int64_t n, const double* __restrict__ scal,
                                                     double* __restrict__ x, double* __restrict__ r,
                                                     const double* __restrict__ p, const double* __restrict__ Ap,
                                                     const double* __restrict__ inv_d, double* __restrict__ z,
                                                     double* partial, unsigned int* ticket, double* out) {
    const double alpha = scal[0] / scal[1];
    double v[2] = {0.0, 0.0};
    for (int64_t i = (int64_t)blockIdx.x * kCgThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kCgThreads) {
        x[i] = fma(alpha, p[i], x[i]);
        const double ri = fma(-alpha, Ap[i], r[i]);
        r[i] = ri;
        const double zi = inv_d ? ri * inv_d[i] : ri;
        if (inv_d) z[i] = zi;
        v[0] = fma(ri, zi, v[0]);
        v[1] = fma(ri, ri, v[1]);
    }
    finish<2>(v, partial, ticket, out);
}

// p = z + (rz_new / rz_old) p with scal = (rz_old, pAp, rz_new, r.r)
__global__ void __launch_bounds__(kCgThreads) k_direction(int64_t n, const double* __restrict__ scal,
                                                          const double* __restrict__ z, double* __restrict__ p) {
    const double beta = scal[2] / scal[0];
    for (int64_t i = (int64_t)blockIdx.x * kCgThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kCgThreads)
        p[i] = fma(beta, p[i], z[i]);
}

}  // namespace
}  // namespace h2b

using namespace h2b;

extern "C" int h2b_cg_workspace_size(int64_t* bytes) {
    if (!bytes) return fail(H2B_ERR_INVALID, "h2b_cg_workspace_size: bad argument");
    *bytes = (int64_t)kCgBlocks * 2 * sizeof(double) + 256;
    return ok();
}

extern "C" int h2b_cg_dot(const double* d_a, const double* d_b, int64_t n, void* d_work, double* d_out,
                          void* stream) {
    if (!d_a || !d_b || !d_work || !d_out || n < 0) return fail(H2B_ERR_INVALID, "h2b_cg_dot: bad argument");
    auto* ticket = reinterpret_cast<unsigned int*>(d_work);
    double* partial = reinterpret_cast<double*>(reinterpret_cast<char*>(d_work) + 256);
    k_dot<<<kCgBlocks, kCgThreads, 0, as_stream(stream)>>>(d_a, d_b, n, partial, ticket, d_out);
    H2B_CUDA_TRY(cudaGetLastError());
    return ok();
}

extern "C" int h2b_cg_step(int64_t n, const double* d_scal, double* d_x, double* d_r, const double* d_p,
                           const double* d_Ap, const double* d_inv_diag, double* d_z, void* d_work, double* d_out,
                           void* stream) {
    if (!d_scal || !d_x || !d_r || !d_p || !d_Ap || !d_work || !d_out || (d_inv_diag && !d_z) || n < 0)
        return fail(H2B_ERR_INVALID, "h2b_cg_step: bad argument");
    auto* ticket = reinterpret_cast<unsigned int*>(d_work);
    double* partial = reinterpret_cast<double*>(reinterpret_cast<char*>(d_work) + 256);
    k_step<<<kCgBlocks, kCgThreads, 0, as_stream(stream)>>>(n, d_scal, d_x, d_r, d_p, d_Ap, d_inv_diag, d_z,
                                                            partial, ticket, d_out);
    H2B_CUDA_TRY(cudaGetLastError());
    return ok();
}

extern "C" int h2b_cg_direction(int64_t n, const double* d_scal, const double* d_z, double* d_p, void* stream) {
    if (!d_scal || !d_z || !d_p || n < 0) return fail(H2B_ERR_INVALID, "h2b_cg_direction: bad argument");
    k_direction<<<kCgBlocks, kCgThreads, 0, as_stream(stream)>>>(n, d_scal, d_z, d_p);
    H2B_CUDA_TRY(cudaGetLastError());
    return ok();
}
