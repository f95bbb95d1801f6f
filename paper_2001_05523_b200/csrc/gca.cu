// Green cross approximation (GCA) cluster bases on the device, one tree level
// (a batch of independent clusters) per call, fp64, sm_100a.
//
//   k_gca_columns  Green-quadrature columns of every cluster of the batch:
//                  L = [sqrt(w) * potentials | sqrt(w) * normal-derivative
//                  potentials] at the 6 m^2 Green points of the inflated
//                  cluster box (gca.green_columns; P0 panel_potentials
//                  K_VALUE / K_DN_Z, P1 p1_potentials K_DN_X / K_DN_X_DN_Z,
//                  reference src/gca.py + src/kernels.py:97-196)
//   k_gca_aca      fully pivoted cross approximation with inverse core on L
//                  (lowrank.aca_inverse_core, src/lowrank.py:154-184): largest
//                  |residual| entry (first in C order), rank-one downdate, stop
//                  when ||R||_F <= eps ||L||_F; then the interpolation matrix
//                  V = L[:, sigma] inv(L[tau, sigma]) (gca.cross_interpolate)
//
// The residual of a cluster lives in shared memory (one CTA per cluster) when
// it fits, else in a global scratch slot (L2-resident); every ACA step is one
// fused pass (downdate + Frobenius norm + argmax) and one block reduction.
#include "device_common.cuh"

namespace h2b {
namespace {

constexpr int kColThreads = 256;
constexpr int kAcaThreads = 512;
constexpr int kAcaWarps = kAcaThreads / 32;
constexpr int kGreenStride = 8;  // x, y, z, sqrt(w), nx, ny, nz, pad

// 1/r to full double precision: hardware seed + two Newton steps
__device__ __forceinline__ double inv_sqrt(double r2) {
    double t = rsqrt_seed(r2);
    t = t * fma(-0.5 * r2, t * t, 1.5);
    t = t * fma(-0.5 * r2, t * t, 1.5);
    return t;
}

template <int FLAVOR>
__global__ void __launch_bounds__(kColThreads) k_gca_columns(const double* __restrict__ P, int64_t F, int Q,
                                                             const int32_t* __restrict__ T,
                                                             const double* __restrict__ Nrm,
                                                             const int64_t* __restrict__ vt_ptr,
                                                             const int32_t* __restrict__ vt_idx,
                                                             const double* __restrict__ lam, h2b_gca_batch b,
                                                             double* __restrict__ L, int* __restrict__ flags) {
    extern __shared__ double sg[];  // k x kGreenStride
    const int c = blockIdx.x;
    const int k = b.n_green;
    const double* g = b.d_green + (int64_t)c * k * kGreenStride;
    for (int i = threadIdx.x; i < k * kGreenStride; i += blockDim.x) sg[i] = g[i];
    __syncthreads();
    const int64_t r0 = b.d_row_ptr[c];
    const int rows = (int)(b.d_row_ptr[c + 1] - r0);
    double* Lc = L + b.d_l_off[c];
    const int64_t FQ = F * Q;
    const double inv4pi = kInv4Pi;
    int bad = 0;
    for (int e = threadIdx.x; e < rows * k; e += blockDim.x) {
        const int r = e / k, j = e - r * k;
        const double zx = sg[j * kGreenStride], zy = sg[j * kGreenStride + 1], zz = sg[j * kGreenStride + 2];
        const double sw = sg[j * kGreenStride + 3];
        const double nzx = sg[j * kGreenStride + 4], nzy = sg[j * kGreenStride + 5], nzz = sg[j * kGreenStride + 6];
        double va = 0.0, vc = 0.0;
        if (FLAVOR == H2B_GCA_P0_SLP) {
            const int64_t p = b.d_rows[r0 + r];
            for (int q = 0; q < Q; ++q) {
                const int64_t gq = p * Q + q;
                const double dx = __ldg(P + gq) - zx, dy = __ldg(P + FQ + gq) - zy, dz = __ldg(P + 2 * FQ + gq) - zz;
                const double w = __ldg(P + 3 * FQ + gq);
                const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
                const double t = inv_sqrt(r2);
                const double wt = w * t;
                va = fma(wt, 1.0, va);
                // (x - z).n_z / r^3
                vc = fma(wt * (t * t), fma(dz, nzz, fma(dy, nzy, dx * nzx)), vc);
            }
        } else if (FLAVOR == H2B_GCA_P1_CURL) {
            // hat of vertex rows[r]: P0 potentials of its incident panels, each
            // weighted by the hat's (constant) surface curl on that panel
            const int v = b.d_rows[r0 + r];
            double a3[3] = {0.0, 0.0, 0.0}, c3[3] = {0.0, 0.0, 0.0};
            for (int64_t ip = vt_ptr[v]; ip < vt_ptr[v + 1]; ++ip) {
                const int p = vt_idx[ip];
                const int l = T[3 * p] == v ? 0 : (T[3 * p + 1] == v ? 1 : 2);
                double pa = 0.0, pc = 0.0;
                for (int q = 0; q < Q; ++q) {
                    const int64_t gq = (int64_t)p * Q + q;
                    const double dx = __ldg(P + gq) - zx, dy = __ldg(P + FQ + gq) - zy,
                                 dz = __ldg(P + 2 * FQ + gq) - zz;
                    const double w = __ldg(P + 3 * FQ + gq);
                    const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
                    const double t = inv_sqrt(r2);
                    const double wt = w * t;
                    pa = fma(wt, 1.0, pa);
                    pc = fma(wt * (t * t), fma(dz, nzz, fma(dy, nzy, dx * nzx)), pc);
                }
                const double* cu = lam + 3 * (3 * (int64_t)p + l);  // curls[p, l, :]
#pragma unroll
                for (int d = 0; d < 3; ++d) {
                    a3[d] = fma(cu[d], pa, a3[d]);
                    c3[d] = fma(cu[d], pc, c3[d]);
                }
            }
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                const double a = a3[d] * inv4pi * sw, cc = c3[d] * inv4pi * sw;
                if (!isfinite(a) || !isfinite(cc)) bad = 1;
                Lc[(int64_t)r * 6 * k + d * k + j] = a;
                Lc[(int64_t)r * 6 * k + (3 + d) * k + j] = cc;
            }
            continue;
        } else {
            // hat function of vertex rows[r]: incident panels, barycentric weight of its corner
            const int v = b.d_rows[r0 + r];
            for (int64_t ip = vt_ptr[v]; ip < vt_ptr[v + 1]; ++ip) {
                const int p = vt_idx[ip];
                const int l = T[3 * p] == v ? 0 : (T[3 * p + 1] == v ? 1 : 2);
                const double nax = Nrm[3 * p], nay = Nrm[3 * p + 1], naz = Nrm[3 * p + 2];
                const double nanz = fma(naz, nzz, fma(nay, nzy, nax * nzx));
                for (int q = 0; q < Q; ++q) {
                    const int64_t gq = (int64_t)p * Q + q;
                    const double dx = __ldg(P + gq) - zx, dy = __ldg(P + FQ + gq) - zy,
                                 dz = __ldg(P + 2 * FQ + gq) - zz;
                    const double w = __ldg(P + 3 * FQ + gq) * lam[3 * q + l];
                    const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
                    const double t = inv_sqrt(r2);
                    const double t3 = t * t * t;
                    const double dna = fma(dz, naz, fma(dy, nay, dx * nax));
                    const double dnz = fma(dz, nzz, fma(dy, nzy, dx * nzx));
                    va = fma(-w * t3, dna, va);
                    vc = fma(w * t3, fma(-3.0 * dna * dnz, t * t, nanz), vc);
                }
            }
        }
        const double a = va * inv4pi * sw, cc = vc * inv4pi * sw;
        if (!isfinite(a) || !isfinite(cc)) bad = 1;
        Lc[(int64_t)r * 2 * k + j] = a;
        Lc[(int64_t)r * 2 * k + k + j] = cc;
    }
    if (bad) atomicOr(flags, 1);
}

// block-wide (sum, max |v| with first index) reduction; all threads get the result
struct Red {
    double sum, best;
    long long idx;
};

__device__ __forceinline__ void red_merge(Red& a, double s, double bv, long long bi) {
    a.sum += s;
    if (bv > a.best || (bv == a.best && bi < a.idx)) {
        a.best = bv;
        a.idx = bi;
    }
}

__device__ Red block_reduce(Red v, double* rs, double* rb, long long* ri) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double s = __shfl_down_sync(0xffffffffu, v.sum, o);
        const double bv = __shfl_down_sync(0xffffffffu, v.best, o);
        const long long bi = __shfl_down_sync(0xffffffffu, v.idx, o);
        red_merge(v, s, bv, bi);
    }
    if (lane == 0) {
        rs[warp] = v.sum;
        rb[warp] = v.best;
        ri[warp] = v.idx;
    }
    __syncthreads();
    if (warp == 0) {
        Red w{0.0, -1.0, 0x7fffffffffffffffll};
        if (lane < kAcaWarps) w = Red{rs[lane], rb[lane], ri[lane]};
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double s = __shfl_down_sync(0xffffffffu, w.sum, o);
            const double bv = __shfl_down_sync(0xffffffffu, w.best, o);
            const long long bi = __shfl_down_sync(0xffffffffu, w.idx, o);
            red_merge(w, s, bv, bi);
        }
        if (lane == 0) {
            rs[kAcaWarps] = w.sum;
            rb[kAcaWarps] = w.best;
            ri[kAcaWarps] = w.idx;
        }
    }
    __syncthreads();
    Red out{rs[kAcaWarps], rb[kAcaWarps], ri[kAcaWarps]};
    __syncthreads();  // the slots are reused by the next reduction
    return out;
}

__global__ void __launch_bounds__(kAcaThreads) k_gca_aca(h2b_gca_batch b, double eps, const double* __restrict__ L,
                                                         double* __restrict__ scratch, int32_t* __restrict__ rank_out,
                                                         int32_t* __restrict__ tau_out, int32_t tau_cap,
                                                         double* __restrict__ V_out, int64_t smem_doubles) {
    extern __shared__ double sm[];
    const int c = blockIdx.x;
    const int64_t r0 = b.d_row_ptr[c];
    const int rows = (int)(b.d_row_ptr[c + 1] - r0);
    const int ncol = b.n_cols > 0 ? b.n_cols : 2 * b.n_green;
    const int64_t n = (int64_t)rows * ncol;
    const double* Lc = L + b.d_l_off[c];
    // shared layout: col[max_rows] | rowp[ncol] | red (3 x (warps+1)) | tau, sigma | R (if it fits)
    double* colb = sm;
    double* rowp = colb + b.max_rows;
    double* rs = rowp + ncol;
    double* rb = rs + kAcaWarps + 1;
    long long* ri = reinterpret_cast<long long*>(rb + kAcaWarps + 1);
    int* tau = reinterpret_cast<int*>(ri + kAcaWarps + 1);
    int* sig = tau + tau_cap;
    const int64_t head = b.max_rows + ncol + 3 * (kAcaWarps + 1) + tau_cap;
    double* R = head + n <= smem_doubles ? sm + head : scratch + b.d_l_off[c];
    const int limit = min(rows, ncol);

    // R = L, ||L||_F, first pivot
    Red acc{0.0, -1.0, 0x7fffffffffffffffll};
    for (int64_t e = threadIdx.x; e < n; e += kAcaThreads) {
        const double v = Lc[e];
        R[e] = v;
        red_merge(acc, v * v, fabs(v), e);
    }
    Red red = block_reduce(acc, rs, rb, ri);
    const double total = sqrt(red.sum);
    const double thr = eps * total;
    int k = 0;
    if (total != 0.0) {
        while (sqrt(red.sum) > thr) {
            const long long idx = red.idx;
            const int i = (int)(idx / ncol), j = (int)(idx - (long long)i * ncol);
            const double piv = R[idx];
            if (piv == 0.0 || k == limit) break;
            if (threadIdx.x == 0) {
                tau[k] = i;
                sig[k] = j;
            }
            ++k;
            for (int a = threadIdx.x; a < rows; a += kAcaThreads) colb[a] = R[(int64_t)a * ncol + j];
            for (int q = threadIdx.x; q < ncol; q += kAcaThreads) rowp[q] = R[(int64_t)i * ncol + q] / piv;
            __syncthreads();
            acc = Red{0.0, -1.0, 0x7fffffffffffffffll};
            for (int64_t e = threadIdx.x; e < n; e += kAcaThreads) {
                const int a = (int)(e / ncol), q = (int)(e - (int64_t)a * ncol);
                const double v = fma(-colb[a], rowp[q], R[e]);
                R[e] = v;
                red_merge(acc, v * v, fabs(v), e);
            }
            red = block_reduce(acc, rs, rb, ri);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) rank_out[c] = k;
    for (int r = threadIdx.x; r < k; r += kAcaThreads) tau_out[(int64_t)c * tau_cap + r] = tau[r];
    if (k == 0) return;

    // C = inv(L[tau, sigma]) in place (Gauss-Jordan, partial pivoting), in R's space (k*k <= rows*ncol)
    double* A = R;
    int* perm = reinterpret_cast<int*>(colb);  // k <= max_rows
    for (int e = threadIdx.x; e < k * k; e += kAcaThreads) {
        const int r = e / k, q = e - r * k;
        A[e] = Lc[(int64_t)tau[r] * ncol + sig[q]];
    }
    __syncthreads();
    for (int p = 0; p < k; ++p) {
        if (threadIdx.x < 32) {
            double bv = -1.0;
            int bi = p;
            for (int r = p + threadIdx.x; r < k; r += 32) {
                const double v = fabs(A[r * k + p]);
                if (v > bv) {
                    bv = v;
                    bi = r;
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double ov = __shfl_down_sync(0xffffffffu, bv, o);
                const int oi = __shfl_down_sync(0xffffffffu, bi, o);
                if (ov > bv || (ov == bv && oi < bi)) {
                    bv = ov;
                    bi = oi;
                }
            }
            if (threadIdx.x == 0) perm[p] = bi;
        }
        __syncthreads();
        const int pr = perm[p];
        if (pr != p)
            for (int q = threadIdx.x; q < k; q += kAcaThreads) {
                const double t = A[p * k + q];
                A[p * k + q] = A[pr * k + q];
                A[pr * k + q] = t;
            }
        __syncthreads();
        const double d = 1.0 / A[p * k + p];
        __syncthreads();
        for (int q = threadIdx.x; q < k; q += kAcaThreads) A[p * k + q] = (q == p ? 1.0 : A[p * k + q]) * d;
        __syncthreads();
        // eliminate column p from every other row (factors staged first)
        for (int r = threadIdx.x; r < k; r += kAcaThreads) rowp[r] = A[r * k + p];
        __syncthreads();
        for (int e = threadIdx.x; e < k * k; e += kAcaThreads) {
            const int r = e / k, q = e - r * k;
            if (r == p) continue;
            const double src = q == p ? 0.0 : A[r * k + q];
            A[r * k + q] = fma(-rowp[r], A[p * k + q], src);
        }
        __syncthreads();
    }
    // undo the row interchanges as column interchanges, last first
    for (int p = k - 1; p >= 0; --p) {
        const int pr = perm[p];
        if (pr != p)
            for (int r = threadIdx.x; r < k; r += kAcaThreads) {
                const double t = A[r * k + p];
                A[r * k + p] = A[r * k + pr];
                A[r * k + pr] = t;
            }
        __syncthreads();
    }
    // V = L[:, sigma] C  (rows x k, row-major)
    double* Vc = V_out + b.d_l_off[c];
    for (int e = threadIdx.x; e < rows * k; e += kAcaThreads) {
        const int a = e / k, q = e - a * k;
        double s = 0.0;
        for (int r = 0; r < k; ++r) s = fma(Lc[(int64_t)a * ncol + sig[r]], A[r * k + q], s);
        Vc[e] = s;
    }
}

}  // namespace
}  // namespace h2b

using namespace h2b;

extern "C" int h2b_gca_columns(const h2b_mesh* m, const double* d_panel_points, int32_t Q, const double* d_lam,
                               int flavor, const h2b_gca_batch* b, double* d_L, void* stream) {
    if (!m || !d_panel_points || !b || !d_L || Q < 1) return fail(H2B_ERR_INVALID, "h2b_gca_columns: bad argument");
    if (flavor != H2B_GCA_P0_SLP && flavor != H2B_GCA_P1_DLP)
        return fail(H2B_ERR_INVALID, "h2b_gca_columns: unknown basis flavor");
    if (flavor == H2B_GCA_P1_DLP && !d_lam) return fail(H2B_ERR_INVALID, "h2b_gca_columns: P1 needs barycentrics");
    if (b->n_clusters == 0) return ok();
    cudaStream_t st = as_stream(stream);
    int* flags;
    H2B_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&flags), sizeof(int), st));
    H2B_CUDA_TRY(cudaMemsetAsync(flags, 0, sizeof(int), st));
    const size_t sm = (size_t)b->n_green * kGreenStride * sizeof(double);
    if (flavor == H2B_GCA_P0_SLP)
        k_gca_columns<H2B_GCA_P0_SLP><<<(unsigned)b->n_clusters, kColThreads, sm, st>>>(
            d_panel_points, m->n_triangles, Q, m->d_triangles, m->d_normals, m->d_vt_ptr, m->d_vt_idx, d_lam, *b, d_L,
            flags);
    else
        k_gca_columns<H2B_GCA_P1_DLP><<<(unsigned)b->n_clusters, kColThreads, sm, st>>>(
            d_panel_points, m->n_triangles, Q, m->d_triangles, m->d_normals, m->d_vt_ptr, m->d_vt_idx, d_lam, *b, d_L,
            flags);
    H2B_CUDA_TRY(cudaGetLastError());
    int h = 0;
    H2B_CUDA_TRY(cudaMemcpyAsync(&h, flags, sizeof(int), cudaMemcpyDeviceToHost, st));
    H2B_CUDA_TRY(cudaStreamSynchronize(st));
    H2B_CUDA_TRY(cudaFreeAsync(flags, st));
    // lowrank.aca_inverse_core raises ValueError on a non-finite matrix
    if (h) return fail(H2B_ERR_INVALID, "matrix contains non-finite entries");
    return ok();
}

extern "C" int h2b_gca_columns_curl(const h2b_mesh* m, const double* d_panel_points, int32_t Q, const double* d_curls,
                                    const h2b_gca_batch* b, double* d_L, void* stream) {
    if (!m || !d_panel_points || !d_curls || !b || !d_L || Q < 1)
        return fail(H2B_ERR_INVALID, "h2b_gca_columns_curl: bad argument");
    if (b->n_clusters == 0) return ok();
    cudaStream_t st = as_stream(stream);
    int* flags;
    H2B_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&flags), sizeof(int), st));
    H2B_CUDA_TRY(cudaMemsetAsync(flags, 0, sizeof(int), st));
    const size_t sm = (size_t)b->n_green * kGreenStride * sizeof(double);
    k_gca_columns<H2B_GCA_P1_CURL><<<(unsigned)b->n_clusters, kColThreads, sm, st>>>(
        d_panel_points, m->n_triangles, Q, m->d_triangles, m->d_normals, m->d_vt_ptr, m->d_vt_idx, d_curls, *b, d_L,
        flags);
    H2B_CUDA_TRY(cudaGetLastError());
    int h = 0;
    H2B_CUDA_TRY(cudaMemcpyAsync(&h, flags, sizeof(int), cudaMemcpyDeviceToHost, st));
    H2B_CUDA_TRY(cudaStreamSynchronize(st));
    H2B_CUDA_TRY(cudaFreeAsync(flags, st));
    if (h) return fail(H2B_ERR_INVALID, "matrix contains non-finite entries");
    return ok();
}

extern "C" int h2b_gca_aca(const h2b_gca_batch* b, double eps, const double* d_L, double* d_scratch, int32_t* d_rank,
                           int32_t* d_tau, int32_t tau_cap, double* d_V, void* stream) {
    const int64_t ncol = b ? (b->n_cols > 0 ? b->n_cols : 2 * (int64_t)b->n_green) : 0;
    if (!b || !d_L || !d_scratch || !d_rank || !d_tau || !d_V || tau_cap < ncol)
        return fail(H2B_ERR_INVALID, "h2b_gca_aca: bad argument");
    if (b->n_clusters == 0) return ok();
    cudaStream_t st = as_stream(stream);
    int dev, max_optin;
    H2B_CUDA_TRY(cudaGetDevice(&dev));
    H2B_CUDA_TRY(cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    const int64_t head = b->max_rows + ncol + 3 * (kAcaWarps + 1) + tau_cap;
    // shared memory: the header plus the largest residual of the batch, capped
    int64_t want = head + (int64_t)b->max_rows * ncol;
    const int64_t cap = max_optin / (int64_t)sizeof(double);
    const int64_t smem_doubles = want < cap ? want : cap;
    if (head > smem_doubles) return fail(H2B_ERR_INVALID, "h2b_gca_aca: cluster too large");
    const size_t bytes = (size_t)smem_doubles * sizeof(double);
    H2B_CUDA_TRY(cudaFuncSetAttribute(k_gca_aca, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    k_gca_aca<<<(unsigned)b->n_clusters, kAcaThreads, bytes, st>>>(*b, eps, d_L, d_scratch, d_rank, d_tau, tau_cap,
                                                                   d_V, smem_doubles);
    H2B_CUDA_TRY(cudaGetLastError());
    return ok();
}
