// Multi-right-hand-side H^2 product Y = A X (X: n_cols x nrhs, nrhs <= 16),
// fp64, sm_100a.  The reference has only the single-vector H2Matrix.matvec
// (src/containers.py:254-270); this applies the same operator -- the same packed
// V / E / S / D arrays and gather lists as the matvec plan -- to a block of
// vectors, so every operator byte streamed from HBM serves nrhs columns.
//
// Every dense product is C (M x R) += A (M x K) B (K x R) with R = 8 or 16
// padded right-hand sides, computed on the FP64 tensor cores:
// mma.sync.m8n8k4.f64 (one 8-row tile per warp, B staged in shared memory).
// Level-synchronous, one launch per stage / tree level:
//   k_mm_fwd_leaf    x_hat_t = V_t^T X|_t                (ClusterBasis.forward, leaves)
//   k_mm_fwd_level   x_hat_p = sum_c E_c^T x_hat_c        (ClusterBasis.forward, upward)
//   k_mm_cpl         y_cpl_t = S_t x_hat|far(t)          (coupling loop)
//   k_mm_bwd_level   v_t = y_cpl_t + E_t v_parent         (ClusterBasis.backward)
//   k_mm_leaf        Y|_t = D_t X|near(t) + V_t v_t       (nearfield loop + leaf expansion)
// Each output entry is produced by one lane in a fixed order: deterministic.
#include <algorithm>
#include <vector>

#include "device_common.cuh"

struct h2b_mmplan {
    h2b_layout L;
    int max_depth_c, max_depth_r;
    int32_t* d_lists;  // all task lists (device)
    std::vector<int64_t> fwd_level_off, bwd_level_off;  // into the lists, per level
    int64_t off_leaf_c, n_leaf_c, off_fwd, off_cpl, n_cpl, off_bwd, off_leaf_r, n_leaf_r;
    int max_c_node;  // largest sum of child ranks (B staging)
    double* xhat;    // xhat_len x 16
    double* ycpl;    // yhat_len x 16
    double* v;       // yhat_len x 16
};

namespace h2b {
namespace {

constexpr int kMmThreads = 256;
constexpr int kMmWarps = kMmThreads / 32;
constexpr int kChunk = 128;  // staged B rows per chunk (gathered right-hand sides)

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

// acc += A[m0:m0+8, k0:k1] B[k0:k1, :] for one warp; fa(m, k) reads A, B is
// staged in shared memory as [k - kb][R] (kb = first staged row).
template <int NT, class FA>
__device__ __forceinline__ void warp_mma(double (&acc)[NT][2], int m0, int M, int k0, int k1, int kb, FA fa,
                                         const double* Bs) {
    constexpr int R = 8 * NT;
    const int lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
    const bool rowok = m0 + g < M;
    int k = k0;
    for (; k + 32 <= k1; k += 32) {
        double a[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) a[u] = rowok ? fa(m0 + g, k + 4 * u + q) : 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int t = 0; t < NT; ++t) dmma(acc[t], a[u], Bs[(k + 4 * u + q - kb) * R + 8 * t + g]);
    }
    for (; k < k1; k += 4) {
        const int kk = k + q;
        const double a = (rowok && kk < k1) ? fa(m0 + g, kk) : 0.0;
#pragma unroll
        for (int t = 0; t < NT; ++t) dmma(acc[t], a, kk < k1 ? Bs[(kk - kb) * R + 8 * t + g] : 0.0);
    }
}

// streaming operand loads (read once): no L1 allocation
__device__ __forceinline__ double ld_stream(const double* p) {
    double v;
    asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}

template <int NT>
__device__ __forceinline__ void zero(double (&acc)[NT][2]) {
#pragma unroll
    for (int t = 0; t < NT; ++t) acc[t][0] = acc[t][1] = 0.0;
}

// store C rows m0 + g, columns 2q, 2q+1 of each n-tile: out(m, n, value)
template <int NT, class FO>
__device__ __forceinline__ void warp_store(const double (&acc)[NT][2], int m0, int M, FO out) {
    const int lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
    if (m0 + g >= M) return;
#pragma unroll
    for (int t = 0; t < NT; ++t) {
        out(m0 + g, 8 * t + 2 * q, acc[t][0]);
        out(m0 + g, 8 * t + 2 * q + 1, acc[t][1]);
    }
}

// ---- forward transform ------------------------------------------------------

template <int NT>
__global__ void __launch_bounds__(kMmThreads) k_mm_fwd_leaf(h2b_layout L, const int32_t* __restrict__ leaves,
                                                            const double* __restrict__ X, int nrhs,
                                                            double* __restrict__ xhat) {
    constexpr int R = 8 * NT;
    extern __shared__ double Bs[];
    const int t = leaves[blockIdx.x];
    const int start = L.c_start[t], size = L.c_size[t], k = L.c_rank[t];
    const double* V = L.c_V + L.c_v_off[t];
    for (int e = threadIdx.x; e < size * R; e += kMmThreads) {
        const int i = e / R, r = e - i * R;
        Bs[e] = r < nrhs ? X[L.col_perm[start + i] * nrhs + r] : 0.0;
    }
    __syncthreads();
    double* out = xhat + L.c_xhat_off[t] * R;
    const int warp = threadIdx.x >> 5;
    for (int m0 = 8 * warp; m0 < k; m0 += 8 * kMmWarps) {
        double acc[NT][2];
        zero(acc);
        warp_mma<NT>(acc, m0, k, 0, size, 0, [&](int m, int kk) { return V[(int64_t)kk * k + m]; }, Bs);
        warp_store<NT>(acc, m0, k, [&](int m, int n, double v) { out[m * R + n] = v; });
    }
}

template <int NT>
__global__ void __launch_bounds__(kMmThreads) k_mm_fwd_level(h2b_layout L, const int32_t* __restrict__ nodes,
                                                             double* __restrict__ xhat) {
    constexpr int R = 8 * NT;
    extern __shared__ double Bs[];
    const int p = nodes[blockIdx.x];
    const int kp = L.c_rank[p];
    const int c0 = L.c_child[2 * p], c1 = L.c_child[2 * p + 1];
    const int k0 = L.c_rank[c0], k1 = L.c_rank[c1];
    // B = [x_hat_c0; x_hat_c1] ((k0 + k1) x R), A = [E_c0^T, E_c1^T] (kp x (k0 + k1))
    for (int e = threadIdx.x; e < (k0 + k1) * R; e += kMmThreads) {
        const int i = e / R, r = e - i * R;
        Bs[e] = i < k0 ? xhat[(L.c_xhat_off[c0] + i) * R + r] : xhat[(L.c_xhat_off[c1] + i - k0) * R + r];
    }
    __syncthreads();
    const double* E0 = L.c_E + L.c_e_off[c0];
    const double* E1 = L.c_E + L.c_e_off[c1];
    double* out = xhat + L.c_xhat_off[p] * R;
    const int warp = threadIdx.x >> 5;
    for (int m0 = 8 * warp; m0 < kp; m0 += 8 * kMmWarps) {
        double acc[NT][2];
        zero(acc);
        warp_mma<NT>(acc, m0, kp, 0, k0, 0, [&](int m, int kk) { return E0[(int64_t)kk * kp + m]; }, Bs);
        warp_mma<NT>(acc, m0, kp, k0, k0 + k1, 0,
                     [&](int m, int kk) { return E1[(int64_t)(kk - k0) * kp + m]; }, Bs);
        warp_store<NT>(acc, m0, kp, [&](int m, int n, double v) { out[m * R + n] = v; });
    }
}

// ---- streamed products: couplings and nearfield -------------------------------
// C (M x R) = A (M x K, row-major, ld) B where B row kk = src[idx[kk]] (R wide,
// or nrhs wide from X when x_src); K staged in chunks of kChunk rows.
template <int NT>
__device__ void streamed_rows(double (&acc)[NT][2], int m0, int M, const double* A, int64_t ld, int K,
                              const int32_t* idx, const double* src, int src_w, int nrhs, double* Bs) {
    constexpr int R = 8 * NT;
    for (int kc = 0; kc < K; kc += kChunk) {
        const int kn = min(kChunk, K - kc);
        __syncthreads();
        for (int e = threadIdx.x; e < kn * R; e += kMmThreads) {
            const int i = e / R, r = e - i * R;
            Bs[e] = r < nrhs ? src[(int64_t)idx[kc + i] * src_w + r] : 0.0;
        }
        __syncthreads();
        if (m0 < M)
            warp_mma<NT>(acc, m0, M, kc, kc + kn, kc, [&](int m, int kk) { return ld_stream(A + (int64_t)m * ld + kk); },
                         Bs);
    }
}

template <int NT>
__global__ void __launch_bounds__(kMmThreads) k_mm_cpl(h2b_layout L, const int32_t* __restrict__ nodes,
                                                       const double* __restrict__ xhat, double* __restrict__ ycpl) {
    constexpr int R = 8 * NT;
    extern __shared__ double Bs[];
    const int t = nodes[blockIdx.x];
    const int k = L.r_rank[t], K = L.s_cols[t];
    const double* S = L.S + L.s_off[t];
    const int32_t* idx = L.s_gidx + L.s_goff[t];
    double* out = ycpl + L.r_yhat_off[t] * R;
    const int warp = threadIdx.x >> 5;
    // every warp takes part in the staging: loop over the same number of tiles
    const int tiles = (k + 7) / 8, rounds = (tiles + kMmWarps - 1) / kMmWarps;
    for (int rd = 0; rd < rounds; ++rd) {
        const int m0 = 8 * (rd * kMmWarps + warp);
        double acc[NT][2];
        zero(acc);
        streamed_rows<NT>(acc, m0, k, S, K, K, idx, xhat, R, R, Bs);
        if (m0 < k) warp_store<NT>(acc, m0, k, [&](int m, int n, double v) { out[m * R + n] = v; });
    }
}

template <int NT>
__global__ void __launch_bounds__(kMmThreads) k_mm_bwd_level(h2b_layout L, const int32_t* __restrict__ nodes,
                                                             const double* __restrict__ ycpl, double* __restrict__ v) {
    constexpr int R = 8 * NT;
    extern __shared__ double Bs[];
    const int t = nodes[blockIdx.x];
    const int k = L.r_rank[t], p = L.r_parent[t];
    const bool cpl = L.s_cols[t] > 0;
    const int kp = p >= 0 ? L.r_rank[p] : 0;
    for (int e = threadIdx.x; e < kp * R; e += kMmThreads) Bs[e] = v[L.r_yhat_off[p] * R + e];
    __syncthreads();
    const double* E = L.r_E + (p >= 0 ? L.r_e_off[t] : 0);
    const double* yc = ycpl + L.r_yhat_off[t] * R;
    double* out = v + L.r_yhat_off[t] * R;
    const int warp = threadIdx.x >> 5;
    for (int m0 = 8 * warp; m0 < k; m0 += 8 * kMmWarps) {
        double acc[NT][2];
        zero(acc);
        if (kp > 0) warp_mma<NT>(acc, m0, k, 0, kp, 0, [&](int m, int kk) { return E[(int64_t)m * kp + kk]; }, Bs);
        warp_store<NT>(acc, m0, k, [&](int m, int n, double val) { out[m * R + n] = val + (cpl ? yc[m * R + n] : 0.0); });
    }
}

template <int NT>
__global__ void __launch_bounds__(kMmThreads) k_mm_leaf(h2b_layout L, const int32_t* __restrict__ leaves,
                                                        const double* __restrict__ X, int nrhs,
                                                        const double* __restrict__ v, double* __restrict__ Y) {
    constexpr int R = 8 * NT;
    extern __shared__ double Bs[];
    const int t = leaves[blockIdx.x];
    const int start = L.r_start[t], size = L.r_size[t], k = L.r_rank[t], C = L.d_cols[t];
    const double* Dm = L.D + L.d_off[t];
    const int32_t* idx = L.d_gidx + L.d_goff[t];
    const double* V = L.r_V + L.r_v_off[t];
    const int warp = threadIdx.x >> 5;
    const int tiles = (size + 7) / 8, rounds = (tiles + kMmWarps - 1) / kMmWarps;
    for (int rd = 0; rd < rounds; ++rd) {
        const int m0 = 8 * (rd * kMmWarps + warp);
        double acc[NT][2];
        zero(acc);
        streamed_rows<NT>(acc, m0, size, Dm, C, C, idx, X, nrhs, nrhs, Bs);
        // + V_t v_t
        __syncthreads();
        for (int e = threadIdx.x; e < k * R; e += kMmThreads) Bs[e] = v[L.r_yhat_off[t] * R + e];
        __syncthreads();
        if (m0 < size) {
            if (k > 0) warp_mma<NT>(acc, m0, size, 0, k, 0, [&](int m, int kk) { return V[(int64_t)m * k + kk]; }, Bs);
            warp_store<NT>(acc, m0, size, [&](int m, int n, double val) {
                if (n < nrhs) Y[L.row_perm[start + m] * nrhs + n] = val;
            });
        }
    }
}

template <typename T>
cudaError_t fetch_mm(const T* d, int64_t n, std::vector<T>& h) {
    h.resize((size_t)std::max<int64_t>(n, 0));
    return n > 0 ? cudaMemcpy(h.data(), d, sizeof(T) * n, cudaMemcpyDeviceToHost) : cudaSuccess;
}

template <int NT>
int run_mm(h2b_mmplan* p, const double* X, int nrhs, double* Y, cudaStream_t st) {
    constexpr int R = 8 * NT;
    const h2b_layout& L = p->L;
    const int32_t* lists = p->d_lists;
    const size_t sm_small = (size_t)std::max(64, p->max_c_node) * R * sizeof(double);
    const size_t sm_chunk = (size_t)std::max(kChunk, 64) * R * sizeof(double);
    const size_t sm_leaf = std::max(sm_chunk, (size_t)512 * R * sizeof(double));
    for (auto* f : {(const void*)k_mm_fwd_leaf<NT>, (const void*)k_mm_fwd_level<NT>, (const void*)k_mm_cpl<NT>,
                    (const void*)k_mm_bwd_level<NT>, (const void*)k_mm_leaf<NT>})
        H2B_CUDA_TRY(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_leaf + (int)sm_small));
    if (p->n_leaf_c > 0)
        k_mm_fwd_leaf<NT><<<(unsigned)p->n_leaf_c, kMmThreads, sm_small, st>>>(L, lists + p->off_leaf_c, X, nrhs,
                                                                              p->xhat);
    for (int lv = 0; lv + 1 < (int)p->fwd_level_off.size(); ++lv) {
        const int64_t a = p->fwd_level_off[lv], b = p->fwd_level_off[lv + 1];
        if (b > a)
            k_mm_fwd_level<NT><<<(unsigned)(b - a), kMmThreads, sm_small, st>>>(L, lists + p->off_fwd + a, p->xhat);
    }
    if (p->n_cpl > 0)
        k_mm_cpl<NT><<<(unsigned)p->n_cpl, kMmThreads, sm_chunk, st>>>(L, lists + p->off_cpl, p->xhat, p->ycpl);
    for (int lv = 0; lv + 1 < (int)p->bwd_level_off.size(); ++lv) {
        const int64_t a = p->bwd_level_off[lv], b = p->bwd_level_off[lv + 1];
        if (b > a)
            k_mm_bwd_level<NT><<<(unsigned)(b - a), kMmThreads, sm_small, st>>>(L, lists + p->off_bwd + a, p->ycpl,
                                                                               p->v);
    }
    if (p->n_leaf_r > 0)
        k_mm_leaf<NT><<<(unsigned)p->n_leaf_r, kMmThreads, sm_leaf, st>>>(L, lists + p->off_leaf_r, X, nrhs, p->v, Y);
    H2B_CUDA_TRY(cudaGetLastError());
    return ok();
}

}  // namespace
}  // namespace h2b

using namespace h2b;

extern "C" int h2b_matmat_create(const h2b_layout* layout, h2b_mmplan** out) {
    if (!layout || !out) return fail(H2B_ERR_INVALID, "h2b_matmat_create: null pointer");
    const h2b_layout& L = *layout;
    if (L.owned) return fail(H2B_ERR_INVALID, "h2b_matmat_create: row-sharded layouts are not supported");
    std::vector<int32_t> cparent, cchild, crank, leaves, rparent, rrank, scols, dcols, csize;
    std::vector<int64_t> rvoff;
    H2B_CUDA_TRY(fetch_mm(L.c_parent, L.c_nodes, cparent));
    H2B_CUDA_TRY(fetch_mm(L.c_child, 2 * (int64_t)L.c_nodes, cchild));
    H2B_CUDA_TRY(fetch_mm(L.c_rank, L.c_nodes, crank));
    H2B_CUDA_TRY(fetch_mm(L.c_leaf_list, L.c_leaves, leaves));
    H2B_CUDA_TRY(fetch_mm(L.r_parent, L.r_nodes, rparent));
    H2B_CUDA_TRY(fetch_mm(L.r_rank, L.r_nodes, rrank));
    H2B_CUDA_TRY(fetch_mm(L.s_cols, L.r_nodes, scols));
    H2B_CUDA_TRY(fetch_mm(L.d_cols, L.r_nodes, dcols));
    H2B_CUDA_TRY(fetch_mm(L.r_v_off, L.r_nodes, rvoff));
    H2B_CUDA_TRY(fetch_mm(L.c_size, L.c_nodes, csize));
    auto depths = [](const std::vector<int32_t>& parent) {
        std::vector<int> d(parent.size(), 0);
        for (size_t u = 0; u < parent.size(); ++u)
            for (int q = parent[u]; q >= 0; q = parent[q]) ++d[u];
        return d;
    };
    const std::vector<int> dc = depths(cparent), dr = depths(rparent);
    const int mc = dc.empty() ? 0 : *std::max_element(dc.begin(), dc.end());
    const int mr = dr.empty() ? 0 : *std::max_element(dr.begin(), dr.end());
    h2b_mmplan* p = new (std::nothrow) h2b_mmplan();
    if (!p) return fail(H2B_ERR_INVALID, "h2b_matmat_create: out of host memory");
    p->L = L;
    p->max_depth_c = mc;
    p->max_depth_r = mr;
    std::vector<int32_t> lists;
    p->off_leaf_c = 0;
    lists.insert(lists.end(), leaves.begin(), leaves.end());
    p->n_leaf_c = (int64_t)leaves.size();
    // upward: non-leaf column nodes, deepest level first
    p->off_fwd = (int64_t)lists.size();
    p->max_c_node = 0;
    p->fwd_level_off.push_back(0);
    for (int d = mc; d >= 0; --d) {
        for (int u = 0; u < L.c_nodes; ++u)
            if (dc[u] == d && cchild[2 * u] >= 0 && cchild[2 * u + 1] >= 0) {
                lists.push_back(u);
                p->max_c_node = std::max(p->max_c_node, crank[cchild[2 * u]] + crank[cchild[2 * u + 1]]);
            }
        p->fwd_level_off.push_back((int64_t)lists.size() - p->off_fwd);
    }
    p->off_cpl = (int64_t)lists.size();
    for (int u = 0; u < L.r_nodes; ++u)
        if (scols[u] > 0 && rrank[u] > 0) lists.push_back(u);
    p->n_cpl = (int64_t)lists.size() - p->off_cpl;
    // downward: every row node with a rank, top level first
    p->off_bwd = (int64_t)lists.size();
    p->bwd_level_off.push_back(0);
    int maxk = 64;
    for (int d = 0; d <= mr; ++d) {
        for (int u = 0; u < L.r_nodes; ++u)
            if (dr[u] == d && rrank[u] > 0) lists.push_back(u);
        p->bwd_level_off.push_back((int64_t)lists.size() - p->off_bwd);
    }
    for (int u = 0; u < L.r_nodes; ++u) maxk = std::max(maxk, rrank[u]);
    p->max_c_node = std::max(p->max_c_node, maxk);
    for (int32_t l : leaves) p->max_c_node = std::max(p->max_c_node, csize[l]);  // B rows of the leaf transform
    p->off_leaf_r = (int64_t)lists.size();
    for (int u = 0; u < L.r_nodes; ++u)
        if (rvoff[u] >= 0) lists.push_back(u);
    p->n_leaf_r = (int64_t)lists.size() - p->off_leaf_r;
    if (maxk > 512) {
        delete p;
        return fail(H2B_ERR_INVALID, "h2b_matmat_create: cluster rank above 512");
    }
    auto alloc = [](void** ptr, size_t bytes) { return cudaMalloc(ptr, bytes ? bytes : 16); };
    H2B_CUDA_TRY(alloc(reinterpret_cast<void**>(&p->d_lists), sizeof(int32_t) * lists.size()));
    H2B_CUDA_TRY(cudaMemcpy(p->d_lists, lists.data(), sizeof(int32_t) * lists.size(), cudaMemcpyHostToDevice));
    H2B_CUDA_TRY(alloc(reinterpret_cast<void**>(&p->xhat), sizeof(double) * 16 * (size_t)L.xhat_len));
    H2B_CUDA_TRY(alloc(reinterpret_cast<void**>(&p->ycpl), sizeof(double) * 16 * (size_t)L.yhat_len));
    H2B_CUDA_TRY(alloc(reinterpret_cast<void**>(&p->v), sizeof(double) * 16 * (size_t)L.yhat_len));
    H2B_CUDA_TRY(cudaMemset(p->ycpl, 0, sizeof(double) * 16 * (size_t)L.yhat_len));
    *out = p;
    return ok();
}

extern "C" int h2b_matmat_destroy(h2b_mmplan* p) {
    if (!p) return ok();
    for (void* q : {(void*)p->d_lists, (void*)p->xhat, (void*)p->ycpl, (void*)p->v})
        if (q) cudaFree(q);
    delete p;
    return ok();
}

extern "C" int h2b_matmat(h2b_mmplan* p, const double* d_X, double* d_Y, int32_t nrhs, void* stream) {
    if (!p || !d_X || !d_Y) return fail(H2B_ERR_INVALID, "h2b_matmat: null pointer");
    if (nrhs < 1 || nrhs > 16) return fail(H2B_ERR_INVALID, "h2b_matmat: 1 <= nrhs <= 16");
    cudaStream_t st = as_stream(stream);
    return nrhs <= 8 ? run_mm<1>(p, d_X, nrhs, d_Y, st) : run_mm<2>(p, d_X, nrhs, d_Y, st);
}
