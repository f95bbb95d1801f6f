// H^2-matrix-vector product y = A x (containers.py:254-270) in two launches.
//
//   k_forward   one CTA per column leaf: gather x_p = x[col_perm] for the leaf,
//               x_hat_t = V_t^T x_p|t, then climb the tree: the second child to
//               arrive at a parent (arrival counter) computes
//               x_hat_parent = sum_ch E_ch^T x_hat_ch in child order
//               (ClusterBasis.forward, containers.py:201-212).  Deterministic:
//               each sum has one fixed order regardless of arrival order.
//   k_backward  one CTA per row cluster, parents first (dynamic tickets over a
//               top-down order guarantee every parent CTA started before its
//               children, so the flag wait below cannot deadlock):
//                 y_hat_t = [S_b1 S_b2 ...] [x_hat_s1; x_hat_s2; ...]   (coupling, :259-264)
//                 leaf: y_near = [D_b1 D_b2 ...] [x_p|s1; x_p|s2; ...]  (nearfield, :266-267)
//                 wait for the parent, y_hat_t += E_t y_hat_parent     (backward, :214-228)
//                 leaf: y[row_perm[i]] = y_near + V_t y_hat_t          (un-permute, :268-269)
//
// All products stream their matrices row-major and coalesced, one warp per
// output row (lanes over columns, double2 loads, shuffle reduction), with the
// gathered right-hand side staged in shared memory.  No atomics on values:
// every output entry is produced by exactly one warp in a fixed order, so the
// result is bitwise reproducible and independent of the number of GPUs.

#include <vector>

#include "device_common.cuh"

struct h2b_plan {
    h2b_layout L;
    int device;
    double* xp;        // n_cols permuted input
    double* xhat;      // xhat_len
    double* yhat;      // yhat_len
    int* arrive;       // c_nodes
    int* flag;         // r_nodes
    int* ticket;       // [0] backward ticket counter, [1] matvec epoch (device-resident: graph-safe)
    int fwd_smem;      // bytes
    int bwd_smem;
    int n_bwd;
    double* hx;        // pinned host staging for h2b_matvec_host
    double* hy;
    double* dx;
    double* dy;
};

namespace h2b {
namespace {

constexpr int kFwdThreads = 128;
constexpr int kBwdThreads = 256;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// out[i] (i < rows) = sum_c M[i*ld + c] * v[c] for c < cols, one warp per row.
// M rows are read with coalesced loads; v is in shared memory.
__device__ __forceinline__ double row_dot(const double* __restrict__ row, const double* __restrict__ v,
                                          int cols, int lane) {
    double acc = 0.0;
    const bool al16 = ((reinterpret_cast<uintptr_t>(row) & 15) == 0);
    if (al16) {
        const double2* r2 = reinterpret_cast<const double2*>(row);
        const int c2 = cols >> 1;
        int c = lane;
        for (; c + 32 < c2; c += 64) {
            const double2 a = __ldcs(r2 + c);
            const double2 b = __ldcs(r2 + c + 32);
            acc = fma(a.x, v[2 * c], acc);
            acc = fma(a.y, v[2 * c + 1], acc);
            acc = fma(b.x, v[2 * c + 64], acc);
            acc = fma(b.y, v[2 * c + 65], acc);
        }
        for (; c < c2; c += 32) {
            const double2 a = __ldcs(r2 + c);
            acc = fma(a.x, v[2 * c], acc);
            acc = fma(a.y, v[2 * c + 1], acc);
        }
        if ((cols & 1) && lane == 0) acc = fma(__ldcs(row + cols - 1), v[cols - 1], acc);
    } else {
        for (int c = lane; c < cols; c += 32) acc = fma(__ldcs(row + c), v[c], acc);
    }
    return warp_sum(acc);
}

// xhat (k) = M^T v for M (rows x k) row-major, all threads of the CTA.
// Threads are split into groups over rows; partial sums reduced in smem.
__device__ void transposed_product(const double* __restrict__ M, const double* __restrict__ v, int rows,
                                   int k, double* __restrict__ red, double* __restrict__ out) {
    const int nt = blockDim.x;
    if (k <= 0) return;
    const int kc = min(k, nt);
    const int groups = max(1, nt / kc);
    for (int c0 = 0; c0 < k; c0 += kc) {
        const int tid = threadIdx.x;
        const int c = tid % kc, g = tid / kc;
        double acc = 0.0;
        if (g < groups && c0 + c < k) {
            for (int r = g; r < rows; r += groups) acc = fma(M[(int64_t)r * k + c0 + c], v[r], acc);
        }
        __syncthreads();
        if (g < groups) red[g * kc + c] = acc;
        __syncthreads();
        if (tid < kc && c0 + tid < k) {
            double s = 0.0;
            for (int gg = 0; gg < groups; ++gg) s += red[gg * kc + tid];
            out[c0 + tid] = s;
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kFwdThreads) k_forward(h2b_layout L, const double* __restrict__ x,
                                                        double* __restrict__ xp, double* __restrict__ xhat,
                                                        int* __restrict__ arrive, int* __restrict__ ticket) {
    extern __shared__ double sm[];
    __shared__ int s_last;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        ticket[0] = 0;  // backward's ticket counter
        ticket[1] += 1; // epoch of this matvec (flags compare against it)
    }
    const int leaf = L.c_leaf_list[blockIdx.x];
    const int start = L.c_start[leaf], size = L.c_size[leaf], k = L.c_rank[leaf];
    double* xs = sm;                 // max leaf size
    double* red = sm + 1024;         // reduction scratch (kFwdThreads)
    double* tmp = red + kFwdThreads; // child-sum staging
    for (int r = threadIdx.x; r < size; r += blockDim.x) {
        const double v = x[L.col_perm[start + r]];
        xs[r] = v;
        xp[start + r] = v;
    }
    __syncthreads();
    transposed_product(L.c_V + L.c_v_off[leaf], xs, size, k, red, xhat + L.c_xhat_off[leaf]);
    int node = leaf;
    while (true) {
        const int parent = L.c_parent[node];
        if (parent < 0) break;
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) {
            const int old = atomicAdd(arrive + parent, 1);
            s_last = (old == 1);
            if (old == 1) arrive[parent] = 0;  // reset for the next matvec
        }
        __syncthreads();
        if (!s_last) break;
        __threadfence();
        const int kp = L.c_rank[parent];
        double* out = xhat + L.c_xhat_off[parent];
        // first child writes, second accumulates (child order, containers.py:209-211)
        for (int ci = 0; ci < 2; ++ci) {
            const int ch = L.c_child[2 * parent + ci];
            const int kc = L.c_rank[ch];
            const double* xc = xhat + L.c_xhat_off[ch];
            for (int r = threadIdx.x; r < kc; r += blockDim.x) tmp[r] = __ldcg(xc + r);
            __syncthreads();
            transposed_product(L.c_E + L.c_e_off[ch], tmp, kc, kp, red, tmp + 1024);
            for (int c = threadIdx.x; c < kp; c += blockDim.x) {
                const double v = tmp[1024 + c];
                out[c] = ci == 0 ? v : __ldcg(out + c) + v;
            }
            __syncthreads();
        }
        node = parent;
    }
}

__global__ void __launch_bounds__(kBwdThreads) k_backward(h2b_layout L, const double* __restrict__ xp,
                                                         const double* __restrict__ xhat,
                                                         double* __restrict__ yhat, double* __restrict__ y,
                                                         int* __restrict__ flag, int* __restrict__ ticket,
                                                         int smem_cols) {
    extern __shared__ double sm[];
    __shared__ int s_node, s_epoch;
    if (threadIdx.x == 0) {
        const int tk = atomicAdd(ticket, 1);
        s_node = L.owned ? L.owned[tk] : L.r_order[tk];
        s_epoch = *reinterpret_cast<volatile int*>(ticket + 1);
    }
    __syncthreads();
    const int node = s_node;
    const int epoch = s_epoch;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const int k = L.r_rank[node];
    const int parent = L.r_parent[node];
    const bool leaf = L.r_v_off[node] >= 0;
    double* vg = sm;                       // gathered right-hand side (smem_cols)
    double* yh = sm + smem_cols;           // y_hat_t (<= 1024)
    double* yp = yh + 1024;                // y_hat_parent (<= 1024)
    double* yn = yp + 1024;                // nearfield rows (<= 1024)

    // 1. coupling y_hat_t = S_t [x_hat_s ...]
    const int K = L.s_cols[node];
    if (K > 0) {
        int off = 0;
        for (int f = L.far_ptr[node]; f < L.far_ptr[node + 1]; ++f) {
            const int s = L.far_col[f];
            const int ks = L.c_rank[s];
            const double* src = xhat + L.c_xhat_off[s];
            for (int c = threadIdx.x; c < ks; c += blockDim.x) vg[off + c] = src[c];
            off += ks;
        }
        __syncthreads();
        const double* S = L.S + L.s_off[node];
        for (int i = warp; i < k; i += nw) {
            const double v = row_dot(S + (int64_t)i * K, vg, K, lane);
            if (lane == 0) yh[i] = v;
        }
    } else {
        for (int i = threadIdx.x; i < k; i += blockDim.x) yh[i] = 0.0;
    }
    __syncthreads();
    // 2. nearfield rows of a leaf (independent of the parent)
    const int start = L.r_start[node], size = L.r_size[node];
    if (leaf) {
        const int C = L.d_cols[node];
        if (C > 0) {
            int off = 0;
            for (int f = L.near_ptr[node]; f < L.near_ptr[node + 1]; ++f) {
                const int s = L.near_col[f];
                const int ss = L.c_start[s], sz = L.c_size[s];
                for (int c = threadIdx.x; c < sz; c += blockDim.x) vg[off + c] = xp[ss + c];
                off += sz;
            }
            __syncthreads();
            const double* D = L.D + L.d_off[node];
            for (int r = warp; r < size; r += nw) {
                const double v = row_dot(D + (int64_t)r * C, vg, C, lane);
                if (lane == 0) yn[r] = v;
            }
        } else {
            for (int r = threadIdx.x; r < size; r += blockDim.x) yn[r] = 0.0;
        }
    }
    // 3. parent contribution
    if (parent >= 0) {
        if (threadIdx.x == 0) {
            volatile int* fp = flag + parent;
            while (*fp != epoch) __nanosleep(64);
        }
        __syncthreads();
        __threadfence();
        const int kp = L.r_rank[parent];
        const double* src = yhat + L.r_yhat_off[parent];
        for (int c = threadIdx.x; c < kp; c += blockDim.x) yp[c] = __ldcg(src + c);
        __syncthreads();
        const double* E = L.r_E + L.r_e_off[node];
        for (int i = warp; i < k; i += nw) {
            const double v = row_dot(E + (int64_t)i * kp, yp, kp, lane);
            if (lane == 0) yh[i] += v;
        }
    }
    __syncthreads();
    // 4. leaf: expand and un-permute; inner node: publish y_hat_t
    if (leaf) {
        const double* Vt = L.r_V + L.r_v_off[node];
        for (int r = warp; r < size; r += nw) {
            const double v = k > 0 ? row_dot(Vt + (int64_t)r * k, yh, k, lane) : 0.0;
            if (lane == 0) y[L.row_perm[start + r]] = yn[r] + v;
        }
    } else {
        double* dst = yhat + L.r_yhat_off[node];
        for (int i = threadIdx.x; i < k; i += blockDim.x) dst[i] = yh[i];
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) atomicExch(flag + node, epoch);
    }
}

__global__ void k_diagonal(h2b_layout L, double* __restrict__ diag) {
    const int node = blockIdx.x * blockDim.x + threadIdx.x;
    if (node >= L.r_nodes || L.r_v_off[node] < 0) return;
    const int ts = L.r_start[node], te = ts + L.r_size[node];
    const int C = L.d_cols[node];
    const double* D = L.D + L.d_off[node];
    for (int r = ts; r < te; ++r) {
        double acc = 0.0;
        int off = 0;
        for (int f = L.near_ptr[node]; f < L.near_ptr[node + 1]; ++f) {
            const int s = L.near_col[f];
            const int ss = L.c_start[s], sz = L.c_size[s];
            if (r >= ss && r < ss + sz) acc += D[(int64_t)(r - ts) * C + off + (r - ss)];
            off += sz;
        }
        diag[L.row_perm[r]] = acc;
    }
}

}  // namespace
}  // namespace h2b

using namespace h2b;

extern "C" int h2b_plan_create(const h2b_layout* layout, h2b_plan** out) {
    if (!layout || !out) return fail(H2B_ERR_INVALID, "h2b_plan_create: null pointer");
    const h2b_layout& L = *layout;
    if (L.c_nodes <= 0 || L.r_nodes <= 0 || L.c_leaves <= 0) return fail(H2B_ERR_INVALID, "h2b_plan_create: empty tree");
    h2b_plan* p = new (std::nothrow) h2b_plan();
    if (!p) return fail(H2B_ERR_INVALID, "h2b_plan_create: out of host memory");
    p->L = L;
    H2B_CUDA_TRY(cudaGetDevice(&p->device));
    auto alloc = [&](void** ptr, size_t bytes) -> cudaError_t {
        return cudaMalloc(ptr, bytes ? bytes : 8);
    };
    H2B_CUDA_TRY(alloc(reinterpret_cast<void**>(&p->xp), sizeof(double) * L.n_cols));
    H2B_CUDA_TRY(alloc(reinterpret_cast<void**>(&p->xhat), sizeof(double) * L.xhat_len));
    H2B_CUDA_TRY(alloc(reinterpret_cast<void**>(&p->yhat), sizeof(double) * L.yhat_len));
    H2B_CUDA_TRY(alloc(reinterpret_cast<void**>(&p->arrive), sizeof(int) * L.c_nodes));
    H2B_CUDA_TRY(alloc(reinterpret_cast<void**>(&p->flag), sizeof(int) * L.r_nodes));
    H2B_CUDA_TRY(alloc(reinterpret_cast<void**>(&p->ticket), 2 * sizeof(int)));
    H2B_CUDA_TRY(cudaMemset(p->arrive, 0, sizeof(int) * L.c_nodes));
    H2B_CUDA_TRY(cudaMemset(p->flag, 0, sizeof(int) * L.r_nodes));
    H2B_CUDA_TRY(cudaMemset(p->ticket, 0, 2 * sizeof(int)));
    // shared memory: largest gathered right-hand side over coupling / nearfield rows
    std::vector<int32_t> scols(L.r_nodes), dcols(L.r_nodes), rsize(L.r_nodes), rrank(L.r_nodes), crank(L.c_nodes),
        csize(L.c_nodes);
    H2B_CUDA_TRY(cudaMemcpy(scols.data(), L.s_cols, sizeof(int32_t) * L.r_nodes, cudaMemcpyDeviceToHost));
    H2B_CUDA_TRY(cudaMemcpy(dcols.data(), L.d_cols, sizeof(int32_t) * L.r_nodes, cudaMemcpyDeviceToHost));
    H2B_CUDA_TRY(cudaMemcpy(rsize.data(), L.r_size, sizeof(int32_t) * L.r_nodes, cudaMemcpyDeviceToHost));
    H2B_CUDA_TRY(cudaMemcpy(rrank.data(), L.r_rank, sizeof(int32_t) * L.r_nodes, cudaMemcpyDeviceToHost));
    H2B_CUDA_TRY(cudaMemcpy(crank.data(), L.c_rank, sizeof(int32_t) * L.c_nodes, cudaMemcpyDeviceToHost));
    H2B_CUDA_TRY(cudaMemcpy(csize.data(), L.c_size, sizeof(int32_t) * L.c_nodes, cudaMemcpyDeviceToHost));
    std::vector<int64_t> rvoff(L.r_nodes);
    H2B_CUDA_TRY(cudaMemcpy(rvoff.data(), L.r_v_off, sizeof(int64_t) * L.r_nodes, cudaMemcpyDeviceToHost));
    int maxcols = 1, maxk = 0, maxleaf = 0;
    for (int i = 0; i < L.r_nodes; ++i) {
        maxcols = std::max(maxcols, std::max(scols[i], dcols[i]));
        maxk = std::max(maxk, rrank[i]);
        if (rvoff[i] >= 0) maxleaf = std::max(maxleaf, rsize[i]);
    }
    for (int i = 0; i < L.c_nodes; ++i) maxk = std::max(maxk, crank[i]);
    std::vector<int32_t> leaves(L.c_leaves);
    H2B_CUDA_TRY(cudaMemcpy(leaves.data(), L.c_leaf_list, sizeof(int32_t) * L.c_leaves, cudaMemcpyDeviceToHost));
    for (int l : leaves) maxleaf = std::max(maxleaf, csize[l]);
    if (maxk > 1024 || maxleaf > 1024) {
        delete p;
        return fail(H2B_ERR_INVALID, "h2b_plan_create: cluster rank or leaf size above 1024");
    }
    p->bwd_smem = (int)sizeof(double) * (maxcols + 3 * 1024);
    p->fwd_smem = (int)sizeof(double) * (1024 + kFwdThreads + 2048);
    p->n_bwd = L.owned ? L.n_owned : L.r_nodes;
    if (p->bwd_smem > 227 * 1024) {
        delete p;
        return fail(H2B_ERR_INVALID, "h2b_plan_create: gathered right-hand side exceeds shared memory");
    }
    H2B_CUDA_TRY(cudaFuncSetAttribute(k_backward, cudaFuncAttributeMaxDynamicSharedMemorySize, p->bwd_smem));
    H2B_CUDA_TRY(cudaFuncSetAttribute(k_forward, cudaFuncAttributeMaxDynamicSharedMemorySize, p->fwd_smem));
    H2B_CUDA_TRY(cudaMallocHost(reinterpret_cast<void**>(&p->hx), sizeof(double) * std::max<int64_t>(1, L.n_cols)));
    H2B_CUDA_TRY(cudaMallocHost(reinterpret_cast<void**>(&p->hy), sizeof(double) * std::max<int64_t>(1, L.n_rows)));
    H2B_CUDA_TRY(alloc(reinterpret_cast<void**>(&p->dx), sizeof(double) * L.n_cols));
    H2B_CUDA_TRY(alloc(reinterpret_cast<void**>(&p->dy), sizeof(double) * L.n_rows));
    *out = p;
    return ok();
}

extern "C" int h2b_plan_destroy(h2b_plan* p) {
    if (!p) return ok();
    cudaFree(p->xp);
    cudaFree(p->xhat);
    cudaFree(p->yhat);
    cudaFree(p->arrive);
    cudaFree(p->flag);
    cudaFree(p->ticket);
    cudaFree(p->dx);
    cudaFree(p->dy);
    cudaFreeHost(p->hx);
    cudaFreeHost(p->hy);
    delete p;
    return ok();
}

extern "C" int h2b_matvec(h2b_plan* p, const double* d_x, double* d_y, void* stream) {
    if (!p || !d_x || !d_y) return fail(H2B_ERR_INVALID, "h2b_matvec: null pointer");
    cudaStream_t st = as_stream(stream);
    k_forward<<<p->L.c_leaves, kFwdThreads, p->fwd_smem, st>>>(p->L, d_x, p->xp, p->xhat, p->arrive, p->ticket);
    H2B_CUDA_TRY(cudaGetLastError());
    int smem_cols = (p->bwd_smem / (int)sizeof(double)) - 3 * 1024;
    k_backward<<<p->n_bwd, kBwdThreads, p->bwd_smem, st>>>(p->L, p->xp, p->xhat, p->yhat, d_y, p->flag,
                                                          p->ticket, smem_cols);
    H2B_CUDA_TRY(cudaGetLastError());
    return ok();
}

extern "C" int h2b_matvec_host(h2b_plan* p, const double* h_x, double* h_y, void* stream) {
    if (!p || !h_x || !h_y) return fail(H2B_ERR_INVALID, "h2b_matvec_host: null pointer");
    cudaStream_t st = as_stream(stream);
    H2B_CUDA_TRY(cudaMemcpyAsync(p->dx, h_x, sizeof(double) * p->L.n_cols, cudaMemcpyHostToDevice, st));
    if (int rc = h2b_matvec(p, p->dx, p->dy, stream)) return rc;
    H2B_CUDA_TRY(cudaMemcpyAsync(h_y, p->dy, sizeof(double) * p->L.n_rows, cudaMemcpyDeviceToHost, st));
    H2B_CUDA_TRY(cudaStreamSynchronize(st));
    return ok();
}

extern "C" int h2b_diagonal(h2b_plan* p, double* d_diag, void* stream) {
    if (!p || !d_diag) return fail(H2B_ERR_INVALID, "h2b_diagonal: null pointer");
    if (p->L.n_rows != p->L.n_cols) return fail(H2B_ERR_INVALID, "diagonal extraction requires a square operator");
    cudaStream_t st = as_stream(stream);
    k_diagonal<<<(p->L.r_nodes + 127) / 128, 128, 0, st>>>(p->L, d_diag);
    H2B_CUDA_TRY(cudaGetLastError());
    return ok();
}
