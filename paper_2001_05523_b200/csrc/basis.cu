// Nested cluster-basis transforms on their own (ClusterBasis.forward /
// ClusterBasis.backward, containers.py:201-228), for callers of the
// reference's basis API.  The H^2 matvec does not use these kernels: it runs
// both transforms inside its single fused launch (matvec.cu).
//
// One launch per tree level (forward: deepest level first; backward: root
// level first), one warp per cluster, lanes over the cluster's coefficients:
//   forward   leaf  x_hat_t[c] = sum_r V_t[r, c] xp[start_t + r]
//             inner x_hat_t[c] = sum_ch sum_r E_ch[r, c] x_hat_ch[r]   (children in order)
//   backward  inner y_hat_ch[r] += sum_c E_ch[r, c] y_hat_t[c]
//             leaf  yp[start_t + i] += sum_c V_t[i, c] y_hat_t[c]
// Every output is written by one lane in a fixed order (deterministic).

#include <algorithm>
#include <vector>

#include "device_common.cuh"

namespace h2b {
namespace {

__global__ void k_basis_fwd(h2b_basis b, const int32_t* __restrict__ nodes, int n, const double* __restrict__ xp,
                            double* __restrict__ xhat) {
    const int w = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
    if (w >= n) return;
    const int u = nodes[w];
    const int k = b.d_rank[u];
    double* out = xhat + b.d_hat_off[u];
    const int l = b.d_left[u];
    if (l < 0) {
        const int size = b.d_size[u];
        const double* V = b.d_V + b.d_v_off[u];
        const double* x = xp + b.d_start[u];
        for (int c = lane; c < k; c += 32) {
            double acc = 0.0;
            for (int r = 0; r < size; ++r) acc = fma(V[(int64_t)r * k + c], x[r], acc);
            out[c] = acc;
        }
        return;
    }
    const int ch[2] = {l, b.d_right[u]};
    for (int c = lane; c < k; c += 32) {
        double acc = 0.0;
        for (int j = 0; j < 2; ++j) {
            const int v = ch[j];
            const int kv = b.d_rank[v];
            const double* E = b.d_E + b.d_e_off[v];
            const double* xv = xhat + b.d_hat_off[v];
            for (int r = 0; r < kv; ++r) acc = fma(E[(int64_t)r * k + c], xv[r], acc);
        }
        out[c] = acc;
    }
}

__global__ void k_basis_bwd(h2b_basis b, const int32_t* __restrict__ nodes, int n, double* __restrict__ yhat,
                            double* __restrict__ yp) {
    const int w = (int)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
    if (w >= n) return;
    const int u = nodes[w];
    const int k = b.d_rank[u];
    const double* v = yhat + b.d_hat_off[u];
    const int l = b.d_left[u];
    if (l < 0) {
        const int size = b.d_size[u];
        const double* V = b.d_V + b.d_v_off[u];
        double* y = yp + b.d_start[u];
        for (int i = lane; i < size; i += 32) {
            double acc = 0.0;
            for (int c = 0; c < k; ++c) acc = fma(V[(int64_t)i * k + c], v[c], acc);
            y[i] += acc;
        }
        return;
    }
    const int ch[2] = {l, b.d_right[u]};
    for (int j = 0; j < 2; ++j) {
        const int q = ch[j];
        const int kq = b.d_rank[q];
        const double* E = b.d_E + b.d_e_off[q];
        double* out = yhat + b.d_hat_off[q];
        for (int r = lane; r < kq; r += 32) {
            double acc = 0.0;
            for (int c = 0; c < k; ++c) acc = fma(E[(int64_t)r * k + c], v[c], acc);
            out[r] += acc;
        }
    }
}

int check_basis(const h2b_basis* b) {
    if (!b || b->n_nodes <= 0 || !b->d_left || !b->d_right || !b->d_start || !b->d_size || !b->d_rank ||
        !b->d_v_off || !b->d_e_off || !b->d_hat_off || !b->d_V || !b->d_E || b->n_levels <= 0 || !b->h_level_off ||
        !b->d_level_nodes)
        return fail(H2B_ERR_INVALID, "h2b_basis: incomplete basis descriptor");
    return ok();
}

// one CTA per block: dst[dst_off + j * dst_ld + i] = src[src_off + i * src_ld + j]
// through a 32 x 33 shared tile (coalesced on both sides)
__global__ void k_transpose_blocks(const int64_t* __restrict__ desc, const double* __restrict__ src,
                                   double* __restrict__ dst) {
    __shared__ double tile[32][33];
    const int64_t* d = desc + 6 * (int64_t)blockIdx.x;
    const int64_t s_off = d[0], s_ld = d[1], rows = d[2], cols = d[3], d_off = d[4], d_ld = d[5];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8 threads
    for (int64_t i0 = 0; i0 < rows; i0 += 32)
        for (int64_t j0 = 0; j0 < cols; j0 += 32) {
            for (int r = ty; r < 32; r += 8) {
                const int64_t i = i0 + r, j = j0 + tx;
                if (i < rows && j < cols) tile[r][tx] = src[s_off + i * s_ld + j];
            }
            __syncthreads();
            for (int r = ty; r < 32; r += 8) {
                const int64_t j = j0 + r, i = i0 + tx;
                if (i < rows && j < cols) dst[d_off + j * d_ld + i] = tile[tx][r];
            }
            __syncthreads();
        }
}

}  // namespace
}  // namespace h2b

using namespace h2b;

extern "C" int h2b_transpose_blocks(int64_t n_blocks, const int64_t* d_desc, const double* d_src, double* d_dst,
                                    void* stream) {
    if (n_blocks < 0 || (n_blocks > 0 && (!d_desc || !d_src || !d_dst)))
        return fail(H2B_ERR_INVALID, "h2b_transpose_blocks: bad argument");
    cudaStream_t st = as_stream(stream);
    for (int64_t b0 = 0; b0 < n_blocks; b0 += 2147483647LL) {
        const unsigned g = (unsigned)std::min<int64_t>(n_blocks - b0, 2147483647LL);
        k_transpose_blocks<<<g, 256, 0, st>>>(d_desc + 6 * b0, d_src, d_dst);
    }
    H2B_CUDA_TRY(cudaGetLastError());
    return ok();
}

extern "C" int h2b_basis_forward(const h2b_basis* b, const double* d_xp, double* d_xhat, void* stream) {
    if (int rc = check_basis(b)) return rc;
    if (!d_xp || !d_xhat) return fail(H2B_ERR_INVALID, "h2b_basis_forward: null vector");
    cudaStream_t st = as_stream(stream);
    for (int lv = b->n_levels - 1; lv >= 0; --lv) {
        const int64_t a = b->h_level_off[lv], e = b->h_level_off[lv + 1];
        if (e <= a) continue;
        const unsigned grid = (unsigned)((32 * (e - a) + 255) / 256);
        k_basis_fwd<<<grid, 256, 0, st>>>(*b, b->d_level_nodes + a, (int)(e - a), d_xp, d_xhat);
    }
    H2B_CUDA_TRY(cudaGetLastError());
    return ok();
}

extern "C" int h2b_basis_backward(const h2b_basis* b, double* d_yhat, double* d_yp, void* stream) {
    if (int rc = check_basis(b)) return rc;
    if (!d_yhat || !d_yp) return fail(H2B_ERR_INVALID, "h2b_basis_backward: null vector");
    cudaStream_t st = as_stream(stream);
    for (int lv = 0; lv < b->n_levels; ++lv) {
        const int64_t a = b->h_level_off[lv], e = b->h_level_off[lv + 1];
        if (e <= a) continue;
        const unsigned grid = (unsigned)((32 * (e - a) + 255) / 256);
        k_basis_bwd<<<grid, 256, 0, st>>>(*b, b->d_level_nodes + a, (int)(e - a), d_yhat, d_yp);
    }
    H2B_CUDA_TRY(cudaGetLastError());
    return ok();
}
