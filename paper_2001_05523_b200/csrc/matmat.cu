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
#include <cstdlib>
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
    uint32_t* flags;  // per column node (forward) then per row node (backward): launch epoch when done
    unsigned long long* ctr;  // ticket counters of the fused forward / backward launches
};

namespace h2b {
namespace {

constexpr int kMmThreads = 256;
constexpr int kMmWarps = kMmThreads / 32;
constexpr int kChunk = 256;  // staged B rows per chunk (gathered right-hand sides)

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    // not volatile: a pure function of its operands, so the compiler may hoist
    // the operand loads of later steps above it
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
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
#pragma unroll 4
    for (; k < k1; k += 4) {
        const int kk = k + q;
        const double a = (rowok && kk < k1) ? fa(m0 + g, kk) : 0.0;
#pragma unroll
        for (int t = 0; t < NT; ++t) dmma(acc[t], a, kk < k1 ? Bs[(kk - kb) * R + 8 * t + g] : 0.0);
    }
}

struct d4 {
    double x, y, z, w;
};
// 32-byte streaming load (LDG.256), read once: no L1 allocation
__device__ __forceinline__ d4 ld_stream4(const double* p) {
    d4 r;
    asm("ld.global.nc.L1::no_allocate.v4.f64 {%0, %1, %2, %3}, [%4];"
                 : "=d"(r.x), "=d"(r.y), "=d"(r.z), "=d"(r.w)
                 : "l"(p));
    return r;
}

// acc += A[m0:m0+8, k0:k1] B for a row-major streamed A (32-byte aligned rows,
// k0 16-aligned): lane (g, q) loads A[m0+g][k + 4q .. k + 4q + 3] with one
// 32-byte load and feeds them to four mma steps whose k index q stands for
// column k + 4q + j (the contraction order is free) -- a quarter of the load
// instructions of the fragment-order loads.  Columns past the last full group
// of 16 take the scalar path.
template <int NT>
__device__ __forceinline__ void warp_mma_stream(double (&acc)[NT][2], int m0, int M, int k0, int k1, int kb,
                                                const double* A, int64_t ld, const double* Bs);

// streaming operand loads (read once): no L1 allocation
__device__ __forceinline__ double ld_stream(const double* p) {
    double v;
    asm("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}

template <int NT>
__device__ __forceinline__ void warp_mma_stream(double (&acc)[NT][2], int m0, int M, int k0, int k1, int kb,
                                                const double* A, int64_t ld, const double* Bs) {
    constexpr int R = 8 * NT;
    const int lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
    const bool rowok = m0 + g < M;
    const double* row = A + (int64_t)(rowok ? m0 + g : m0) * ld;
    int k = k0;
    for (; k + 64 <= k1; k += 64) {
        d4 a[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) a[u] = rowok ? ld_stream4(row + k + 16 * u + 4 * q) : d4{0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const double* b = Bs + (k + 16 * u + 4 * q - kb) * R + g;
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                dmma(acc[t], a[u].x, b[8 * t]);
                dmma(acc[t], a[u].y, b[R + 8 * t]);
                dmma(acc[t], a[u].z, b[2 * R + 8 * t]);
                dmma(acc[t], a[u].w, b[3 * R + 8 * t]);
            }
        }
    }
    for (; k + 16 <= k1; k += 16) {
        const d4 a = rowok ? ld_stream4(row + k + 4 * q) : d4{0.0, 0.0, 0.0, 0.0};
        const double* b = Bs + (k + 4 * q - kb) * R + g;
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            dmma(acc[t], a.x, b[8 * t]);
            dmma(acc[t], a.y, b[R + 8 * t]);
            dmma(acc[t], a.z, b[2 * R + 8 * t]);
            dmma(acc[t], a.w, b[3 * R + 8 * t]);
        }
    }
#pragma unroll 4
    for (; k < k1; k += 4) {
        const int kk = k + q;
        const double a = (rowok && kk < k1) ? ld_stream(row + kk) : 0.0;
#pragma unroll
        for (int t = 0; t < NT; ++t) dmma(acc[t], a, kk < k1 ? Bs[(kk - kb) * R + 8 * t + g] : 0.0);
    }
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

// ---- work split over the CTA's warps -------------------------------------------
// Row tiles of 8; with fewer tiles than warps the K range of each tile is split
// over nsplit warps and the partial sums are added in split order (fixed:
// deterministic).  Every warp runs the same number of rounds (block barriers).
struct Split {
    int tiles, nsplit, per_round, rounds;
};

__device__ __forceinline__ Split make_split(int M) {
    Split s;
    s.tiles = (M + 7) / 8;
    s.nsplit = s.tiles >= kMmWarps ? 1 : kMmWarps / max(s.tiles, 1);
    s.per_round = kMmWarps / s.nsplit;
    s.rounds = (s.tiles + s.per_round - 1) / s.per_round;
    return s;
}

// [lo, hi) of split `sp` inside [a, b) (4-aligned pieces)
__device__ __forceinline__ void split_range(int a, int b, int nsplit, int sp, int& lo, int& hi, int align = 4) {
    const int per = (((b - a) + nsplit - 1) / nsplit + align - 1) / align * align;
    lo = min(b, a + sp * per);
    hi = min(b, lo + per);
}

// add the split partials (split 0 keeps the sum); all warps call it
template <int NT>
__device__ __forceinline__ void reduce_splits(double (&acc)[NT][2], const Split& s, double* red) {
    if (s.nsplit == 1) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int sp = warp / s.per_round;
    double* mine = red + ((size_t)warp * 32 + lane) * 2 * NT;
    __syncthreads();
    if (sp > 0)
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            mine[2 * t] = acc[t][0];
            mine[2 * t + 1] = acc[t][1];
        }
    __syncthreads();
    if (sp == 0)
        for (int q = 1; q < s.nsplit; ++q) {
            const double* o = red + ((size_t)(warp + q * s.per_round) * 32 + lane) * 2 * NT;
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                acc[t][0] += o[2 * t];
                acc[t][1] += o[2 * t + 1];
            }
        }
}

// C (M x R) = A (M x K) B with B (K x R) fully staged in Bs; out(m, n, value)
template <int NT, class FA, class FO>
__device__ void cta_product(int M, int K, FA fa, const double* Bs, double* red, FO out) {
    const Split s = make_split(M);
    const int warp = threadIdx.x >> 5;
    const int sp = warp / s.per_round;
    for (int rd = 0; rd < s.rounds; ++rd) {
        const int tile = rd * s.per_round + warp % s.per_round;
        double acc[NT][2];
        zero(acc);
        int lo, hi;
        split_range(0, K, s.nsplit, sp, lo, hi);
        if (tile < s.tiles && lo < hi) warp_mma<NT>(acc, 8 * tile, M, lo, hi, 0, fa, Bs);
        reduce_splits<NT>(acc, s, red);
        if (tile < s.tiles && sp == 0) warp_store<NT>(acc, 8 * tile, M, out);
    }
}

// C (M x R) = A (M x K, row-major, ld, streamed once) B with B row kk =
// src[idx[kk]] (src_w wide, first nrhs columns), staged kChunk rows at a time;
// then C += A2 (M x K2) B2 with B2 (K2 x R) contiguous at src2 (leaf expansion);
// out(m, n, value)
template <int NT, class FA2, class FO>
__device__ void cta_streamed(int M, const double* A, int64_t ld, int K, const int32_t* idx, const double* src,
                             int src_w, int nrhs, int K2, FA2 fa2, const double* src2, double* Bs, double* red,
                             FO out) {
    constexpr int R = 8 * NT;
    const Split s = make_split(M);
    const int warp = threadIdx.x >> 5;
    const int sp = warp / s.per_round;
    for (int rd = 0; rd < s.rounds; ++rd) {
        const int tile = rd * s.per_round + warp % s.per_round;
        const bool act = tile < s.tiles;
        double acc[NT][2];
        zero(acc);
        for (int kc = 0; kc < K; kc += kChunk) {
            const int kn = min(kChunk, K - kc);
            __syncthreads();
            for (int e = threadIdx.x; e < kn * R; e += kMmThreads) {
                const int i = e / R, r = e - i * R;
                Bs[e] = r < nrhs ? src[(int64_t)idx[kc + i] * src_w + r] : 0.0;
            }
            __syncthreads();
            int lo, hi;
            split_range(kc, kc + kn, s.nsplit, sp, lo, hi, 16);
            if (act && lo < hi) warp_mma_stream<NT>(acc, 8 * tile, M, lo, hi, kc, A, ld, Bs);
        }
        if (K2 > 0) {
            __syncthreads();
            for (int e = threadIdx.x; e < K2 * R; e += kMmThreads) Bs[e] = src2[e];
            __syncthreads();
            int lo, hi;
            split_range(0, K2, s.nsplit, sp, lo, hi);
            if (act && lo < hi) warp_mma<NT>(acc, 8 * tile, M, lo, hi, 0, fa2, Bs);
        }
        reduce_splits<NT>(acc, s, red);
        if (act && sp == 0) warp_store<NT>(acc, 8 * tile, M, out);
    }
}

// ---- tree transforms: one warp per cluster ---------------------------------------
// The per-cluster products are small (ranks ~25-50): a warp stages its B in a
// private shared-memory slice and runs all row tiles itself, so a CTA keeps
// kMmWarps clusters in flight without block barriers.

// all row tiles of C (M x R) = A (M x K) B, B staged at Bw; out(m, n, value)
template <int NT, class FA, class FO>
__device__ __forceinline__ void warp_product(int M, int K, FA fa, const double* Bw, FO out) {
    for (int m0 = 0; m0 < M; m0 += 8) {
        double acc[NT][2];
        zero(acc);
        warp_mma<NT>(acc, m0, M, 0, K, 0, fa, Bw);
        warp_store<NT>(acc, m0, M, out);
    }
}

template <int NT>
__global__ void __launch_bounds__(kMmThreads) k_mm_fwd_leaf(h2b_layout L, const int32_t* __restrict__ leaves, int n,
                                                            const double* __restrict__ X, int nrhs,
                                                            double* __restrict__ xhat, int slice) {
    constexpr int R = 8 * NT;
    extern __shared__ double Bs[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int i = blockIdx.x * kMmWarps + warp;
    if (i >= n) return;
    double* Bw = Bs + (size_t)warp * slice;
    const int t = leaves[i];
    const int start = L.c_start[t], size = L.c_size[t], k = L.c_rank[t];
    const double* V = L.c_V + L.c_v_off[t];
    for (int e = lane; e < size * R; e += 32) {
        const int r = e % R;
        Bw[e] = r < nrhs ? X[L.col_perm[start + e / R] * nrhs + r] : 0.0;
    }
    __syncwarp();
    double* out = xhat + L.c_xhat_off[t] * R;
    warp_product<NT>(k, size, [&](int m, int kk) { return V[(int64_t)kk * k + m]; }, Bw,
                     [&](int m, int c, double v) { out[m * R + c] = v; });
}

// inner levels: one CTA per cluster (split-K over the warps measured faster
// than a warp per cluster for the transfer products)
template <int NT>
__global__ void __launch_bounds__(kMmThreads) k_mm_fwd_level(h2b_layout L, const int32_t* __restrict__ nodes,
                                                             double* __restrict__ xhat, int bs_doubles) {
    constexpr int R = 8 * NT;
    extern __shared__ double Bs[];
    double* red = Bs + bs_doubles;
    const int p = nodes[blockIdx.x];
    const int kp = L.c_rank[p];
    const int c0 = L.c_child[2 * p], c1 = L.c_child[2 * p + 1];
    const int k0 = L.c_rank[c0], k1 = L.c_rank[c1];
    // B = [x_hat_c0; x_hat_c1] ((k0 + k1) x R), A = [E_c0^T, E_c1^T] (kp x (k0 + k1))
    const double* x0 = xhat + L.c_xhat_off[c0] * R;
    const double* x1 = xhat + L.c_xhat_off[c1] * R;
    for (int e = threadIdx.x; e < (k0 + k1) * R; e += kMmThreads) Bs[e] = e < k0 * R ? x0[e] : x1[e - k0 * R];
    __syncthreads();
    const double* E0 = L.c_E + L.c_e_off[c0];
    const double* E1 = L.c_E + L.c_e_off[c1];
    double* out = xhat + L.c_xhat_off[p] * R;
    cta_product<NT>(kp, k0 + k1,
                    [&](int m, int kk) { return kk < k0 ? E0[(int64_t)kk * kp + m] : E1[(int64_t)(kk - k0) * kp + m]; },
                    Bs, red, [&](int m, int n, double v) { out[m * R + n] = v; });
}

template <int NT>
__global__ void __launch_bounds__(kMmThreads) k_mm_bwd_level(h2b_layout L, const int32_t* __restrict__ nodes,
                                                             const double* __restrict__ ycpl, double* __restrict__ v,
                                                             int bs_doubles) {
    constexpr int R = 8 * NT;
    extern __shared__ double Bs[];
    double* red = Bs + bs_doubles;
    const int t = nodes[blockIdx.x];
    const int k = L.r_rank[t], p = L.r_parent[t];
    const bool cpl = L.s_cols[t] > 0;
    const int kp = p >= 0 ? L.r_rank[p] : 0;
    if (kp > 0) {
        const double* vp = v + L.r_yhat_off[p] * R;
        for (int e = threadIdx.x; e < kp * R; e += kMmThreads) Bs[e] = vp[e];
    }
    __syncthreads();
    const double* E = L.r_E + (p >= 0 ? L.r_e_off[t] : 0);
    const double* yc = ycpl + L.r_yhat_off[t] * R;
    double* out = v + L.r_yhat_off[t] * R;
    cta_product<NT>(k, kp, [&](int m, int kk) { return E[(int64_t)m * kp + kk]; }, Bs, red,
                    [&](int m, int n, double val) { out[m * R + n] = val + (cpl ? yc[m * R + n] : 0.0); });
}

// ---- fused tree transforms (one launch each) --------------------------------------
// Tasks are ticketed (atomic counter, monotonic over launches: epoch = t / n + 1)
// in dependency order -- leaves, then inner clusters deepest first (forward);
// parents first (backward) -- and a task waits only on flags of smaller
// tickets, so any residency makes progress.  A finished cluster publishes its
// coefficients with a release store of the epoch into its flag.
__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release_u32(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void wait_flag(const uint32_t* f, uint32_t ep) {
    while (ld_acquire_u32(f) != ep) __nanosleep(64);
}

template <int NT>
__global__ void __launch_bounds__(kMmThreads) k_mm_fwd_fused(h2b_layout L, const int32_t* __restrict__ leaves,
                                                             int n_leaves, const int32_t* __restrict__ inner,
                                                             int n_inner, const double* __restrict__ X, int nrhs,
                                                             double* xhat, uint32_t* flags,
                                                             unsigned long long* ctr, int bs_doubles) {
    constexpr int R = 8 * NT;
    extern __shared__ double Bs[];
    double* red = Bs + bs_doubles;
    __shared__ int s_task;
    __shared__ uint32_t s_ep;
    const int n = n_leaves + n_inner;
    if (threadIdx.x == 0) {
        const unsigned long long t = atomicAdd(ctr, 1ull);
        s_task = (int)(t % (unsigned long long)n);
        s_ep = (uint32_t)(t / (unsigned long long)n) + 1u;
    }
    __syncthreads();
    const int task = s_task;
    const uint32_t ep = s_ep;
    int node;
    if (task < n_leaves) {
        node = leaves[task];
        const int start = L.c_start[node], size = L.c_size[node], k = L.c_rank[node];
        const double* V = L.c_V + L.c_v_off[node];
        for (int e = threadIdx.x; e < size * R; e += kMmThreads) {
            const int r = e % R;
            Bs[e] = r < nrhs ? X[L.col_perm[start + e / R] * nrhs + r] : 0.0;
        }
        __syncthreads();
        double* out = xhat + L.c_xhat_off[node] * R;
        cta_product<NT>(k, size, [&](int m, int kk) { return V[(int64_t)kk * k + m]; }, Bs, red,
                        [&](int m, int c, double v) { out[m * R + c] = v; });
    } else {
        node = inner[task - n_leaves];
        const int kp = L.c_rank[node];
        const int c0 = L.c_child[2 * node], c1 = L.c_child[2 * node + 1];
        const int k0 = L.c_rank[c0], k1 = L.c_rank[c1];
        if (threadIdx.x == 0) {
            wait_flag(flags + c0, ep);
            wait_flag(flags + c1, ep);
        }
        __syncthreads();
        const double* x0 = xhat + L.c_xhat_off[c0] * R;
        const double* x1 = xhat + L.c_xhat_off[c1] * R;
        for (int e = threadIdx.x; e < (k0 + k1) * R; e += kMmThreads)
            Bs[e] = e < k0 * R ? __ldcg(x0 + e) : __ldcg(x1 + e - k0 * R);
        __syncthreads();
        const double* E0 = L.c_E + L.c_e_off[c0];
        const double* E1 = L.c_E + L.c_e_off[c1];
        double* out = xhat + L.c_xhat_off[node] * R;
        cta_product<NT>(kp, k0 + k1,
                        [&](int m, int kk) {
                            return kk < k0 ? E0[(int64_t)kk * kp + m] : E1[(int64_t)(kk - k0) * kp + m];
                        },
                        Bs, red, [&](int m, int c, double v) { out[m * R + c] = v; });
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        st_release_u32(flags + node, ep);
    }
}

template <int NT>
__global__ void __launch_bounds__(kMmThreads) k_mm_bwd_fused(h2b_layout L, const int32_t* __restrict__ nodes, int n,
                                                             const double* __restrict__ ycpl, double* v,
                                                             uint32_t* flags, unsigned long long* ctr,
                                                             int bs_doubles) {
    constexpr int R = 8 * NT;
    extern __shared__ double Bs[];
    double* red = Bs + bs_doubles;
    __shared__ int s_task;
    __shared__ uint32_t s_ep;
    if (threadIdx.x == 0) {
        const unsigned long long t = atomicAdd(ctr, 1ull);
        s_task = (int)(t % (unsigned long long)n);
        s_ep = (uint32_t)(t / (unsigned long long)n) + 1u;
    }
    __syncthreads();
    const int t = nodes[s_task];
    const uint32_t ep = s_ep;
    const int k = L.r_rank[t], p = L.r_parent[t];
    const bool cpl = L.s_cols[t] > 0;
    const int kp = p >= 0 ? L.r_rank[p] : 0;
    if (kp > 0) {
        if (threadIdx.x == 0) wait_flag(flags + p, ep);
        __syncthreads();
        const double* vp = v + L.r_yhat_off[p] * R;
        for (int e = threadIdx.x; e < kp * R; e += kMmThreads) Bs[e] = __ldcg(vp + e);
    }
    __syncthreads();
    const double* E = L.r_E + (p >= 0 ? L.r_e_off[t] : 0);
    const double* yc = ycpl + L.r_yhat_off[t] * R;
    double* out = v + L.r_yhat_off[t] * R;
    cta_product<NT>(k, kp, [&](int m, int kk) { return E[(int64_t)m * kp + kk]; }, Bs, red,
                    [&](int m, int c, double val) { out[m * R + c] = val + (cpl ? yc[m * R + c] : 0.0); });
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        st_release_u32(flags + t, ep);
    }
}

// ---- couplings, downward transform, nearfield ------------------------------------

template <int NT>
__global__ void __launch_bounds__(kMmThreads) k_mm_cpl(h2b_layout L, const int32_t* __restrict__ nodes,
                                                       const double* __restrict__ xhat, double* __restrict__ ycpl,
                                                       int bs_doubles) {
    constexpr int R = 8 * NT;
    extern __shared__ double Bs[];
    double* red = Bs + bs_doubles;
    const int t = nodes[blockIdx.x];
    const int k = L.r_rank[t], K = L.s_cols[t];
    double* out = ycpl + L.r_yhat_off[t] * R;
    cta_streamed<NT>(k, L.S + L.s_off[t], K, K, L.s_gidx + L.s_goff[t], xhat, R, R, 0,
                     [](int, int) { return 0.0; }, nullptr, Bs, red,
                     [&](int m, int n, double v) { out[m * R + n] = v; });
}

template <int NT>
__global__ void __launch_bounds__(kMmThreads) k_mm_leaf(h2b_layout L, const int32_t* __restrict__ leaves,
                                                        const double* __restrict__ X, int nrhs,
                                                        const double* __restrict__ v, double* __restrict__ Y,
                                                        int bs_doubles) {
    constexpr int R = 8 * NT;
    extern __shared__ double Bs[];
    double* red = Bs + bs_doubles;
    const int t = leaves[blockIdx.x];
    const int start = L.r_start[t], size = L.r_size[t], k = L.r_rank[t], C = L.d_cols[t];
    const double* V = L.r_V + L.r_v_off[t];
    cta_streamed<NT>(size, L.D + L.d_off[t], C, C, L.d_gidx + L.d_goff[t], X, nrhs, nrhs, k,
                     [&](int m, int kk) { return V[(int64_t)m * k + kk]; }, v + L.r_yhat_off[t] * R, Bs, red,
                     [&](int m, int n, double val) {
                         if (n < nrhs) Y[L.row_perm[start + m] * nrhs + n] = val;
                     });
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
    // streamed products: a chunk of gathered rows (or a leaf's ranks) + the
    // split-reduction buffer; tree transforms: one B slice per warp
    const int bs = std::max(std::max(kChunk, p->max_c_node), 64) * R;
    const size_t sm = (size_t)(bs + kMmWarps * 32 * 2 * NT) * sizeof(double);
    const int slice = std::max(p->max_c_node, 64) * R;
    const size_t sm_tree = (size_t)kMmWarps * slice * sizeof(double);
    for (auto* f : {(const void*)k_mm_cpl<NT>, (const void*)k_mm_leaf<NT>, (const void*)k_mm_fwd_level<NT>,
                    (const void*)k_mm_bwd_level<NT>})
        H2B_CUDA_TRY(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    for (auto* f : {(const void*)k_mm_fwd_leaf<NT>})
        H2B_CUDA_TRY(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_tree));
    auto blocks = [](int64_t n) { return (unsigned)((n + kMmWarps - 1) / kMmWarps); };
    // fused tree launches pay off where launches dominate (config 1: 0.26 -> 0.21 ms
    // for 8 RHS); on large trees the waiting tasks cost more than the level
    // launches (sphere L8: 1.44 vs 1.52 ms), so the level kernels are kept there
    // (H2B_MM_LEVELS=0/1 forces either)
    const int64_t n_inner = p->fwd_level_off.back(), n_bwd = p->bwd_level_off.back();
    const char* lv_env = getenv("H2B_MM_LEVELS");
    const bool levels = lv_env ? lv_env[0] == '1' : (p->n_leaf_c + n_inner > 8192);
    if (!levels) {
        for (auto* f : {(const void*)k_mm_fwd_fused<NT>, (const void*)k_mm_bwd_fused<NT>})
            H2B_CUDA_TRY(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        if (p->n_leaf_c + n_inner > 0)
            k_mm_fwd_fused<NT><<<(unsigned)(p->n_leaf_c + n_inner), kMmThreads, sm, st>>>(
                L, lists + p->off_leaf_c, (int)p->n_leaf_c, lists + p->off_fwd, (int)n_inner, X, nrhs, p->xhat,
                p->flags, p->ctr, bs);
        if (p->n_cpl > 0)
            k_mm_cpl<NT><<<(unsigned)p->n_cpl, kMmThreads, sm, st>>>(L, lists + p->off_cpl, p->xhat, p->ycpl, bs);
        if (n_bwd > 0)
            k_mm_bwd_fused<NT><<<(unsigned)n_bwd, kMmThreads, sm, st>>>(L, lists + p->off_bwd, (int)n_bwd, p->ycpl,
                                                                       p->v, p->flags + L.c_nodes, p->ctr + 1, bs);
    } else {
    if (p->n_leaf_c > 0)
        k_mm_fwd_leaf<NT><<<blocks(p->n_leaf_c), kMmThreads, sm_tree, st>>>(L, lists + p->off_leaf_c,
                                                                           (int)p->n_leaf_c, X, nrhs, p->xhat, slice);
    for (int lv = 0; lv + 1 < (int)p->fwd_level_off.size(); ++lv) {
        const int64_t a = p->fwd_level_off[lv], b = p->fwd_level_off[lv + 1];
        if (b > a)
            k_mm_fwd_level<NT><<<(unsigned)(b - a), kMmThreads, sm, st>>>(L, lists + p->off_fwd + a, p->xhat, bs);
    }
    if (p->n_cpl > 0)
        k_mm_cpl<NT><<<(unsigned)p->n_cpl, kMmThreads, sm, st>>>(L, lists + p->off_cpl, p->xhat, p->ycpl, bs);
    for (int lv = 0; lv + 1 < (int)p->bwd_level_off.size(); ++lv) {
        const int64_t a = p->bwd_level_off[lv], b = p->bwd_level_off[lv + 1];
        if (b > a)
            k_mm_bwd_level<NT><<<(unsigned)(b - a), kMmThreads, sm, st>>>(L, lists + p->off_bwd + a, p->ycpl, p->v,
                                                                         bs);
    }
    }
    if (p->n_leaf_r > 0)
        k_mm_leaf<NT><<<(unsigned)p->n_leaf_r, kMmThreads, sm, st>>>(L, lists + p->off_leaf_r, X, nrhs, p->v, Y, bs);
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
    H2B_CUDA_TRY(alloc(reinterpret_cast<void**>(&p->flags), sizeof(uint32_t) * ((size_t)L.c_nodes + L.r_nodes)));
    H2B_CUDA_TRY(cudaMemset(p->flags, 0, sizeof(uint32_t) * ((size_t)L.c_nodes + L.r_nodes)));
    H2B_CUDA_TRY(alloc(reinterpret_cast<void**>(&p->ctr), 2 * sizeof(unsigned long long)));
    H2B_CUDA_TRY(cudaMemset(p->ctr, 0, 2 * sizeof(unsigned long long)));
    *out = p;
    return ok();
}

extern "C" int h2b_matmat_destroy(h2b_mmplan* p) {
    if (!p) return ok();
    for (void* q : {(void*)p->d_lists, (void*)p->xhat, (void*)p->ycpl, (void*)p->v, (void*)p->flags, (void*)p->ctr})
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
