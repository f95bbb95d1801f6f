// Galerkin panel-pair quadrature for the Laplace single- and double-layer
// operators on flat triangles, fp64, sm_100a.
//
//   k_panel_points   regular Duffy tensor rule on every panel   (quadrature.py:58-87)
//   k_touch_*        touching-pair enumeration + Sauter-Schwab case/permutation
//                    classification                               (kernels.py:246-254,333-343;
//                                                                  quadrature.py:90-118)
//   k_singular       Sauter-Schwab integrals of all touching pairs (kernels.py:260-319)
//   k_blocks_slp     dense SLP blocks: regular tensor rule, touching pairs patched
//                    from the singular table                      (kernels.py:365-445)
//   k_blocks_dlp     dense DLP blocks with the P1 vertex scatter  (kernels.py:365-434,448-468)
//
// All quadrature loops are FP64-pipe bound.  1/r is a hardware rsqrt seed plus
// one Newton correction folded into the accumulation; squared distances of
// regular pairs use the Gram form on block-centred coordinates (the
// reference's _dist2, kernels.py:75-85, without its cancellation because both
// point sets are shifted to a block-local origin first).

#include <climits>
#include <cstdlib>

#include <cub/device/device_scan.cuh>

#include "device_common.cuh"

// tuning knobs of the regular SLP kernel (see launch_slp)
#ifndef H2B_SLP_UNROLL_OUTER
#define H2B_SLP_UNROLL_OUTER 16
#endif
constexpr int kSlpUnroll = H2B_SLP_UNROLL_OUTER;
#ifndef H2B_DLP_XN_REG
#define H2B_DLP_XN_REG 0  // x'.n of the row points in registers per pair (needs the row loop unrolled)
#endif
#ifndef H2B_DLP_UI
#define H2B_DLP_UI 3      // unroll of the row-point loop (sphere L8 DLP regular: 52.4 ms at 3, 55.2 ms at 1)
#endif
constexpr int kDlpUnroll = H2B_DLP_UI;
#ifndef H2B_SLP_THREADS
#define H2B_SLP_THREADS 128  // threads per pair-block CTA (128 x 4 CTAs/SM measured 2 % faster than 256 x 2)
#endif

namespace h2b {
namespace {

constexpr int kTile = 64;       // max rows / columns of one pair-block job
constexpr int kSlpLd = kTile + 1;  // padded point stride of the SLP stage (staging stores ~2-way, not 9-way, bank conflicts)
constexpr int kDlpMaxPanels = 128;  // max column panels of one DLP job
constexpr int kDlpRowChunk = 8;

// flags bits (reduced per launch, mapped to the reference's exceptions)
constexpr int kFlagNonFinite = 1;
constexpr int kFlagTouching = 2;
constexpr int kFlagMissing = 4;
constexpr int kFlagShape = 8;
constexpr int kFlagCandidates = 16;

// ----------------------------------------------------------------------------
// regular panel points
__global__ void k_panel_points(const double* __restrict__ V, const int32_t* __restrict__ T,
                               const double* __restrict__ A, int64_t F,
                               const double* __restrict__ rxy, const double* __restrict__ rw, int Q,
                               double* __restrict__ out) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= F * Q) return;
    const int64_t f = e / Q;
    const int j = (int)(e - f * Q);
    const int i0 = T[3 * f], i1 = T[3 * f + 1], i2 = T[3 * f + 2];
    const double x = rxy[2 * j], y = rxy[2 * j + 1];
    const int64_t FQ = F * Q;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const double c0 = V[3 * i0 + k], c1 = V[3 * i1 + k], c2 = V[3 * i2 + k];
        // c0 + x (c1 - c0) + y (c2 - c0), evaluated as written (no contraction)
        out[k * FQ + e] = __dadd_rn(__dadd_rn(c0, __dmul_rn(x, c1 - c0)), __dmul_rn(y, c2 - c0));
    }
    out[3 * FQ + e] = rw[j] * (2.0 * A[f]);
}

// ----------------------------------------------------------------------------
// touching pairs
// The touching panels of panel a (sharing >= 1 vertex, a itself included),
// ascending and unique: a three-way merge of its vertices' incident-triangle
// lists (each ascending, Mesh.vertex_triangle_csr), streamed to f(b, i) with
// no per-thread candidate array.
template <class Fn>
__device__ __forceinline__ int for_each_touching(const int32_t* __restrict__ T, const int64_t* __restrict__ vt_ptr,
                                                 const int32_t* __restrict__ vt_idx, int64_t a, Fn&& f) {
    int64_t p[3], e[3];
    int h[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const int v = T[3 * a + k];
        p[k] = vt_ptr[v];
        e[k] = vt_ptr[v + 1];
        h[k] = p[k] < e[k] ? vt_idx[p[k]] : INT_MAX;
    }
    int n = 0, last = -1;
    while (true) {
        const int m = min(h[0], min(h[1], h[2]));
        if (m == INT_MAX) break;
#pragma unroll
        for (int k = 0; k < 3; ++k)
            if (h[k] == m) {
                ++p[k];
                h[k] = p[k] < e[k] ? vt_idx[p[k]] : INT_MAX;
            }
        if (m != last) {
            f(m, n);
            ++n;
            last = m;
        }
    }
    return n;
}

// quadrature.py:90-118: case = #shared vertices (3 when identical); shared
// vertices first in ascending global id, remaining local vertices in order.
__device__ int classify(const int* ta, const int* tb, bool same) {
    if (same) return H2B_IDENTICAL | (0 << 2) | (1 << 4) | (2 << 6) | (0 << 8) | (1 << 10) | (2 << 12);
    int sa[3], sb[3], ns = 0;
    // shared vertices, ascending global id
    int sh[3];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            if (ta[i] == tb[j]) sh[ns++] = ta[i];
    if (ns == 2 && sh[0] > sh[1]) {
        const int t = sh[0];
        sh[0] = sh[1];
        sh[1] = t;
    }
    if (ns == 0) return H2B_DISJOINT | (0 << 2) | (1 << 4) | (2 << 6) | (0 << 8) | (1 << 10) | (2 << 12);
    int pa[3], pb[3];
    for (int s = 0; s < ns; ++s) {
        for (int i = 0; i < 3; ++i) {
            if (ta[i] == sh[s]) sa[s] = i;
            if (tb[i] == sh[s]) sb[s] = i;
        }
        pa[s] = sa[s];
        pb[s] = sb[s];
    }
    int ka = ns, kb = ns;
    for (int i = 0; i < 3; ++i) {
        bool ua = false, ub = false;
        for (int s = 0; s < ns; ++s) {
            ua |= (sa[s] == i);
            ub |= (sb[s] == i);
        }
        if (!ua) pa[ka++] = i;
        if (!ub) pb[kb++] = i;
    }
    const int code = ns == 2 ? H2B_EDGE : H2B_VERTEX;
    return code | (pa[0] << 2) | (pa[1] << 4) | (pa[2] << 6) | (pb[0] << 8) | (pb[1] << 10) |
           (pb[2] << 12);
}

__global__ void k_touch_count(const int32_t* __restrict__ T, int64_t F,
                              const int64_t* __restrict__ vt_ptr, const int32_t* __restrict__ vt_idx,
                              int64_t* __restrict__ counts, unsigned long long* __restrict__ case_count,
                              int* flags) {
    const int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    __shared__ unsigned long long sc[4];
    if (threadIdx.x < 4) sc[threadIdx.x] = 0;
    __syncthreads();
    if (a < F) {
        const int ta[3] = {T[3 * a], T[3 * a + 1], T[3 * a + 2]};
        int c[4] = {0, 0, 0, 0};
        const int m = for_each_touching(T, vt_ptr, vt_idx, a, [&](int b, int) {
            const int tb[3] = {T[3 * b], T[3 * b + 1], T[3 * b + 2]};
            c[classify(ta, tb, b == a) & 3]++;
        });
        counts[a] = m;
        for (int k = 1; k < 4; ++k)
            if (c[k]) atomicAdd(&sc[k], (unsigned long long)c[k]);
        if (c[0]) atomicOr(flags, kFlagCandidates);  // cannot happen on a valid mesh
    }
    __syncthreads();
    if (threadIdx.x > 0 && threadIdx.x < 4 && sc[threadIdx.x]) atomicAdd(&case_count[threadIdx.x], sc[threadIdx.x]);
}

__global__ void k_touch_fill(const int32_t* __restrict__ T, int64_t F,
                             const int64_t* __restrict__ vt_ptr, const int32_t* __restrict__ vt_idx,
                             const int64_t* __restrict__ row_ptr, int32_t* __restrict__ col,
                             int32_t* __restrict__ info, int32_t* __restrict__ seg_count, int* flags) {
    const int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= F) return;
    const int ta[3] = {T[3 * a], T[3 * a + 1], T[3 * a + 2]};
    const int64_t base = row_ptr[a];
    int c[3] = {0, 0, 0};
    for_each_touching(T, vt_ptr, vt_idx, a, [&](int b, int i) {
        const int tb[3] = {T[3 * b], T[3 * b + 1], T[3 * b + 2]};
        const int inf = classify(ta, tb, b == a);
        col[base + i] = b;
        info[base + i] = inf;
        const int code = inf & 3;
        c[code == H2B_IDENTICAL ? 0 : (code == H2B_EDGE ? 1 : 2)]++;
    });
    // per-panel case counts, segment-major: one scan over [3][F] gives every
    // pair its slot in the case-grouped list (no contended atomics: a global
    // cursor per case serialised ~27 M atomics at config 3)
    seg_count[a] = c[0];
    seg_count[F + a] = c[1];
    seg_count[2 * F + a] = c[2];
}

// case-grouped pair list: segment k, rows ascending, columns ascending
__global__ void k_touch_list(const int64_t* __restrict__ row_ptr, int64_t F, const int32_t* __restrict__ info,
                             const int32_t* __restrict__ seg_pos, int32_t* __restrict__ case_list) {
    const int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= F) return;
    int pos[3] = {seg_pos[a], seg_pos[F + a], seg_pos[2 * F + a]};
    for (int64_t p = row_ptr[a]; p < row_ptr[a + 1]; ++p) {
        const int code = info[p] & 3;
        const int seg = code == H2B_IDENTICAL ? 0 : (code == H2B_EDGE ? 1 : 2);
        case_list[pos[seg]++] = (int32_t)p;
    }
}

// unordered (a < b) edge / vertex pairs per row panel, segment-major [2][F]
__global__ void k_half_count(const int64_t* __restrict__ row_ptr, int64_t F, const int32_t* __restrict__ col,
                             const int32_t* __restrict__ info, int32_t* __restrict__ cnt) {
    const int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= F) return;
    int ce = 0, cv = 0;
    for (int64_t p = row_ptr[a]; p < row_ptr[a + 1]; ++p) {
        if (col[p] <= a) continue;
        const int code = info[p] & 3;
        ce += code == H2B_EDGE;
        cv += code == H2B_VERTEX;
    }
    cnt[a] = ce;
    cnt[F + a] = cv;
}

__global__ void k_half_fill(const int64_t* __restrict__ row_ptr, int64_t F, const int32_t* __restrict__ col,
                            const int32_t* __restrict__ info, const int32_t* __restrict__ pos_in,
                            int64_t base, int32_t* __restrict__ half) {
    const int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= F) return;
    int64_t pe = base + pos_in[a], pv = base + pos_in[F + a];
    for (int64_t p = row_ptr[a]; p < row_ptr[a + 1]; ++p) {
        if (col[p] <= a) continue;
        const int code = info[p] & 3;
        if (code == H2B_EDGE) half[pe++] = (int32_t)p;
        else if (code == H2B_VERTEX) half[pv++] = (int32_t)p;
    }
}


// case code + permutations of arbitrary pairs (kernels.pair_integrals),
// counted per segment: 0 identical, 1 edge, 2 vertex, 3 disjoint
__device__ __forceinline__ int seg_of(int code) {
    return code == H2B_IDENTICAL ? 0 : code == H2B_EDGE ? 1 : code == H2B_VERTEX ? 2 : 3;
}

__global__ void k_classify_list(const int32_t* __restrict__ T, int64_t n, const int32_t* __restrict__ pa,
                                const int32_t* __restrict__ pb, int32_t* __restrict__ info,
                                unsigned long long* __restrict__ count) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int a = pa[i], b = pb[i];
    const int ta[3] = {T[3 * a], T[3 * a + 1], T[3 * a + 2]};
    const int tb[3] = {T[3 * b], T[3 * b + 1], T[3 * b + 2]};
    const int inf = classify(ta, tb, a == b);
    info[i] = inf;
    atomicAdd(&count[seg_of(inf & 3)], 1ull);
}

__global__ void k_bucket_list(int64_t n, const int32_t* __restrict__ info, int32_t* __restrict__ list,
                              unsigned long long* __restrict__ cursor) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    list[atomicAdd(&cursor[seg_of(info[i] & 3)], 1ull)] = (int32_t)i;
}

// ----------------------------------------------------------------------------
// Sauter-Schwab integrals
struct SegDesc {
    int64_t list_off, count;
    int32_t first_block, n_blocks;
    const double* p;
    const double* w;
    int64_t n;
    int kase;  // H2B_IDENTICAL / H2B_EDGE / H2B_VERTEX / H2B_DISJOINT
};

struct SegSet {
    SegDesc s[4];
    int nseg;
};

constexpr int kRuleChunk = 256;
constexpr int kRuleStride = 8;

__device__ __forceinline__ int64_t find_row(const int64_t* __restrict__ row_ptr, int64_t F, int64_t pid) {
    int64_t lo = 0, hi = F;  // row_ptr[lo] <= pid < row_ptr[hi]
    while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (row_ptr[mid] <= pid) lo = mid; else hi = mid;
    }
    return lo;
}

template <int KIND>
__global__ void __launch_bounds__(128) k_singular(const double* __restrict__ V, const int32_t* __restrict__ T,
                                                 const double* __restrict__ Nrm, const double* __restrict__ Ar,
                                                 const int64_t* __restrict__ row_ptr, int64_t F,
                                                 const int32_t* __restrict__ col, const int32_t* __restrict__ info,
                                                 const int32_t* __restrict__ case_list, SegSet segs,
                                                 double* __restrict__ values, int mirror,
                                                 const int32_t* __restrict__ pa_list) {
    __shared__ double srule[kRuleChunk * kRuleStride];
    int si = 0;
    while (si + 1 < segs.nseg && (int)blockIdx.x >= segs.s[si + 1].first_block) ++si;
    const SegDesc sd = segs.s[si];
    const int kase = sd.kase;
    const int64_t local = (int64_t)(blockIdx.x - sd.first_block) * blockDim.x + threadIdx.x;
    const bool active = local < sd.count;

    double base[3] = {0, 0, 0}, ea1[3] = {0, 0, 0}, ea2[3] = {0, 0, 0}, eb1[3] = {0, 0, 0},
           eb2[3] = {0, 0, 0}, nb[3] = {0, 0, 0};
    double scale = 0.0;
    int64_t pid = 0, a = 0;
    int inf = 0, b = 0;
    if (active) {
        pid = case_list[sd.list_off + local];
        // touching table: the row panel from the CSR; pair list: given
        a = pa_list ? (int64_t)pa_list[pid] : find_row(row_ptr, F, pid);
        b = col[pid];
        inf = info[pid];
        int pa[3] = {(inf >> 2) & 3, (inf >> 4) & 3, (inf >> 6) & 3};
        int pb[3] = {(inf >> 8) & 3, (inf >> 10) & 3, (inf >> 12) & 3};
        double ca[3][3], cb[3][3];
        for (int r = 0; r < 3; ++r) {
            const int va = T[3 * a + pa[r]], vb = T[3 * b + pb[r]];
            for (int k = 0; k < 3; ++k) {
                ca[r][k] = V[3 * va + k];
                cb[r][k] = V[3 * vb + k];
            }
        }
        for (int k = 0; k < 3; ++k) {
            base[k] = ca[0][k] - cb[0][k];
            ea1[k] = ca[1][k] - ca[0][k];
            ea2[k] = ca[2][k] - ca[1][k];
            eb1[k] = -(cb[1][k] - cb[0][k]);
            eb2[k] = -(cb[2][k] - cb[1][k]);
            nb[k] = Nrm[3 * b + k];
        }
        scale = 4.0 * Ar[a] * Ar[b];
    }

    double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0;
    const bool sym = (KIND == H2B_SLP) && (kase == H2B_EDGE || kase == H2B_VERTEX);
    for (int64_t c0 = 0; c0 < sd.n; c0 += kRuleChunk) {
        const int cn = (int)min((int64_t)kRuleChunk, sd.n - c0);
        __syncthreads();
        for (int e = threadIdx.x; e < cn; e += blockDim.x) {
            const double* p = sd.p + 4 * (c0 + e);
            const double w = sd.w[c0 + e];
            double* d = srule + e * kRuleStride;
            if (KIND == H2B_SLP && kase != H2B_DISJOINT) {
                // sums and differences of the two charts' coordinates: both
                // orientations of a symmetrised pair share the sum terms.
                // Scaled by 1/w: the distance vectors come out divided by the
                // weight, so the rsqrt seed of r^2/w^2 is already w t (the
                // weight costs no product per evaluation; w > 0)
                const double iw = 1.0 / w;
                d[0] = (p[0] + p[2]) * iw;
                d[1] = (p[1] + p[3]) * iw;
                d[2] = (p[0] - p[2]) * iw;
                d[3] = (p[1] - p[3]) * iw;
                d[4] = w;
            } else {
                d[0] = p[0];
                d[1] = p[1];
                d[2] = p[2];
                d[3] = p[3];
                d[4] = w;
                d[5] = w * (1.0 - p[2]);
                d[6] = w * (p[2] - p[3]);
                d[7] = w * p[3];
            }
        }
        __syncthreads();
        if (!active) continue;
        if (kase == H2B_DISJOINT) {
            // pair list only (kernels.pair_integrals on separated panels): the
            // tensor rule of quadrature.py:171-180 through both charts,
            // d = (A1 - B1) + u1 E_a1 + v1 E_a2 - u2 E_b1 - v2 E_b2
#pragma unroll 2
            for (int e = 0; e < cn; ++e) {
                const double* d = srule + e * kRuleStride;
                const double u1 = d[0], v1 = d[1], u2 = d[2], v2 = d[3], w = d[4];
                double dd[3];
#pragma unroll
                for (int k = 0; k < 3; ++k)
                    dd[k] = fma(v2, eb2[k], fma(u2, eb1[k], fma(v1, ea2[k], fma(u1, ea1[k], base[k]))));
                const double r2 = fma(dd[2], dd[2], fma(dd[1], dd[1], dd[0] * dd[0]));
                const double t = rsqrt_seed(r2);
                const double sq = t * t;
                if (KIND == H2B_SLP) {
                    acc0 = fma(w * t, fma(-r2, sq, 3.0), acc0);
                } else {
                    const double num = fma(dd[2], nb[2], fma(dd[1], nb[1], dd[0] * nb[0]));
                    const double k = (num * fma(-r2, sq, 5.0 / 3.0)) * (sq * t);
                    acc0 = fma(k, d[5], acc0);
                    acc1 = fma(k, d[6], acc1);
                    acc2 = fma(k, d[7], acc2);
                }
            }
        } else if (KIND == H2B_SLP) {
            if (kase == H2B_IDENTICAL) {
                // same panel: d = (u1-u2) E1 + (v1-v2) E2 (base = 0), so
                // r^2 = du (du |E1|^2 + 2 dv E1.E2) + dv^2 |E2|^2 (a 2x2 Gram form)
                const double g11 = fma(ea1[2], ea1[2], fma(ea1[1], ea1[1], ea1[0] * ea1[0]));
                const double g12 = 2.0 * fma(ea1[2], ea2[2], fma(ea1[1], ea2[1], ea1[0] * ea2[0]));
                const double g22 = fma(ea2[2], ea2[2], fma(ea2[1], ea2[1], ea2[0] * ea2[0]));
#pragma unroll 4
                for (int e = 0; e < cn; ++e) {
                    const double* d = srule + e * kRuleStride;
                    const double du = d[2], dv = d[3];  // u1 - u2, v1 - v2
                    const double r2 = fma(du, fma(du, g11, dv * g12), (dv * dv) * g22);  // r^2 / w^2
                    const double t = rsqrt_seed(r2);
                    const double s = t * t;
                    const double c = fma(-r2, s, 3.0);
                    acc0 = fma(t, c, acc0);
                }
            } else {
                // shared vertex first in both charts, so base = 0 and
                //   d  = u1 E_a1 + v1 E_a2 + u2 E_b1 + v2 E_b2      (E_b negated)
                //   d' = u2 E_a1 + v2 E_a2 + u1 E_b1 + v1 E_b2      (swapped rule)
                // = c +- e with c = s P + s' Q, e = m M + m' N over the sums
                // s = u1 + u2, s' = v1 + v2 and differences m = u1 - u2, m' = v1 - v2
                double P[3], M[3], Qv[3], N[3];
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    P[k] = 0.5 * (ea1[k] + eb1[k]);
                    M[k] = 0.5 * (ea1[k] - eb1[k]);
                    Qv[k] = 0.5 * (ea2[k] + eb2[k]);
                    N[k] = 0.5 * (ea2[k] - eb2[k]);
                }
#pragma unroll 2
                for (int e = 0; e < cn; ++e) {
                    const double* d = srule + e * kRuleStride;
                    const double su = d[0], sv = d[1], mu = d[2], mv = d[3];  // scaled by 1/w
                    double dp[3], dm[3];
#pragma unroll
                    for (int k = 0; k < 3; ++k) {
                        const double c = fma(sv, Qv[k], su * P[k]);
                        const double ee = fma(mv, N[k], mu * M[k]);
                        dp[k] = c + ee;
                        dm[k] = c - ee;
                    }
                    double r2 = fma(dp[2], dp[2], fma(dp[1], dp[1], dp[0] * dp[0]));
                    double t = rsqrt_seed(r2);
                    double sq = t * t;
                    double cc = fma(-r2, sq, 3.0);
                    acc0 = fma(t, cc, acc0);
                    // orientation-swapped rule (kernels.py:303-309)
                    r2 = fma(dm[2], dm[2], fma(dm[1], dm[1], dm[0] * dm[0]));
                    t = rsqrt_seed(r2);
                    sq = t * t;
                    cc = fma(-r2, sq, 3.0);
                    acc1 = fma(t, cc, acc1);
                }
            }
        } else {
            // DLP: <x - y, n_b> / r^3 weighted by the column chart barycentrics.
            // The shared vertex comes first in both charts (base = 0) and E_b1,
            // E_b2 lie in panel b's plane, so <x - y, n_b> = u1 <E_a1, n_b> +
            // v1 <E_a2, n_b> (the E_b terms are rounding noise)
            const double al = fma(ea1[2], nb[2], fma(ea1[1], nb[1], ea1[0] * nb[0]));
            const double be = fma(ea2[2], nb[2], fma(ea2[1], nb[1], ea2[0] * nb[0]));
#pragma unroll 2
            for (int e = 0; e < cn; ++e) {
                const double* d = srule + e * kRuleStride;
                const double u1 = d[0], v1 = d[1], u2 = d[2], v2 = d[3];
                const double dx = fma(v2, eb2[0], fma(u2, eb1[0], fma(v1, ea2[0], u1 * ea1[0])));
                const double dy = fma(v2, eb2[1], fma(u2, eb1[1], fma(v1, ea2[1], u1 * ea1[1])));
                const double dz = fma(v2, eb2[2], fma(u2, eb1[2], fma(v1, ea2[2], u1 * ea1[2])));
                const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
                const double t = rsqrt_seed(r2);
                const double s = t * t;
                const double c3 = fma(-r2, s, 5.0 / 3.0);
                const double num = fma(v1, be, u1 * al);
                const double k = (num * c3) * (s * t);
                acc0 = fma(k, d[5], acc0);
                acc1 = fma(k, d[6], acc1);
                acc2 = fma(k, d[7], acc2);
            }
        }
    }
    if (!active) return;
    if (KIND == H2B_SLP) {
        // 1/r = t (3 - r^2 t^2) / 2; symmetrised pairs average both orientations
        double v = sym ? 0.25 * (acc0 + acc1) : 0.5 * acc0;
        v *= kInv4Pi * scale;
        values[pid] = v;
        if (mirror && kase != H2B_IDENTICAL) {
            // unordered pair {a, b}: the same value for (b, a) (symmetric SLP)
            for (int64_t q = row_ptr[b]; q < row_ptr[b + 1]; ++q)
                if (col[q] == (int32_t)a) values[q] = v;
        }
    } else {
        // 1/r^3 = 1.5 t^3 (5/3 - r^2 t^2); scatter back to original local vertices
        const double f = 1.5 * kInv4Pi * scale;
        double out[3];
        const int pb0 = (inf >> 8) & 3, pb1 = (inf >> 10) & 3, pb2 = (inf >> 12) & 3;
        out[pb0] = acc0 * f;
        out[pb1] = acc1 * f;
        out[pb2] = acc2 * f;
        values[3 * pid] = out[0];
        values[3 * pid + 1] = out[1];
        values[3 * pid + 2] = out[2];
    }
}

// ----------------------------------------------------------------------------
// regular SLP pair blocks
__device__ __forceinline__ bool shares_vertex(const int* ra, const int* cb) {
    bool h = false;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) h |= (ra[i] == cb[j]);
    return h;
}

__device__ __forceinline__ int64_t touch_find(const int64_t* __restrict__ row_ptr,
                                              const int32_t* __restrict__ col, int a, int b) {
    // (a row holds the ~12 panels touching panel a: eight independent loads
    // per step instead of one dependent load per entry)
    const int64_t p0 = row_ptr[a], p1 = row_ptr[a + 1];
    for (int64_t p = p0; p < p1; p += 8) {
        int c[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) c[u] = p + u < p1 ? __ldg(col + p + u) : -1;
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (c[u] == b) return p + u;
    }
    return -1;
}

// constant factor of the folded Newton step: with p = r^2/2 and t ~ rsqrt(p),
// 1/(4 pi r) = t (3 - p t^2) / (8 sqrt(2) pi)
constexpr double kSlpFold = 1.0 / (8.0 * 1.4142135623730950488016887 * kPi);

template <int Q, int JC, int MINB, int R, int UJ>
__global__ void __launch_bounds__(H2B_SLP_THREADS, MINB) k_blocks_slp(const double* __restrict__ P, int64_t F,
                                                   const int32_t* __restrict__ T,
                                                   const int64_t* __restrict__ jobs,
                                                   const int32_t* __restrict__ row_idx,
                                                   const int32_t* __restrict__ col_idx,
                                                   const int64_t* __restrict__ t_row_ptr,
                                                   const int32_t* __restrict__ t_col,
                                                   const double* __restrict__ t_val,
                                                   double* __restrict__ out, int* __restrict__ flags) {
    extern __shared__ double smem[];
    double* rx = smem;                 // [5][Q][kSlpLd]: x', y', z', -|x'|^2/2, W
    double* cx = smem + 5 * Q * kSlpLd; // [5][Q][kSlpLd]: y', ..., W / (8 sqrt2 pi)
    int* rv = reinterpret_cast<int*>(cx + 5 * Q * kSlpLd);  // [kTile][3]
    int* cv = rv + 3 * kTile;
    int* rp = cv + 3 * kTile;
    int* cp = rp + kTile;

    const int64_t* jb = jobs + 8 * (int64_t)blockIdx.x;
    const int64_t row_off = jb[0], col_off = jb[2], out_off = jb[4], ld = jb[5];
    const int64_t m_off = jb[6], m_ld = jb[7];
    const int nr = (int)jb[1], nc = (int)jb[3];
    // diagonal tile of a symmetric block: upper triangle only, mirrored
    const bool tri = m_off == out_off;
    if (nr > kTile || nc > kTile) {
        if (threadIdx.x == 0) atomicOr(flags, kFlagShape);
        return;
    }
    if (nr == 0 || nc == 0) return;
    const int64_t FQ = F * Q;
    const int64_t o_idx = (int64_t)row_idx[row_off] * Q;
    const double ox = P[o_idx], oy = P[FQ + o_idx], oz = P[2 * FQ + o_idx];

    for (int e = threadIdx.x; e < nr * Q; e += blockDim.x) {
        const int r = e / Q, i = e - r * Q;
        const int pnl = row_idx[row_off + r];
        const int64_t g = (int64_t)pnl * Q + i;
        const double x = P[g] - ox, y = P[FQ + g] - oy, z = P[2 * FQ + g] - oz;
        const int s = i * kSlpLd + r;
        rx[s] = -x;  // negated: r^2/2 = |x'|^2/2 + |y'|^2/2 + (-x').y'
        rx[Q * kSlpLd + s] = -y;
        rx[2 * Q * kSlpLd + s] = -z;
        rx[3 * Q * kSlpLd + s] = 0.5 * fma(z, z, fma(y, y, x * x));
        rx[4 * Q * kSlpLd + s] = P[3 * FQ + g];
        if (i == 0) {
            rp[r] = pnl;
            rv[3 * r] = T[3 * pnl];
            rv[3 * r + 1] = T[3 * pnl + 1];
            rv[3 * r + 2] = T[3 * pnl + 2];
        }
    }
    for (int e = threadIdx.x; e < nc * Q; e += blockDim.x) {
        const int c = e / Q, j = e - c * Q;
        const int pnl = col_idx[col_off + c];
        const int64_t g = (int64_t)pnl * Q + j;
        const double x = P[g] - ox, y = P[FQ + g] - oy, z = P[2 * FQ + g] - oz;
        const int s = j * kSlpLd + c;
        // column point scaled by cw = 1 / w^2 (w = W kSlpFold > 0): the seed of
        // rsqrt(cw p) is already w t, so the weight costs no product per pair
        const double w = P[3 * FQ + g] * kSlpFold;
        const double cw = 1.0 / (w * w);
        cx[s] = cw * x;
        cx[Q * kSlpLd + s] = cw * y;
        cx[2 * Q * kSlpLd + s] = cw * z;
        cx[3 * Q * kSlpLd + s] = cw * (0.5 * fma(z, z, fma(y, y, x * x)));
        cx[4 * Q * kSlpLd + s] = cw;
        if (j == 0) {
            cp[c] = pnl;
            cv[3 * c] = T[3 * pnl];
            cv[3 * c + 1] = T[3 * pnl + 1];
            cv[3 * c + 2] = T[3 * pnl + 2];
        }
    }
    __syncthreads();

    int lflags = 0;
    const int np = tri ? nc * (nc + 1) / 2 : nr * nc;
    for (int p = threadIdx.x; p < np; p += blockDim.x) {
        int a, b;
        if (tri) {
            // p = b (b + 1) / 2 + a, 0 <= a <= b
            // single-precision root (p < 2080: exact after the corrections)
            b = (int)((sqrtf(8.0f * (float)p + 1.0f) - 1.0f) * 0.5f);
            if ((b + 1) * (b + 2) / 2 <= p) ++b;
            if (b * (b + 1) / 2 > p) --b;
            a = p - b * (b + 1) / 2;
        } else {
            a = p / nc;
            b = p - a * nc;
        }
        double val;
        if (shares_vertex(rv + 3 * a, cv + 3 * b)) {
            if (t_row_ptr == nullptr) {
                lflags |= kFlagTouching;
                val = 0.0;
            } else {
                const int64_t k = touch_find(t_row_ptr, t_col, rp[a], cp[b]);
                if (k < 0) {
                    lflags |= kFlagMissing;
                    val = 0.0;
                } else {
                    val = t_val[k];
                }
            }
        } else {
            double tot = 0.0;
#pragma unroll UJ
            for (int j0 = 0; j0 < Q; j0 += JC) {
                double y0[JC], y1[JC], y2[JC], yh[JC], yw[JC];
#pragma unroll
                for (int j = 0; j < JC; ++j) {
                    if (j0 + j < Q) {
                        const int s = (j0 + j) * kSlpLd + b;
                        y0[j] = cx[s];
                        y1[j] = cx[Q * kSlpLd + s];
                        y2[j] = cx[2 * Q * kSlpLd + s];
                        yh[j] = cx[3 * Q * kSlpLd + s];
                        yw[j] = cx[4 * Q * kSlpLd + s];
                    }
                }
                // R row points per step: R independent accumulation chains
#pragma unroll kSlpUnroll
                for (int i0 = 0; i0 < Q; i0 += R) {
                    double xa[R][5], acc[R];
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        const int si = (i0 + r < Q ? i0 + r : Q - 1) * kSlpLd + a;
#pragma unroll
                        for (int f = 0; f < 5; ++f) xa[r][f] = rx[f * Q * kSlpLd + si];
                        acc[r] = 0.0;
                    }
#pragma unroll
                    for (int j = 0; j < JC; ++j) {
                        if (j0 + j < Q) {
#pragma unroll
                            for (int r = 0; r < R; ++r) {
                                if (i0 + r < Q) {
                                    // p = c (|x'|^2/2 + |y'|^2/2 - x'.y') = c r^2/2 (4 FMA),
                                    // t ~ rsqrt(p) = w sqrt(2) / r; one Newton step folded:
                                    // w / r ~ t (3 - p t^2) / (2 sqrt 2)  (7 FP64 ops per point pair)
                                    const double pa = fma(xa[r][0], y0[j], fma(xa[r][1], y1[j],
                                                      fma(xa[r][2], y2[j], fma(xa[r][3], yw[j], yh[j]))));
                                    const double ta = rsqrt_seed(pa);
                                    acc[r] = fma(ta, fma(-pa, ta * ta, 3.0), acc[r]);
                                }
                            }
                        }
                    }
#pragma unroll
                    for (int r = 0; r < R; ++r)
                        if (i0 + r < Q) tot = fma(xa[r][4], acc[r], tot);
                }
            }
            val = tot;
        }
        if (!isfinite(val)) lflags |= kFlagNonFinite;
        // out_off < 0: mirror-only job (a sharded rank integrates a block pair
        // in the orientation one GPU uses and keeps only the transposed copy)
        if (out_off >= 0) out[out_off + (int64_t)a * ld + b] = val;
        if (m_off >= 0 && !(tri && a == b)) out[m_off + (int64_t)b * m_ld + a] = val;
    }
    if (lflags) atomicOr(flags, lflags);
}

// ----------------------------------------------------------------------------
// regular DLP pair blocks (P0 rows x P1 columns) with the vertex scatter
template <int Q>
struct DlpLam {
    double v[Q * 3];
};
__constant__ double c_lam[64 * 3];  // barycentrics of the regular rule, Q <= 64

// 1/r^3 = 1.5 (1/2)^(3/2) t^3 (5/3 + g t^2) with g = -r^2/2, t ~ rsqrt(-g)
constexpr double kDlpFold = 1.5 * 0.35355339059327376220042218 / (4.0 * kPi);

// JC column points per register chunk (fewer registers -> more resident CTAs)
template <int Q, int JC = Q, int MINB = 1>
__global__ void __launch_bounds__(256, MINB) k_blocks_dlp(const double* __restrict__ P, int64_t F,
                                                   const int32_t* __restrict__ T,
                                                   const double* __restrict__ Nrm,
                                                   const int64_t* __restrict__ jobs,
                                                   const int32_t* __restrict__ row_idx,
                                                   const int32_t* __restrict__ pan_idx,
                                                   const int32_t* __restrict__ inc_ptr,
                                                   const int32_t* __restrict__ inc,
                                                   const int64_t* __restrict__ inc_base,
                                                   const int64_t* __restrict__ t_row_ptr,
                                                   const int32_t* __restrict__ t_col,
                                                   const double* __restrict__ t_val,
                                                   double* __restrict__ out, int* __restrict__ flags) {
    extern __shared__ double smem[];
    constexpr int RT = kTile, PT = kDlpMaxPanels;
    double* rx = smem;                  // [6][Q][RT]: ci x', ci (-|x'|^2/2), ci, 1/ci
    double* px = rx + 6 * Q * RT;       // [6][Q][PT]: y', -|y'|^2/2, W, (y'.n) W
    double* pn = px + 6 * Q * PT;       // [3][PT]
    double* scr = pn + 3 * PT;          // [kDlpRowChunk][PT][3]
    int* rv = reinterpret_cast<int*>(scr + kDlpRowChunk * PT * 3);
    int* pv = rv + 3 * RT;
    int* rp = pv + 3 * PT;
    int* pp = rp + RT;

    const int64_t* jb = jobs + 8 * (int64_t)blockIdx.x;
    const int64_t row_off = jb[0], pan_off = jb[2], out_off = jb[6], ld = jb[7];
    const int nr = (int)jb[1], npn = (int)jb[3], nc = (int)jb[5];
    const int64_t ibase = inc_base[blockIdx.x];
    if (nr > RT || npn > PT || nc > kTile) {
        if (threadIdx.x == 0) atomicOr(flags, kFlagShape);
        return;
    }
    if (nr == 0 || nc == 0) return;
    const int64_t FQ = F * Q;
    const int64_t o_idx = (int64_t)row_idx[row_off] * Q;
    const double ox = P[o_idx], oy = P[FQ + o_idx], oz = P[2 * FQ + o_idx];

    for (int e = threadIdx.x; e < nr * Q; e += blockDim.x) {
        const int r = e / Q, i = e - r * Q;
        const int pnl = row_idx[row_off + r];
        const int64_t g = (int64_t)pnl * Q + i;
        const double x = P[g] - ox, y = P[FQ + g] - oy, z = P[2 * FQ + g] - oz;
        const int s = i * RT + r;
        // row point scaled by ci = w^(-2/3): rsqrt(-ci g)^3 = w t^3, so the
        // row weight rides in the seed (no product per point pair)
        const double ci = 1.0 / cbrt(P[3 * FQ + g] * P[3 * FQ + g]);
        rx[s] = ci * x;
        rx[Q * RT + s] = ci * y;
        rx[2 * Q * RT + s] = ci * z;
        rx[3 * Q * RT + s] = ci * (-0.5 * fma(z, z, fma(y, y, x * x)));
        rx[4 * Q * RT + s] = ci;
        rx[5 * Q * RT + s] = 1.0 / ci;
        if (i == 0) {
            rp[r] = pnl;
            rv[3 * r] = T[3 * pnl];
            rv[3 * r + 1] = T[3 * pnl + 1];
            rv[3 * r + 2] = T[3 * pnl + 2];
        }
    }
    for (int e = threadIdx.x; e < npn * Q; e += blockDim.x) {
        const int c = e / Q, j = e - c * Q;
        const int pnl = pan_idx[pan_off + c];
        const int64_t g = (int64_t)pnl * Q + j;
        const double x = P[g] - ox, y = P[FQ + g] - oy, z = P[2 * FQ + g] - oz;
        const double n0 = Nrm[3 * pnl], n1 = Nrm[3 * pnl + 1], n2 = Nrm[3 * pnl + 2];
        const int s = j * PT + c;
        px[s] = x;
        px[Q * PT + s] = y;
        px[2 * Q * PT + s] = z;
        px[3 * Q * PT + s] = -0.5 * fma(z, z, fma(y, y, x * x));
        const double wf = P[3 * FQ + g] * kDlpFold;
        px[4 * Q * PT + s] = wf;
        px[5 * Q * PT + s] = fma(z, n2, fma(y, n1, x * n0)) * wf;  // (y'.n) w: folds a product per evaluation
        if (j == 0) {
            pp[c] = pnl;
            pn[c] = n0;
            pn[PT + c] = n1;
            pn[2 * PT + c] = n2;
            pv[3 * c] = T[3 * pnl];
            pv[3 * c + 1] = T[3 * pnl + 1];
            pv[3 * c + 2] = T[3 * pnl + 2];
        }
    }
    __syncthreads();

    int lflags = 0;
    for (int r0 = 0; r0 < nr; r0 += kDlpRowChunk) {
        const int rc = min(kDlpRowChunk, nr - r0);
        const int np = rc * npn;
        for (int p = threadIdx.x; p < np; p += blockDim.x) {
            const int al = p / npn, b = p - al * npn;
            const int a = r0 + al;
            double v0, v1, v2;
            if (shares_vertex(rv + 3 * a, pv + 3 * b)) {
                v0 = v1 = v2 = 0.0;
                if (t_row_ptr == nullptr) {
                    lflags |= kFlagTouching;
                } else {
                    const int64_t k = touch_find(t_row_ptr, t_col, rp[a], pp[b]);
                    if (k < 0) {
                        lflags |= kFlagMissing;
                    } else {
                        v0 = t_val[3 * k];
                        v1 = t_val[3 * k + 1];
                        v2 = t_val[3 * k + 2];
                    }
                }
            } else {
                const double n0 = pn[b], n1 = pn[PT + b], n2 = pn[2 * PT + b];
#if H2B_DLP_XN_REG
                // x'.n per row point (unscaled), once per pair
                double xn[Q];
#pragma unroll
                for (int i = 0; i < Q; ++i) {
                    const int s = i * RT + a;
                    xn[i] = rx[5 * Q * RT + s] * fma(rx[2 * Q * RT + s], n2, fma(rx[Q * RT + s], n1, rx[s] * n0));
                }
#endif
                double t0 = 0.0, t1 = 0.0, t2 = 0.0;
#pragma unroll 1
                for (int j0 = 0; j0 < Q; j0 += JC) {
                    double y0[JC], y1[JC], y2[JC], yh[JC], yw[JC], yn[JC], K[JC];
#pragma unroll
                    for (int j = 0; j < JC; ++j) {
                        K[j] = 0.0;
                        if (j0 + j < Q) {
                            const int s = (j0 + j) * PT + b;
                            y0[j] = px[s];
                            y1[j] = px[Q * PT + s];
                            y2[j] = px[2 * Q * PT + s];
                            yh[j] = px[3 * Q * PT + s];
                            yw[j] = px[4 * Q * PT + s];
                            yn[j] = px[5 * Q * PT + s];
                        }
                    }
                    // K_j = sum_i w_i k_ij: g' = ci g (4 FMA), u = rsqrt(-g')^3 = w_i t^3,
                    // 1/r^3 Newton factor (5/3 + g t^2), (x' - y').n w_j (10 FP64 ops)
#pragma unroll kDlpUnroll
                    for (int i = 0; i < Q; ++i) {
                        const int s = i * RT + a;
                        const double x0 = rx[s], x1 = rx[Q * RT + s], x2 = rx[2 * Q * RT + s];
                        const double xh = rx[3 * Q * RT + s], ci = rx[4 * Q * RT + s];
#if H2B_DLP_XN_REG
                        const double xni = xn[i];
#else
                        const double xni = rx[5 * Q * RT + s] * fma(x2, n2, fma(x1, n1, x0 * n0));
#endif
#pragma unroll
                        for (int j = 0; j < JC; ++j) {
                            if (j0 + j < Q) {
                                const double g = fma(x0, y0[j], fma(x1, y1[j], fma(x2, y2[j], fma(ci, yh[j], xh))));
                                const double t = rsqrt_seed(-g);
                                const double s2 = t * t;
                                const double c3 = fma(g, s2, 5.0 / 3.0);
                                K[j] = fma(fma(xni, yw[j], -yn[j]) * c3, s2 * t, K[j]);
                            }
                        }
                    }
#pragma unroll
                    for (int j = 0; j < JC; ++j) {
                        if (j0 + j < Q) {
                            t0 = fma(K[j], c_lam[3 * (j0 + j)], t0);
                            t1 = fma(K[j], c_lam[3 * (j0 + j) + 1], t1);
                            t2 = fma(K[j], c_lam[3 * (j0 + j) + 2], t2);
                        }
                    }
                }
                v0 = t0;
                v1 = t1;
                v2 = t2;
            }
            double* sp = scr + (al * PT + b) * 3;
            sp[0] = v0;
            sp[1] = v1;
            sp[2] = v2;
        }
        __syncthreads();
        // vertex scatter, fixed order per column (l-major, ascending panel:
        // the order np.add.at applies in kernels.dlp_block)
        for (int p = threadIdx.x; p < rc * nc; p += blockDim.x) {
            const int al = p / nc, c = p - al * nc;
            const int32_t* ip = inc_ptr + ibase + c;
            double s = 0.0;
            for (int k = ip[0]; k < ip[1]; ++k) {
                const int code = inc[k];
                s += scr[(al * PT + (code >> 2)) * 3 + (code & 3)];
            }
            if (!isfinite(s)) lflags |= kFlagNonFinite;
            out[out_off + (int64_t)(r0 + al) * ld + c] = s;
        }
        __syncthreads();
    }
    if (lflags) atomicOr(flags, lflags);
}


// ----------------------------------------------------------------------------
// hypersingular P1 x P1 blocks through the surface-curl representation
// (kernels.py:471-511): w_ij = sum over the incident panels a of i and b of j
// of <curl_a(i), curl_b(j)> V_ab, V_ab the single-layer panel-pair integrals
// (k_blocks_slp into a scratch buffer first).  One CTA per block, one thread
// per entry; contributions added in the reference's np.add.at order (local
// vertex of i, local vertex of j, then row panel, then column panel).
// desc per block (int64 x 8): nr, nc, v_off, n_pb, r_inc, c_inc, out_off, ld.
// Incidence entries: pos (panel position in the block's row / column panel
// list) and cl = 3 * panel + local vertex (row of the (3F, 3) curl table).
__global__ void k_hyp_scatter(const int64_t* __restrict__ desc, const int32_t* __restrict__ r_ptr,
                              const int32_t* __restrict__ r_pos, const int32_t* __restrict__ r_cl,
                              const int32_t* __restrict__ c_ptr, const int32_t* __restrict__ c_pos,
                              const int32_t* __restrict__ c_cl, const double* __restrict__ curls,
                              const double* __restrict__ vals, double* __restrict__ out, int* __restrict__ flags) {
    const int64_t* d = desc + 8 * (int64_t)blockIdx.x;
    const int nr = (int)d[0], nc = (int)d[1];
    const int64_t v_off = d[2], npb = d[3], ri = d[4], ci = d[5], o_off = d[6], ld = d[7];
    int lflags = 0;
    for (int e = threadIdx.x; e < nr * nc; e += blockDim.x) {
        const int i = e / nc, j = e - i * nc;
        const int ra = r_ptr[ri + i], re = r_ptr[ri + i + 1], ca = c_ptr[ci + j], ce = c_ptr[ci + j + 1];
        double sum = 0.0;
        for (int la = 0; la < 3; ++la)
            for (int lb = 0; lb < 3; ++lb)
                for (int p = ra; p < re; ++p) {
                    const int cla = r_cl[p];
                    if (cla % 3 != la) continue;
                    const double x0 = curls[3 * cla], x1 = curls[3 * cla + 1], x2 = curls[3 * cla + 2];
                    const double* vrow = vals + v_off + (int64_t)r_pos[p] * npb;
                    for (int q = ca; q < ce; ++q) {
                        const int clb = c_cl[q];
                        if (clb % 3 != lb) continue;
                        const double dot = fma(x2, curls[3 * clb + 2], fma(x1, curls[3 * clb + 1], x0 * curls[3 * clb]));
                        sum += vrow[c_pos[q]] * dot;
                    }
                }
        if (!isfinite(sum)) lflags |= kFlagNonFinite;
        out[o_off + (int64_t)i * ld + j] = sum;
    }
    if (lflags) atomicOr(flags, lflags);
}

int check_flags(int* d_flags, cudaStream_t st) {
    int h = 0;
    H2B_CUDA_TRY(cudaMemcpyAsync(&h, d_flags, sizeof(int), cudaMemcpyDeviceToHost, st));
    H2B_CUDA_TRY(cudaStreamSynchronize(st));
    H2B_CUDA_TRY(cudaFreeAsync(d_flags, st));
    if (h & kFlagShape) return fail(H2B_ERR_INVALID, "pair-block job exceeds the tile size");
    if (h & kFlagCandidates) return fail(H2B_ERR_INVALID, "vertex valence too large or invalid mesh topology");
    if (h & kFlagTouching) return fail(H2B_ERR_TOUCHING, "expected well-separated panels, found touching pair");
    if (h & kFlagMissing) return fail(H2B_ERR_MISSING, "panel pair missing from the singular table");
    if (h & kFlagNonFinite) return fail(H2B_ERR_NONFINITE, "non-finite nearfield entries");
    return ok();
}

int alloc_flags(int** d, cudaStream_t st) {
    H2B_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(d), sizeof(int), st));
    H2B_CUDA_TRY(cudaMemsetAsync(*d, 0, sizeof(int), st));
    return ok();
}

#ifndef H2B_SLP9_JC
#define H2B_SLP9_JC 9
#endif
#ifndef H2B_SLP9_MINB
#define H2B_SLP9_MINB 4
#endif
#ifndef H2B_SLP9_R
#define H2B_SLP9_R 3  // row points per step (sphere L8: 3 rows 5.85 ms, 2 rows 6.09 ms, 1 row 5.96 ms)
#endif
#ifndef H2B_SLP9_UJ
#define H2B_SLP9_UJ 16  // unroll of the column-chunk loop (16: fully)
#endif

template <int Q, int JC, int MINB = 2, int R = 2, int UJ = 16>
int launch_slp(const h2b_mesh* m, const double* P, const h2b_jobs* jobs, const h2b_touch* t,
               const double* tv, double* out, int* flags, cudaStream_t st) {
    const size_t sm = (size_t)10 * Q * kSlpLd * sizeof(double) + (size_t)8 * kTile * sizeof(int);
    auto kern = k_blocks_slp<Q, JC, MINB, R, UJ>;
    H2B_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    const int64_t nj = jobs->n_jobs;
    for (int64_t j0 = 0; j0 < nj; j0 += 2147483647LL) {
        const unsigned g = (unsigned)std::min<int64_t>(nj - j0, 2147483647LL);
        kern<<<g, H2B_SLP_THREADS, sm, st>>>(P, m->n_triangles, m->d_triangles, jobs->d_jobs + 8 * j0, jobs->d_row_idx,
                                 jobs->d_col_idx, t ? t->d_row_ptr : nullptr, t ? t->d_col : nullptr, tv,
                                 out, flags);
    }
    H2B_CUDA_TRY(cudaGetLastError());
    return ok();
}

#ifndef H2B_DLP9_JC
#define H2B_DLP9_JC 3  // measured: 5.0 -> 4.3 ms at config 1 (114 registers, 2 CTAs/SM)
#endif
#ifndef H2B_DLP9_MINB
#define H2B_DLP9_MINB 1
#endif

template <int Q, int JC = Q, int MINB = 1>
int launch_dlp(const h2b_mesh* m, const double* P, const h2b_dlp_jobs* jobs, const h2b_touch* t,
               const double* tv, double* out, int* flags, cudaStream_t st) {
    const size_t sm = (size_t)(6 * Q * kTile + 6 * Q * kDlpMaxPanels + 3 * kDlpMaxPanels +
                               kDlpRowChunk * kDlpMaxPanels * 3) * sizeof(double) +
                      (size_t)(4 * kTile + 4 * kDlpMaxPanels) * sizeof(int);
    auto kern = k_blocks_dlp<Q, JC, MINB>;
    H2B_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    if (jobs->n_jobs > 0)
        kern<<<(unsigned)jobs->n_jobs, 256, sm, st>>>(P, m->n_triangles, m->d_triangles, m->d_normals,
                                                      jobs->d_jobs, jobs->d_row_idx, jobs->d_pan_idx,
                                                      jobs->d_inc_ptr, jobs->d_inc, jobs->d_inc_base,
                                                      t ? t->d_row_ptr : nullptr, t ? t->d_col : nullptr,
                                                      tv, out, flags);
    H2B_CUDA_TRY(cudaGetLastError());
    return ok();
}

}  // namespace
}  // namespace h2b

using namespace h2b;

extern "C" int h2b_panel_points(const h2b_mesh* m, const double* d_rule_xy, const double* d_rule_w,
                                int32_t Q, double* d_out, void* stream) {
    if (!m || !d_rule_xy || !d_rule_w || !d_out || Q < 1) return fail(H2B_ERR_INVALID, "h2b_panel_points: bad argument");
    const int64_t n = m->n_triangles * Q;
    if (n == 0) return ok();
    k_panel_points<<<(unsigned)((n + 255) / 256), 256, 0, as_stream(stream)>>>(
        m->d_vertices, m->d_triangles, m->d_areas, m->n_triangles, d_rule_xy, d_rule_w, Q, d_out);
    H2B_CUDA_TRY(cudaGetLastError());
    return ok();
}

extern "C" int h2b_touch_count(const h2b_mesh* m, int64_t* d_row_ptr, int64_t* h_case_count, void* stream) {
    if (!m || !d_row_ptr || !h_case_count) return fail(H2B_ERR_INVALID, "h2b_touch_count: bad argument");
    cudaStream_t st = as_stream(stream);
    const int64_t F = m->n_triangles;
    int* flags;
    if (int rc = alloc_flags(&flags, st)) return rc;
    unsigned long long* cc;
    int64_t* counts;
    H2B_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&cc), 4 * sizeof(unsigned long long), st));
    H2B_CUDA_TRY(cudaMemsetAsync(cc, 0, 4 * sizeof(unsigned long long), st));
    H2B_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&counts), (F + 1) * sizeof(int64_t), st));
    H2B_CUDA_TRY(cudaMemsetAsync(counts, 0, (F + 1) * sizeof(int64_t), st));
    if (F > 0)
        k_touch_count<<<(unsigned)((F + 127) / 128), 128, 0, st>>>(m->d_triangles, F, m->d_vt_ptr, m->d_vt_idx,
                                                                  counts, cc, flags);
    H2B_CUDA_TRY(cudaGetLastError());
    size_t tmp_bytes = 0;
    H2B_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, counts, d_row_ptr, F + 1, st));
    void* tmp;
    H2B_CUDA_TRY(cudaMallocAsync(&tmp, tmp_bytes, st));
    H2B_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, counts, d_row_ptr, F + 1, st));
    unsigned long long hc[4];
    H2B_CUDA_TRY(cudaMemcpyAsync(hc, cc, sizeof(hc), cudaMemcpyDeviceToHost, st));
    H2B_CUDA_TRY(cudaFreeAsync(tmp, st));
    H2B_CUDA_TRY(cudaFreeAsync(counts, st));
    H2B_CUDA_TRY(cudaFreeAsync(cc, st));
    if (int rc = check_flags(flags, st)) return rc;  // synchronises
    h_case_count[0] = (int64_t)hc[H2B_IDENTICAL];
    h_case_count[1] = (int64_t)hc[H2B_EDGE];
    h_case_count[2] = (int64_t)hc[H2B_VERTEX];
    h_case_count[3] = (int64_t)(hc[1] + hc[2] + hc[3]);
    return ok();
}

// exclusive scan of n int32 counts into d_pos (n + 1 entries, int32)
static int scan_counts(const int32_t* d_cnt, int32_t* d_pos, int64_t n, cudaStream_t st) {
    size_t tmp_bytes = 0;
    H2B_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, d_cnt, d_pos, n + 1, st));
    void* tmp;
    H2B_CUDA_TRY(cudaMallocAsync(&tmp, tmp_bytes, st));
    H2B_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, d_cnt, d_pos, n + 1, st));
    H2B_CUDA_TRY(cudaFreeAsync(tmp, st));
    return 0;
}

extern "C" int h2b_touch_fill(const h2b_mesh* m, const int64_t* d_row_ptr, const int64_t* h_case_count,
                              int32_t* d_col, int32_t* d_info, int32_t* d_case_list, void* stream) {
    if (!m || !d_row_ptr || !h_case_count || !d_col || !d_info || !d_case_list)
        return fail(H2B_ERR_INVALID, "h2b_touch_fill: bad argument");
    cudaStream_t st = as_stream(stream);
    const int64_t F = m->n_triangles;
    if (h_case_count[3] >= (int64_t)INT32_MAX) return fail(H2B_ERR_INVALID, "h2b_touch_fill: > 2^31 touching pairs");
    int* flags;
    if (int rc = alloc_flags(&flags, st)) return rc;
    if (F > 0) {
        int32_t *cnt, *pos;
        H2B_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&cnt), (3 * F + 1) * sizeof(int32_t), st));
        H2B_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&pos), (3 * F + 1) * sizeof(int32_t), st));
        H2B_CUDA_TRY(cudaMemsetAsync(cnt + 3 * F, 0, sizeof(int32_t), st));
        const unsigned g = (unsigned)((F + 127) / 128);
        k_touch_fill<<<g, 128, 0, st>>>(m->d_triangles, F, m->d_vt_ptr, m->d_vt_idx, d_row_ptr, d_col, d_info, cnt,
                                         flags);
        H2B_CUDA_TRY(cudaGetLastError());
        if (int rc = scan_counts(cnt, pos, 3 * F, st)) return rc;
        k_touch_list<<<g, 128, 0, st>>>(d_row_ptr, F, d_info, pos, d_case_list);
        H2B_CUDA_TRY(cudaGetLastError());
        H2B_CUDA_TRY(cudaFreeAsync(pos, st));
        H2B_CUDA_TRY(cudaFreeAsync(cnt, st));
    }
    return check_flags(flags, st);
}

extern "C" int h2b_touch_half(const h2b_touch* t, int32_t* d_half_list, int64_t* h_half_off, void* stream) {
    if (!t || !d_half_list || !h_half_off || !t->h_case_off) return fail(H2B_ERR_INVALID, "h2b_touch_half: bad argument");
    cudaStream_t st = as_stream(stream);
    const int64_t* co = t->h_case_off;
    const int64_t F = t->n_panels;
    const int64_t n_id = co[1] - co[0], n_edge = co[2] - co[1], n_vert = co[3] - co[2];
    if ((n_edge & 1) || (n_vert & 1)) return fail(H2B_ERR_INVALID, "h2b_touch_half: touching relation not symmetric");
    const int64_t off[4] = {0, n_id, n_id + n_edge / 2, n_id + n_edge / 2 + n_vert / 2};
    if (n_id > 0)
        H2B_CUDA_TRY(cudaMemcpyAsync(d_half_list, t->d_case_list + co[0], n_id * sizeof(int32_t),
                                     cudaMemcpyDeviceToDevice, st));
    if (F > 0 && n_edge + n_vert > 0) {
        // per row panel: its (a < b) edge and vertex pairs, segment-major;
        // one scan places them (rows ascending, columns ascending)
        int32_t *cnt, *pos;
        H2B_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&cnt), (2 * F + 1) * sizeof(int32_t), st));
        H2B_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&pos), (2 * F + 1) * sizeof(int32_t), st));
        H2B_CUDA_TRY(cudaMemsetAsync(cnt + 2 * F, 0, sizeof(int32_t), st));
        const unsigned g = (unsigned)((F + 127) / 128);
        k_half_count<<<g, 128, 0, st>>>(t->d_row_ptr, F, t->d_col, t->d_info, cnt);
        H2B_CUDA_TRY(cudaGetLastError());
        if (int rc = scan_counts(cnt, pos, 2 * F, st)) return rc;
        int32_t hpos[2];  // start of the vertex part, total
        H2B_CUDA_TRY(cudaMemcpyAsync(hpos, pos + F, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
        H2B_CUDA_TRY(cudaMemcpyAsync(hpos + 1, pos + 2 * F, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
        k_half_fill<<<g, 128, 0, st>>>(t->d_row_ptr, F, t->d_col, t->d_info, pos, off[1], d_half_list);
        H2B_CUDA_TRY(cudaGetLastError());
        H2B_CUDA_TRY(cudaFreeAsync(pos, st));
        H2B_CUDA_TRY(cudaFreeAsync(cnt, st));
        H2B_CUDA_TRY(cudaStreamSynchronize(st));
        if ((int64_t)hpos[0] != n_edge / 2 || (int64_t)hpos[1] != n_edge / 2 + n_vert / 2)
            return fail(H2B_ERR_INVALID, "h2b_touch_half: touching relation not symmetric");
    }
    for (int i = 0; i < 4; ++i) h_half_off[i] = off[i];
    return ok();
}

extern "C" int h2b_singular(const h2b_mesh* m, const h2b_touch* t, int kind, const h2b_rule* rules,
                            double* d_values, void* stream) {
    if (!m || !t || !rules || !d_values || !t->h_case_off) return fail(H2B_ERR_INVALID, "h2b_singular: bad argument");
    if (kind != H2B_SLP && kind != H2B_DLP) return fail(H2B_ERR_INVALID, "h2b_singular: unknown kind");
    cudaStream_t st = as_stream(stream);
    if (kind == H2B_DLP) {
        // identical flat panels: <x - y, n> = 0 identically (kernels.py:278-279)
        H2B_CUDA_TRY(cudaMemsetAsync(d_values, 0, 3 * sizeof(double) * t->n_pairs, st));
    }
    // symmetric single-layer table: one thread per unordered pair
    const bool half = kind == H2B_SLP && t->d_half_list && t->h_half_off;
    const int64_t* segoff = half ? t->h_half_off : t->h_case_off;
    const int32_t* list = half ? t->d_half_list : t->d_case_list;
    SegSet ss;
    ss.nseg = 0;
    int32_t block = 0;
    // heaviest case first (edge: 5 q^4 points x 2 orientations)
    const int order[3] = {1, 0, 2};
    const int kases[3] = {H2B_IDENTICAL, H2B_EDGE, H2B_VERTEX};
    for (int oi = 0; oi < 3; ++oi) {
        const int c = order[oi];
        if (kind == H2B_DLP && c == 0) continue;
        const int64_t cnt = segoff[c + 1] - segoff[c];
        if (cnt <= 0) continue;
        SegDesc& sd = ss.s[ss.nseg++];
        sd.list_off = segoff[c];
        sd.count = cnt;
        sd.first_block = block;
        sd.n_blocks = (int32_t)((cnt + 127) / 128);
        sd.p = rules[c].d_p;
        sd.w = rules[c].d_w;
        sd.n = rules[c].n;
        sd.kase = kases[c];
        block += sd.n_blocks;
    }
    if (block > 0) {
        if (kind == H2B_SLP)
            k_singular<H2B_SLP><<<block, 128, 0, st>>>(m->d_vertices, m->d_triangles, m->d_normals, m->d_areas,
                                                       t->d_row_ptr, t->n_panels, t->d_col, t->d_info,
                                                       list, ss, d_values, half ? 1 : 0, nullptr);
        else
            k_singular<H2B_DLP><<<block, 128, 0, st>>>(m->d_vertices, m->d_triangles, m->d_normals, m->d_areas,
                                                       t->d_row_ptr, t->n_panels, t->d_col, t->d_info,
                                                       list, ss, d_values, 0, nullptr);
        H2B_CUDA_TRY(cudaGetLastError());
    }
    return ok();
}

extern "C" int h2b_pair_blocks_slp(const h2b_mesh* m, const double* d_panel_points, int32_t Q,
                                   const h2b_jobs* jobs, const h2b_touch* t, const double* d_touch_values,
                                   double* d_out, void* stream) {
    if (!m || !d_panel_points || !jobs || !d_out) return fail(H2B_ERR_INVALID, "h2b_pair_blocks_slp: bad argument");
    if (t && !d_touch_values) return fail(H2B_ERR_INVALID, "h2b_pair_blocks_slp: table without values");
    if (jobs->n_jobs == 0) return ok();
    cudaStream_t st = as_stream(stream);
    int* flags;
    if (int rc = alloc_flags(&flags, st)) return rc;
    int rc;
    switch (Q) {
        case 1: rc = launch_slp<1, 1>(m, d_panel_points, jobs, t, d_touch_values, d_out, flags, st); break;
        case 4: rc = launch_slp<4, 4>(m, d_panel_points, jobs, t, d_touch_values, d_out, flags, st); break;
        case 9: rc = launch_slp<9, H2B_SLP9_JC, H2B_SLP9_MINB, H2B_SLP9_R, H2B_SLP9_UJ>(m, d_panel_points, jobs, t, d_touch_values, d_out,
                                                                        flags, st);
            break;
        case 16: rc = launch_slp<16, 8>(m, d_panel_points, jobs, t, d_touch_values, d_out, flags, st); break;
        case 25: rc = launch_slp<25, 5>(m, d_panel_points, jobs, t, d_touch_values, d_out, flags, st); break;
        default: rc = fail(H2B_ERR_INVALID, "h2b_pair_blocks_slp: supported regular orders q = 1..5");
    }
    if (rc) return rc;
    return check_flags(flags, st);
}

extern "C" int h2b_pair_blocks_dlp(const h2b_mesh* m, const double* d_panel_points, const double* d_lam,
                                   int32_t Q, const h2b_dlp_jobs* jobs, const h2b_touch* t,
                                   const double* d_touch_values, double* d_out, void* stream) {
    if (!m || !d_panel_points || !jobs || !d_out || !d_lam) return fail(H2B_ERR_INVALID, "h2b_pair_blocks_dlp: bad argument");
    if (t && !d_touch_values) return fail(H2B_ERR_INVALID, "h2b_pair_blocks_dlp: table without values");
    if (Q > 64) return fail(H2B_ERR_INVALID, "h2b_pair_blocks_dlp: Q > 64");
    if (jobs->n_jobs == 0) return ok();
    cudaStream_t st = as_stream(stream);
    H2B_CUDA_TRY(cudaMemcpyToSymbolAsync(c_lam, d_lam, sizeof(double) * 3 * Q, 0, cudaMemcpyDeviceToDevice, st));
    int* flags;
    if (int rc = alloc_flags(&flags, st)) return rc;
    int rc;
    switch (Q) {
        case 1: rc = launch_dlp<1>(m, d_panel_points, jobs, t, d_touch_values, d_out, flags, st); break;
        case 4: rc = launch_dlp<4>(m, d_panel_points, jobs, t, d_touch_values, d_out, flags, st); break;
        case 9:
            rc = launch_dlp<9, H2B_DLP9_JC, H2B_DLP9_MINB>(m, d_panel_points, jobs, t, d_touch_values, d_out, flags, st);
            break;
        case 16: rc = launch_dlp<16, 4>(m, d_panel_points, jobs, t, d_touch_values, d_out, flags, st); break;
        default: rc = fail(H2B_ERR_INVALID, "h2b_pair_blocks_dlp: supported regular orders q = 1..4");
    }
    if (rc) return rc;
    return check_flags(flags, st);
}

// kernels.pair_integrals (kernels.py:260-319) on an arbitrary list of panel
// pairs: classification on the device, then the Sauter-Schwab kernel with the
// rule of each pair's case (rules[0..3] = identical, edge, vertex, disjoint).
extern "C" int h2b_pair_integrals(const h2b_mesh* m, int64_t n, const int32_t* d_pa, const int32_t* d_pb, int kind,
                                  const h2b_rule* rules, double* d_values, void* stream) {
    if (!m || (n > 0 && (!d_pa || !d_pb || !d_values)) || !rules || n < 0)
        return fail(H2B_ERR_INVALID, "h2b_pair_integrals: bad argument");
    if (kind != H2B_SLP && kind != H2B_DLP) return fail(H2B_ERR_INVALID, "h2b_pair_integrals: unknown kind");
    if (n == 0) return ok();
    if (n > 2147483647LL) return fail(H2B_ERR_INVALID, "h2b_pair_integrals: more than 2^31 pairs");
    cudaStream_t st = as_stream(stream);
    H2B_CUDA_TRY(cudaMemsetAsync(d_values, 0, (kind == H2B_DLP ? 3 : 1) * sizeof(double) * n, st));
    int32_t *info, *list;
    unsigned long long* cnt;
    H2B_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&info), n * sizeof(int32_t), st));
    H2B_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&list), n * sizeof(int32_t), st));
    H2B_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&cnt), 4 * sizeof(unsigned long long), st));
    H2B_CUDA_TRY(cudaMemsetAsync(cnt, 0, 4 * sizeof(unsigned long long), st));
    const unsigned g = (unsigned)((n + 255) / 256);
    k_classify_list<<<g, 256, 0, st>>>(m->d_triangles, n, d_pa, d_pb, info, cnt);
    H2B_CUDA_TRY(cudaGetLastError());
    unsigned long long hc[4];
    H2B_CUDA_TRY(cudaMemcpyAsync(hc, cnt, sizeof(hc), cudaMemcpyDeviceToHost, st));
    H2B_CUDA_TRY(cudaStreamSynchronize(st));
    int64_t off[5] = {0, 0, 0, 0, 0};
    for (int c = 0; c < 4; ++c) off[c + 1] = off[c] + (int64_t)hc[c];
    unsigned long long cur[4] = {(unsigned long long)off[0], (unsigned long long)off[1], (unsigned long long)off[2],
                                 (unsigned long long)off[3]};
    H2B_CUDA_TRY(cudaMemcpyAsync(cnt, cur, sizeof(cur), cudaMemcpyHostToDevice, st));
    k_bucket_list<<<g, 256, 0, st>>>(n, info, list, cnt);
    H2B_CUDA_TRY(cudaGetLastError());
    SegSet ss;
    ss.nseg = 0;
    int32_t block = 0;
    const int order[4] = {1, 0, 2, 3};
    const int kases[4] = {H2B_IDENTICAL, H2B_EDGE, H2B_VERTEX, H2B_DISJOINT};
    for (int oi = 0; oi < 4; ++oi) {
        const int c = order[oi];
        if (kind == H2B_DLP && c == 0) continue;  // identical flat panels: 0 (kernels.py:278-279)
        const int64_t cn = off[c + 1] - off[c];
        if (cn <= 0) continue;
        if (!rules[c].d_p || !rules[c].d_w || rules[c].n <= 0) return fail(H2B_ERR_INVALID, "h2b_pair_integrals: rule missing");
        SegDesc& sd = ss.s[ss.nseg++];
        sd.list_off = off[c];
        sd.count = cn;
        sd.first_block = block;
        sd.n_blocks = (int32_t)((cn + 127) / 128);
        sd.p = rules[c].d_p;
        sd.w = rules[c].d_w;
        sd.n = rules[c].n;
        sd.kase = kases[c];
        block += sd.n_blocks;
    }
    if (block > 0) {
        if (kind == H2B_SLP)
            k_singular<H2B_SLP><<<block, 128, 0, st>>>(m->d_vertices, m->d_triangles, m->d_normals, m->d_areas,
                                                       nullptr, m->n_triangles, d_pb, info, list, ss, d_values, 0,
                                                       d_pa);
        else
            k_singular<H2B_DLP><<<block, 128, 0, st>>>(m->d_vertices, m->d_triangles, m->d_normals, m->d_areas,
                                                       nullptr, m->n_triangles, d_pb, info, list, ss, d_values, 0,
                                                       d_pa);
        H2B_CUDA_TRY(cudaGetLastError());
    }
    H2B_CUDA_TRY(cudaFreeAsync(info, st));
    H2B_CUDA_TRY(cudaFreeAsync(list, st));
    H2B_CUDA_TRY(cudaFreeAsync(cnt, st));
    return ok();
}

extern "C" int h2b_hyp_scatter(int64_t n_blocks, const int64_t* d_desc, const int32_t* d_r_ptr,
                               const int32_t* d_r_pos, const int32_t* d_r_cl, const int32_t* d_c_ptr,
                               const int32_t* d_c_pos, const int32_t* d_c_cl, const double* d_curls,
                               const double* d_vals, double* d_out, void* stream) {
    if (n_blocks < 0 || (n_blocks > 0 && (!d_desc || !d_r_ptr || !d_r_pos || !d_r_cl || !d_c_ptr || !d_c_pos ||
                                          !d_c_cl || !d_curls || !d_vals || !d_out)))
        return fail(H2B_ERR_INVALID, "h2b_hyp_scatter: bad argument");
    if (n_blocks == 0) return ok();
    cudaStream_t st = as_stream(stream);
    int* flags;
    if (int rc = alloc_flags(&flags, st)) return rc;
    for (int64_t b0 = 0; b0 < n_blocks; b0 += 2147483647LL) {
        const unsigned g = (unsigned)std::min<int64_t>(n_blocks - b0, 2147483647LL);
        k_hyp_scatter<<<g, 256, 0, st>>>(d_desc + 8 * b0, d_r_ptr, d_r_pos, d_r_cl, d_c_ptr, d_c_pos, d_c_cl,
                                          d_curls, d_vals, d_out, flags);
    }
    H2B_CUDA_TRY(cudaGetLastError());
    return check_flags(flags, st);
}
