// Cluster tree and block tree on the device (the level-9
// structure without the host recursion), bit-exact with the reference's
// clustering.py:78-160 and with the host builder (structure.cpp).
//
// Cluster tree (build_cluster_tree, clustering.py:78-121), one tree level per
// step: every node of the level gets its tight box, longest axis and centre
// midpoint from a block reduction (min / max are exact in any order); each
// dof of a node that splits is flagged `c <= mid`, one device-wide exclusive
// scan of the flags gives every dof its slot (left part in input order, then
// the right part: the reference's stable mask split); the rare nodes whose
// centres do not separate take the stable-median fallback on the host.  Node
// uids (preorder creation counter) follow from the subtree sizes afterwards.
//
// Block tree (BlockTree._descend, clustering.py:149-160), one recursion level
// per step: every frontier pair is admissible (far leaf), leaf x leaf (near
// leaf) or expands into its children pairs in row-major order.  The far and
// near lists come out in the reference's depth-first order: subtree far /
// near counts bottom-up, then each child's offset from its parent's and its
// elder siblings' counts top-down.
//
// Floating point: the same IEEE operations as structure.cpp, written with
// explicit round-to-nearest intrinsics (no contraction), the admissibility
// norm as fma(c, c, fma(b, b, a*a)).

#include <algorithm>
#include <numeric>
#include <vector>

#include <cub/device/device_scan.cuh>

#include "device_common.cuh"

namespace h2b {
namespace {

constexpr int kTB = 256;

__device__ __forceinline__ double dmin(double a, double b) { return a < b ? a : (b < a ? b : a); }
__device__ __forceinline__ double dmax(double a, double b) { return a > b ? a : (b > a ? b : a); }

// one CTA per node of the level: box, and for nodes that split the axis and
// the centre midpoint; also tags every position of the node with its index
__global__ void k_node_stats(const double* __restrict__ boxes, const double* __restrict__ centers,
                             const int32_t* __restrict__ ids, const int64_t* __restrict__ nstart,
                             const int64_t* __restrict__ ncnt, int64_t r_leaf, double* __restrict__ nbox,
                             double* __restrict__ nmid, int32_t* __restrict__ naxis, int32_t* __restrict__ pos_node) {
    __shared__ double red[6][kTB / 32];
    const int node = blockIdx.x;
    const int64_t s = nstart[node], cnt = ncnt[node];
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int64_t i = threadIdx.x; i < cnt; i += blockDim.x) {
        const int32_t d = ids[s + i];
        pos_node[s + i] = node;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            lo[k] = dmin(lo[k], boxes[6 * (int64_t)d + k]);
            hi[k] = dmax(hi[k], boxes[6 * (int64_t)d + 3 + k]);
        }
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < 3; ++k)
        for (int o = 16; o > 0; o >>= 1) {
            lo[k] = dmin(lo[k], __shfl_xor_sync(0xffffffffu, lo[k], o));
            hi[k] = dmax(hi[k], __shfl_xor_sync(0xffffffffu, hi[k], o));
        }
    if (lane == 0)
        for (int k = 0; k < 3; ++k) {
            red[k][warp] = lo[k];
            red[3 + k][warp] = hi[k];
        }
    __syncthreads();
    __shared__ double box[6];
    __shared__ int axis_s;
    if (threadIdx.x == 0) {
        for (int k = 0; k < 3; ++k) {
            double a = red[k][0], b = red[3 + k][0];
            for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
                a = dmin(a, red[k][w]);
                b = dmax(b, red[3 + k][w]);
            }
            box[k] = a;
            box[3 + k] = b;
            nbox[6 * node + k] = a;
            nbox[6 * node + 3 + k] = b;
        }
        // np.argmax of the extents: the first maximum
        int ax = 0;
        double best = __dsub_rn(box[3], box[0]);
        for (int k = 1; k < 3; ++k) {
            const double e = __dsub_rn(box[3 + k], box[k]);
            if (e > best) {
                best = e;
                ax = k;
            }
        }
        axis_s = ax;
        naxis[node] = cnt > r_leaf ? ax : -1;
    }
    __syncthreads();
    if (cnt <= r_leaf) return;
    const int ax = axis_s;
    double cmin = INFINITY, cmax = -INFINITY;
    for (int64_t i = threadIdx.x; i < cnt; i += blockDim.x) {
        const double c = centers[3 * (int64_t)ids[s + i] + ax];
        cmin = dmin(cmin, c);
        cmax = dmax(cmax, c);
    }
    for (int o = 16; o > 0; o >>= 1) {
        cmin = dmin(cmin, __shfl_xor_sync(0xffffffffu, cmin, o));
        cmax = dmax(cmax, __shfl_xor_sync(0xffffffffu, cmax, o));
    }
    if (lane == 0) {
        red[0][warp] = cmin;
        red[1][warp] = cmax;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = red[0][0], b = red[1][0];
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
            a = dmin(a, red[0][w]);
            b = dmax(b, red[1][w]);
        }
        nmid[node] = __dmul_rn(0.5, __dadd_rn(a, b));
    }
}

__global__ void k_centers(const double* __restrict__ boxes, int64_t n, double* __restrict__ centers) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= 3 * n) return;
    const int64_t d = i / 3, k = i - 3 * d;
    centers[i] = __dmul_rn(0.5, __dadd_rn(boxes[6 * d + k], boxes[6 * d + 3 + k]));
}

// left flag of every position (0 for positions of nodes that do not split)
__global__ void k_split_flags(const double* __restrict__ centers, const int32_t* __restrict__ ids, int64_t n,
                              const int32_t* __restrict__ pos_node, const int32_t* __restrict__ naxis,
                              const double* __restrict__ nmid, int32_t* __restrict__ flag) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const int node = pos_node[p];
    int f = 0;
    if (node >= 0) {
        const int ax = naxis[node];
        if (ax >= 0) f = centers[3 * (int64_t)ids[p] + ax] <= nmid[node] ? 1 : 0;
    }
    flag[p] = f;
}

__global__ void k_node_left(const int64_t* __restrict__ nstart, const int64_t* __restrict__ ncnt, int m,
                            const int32_t* __restrict__ scan, int64_t* __restrict__ nleft) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    nleft[i] = (int64_t)scan[nstart[i] + ncnt[i]] - scan[nstart[i]];
}

// stable split: left part in input order, then the right part
__global__ void k_split_scatter(const int32_t* __restrict__ ids, int64_t n, const int32_t* __restrict__ pos_node,
                                const int32_t* __restrict__ naxis, const int64_t* __restrict__ nstart,
                                const int64_t* __restrict__ nleft, const int32_t* __restrict__ flag,
                                const int32_t* __restrict__ scan, int32_t* __restrict__ out) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const int node = pos_node[p];
    if (node < 0 || naxis[node] < 0) {
        out[p] = ids[p];
        return;
    }
    const int64_t s = nstart[node];
    const int64_t before = (int64_t)scan[p] - scan[s];  // left flags before p in the node
    const int64_t q = flag[p] ? s + before : s + nleft[node] + (p - s - before);
    out[q] = ids[p];
}

// ---------------------------------------------------------------------------
// block tree

__device__ __forceinline__ double norm3(double a, double b, double c) {
    return __dsqrt_rn(__fma_rn(c, c, __fma_rn(b, b, __dmul_rn(a, a))));
}

struct DevTree {
    const int64_t* left;
    const int64_t* right;
    const double* boxes;
    const double* diam;
};

// frontier pair -> 0 far, 1 near, else the number of children pairs (2 or 4
// or 2) + 2 encoded as 2 + count
__global__ void k_pair_kind(DevTree R, DevTree C, double two_eta, const int32_t* __restrict__ ft,
                            const int32_t* __restrict__ fs, int64_t m, int32_t* __restrict__ kind,
                            int32_t* __restrict__ nchild) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    const int t = ft[i], s = fs[i];
    const double* a = R.boxes + 6 * (int64_t)t;
    const double* b = C.boxes + 6 * (int64_t)s;
    double g[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const double u = __dsub_rn(a[k], b[3 + k]);
        const double v = __dsub_rn(b[k], a[3 + k]);
        const double mm = (u >= v) ? u : v;
        g[k] = (0.0 >= mm) ? 0.0 : mm;
    }
    const double dist = norm3(g[0], g[1], g[2]);
    const double dt = R.diam[t], ds = C.diam[s];
    const double diam = dt < ds ? ds : dt;  // max(rdiam, cdiam)
    int kd, nc = 0;
    if (diam <= __dmul_rn(two_eta, dist)) {
        kd = 0;
    } else {
        const bool tl = R.left[t] < 0, sl = C.left[s] < 0;
        if (tl && sl) {
            kd = 1;
        } else {
            kd = 2;
            nc = (tl ? 1 : 2) * (sl ? 1 : 2);
        }
    }
    kind[i] = kd;
    nchild[i] = nc;
}

__global__ void k_pair_expand(DevTree R, DevTree C, const int32_t* __restrict__ ft, const int32_t* __restrict__ fs,
                              int64_t m, const int32_t* __restrict__ nchild, const int32_t* __restrict__ coff,
                              int32_t* __restrict__ nt, int32_t* __restrict__ ns) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m || nchild[i] == 0) return;
    const int t = ft[i], s = fs[i];
    int ts[2] = {t, -1}, ss[2] = {s, -1};
    int ntc = 1, nsc = 1;
    if (R.left[t] >= 0) {
        ts[0] = (int)R.left[t];
        ts[1] = (int)R.right[t];
        ntc = 2;
    }
    if (C.left[s] >= 0) {
        ss[0] = (int)C.left[s];
        ss[1] = (int)C.right[s];
        nsc = 2;
    }
    int o = coff[i];
    for (int a = 0; a < ntc; ++a)
        for (int b = 0; b < nsc; ++b) {
            nt[o] = ts[a];
            ns[o] = ss[b];
            ++o;
        }
}


// bottom-up: far / near leaves below every pair of a recursion level
__global__ void k_dfs_count(int64_t m, const int32_t* __restrict__ kind, const int32_t* __restrict__ coff,
                            const int64_t* __restrict__ cf_next, const int64_t* __restrict__ cn_next,
                            int64_t* __restrict__ cf, int64_t* __restrict__ cn) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    int64_t f = kind[i] == 0 ? 1 : 0, q = kind[i] == 1 ? 1 : 0;
    for (int32_t c = coff[i]; c < coff[i + 1]; ++c) {
        f += cf_next[c];
        q += cn_next[c];
    }
    cf[i] = f;
    cn[i] = q;
}

// top-down: a leaf pair writes itself at its offset; an inner pair hands its
// children their offsets (its own plus the elder siblings' counts)
__global__ void k_dfs_place(int64_t m, const int32_t* __restrict__ ft, const int32_t* __restrict__ fs,
                            const int32_t* __restrict__ kind, const int32_t* __restrict__ coff,
                            const int64_t* __restrict__ of, const int64_t* __restrict__ on,
                            const int64_t* __restrict__ cf_next, const int64_t* __restrict__ cn_next,
                            int64_t* __restrict__ of_next, int64_t* __restrict__ on_next, int64_t* __restrict__ far,
                            int64_t* __restrict__ near) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    if (kind[i] == 0) {
        far[2 * of[i]] = ft[i];
        far[2 * of[i] + 1] = fs[i];
    } else if (kind[i] == 1) {
        near[2 * on[i]] = ft[i];
        near[2 * on[i] + 1] = fs[i];
    } else {
        int64_t f = of[i], q = on[i];
        for (int32_t c = coff[i]; c < coff[i + 1]; ++c) {
            of_next[c] = f;
            on_next[c] = q;
            f += cf_next[c];
            q += cn_next[c];
        }
    }
}

__global__ void k_box_diam(const double* __restrict__ boxes, int64_t n, double* __restrict__ diam) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double* b = boxes + 6 * i;
    diam[i] = norm3(__dsub_rn(b[3], b[0]), __dsub_rn(b[4], b[1]), __dsub_rn(b[5], b[2]));
}

template <class T>
int dalloc(T** p, int64_t n) {
    H2B_CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(p), sizeof(T) * std::max<int64_t>(n, 1)));
    return 0;
}

int exclusive_scan(const int32_t* in, int32_t* out, int64_t n, void*& tmp, size_t& tmp_bytes) {
    size_t need = 0;
    H2B_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, need, in, out, n));
    if (need > tmp_bytes) {
        if (tmp) cudaFree(tmp);
        H2B_CUDA_TRY(cudaMalloc(&tmp, need));
        tmp_bytes = need;
    }
    H2B_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, in, out, n));
    return 0;
}

struct Freer {
    std::vector<void*> p;
    ~Freer() {
        for (void* q : p)
            if (q) cudaFree(q);
    }
    template <class T>
    T* add(T* q) {
        p.push_back(q);
        return q;
    }
};

}  // namespace
}  // namespace h2b

using namespace h2b;

extern "C" int h2b_cluster_tree_device(const double* h_boxes, int64_t n, int64_t r_leaf, int64_t* h_perm,
                                       int64_t* h_n_nodes, int64_t* h_start, int64_t* h_end, int64_t* h_depth,
                                       int64_t* h_left, int64_t* h_right, double* h_node_boxes) {
    if (n <= 0) return fail(H2B_ERR_INVALID, "cannot build a cluster tree over an empty index set");
    if (r_leaf < 1) return fail(H2B_ERR_INVALID, "r_leaf must be >= 1");
    if (n >= (int64_t)INT32_MAX) return fail(H2B_ERR_INVALID, "h2b_cluster_tree_device: more than 2^31 dofs");
    if (!h_boxes || !h_perm || !h_n_nodes || !h_start || !h_end || !h_depth || !h_left || !h_right || !h_node_boxes)
        return fail(H2B_ERR_INVALID, "h2b_cluster_tree_device: null pointer");
    Freer F;
    double *boxes, *centers;
    int32_t *ids, *ids2, *pos_node, *flag, *scan;
    if (dalloc(&boxes, 6 * n) || dalloc(&centers, 3 * n) || dalloc(&ids, n) || dalloc(&ids2, n) ||
        dalloc(&pos_node, n) || dalloc(&flag, n + 1) || dalloc(&scan, n + 1))
        return H2B_ERR_CUDA;
    F.add(boxes), F.add(centers), F.add(ids), F.add(ids2), F.add(pos_node), F.add(flag), F.add(scan);
    H2B_CUDA_TRY(cudaMemcpy(boxes, h_boxes, sizeof(double) * 6 * n, cudaMemcpyHostToDevice));
    k_centers<<<(unsigned)((3 * n + kTB - 1) / kTB), kTB>>>(boxes, n, centers);
    {
        std::vector<int32_t> iota(n);
        std::iota(iota.begin(), iota.end(), 0);
        H2B_CUDA_TRY(cudaMemcpy(ids, iota.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice));
    }
    void* tmp = nullptr;
    size_t tmp_bytes = 0;
    // nodes in creation-by-level order; per node: start, cnt, depth, parent, is-right-child
    std::vector<int64_t> g_start, g_cnt, g_depth, g_parent, g_left, g_right;
    std::vector<double> g_box;
    std::vector<int64_t> lvl_start = {0}, lvl_cnt = {n}, lvl_parent = {-1};
    std::vector<int> lvl_side = {0};
    int64_t depth = 0;
    int64_t cap = 0;
    int64_t *d_nstart = nullptr, *d_ncnt = nullptr, *d_nleft = nullptr;
    double *d_nbox = nullptr, *d_nmid = nullptr;
    int32_t* d_naxis = nullptr;
    auto freeall = [&]() {
        for (void* q : {(void*)d_nstart, (void*)d_ncnt, (void*)d_nleft, (void*)d_nbox, (void*)d_nmid, (void*)d_naxis})
            if (q) cudaFree(q);
        if (tmp) cudaFree(tmp);
    };
    int rc = 0;
    while (!lvl_start.empty() && rc == 0) {
        const int64_t m = (int64_t)lvl_start.size();
        if (m > cap) {
            for (void* q : {(void*)d_nstart, (void*)d_ncnt, (void*)d_nleft, (void*)d_nbox, (void*)d_nmid,
                            (void*)d_naxis})
                if (q) cudaFree(q);
            cap = 2 * m;
            if (dalloc(&d_nstart, cap) || dalloc(&d_ncnt, cap) || dalloc(&d_nleft, cap) || dalloc(&d_nbox, 6 * cap) ||
                dalloc(&d_nmid, cap) || dalloc(&d_naxis, cap)) {
                rc = H2B_ERR_CUDA;
                break;
            }
        }
        cudaMemcpy(d_nstart, lvl_start.data(), sizeof(int64_t) * m, cudaMemcpyHostToDevice);
        cudaMemcpy(d_ncnt, lvl_cnt.data(), sizeof(int64_t) * m, cudaMemcpyHostToDevice);
        cudaMemset(pos_node, 0xff, sizeof(int32_t) * n);  // -1: finished leaves
        k_node_stats<<<(unsigned)m, kTB>>>(boxes, centers, ids, d_nstart, d_ncnt, r_leaf, d_nbox, d_nmid, d_naxis,
                                            pos_node);
        const unsigned gn = (unsigned)((n + kTB - 1) / kTB);
        k_split_flags<<<gn, kTB>>>(centers, ids, n, pos_node, d_naxis, d_nmid, flag);
        cudaMemset(flag + n, 0, sizeof(int32_t));
        if ((rc = exclusive_scan(flag, scan, n + 1, tmp, tmp_bytes))) break;
        k_node_left<<<(unsigned)((m + kTB - 1) / kTB), kTB>>>(d_nstart, d_ncnt, (int)m, scan, d_nleft);
        std::vector<int64_t> nleft(m);
        std::vector<int32_t> naxis(m);
        std::vector<double> nbox(6 * m);
        cudaMemcpy(nleft.data(), d_nleft, sizeof(int64_t) * m, cudaMemcpyDeviceToHost);
        cudaMemcpy(naxis.data(), d_naxis, sizeof(int32_t) * m, cudaMemcpyDeviceToHost);
        const cudaError_t e = cudaMemcpy(nbox.data(), d_nbox, sizeof(double) * 6 * m, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) {
            rc = fail(H2B_ERR_CUDA, std::string("h2b_cluster_tree_device: ") + cudaGetErrorString(e));
            break;
        }
        // stable-median fallback (clustering.py:110-114) where the centres do not separate
        bool refix = false;
        std::vector<double> hcent;
        for (int64_t i = 0; i < m; ++i) {
            if (naxis[i] < 0 || (nleft[i] > 0 && nleft[i] < lvl_cnt[i])) continue;
            const int64_t s = lvl_start[i], cnt = lvl_cnt[i];
            if (hcent.empty()) {
                hcent.resize(3 * n);
                cudaMemcpy(hcent.data(), centers, sizeof(double) * 3 * n, cudaMemcpyDeviceToHost);
            }
            std::vector<int32_t> hid(cnt);
            cudaMemcpy(hid.data(), ids + s, sizeof(int32_t) * cnt, cudaMemcpyDeviceToHost);
            std::vector<double> c(cnt);
            for (int64_t j = 0; j < cnt; ++j) c[j] = hcent[3 * (int64_t)hid[j] + naxis[i]];
            std::vector<int64_t> order(cnt);
            std::iota(order.begin(), order.end(), 0);
            std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return c[a] < c[b]; });
            std::vector<int32_t> f(cnt, 0);
            for (int64_t j = 0; j < cnt / 2; ++j) f[order[j]] = 1;
            cudaMemcpy(flag + s, f.data(), sizeof(int32_t) * cnt, cudaMemcpyHostToDevice);
            refix = true;
        }
        if (refix) {
            if ((rc = exclusive_scan(flag, scan, n + 1, tmp, tmp_bytes))) break;
            k_node_left<<<(unsigned)((m + kTB - 1) / kTB), kTB>>>(d_nstart, d_ncnt, (int)m, scan, d_nleft);
            cudaMemcpy(nleft.data(), d_nleft, sizeof(int64_t) * m, cudaMemcpyDeviceToHost);
        }
        k_split_scatter<<<gn, kTB>>>(ids, n, pos_node, d_naxis, d_nstart, d_nleft, flag, scan, ids2);
        std::swap(ids, ids2);
        // record this level's nodes; the next level's
        std::vector<int64_t> ns, nc, np;
        std::vector<int> sd;
        for (int64_t i = 0; i < m; ++i) {
            const int64_t g = (int64_t)g_start.size();
            g_start.push_back(lvl_start[i]);
            g_cnt.push_back(lvl_cnt[i]);
            g_depth.push_back(depth);
            g_parent.push_back(lvl_parent[i]);
            g_left.push_back(-1);
            g_right.push_back(-1);
            for (int k = 0; k < 6; ++k) g_box.push_back(nbox[6 * i + k]);
            if (lvl_parent[i] >= 0) (lvl_side[i] ? g_right : g_left)[lvl_parent[i]] = g;
            if (naxis[i] >= 0) {
                ns.push_back(lvl_start[i]);
                nc.push_back(nleft[i]);
                np.push_back(g);
                sd.push_back(0);
                ns.push_back(lvl_start[i] + nleft[i]);
                nc.push_back(lvl_cnt[i] - nleft[i]);
                np.push_back(g);
                sd.push_back(1);
            }
        }
        lvl_start.swap(ns);
        lvl_cnt.swap(nc);
        lvl_parent.swap(np);
        lvl_side.swap(sd);
        ++depth;
    }
    if (rc == 0) {
        const cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) rc = fail(H2B_ERR_CUDA, std::string("h2b_cluster_tree_device: ") + cudaGetErrorString(e));
    }
    if (rc == 0) {
        // preorder uids (the reference's creation counter): subtree sizes, then
        // left child = parent + 1, right child = parent + 1 + |left subtree|
        const int64_t G = (int64_t)g_start.size();
        std::vector<int64_t> size(G, 1), uid(G, 0);
        for (int64_t g = G - 1; g >= 0; --g)
            if (g_parent[g] >= 0) size[g_parent[g]] += size[g];
        for (int64_t g = 0; g < G; ++g) {
            if (g_left[g] >= 0) uid[g_left[g]] = uid[g] + 1;
            if (g_right[g] >= 0) uid[g_right[g]] = uid[g] + 1 + (g_left[g] >= 0 ? size[g_left[g]] : 0);
        }
        for (int64_t g = 0; g < G; ++g) {
            const int64_t u = uid[g];
            h_start[u] = g_start[g];
            h_end[u] = g_start[g] + g_cnt[g];
            h_depth[u] = g_depth[g];
            h_left[u] = g_left[g] >= 0 ? uid[g_left[g]] : -1;
            h_right[u] = g_right[g] >= 0 ? uid[g_right[g]] : -1;
            for (int k = 0; k < 6; ++k) h_node_boxes[6 * u + k] = g_box[6 * g + k];
        }
        *h_n_nodes = G;
        std::vector<int32_t> perm(n);
        const cudaError_t e = cudaMemcpy(perm.data(), ids, sizeof(int32_t) * n, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) rc = fail(H2B_ERR_CUDA, std::string("h2b_cluster_tree_device: ") + cudaGetErrorString(e));
        for (int64_t i = 0; i < n; ++i) h_perm[i] = perm[i];
    }
    freeall();
    return rc ? rc : ok();
}

extern "C" int h2b_block_tree_device(const h2b_tree* row, const h2b_tree* col, double eta, int64_t* h_far,
                                     int64_t far_cap, int64_t* h_near, int64_t near_cap, int64_t* h_n_far,
                                     int64_t* h_n_near) {
    if (!row || !col || !h_n_far || !h_n_near) return fail(H2B_ERR_INVALID, "h2b_block_tree_device: null pointer");
    if (!(eta > 0.0)) return fail(H2B_ERR_INVALID, "eta must be positive");
    Freer F;
    DevTree R, C;
    const h2b_tree* tr[2] = {row, col};
    DevTree* dt[2] = {&R, &C};
    for (int w = 0; w < 2; ++w) {
        const int64_t nn = tr[w]->n_nodes;
        int64_t *l, *r;
        double *b, *d;
        if (dalloc(&l, nn) || dalloc(&r, nn) || dalloc(&b, 6 * nn) || dalloc(&d, nn)) return H2B_ERR_CUDA;
        F.add(l), F.add(r), F.add(b), F.add(d);
        H2B_CUDA_TRY(cudaMemcpy(l, tr[w]->left, sizeof(int64_t) * nn, cudaMemcpyHostToDevice));
        H2B_CUDA_TRY(cudaMemcpy(r, tr[w]->right, sizeof(int64_t) * nn, cudaMemcpyHostToDevice));
        H2B_CUDA_TRY(cudaMemcpy(b, tr[w]->boxes, sizeof(double) * 6 * nn, cudaMemcpyHostToDevice));
        k_box_diam<<<(unsigned)((nn + kTB - 1) / kTB), kTB>>>(b, nn, d);
        *dt[w] = DevTree{l, r, b, d};
    }
    const double two_eta = 2.0 * eta;
    // levels of the recursion: pairs (device), their kind, their children offsets
    std::vector<int32_t*> lt, ls, lkind, lcoff;
    std::vector<int64_t> lm;
    int32_t *t0, *s0;
    if (dalloc(&t0, 1) || dalloc(&s0, 1)) return H2B_ERR_CUDA;
    F.add(t0), F.add(s0);
    H2B_CUDA_TRY(cudaMemset(t0, 0, sizeof(int32_t)));
    H2B_CUDA_TRY(cudaMemset(s0, 0, sizeof(int32_t)));
    void* tmp = nullptr;
    size_t tmp_bytes = 0;
    int32_t *ft = t0, *fs = s0;
    int64_t m = 1;
    while (m > 0) {
        int32_t *kind, *nch, *coff;
        if (dalloc(&kind, m) || dalloc(&nch, m + 1) || dalloc(&coff, m + 1)) return H2B_ERR_CUDA;
        F.add(kind), F.add(nch), F.add(coff);
        const unsigned g = (unsigned)((m + kTB - 1) / kTB);
        k_pair_kind<<<g, kTB>>>(R, C, two_eta, ft, fs, m, kind, nch);
        H2B_CUDA_TRY(cudaMemset(nch + m, 0, sizeof(int32_t)));
        if (int rc = exclusive_scan(nch, coff, m + 1, tmp, tmp_bytes)) {
            if (tmp) cudaFree(tmp);
            return rc;
        }
        int32_t total;
        H2B_CUDA_TRY(cudaMemcpy(&total, coff + m, sizeof(int32_t), cudaMemcpyDeviceToHost));
        lt.push_back(ft);
        ls.push_back(fs);
        lkind.push_back(kind);
        lcoff.push_back(coff);
        lm.push_back(m);
        int32_t *nt = nullptr, *ns = nullptr;
        if (total > 0) {
            if (dalloc(&nt, total) || dalloc(&ns, total)) return H2B_ERR_CUDA;
            F.add(nt), F.add(ns);
            k_pair_expand<<<g, kTB>>>(R, C, ft, fs, m, nch, coff, nt, ns);
        }
        ft = nt;
        fs = ns;
        m = total;
    }
    if (tmp) cudaFree(tmp);
    H2B_CUDA_TRY(cudaDeviceSynchronize());
    // depth-first order (the recursion tree, level by level on the device):
    // subtree far / near counts bottom-up, then offsets top-down
    const int L = (int)lm.size();
    std::vector<int64_t*> cf(L), cn(L), of(L), on(L);
    for (int l = 0; l < L; ++l) {
        if (dalloc(&cf[l], lm[l]) || dalloc(&cn[l], lm[l]) || dalloc(&of[l], lm[l]) || dalloc(&on[l], lm[l]))
            return H2B_ERR_CUDA;
        F.add(cf[l]), F.add(cn[l]), F.add(of[l]), F.add(on[l]);
    }
    for (int l = L - 1; l >= 0; --l) {
        const unsigned g = (unsigned)((lm[l] + kTB - 1) / kTB);
        k_dfs_count<<<g, kTB>>>(lm[l], lkind[l], lcoff[l], l + 1 < L ? cf[l + 1] : nullptr,
                                l + 1 < L ? cn[l + 1] : nullptr, cf[l], cn[l]);
    }
    int64_t tot[2];
    H2B_CUDA_TRY(cudaMemcpy(&tot[0], cf[0], sizeof(int64_t), cudaMemcpyDeviceToHost));
    H2B_CUDA_TRY(cudaMemcpy(&tot[1], cn[0], sizeof(int64_t), cudaMemcpyDeviceToHost));
    const int64_t nf = tot[0], nn = tot[1];
    *h_n_far = nf;
    *h_n_near = nn;
    if (nf > far_cap || nn > near_cap || (nf && !h_far) || (nn && !h_near))
        return fail(H2B_ERR_CAPACITY, "h2b_block_tree_device: output capacity too small");
    int64_t *dfar, *dnear;
    if (dalloc(&dfar, 2 * nf) || dalloc(&dnear, 2 * nn)) return H2B_ERR_CUDA;
    F.add(dfar), F.add(dnear);
    H2B_CUDA_TRY(cudaMemset(of[0], 0, sizeof(int64_t)));
    H2B_CUDA_TRY(cudaMemset(on[0], 0, sizeof(int64_t)));
    for (int l = 0; l < L; ++l) {
        const unsigned g = (unsigned)((lm[l] + kTB - 1) / kTB);
        k_dfs_place<<<g, kTB>>>(lm[l], lt[l], ls[l], lkind[l], lcoff[l], of[l], on[l],
                                l + 1 < L ? cf[l + 1] : nullptr, l + 1 < L ? cn[l + 1] : nullptr,
                                l + 1 < L ? of[l + 1] : nullptr, l + 1 < L ? on[l + 1] : nullptr, dfar, dnear);
    }
    H2B_CUDA_TRY(cudaGetLastError());
    if (nf) H2B_CUDA_TRY(cudaMemcpy(h_far, dfar, sizeof(int64_t) * 2 * nf, cudaMemcpyDeviceToHost));
    if (nn) H2B_CUDA_TRY(cudaMemcpy(h_near, dnear, sizeof(int64_t) * 2 * nn, cudaMemcpyDeviceToHost));
    return ok();
}
