// Host-side structure layer: geometric cluster tree and admissibility block
// tree, bit-exact with the reference (`h2bem.clustering`).
//
// Compiled with -ffp-contract=off: every floating-point expression below is
// evaluated exactly as written (IEEE binary64, round-to-nearest), which is what
// makes the integer outputs (perm, node ranges, far/near lists) identical to
// the numpy reference.  The one place the reference goes through BLAS is the
// Euclidean norm of a 3-vector inside admissibility (np.linalg.norm -> ddot);
// on the reference host that is fma(c, c, fma(b, b, a*a)) and we spell it out.

#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "h2b_internal.h"

namespace {

struct TreeBuilder {
    const double* boxes;  // n x 2 x 3
    int64_t r_leaf;
    std::vector<double> centers;  // n x 3
    int64_t* perm;
    int64_t* start;
    int64_t* end;
    int64_t* depth;
    int64_t* left;
    int64_t* right;
    double* node_boxes;
    int64_t counter = 0;

    // clustering.py:96-118 (build): tight box, longest axis, midpoint of the
    // centre coordinates, `c <= mid` to the left in input order, stable-median
    // fallback when one side would be empty; uid = preorder creation counter.
    int64_t build(std::vector<int64_t>& ids, int64_t s, int64_t d) {
        const int64_t cnt = (int64_t)ids.size();
        double lo[3], hi[3];
        for (int k = 0; k < 3; ++k) {
            lo[k] = boxes[ids[0] * 6 + k];
            hi[k] = boxes[ids[0] * 6 + 3 + k];
        }
        for (int64_t i = 1; i < cnt; ++i) {
            const double* b = boxes + ids[i] * 6;
            for (int k = 0; k < 3; ++k) {
                lo[k] = std::min(lo[k], b[k]);
                hi[k] = std::max(hi[k], b[3 + k]);
            }
        }
        const int64_t uid = counter++;
        start[uid] = s;
        end[uid] = s + cnt;
        depth[uid] = d;
        left[uid] = right[uid] = -1;
        for (int k = 0; k < 3; ++k) {
            node_boxes[uid * 6 + k] = lo[k];
            node_boxes[uid * 6 + 3 + k] = hi[k];
        }
        if (cnt <= r_leaf) {
            std::copy(ids.begin(), ids.end(), perm + s);
            return uid;
        }
        int axis = 0;
        double best = hi[0] - lo[0];
        for (int k = 1; k < 3; ++k) {
            const double e = hi[k] - lo[k];
            if (e > best) {
                best = e;
                axis = k;
            }
        }
        std::vector<double> c(cnt);
        double cmin = INFINITY, cmax = -INFINITY;
        for (int64_t i = 0; i < cnt; ++i) {
            c[i] = centers[ids[i] * 3 + axis];
            cmin = std::min(cmin, c[i]);
            cmax = std::max(cmax, c[i]);
        }
        const double mid = 0.5 * (cmin + cmax);
        std::vector<char> mask(cnt);
        int64_t nl = 0;
        for (int64_t i = 0; i < cnt; ++i) {
            mask[i] = c[i] <= mid;
            nl += mask[i];
        }
        if (nl == 0 || nl == cnt) {
            std::vector<int64_t> order(cnt);
            std::iota(order.begin(), order.end(), 0);
            std::stable_sort(order.begin(), order.end(),
                             [&](int64_t a, int64_t b) { return c[a] < c[b]; });
            std::fill(mask.begin(), mask.end(), 0);
            const int64_t half = cnt / 2;
            for (int64_t i = 0; i < half; ++i) mask[order[i]] = 1;
            nl = half;
        }
        std::vector<int64_t> lids, rids;
        lids.reserve(nl);
        rids.reserve(cnt - nl);
        for (int64_t i = 0; i < cnt; ++i) (mask[i] ? lids : rids).push_back(ids[i]);
        ids.clear();
        ids.shrink_to_fit();
        const int64_t l = build(lids, s, d + 1);
        const int64_t r = build(rids, s + nl, d + 1);
        left[uid] = l;
        right[uid] = r;
        return uid;
    }
};

// clustering.py:7-21 with the host BLAS ddot spelled out.
inline double norm3(double a, double b, double c) {
    return std::sqrt(std::fma(c, c, std::fma(b, b, a * a)));
}

inline double box_diameter(const double* bx) {
    return norm3(bx[3] - bx[0], bx[4] - bx[1], bx[5] - bx[2]);
}

inline double box_distance(const double* a, const double* b) {
    double g[3];
    for (int k = 0; k < 3; ++k) {
        const double u = a[k] - b[3 + k];
        const double v = b[k] - a[3 + k];
        const double m = (u >= v) ? u : v;  // np.maximum (no NaNs here)
        g[k] = (0.0 >= m) ? 0.0 : m;
    }
    return norm3(g[0], g[1], g[2]);
}

struct BlockBuilder {
    const h2b_tree* row;
    const h2b_tree* col;
    double two_eta;
    std::vector<double> rdiam, cdiam;
    std::vector<int64_t> far, near;

    // clustering.py:149-160: admissible first, then leaf x leaf -> near, else the
    // children product in row-major order (a leaf stands in for itself).
    void descend(int64_t t, int64_t s) {
        const double* bt = row->boxes + t * 6;
        const double* bs = col->boxes + s * 6;
        const double diam = std::max(rdiam[t], cdiam[s]);
        if (diam <= two_eta * box_distance(bt, bs)) {
            far.push_back(t);
            far.push_back(s);
            return;
        }
        const bool tl = row->left[t] < 0, sl = col->left[s] < 0;
        if (tl && sl) {
            near.push_back(t);
            near.push_back(s);
            return;
        }
        int64_t ts[2] = {t, -1}, ss[2] = {s, -1};
        int nt = 1, ns = 1;
        if (!tl) {
            ts[0] = row->left[t];
            ts[1] = row->right[t];
            nt = 2;
        }
        if (!sl) {
            ss[0] = col->left[s];
            ss[1] = col->right[s];
            ns = 2;
        }
        for (int i = 0; i < nt; ++i)
            for (int j = 0; j < ns; ++j) descend(ts[i], ss[j]);
    }
};

}  // namespace

extern "C" int h2b_cluster_tree(const double* h_boxes, int64_t n, int64_t r_leaf, int64_t* h_perm,
                                int64_t* h_n_nodes, int64_t* h_start, int64_t* h_end,
                                int64_t* h_depth, int64_t* h_left, int64_t* h_right,
                                double* h_node_boxes) {
    if (n <= 0) return h2b::fail(H2B_ERR_INVALID, "cannot build a cluster tree over an empty index set");
    if (r_leaf < 1) return h2b::fail(H2B_ERR_INVALID, "r_leaf must be >= 1");
    if (!h_boxes || !h_perm || !h_n_nodes || !h_start || !h_end || !h_depth || !h_left || !h_right ||
        !h_node_boxes)
        return h2b::fail(H2B_ERR_INVALID, "h2b_cluster_tree: null pointer");
    try {
        TreeBuilder tb;
        tb.boxes = h_boxes;
        tb.r_leaf = r_leaf;
        tb.centers.resize(n * 3);
        for (int64_t i = 0; i < n; ++i)
            for (int k = 0; k < 3; ++k)
                tb.centers[i * 3 + k] = 0.5 * (h_boxes[i * 6 + k] + h_boxes[i * 6 + 3 + k]);
        tb.perm = h_perm;
        tb.start = h_start;
        tb.end = h_end;
        tb.depth = h_depth;
        tb.left = h_left;
        tb.right = h_right;
        tb.node_boxes = h_node_boxes;
        std::vector<int64_t> ids(n);
        std::iota(ids.begin(), ids.end(), 0);
        tb.build(ids, 0, 0);
        *h_n_nodes = tb.counter;
    } catch (const std::exception& e) {
        return h2b::fail(H2B_ERR_INVALID, std::string("h2b_cluster_tree: ") + e.what());
    }
    return h2b::ok();
}

extern "C" int h2b_block_tree(const h2b_tree* row, const h2b_tree* col, double eta, int64_t* h_far,
                              int64_t far_cap, int64_t* h_near, int64_t near_cap,
                              int64_t* h_n_far, int64_t* h_n_near) {
    if (!row || !col || !h_n_far || !h_n_near) return h2b::fail(H2B_ERR_INVALID, "h2b_block_tree: null pointer");
    if (!(eta > 0.0)) return h2b::fail(H2B_ERR_INVALID, "eta must be positive");
    try {
        BlockBuilder bb;
        bb.row = row;
        bb.col = col;
        bb.two_eta = 2.0 * eta;
        bb.rdiam.resize(row->n_nodes);
        bb.cdiam.resize(col->n_nodes);
        for (int64_t i = 0; i < row->n_nodes; ++i) bb.rdiam[i] = box_diameter(row->boxes + 6 * i);
        for (int64_t i = 0; i < col->n_nodes; ++i) bb.cdiam[i] = box_diameter(col->boxes + 6 * i);
        bb.descend(0, 0);
        const int64_t nf = (int64_t)bb.far.size() / 2, nn = (int64_t)bb.near.size() / 2;
        *h_n_far = nf;
        *h_n_near = nn;
        if (nf > far_cap || nn > near_cap || (nf && !h_far) || (nn && !h_near))
            return h2b::fail(H2B_ERR_CAPACITY, "h2b_block_tree: output capacity too small");
        if (nf) std::memcpy(h_far, bb.far.data(), sizeof(int64_t) * 2 * nf);
        if (nn) std::memcpy(h_near, bb.near.data(), sizeof(int64_t) * 2 * nn);
    } catch (const std::exception& e) {
        return h2b::fail(H2B_ERR_INVALID, std::string("h2b_block_tree: ") + e.what());
    }
    return h2b::ok();
}
