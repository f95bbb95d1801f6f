/*
 * h2b.h — C ABI of the B200-native H^2-matvec + Galerkin nearfield quadrature
 * library (libh2b.so), the drop-in boundary for the hot path of the reference
 * package `h2bem` (arXiv 2001.05523).
 *
 * Every entry point is `extern "C"`, takes plain pointers and sizes, returns an
 * int status (H2B_OK == 0) and never throws.  The message of the last failure
 * on the calling thread is available through h2b_last_error().  Pointers named
 * d_* are DEVICE pointers (owned by the caller, e.g. torch tensors); h_* are
 * host pointers.  `stream` is a cudaStream_t passed as void* (NULL = legacy
 * default stream).  All device work is stream-ordered; functions that must
 * return host-visible sizes synchronise the stream and say so.
 *
 * Reference interfaces replaced (paths relative to /root/reference/pkg/src/h2bem):
 *   h2b_cluster_tree     <- clustering.build_cluster_tree          clustering.py:78-121
 *   h2b_block_tree       <- clustering.BlockTree._descend          clustering.py:137-160
 *   h2b_panel_points     <- quadrature.triangle_points             quadrature.py:71-87
 *   h2b_touch_count/fill <- kernels.touching_pairs/_classify_pairs  kernels.py:246-254,333-343
 *                           + quadrature.classify_panel_pair        quadrature.py:90-118
 *   h2b_singular         <- kernels.SingularTable (all touching pairs) kernels.py:346-362
 *   h2b_pair_integrals   <- kernels.pair_integrals (any pair list)  kernels.py:260-319
 *   h2b_pair_blocks_slp  <- kernels.panel_pair_matrix(SLP)+slp_block kernels.py:365-445
 *   h2b_pair_blocks_dlp  <- kernels.panel_pair_matrix(DLP)+dlp_block kernels.py:365-434,448-468
 *   h2b_plan_create /
 *   h2b_matvec           <- containers.H2Matrix.matvec             containers.py:254-270
 *                           (ClusterBasis.forward/backward          containers.py:201-228)
 *   h2b_diagonal         <- containers.H2Matrix.diagonal           containers.py:290-301
 *   h2b_basis_forward /
 *   h2b_basis_backward   <- containers.ClusterBasis.forward/backward containers.py:201-228
 *   h2b_matmat           <- (no reference counterpart: H2Matrix.matvec per column, containers.py:254-270)
 *   h2b_cg_*             <- solver.cg (vector updates, dots)      solver.py:22-59
 *   h2b_gca_columns /
 *   h2b_gca_aca          <- gca.build_basis (green_columns, cross_interpolate) gca.py:149-179,
 *                           lowrank.aca_inverse_core               lowrank.py:154-184
 */
#ifndef H2B_H
#define H2B_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (mapped to the reference's Python exceptions) ---------- */
#define H2B_OK 0
#define H2B_ERR_INVALID 1   /* ValueError: bad argument                         */
#define H2B_ERR_CUDA 2      /* RuntimeError: CUDA failure                       */
#define H2B_ERR_NONFINITE 3 /* FloatingPointError: non-finite nearfield entry   */
#define H2B_ERR_TOUCHING 4  /* ValueError: touching pair with require_disjoint  */
#define H2B_ERR_MISSING 5   /* KeyError: pair missing from the singular table   */
#define H2B_ERR_CAPACITY 6  /* output capacity too small; sizes were returned   */

/* operator kinds (kernels.SLP / kernels.DLP) */
#define H2B_SLP 0
#define H2B_DLP 1

/* touching-pair case codes = number of shared vertices (kernels.py:246-254) */
#define H2B_DISJOINT 0
#define H2B_VERTEX 1
#define H2B_EDGE 2
#define H2B_IDENTICAL 3

int h2b_last_error(char* buf, size_t n);
int h2b_abi_version(void);

/* ======================= structure (host, bit-exact) ======================= */

/* Geometric bisection tree over support boxes (n x 2 x 3, [min; max]).
 * Node arrays have capacity 2n-1 and are filled in preorder (uid order);
 * left/right = -1 for leaves, node_boxes is (2n-1) x 2 x 3. */
int h2b_cluster_tree(const double* h_boxes, int64_t n, int64_t r_leaf, int64_t* h_perm,
                     int64_t* h_n_nodes, int64_t* h_start, int64_t* h_end, int64_t* h_depth,
                     int64_t* h_left, int64_t* h_right, double* h_node_boxes);

typedef struct {
    int64_t n_nodes;
    const int64_t* left;  /* child uids, -1 for leaves (root = uid 0) */
    const int64_t* right;
    const double* boxes;  /* n_nodes x 2 x 3 */
} h2b_tree;

/* Admissibility-driven leaf partition in the reference's depth-first order.
 * far/near are (cap x 2) [row uid, col uid].  On H2B_ERR_CAPACITY the counts
 * are still written and the call may be repeated with larger buffers. */
int h2b_block_tree(const h2b_tree* row, const h2b_tree* col, double eta, int64_t* h_far,
                   int64_t far_cap, int64_t* h_near, int64_t near_cap, int64_t* h_n_far,
                   int64_t* h_n_near);
/* The same two builders on the device, same arguments and
 * outputs (host arrays), bit-exact with the host builders: the cluster tree
 * level by level (block reductions for boxes and midpoints, one scan for the
 * stable split), the block tree one recursion level at a time with the
 * depth-first order restored from subtree counts. */
int h2b_cluster_tree_device(const double* h_boxes, int64_t n, int64_t r_leaf, int64_t* h_perm,
                            int64_t* h_n_nodes, int64_t* h_start, int64_t* h_end, int64_t* h_depth,
                            int64_t* h_left, int64_t* h_right, double* h_node_boxes);
int h2b_block_tree_device(const h2b_tree* row, const h2b_tree* col, double eta, int64_t* h_far,
                          int64_t far_cap, int64_t* h_near, int64_t near_cap, int64_t* h_n_far,
                          int64_t* h_n_near);

/* ======================= Galerkin quadrature (device) ====================== */

typedef struct {
    int64_t n_vertices, n_triangles;
    const double* d_vertices;   /* V x 3 */
    const int32_t* d_triangles; /* F x 3 */
    const double* d_normals;    /* F x 3 */
    const double* d_areas;      /* F     */
    const int64_t* d_vt_ptr;    /* V+1: vertex -> incident triangles (CSR) */
    const int32_t* d_vt_idx;    /* 3F  */
} h2b_mesh;

/* Regular (Duffy tensor) rule points on every panel: out = SoA [4][F][Q]
 * (x, y, z, weight incl. 2*area).  rule_xy: Q x 2 reference points, rule_w: Q. */
int h2b_panel_points(const h2b_mesh* m, const double* d_rule_xy, const double* d_rule_w,
                     int32_t Q, double* d_out, void* stream);

typedef struct {
    int64_t n_panels, n_pairs;
    const int64_t* d_row_ptr; /* F+1, CSR over row panel                      */
    const int32_t* d_col;     /* n_pairs, ascending within a row              */
    const int32_t* d_info;    /* code | perm_a << 2 | perm_b << 8 (2 bits/idx) */
    const int32_t* d_case_list; /* n_pairs pair ids grouped by case          */
    const int64_t* h_case_off;  /* 4: start of identical/edge/vertex/end in case_list */
    /* optional (NULL if absent, see h2b_touch_half): one pair id per unordered
     * touching pair {a, b} (a < b; identical pairs once), grouped by case */
    const int32_t* d_half_list;
    const int64_t* h_half_off;  /* 4: segment starts in d_half_list + end */
} h2b_touch;

/* Pass 1: per row panel touching count -> exclusive scan in d_row_ptr (F+1),
 * per-case counts in h_case_count[4] (identical, edge, vertex, total).
 * Synchronises the stream. */
int h2b_touch_count(const h2b_mesh* m, int64_t* d_row_ptr, int64_t* h_case_count, void* stream);
/* Pass 2: sorted columns, case/permutation info and the case-grouped pair list. */
int h2b_touch_fill(const h2b_mesh* m, const int64_t* d_row_ptr, const int64_t* h_case_count,
                   int32_t* d_col, int32_t* d_info, int32_t* d_case_list, void* stream);

/* Pass 3 (optional): the unordered-pair list of the symmetric single-layer
 * table.  Every touching relation is symmetric, so the edge and vertex
 * segments hold exactly half of the ordered pairs (checked; H2B_ERR_INVALID
 * otherwise).  d_half_list: n_identical + (n_edge + n_vertex) / 2 entries,
 * h_half_off[4] receives its segment offsets.  Synchronises. */
int h2b_touch_half(const h2b_touch* t, int32_t* d_half_list, int64_t* h_half_off, void* stream);

typedef struct {
    int64_t n;         /* number of rule points */
    const double* d_p; /* n x 4: (u1, v1, u2, v2) */
    const double* d_w; /* n */
} h2b_rule;

/* Sauter-Schwab integrals of every touching pair.  rules[0..2] = identical,
 * edge, vertex rules (quadrature.sauter_schwab_rule).  values: n_pairs (SLP)
 * or n_pairs x 3 (DLP, original local vertex order of the column panel).
 * SLP with t->d_half_list set: each unordered pair is integrated once (the
 * reference symmetrises edge/vertex pairs over both orientations,
 * kernels.py:303-309, so G(a,b) = G(b,a)) and written to both ordered ids. */
int h2b_singular(const h2b_mesh* m, const h2b_touch* t, int kind, const h2b_rule* rules,
                 double* d_values, void* stream);

/* kernels.pair_integrals (kernels.py:260-319) on an arbitrary list of n
 * panel pairs (d_pa[i], d_pb[i]): each pair is classified on the device
 * (quadrature.classify_panel_pair) and integrated with the Sauter-Schwab rule
 * of its case, rules[0..3] = identical, edge, vertex, disjoint
 * (quadrature.sauter_schwab_rule).  values: n (SLP; edge/vertex pairs
 * averaged over both orientations) or n x 3 (DLP, original local vertex
 * order of the column panel; identical pairs 0).  Synchronises. */
int h2b_pair_integrals(const h2b_mesh* m, int64_t n, const int32_t* d_pa, const int32_t* d_pb, int kind,
                       const h2b_rule* rules, double* d_values, void* stream);

typedef struct {
    int64_t n_jobs;
    const int64_t* d_jobs;    /* n_jobs x 8: row_off, n_rows, col_off, n_cols, out_off, out_ld,
                               * mirror_off, mirror_ld (mirror_off = -1: none) */
    const int32_t* d_row_idx; /* row panels */
    const int32_t* d_col_idx; /* column panels (SLP) */
} h2b_jobs;

/* Dense SLP blocks out[out_off + r*ld + c] = G(row_idx[row_off+r], col_idx[col_off+c]).
 * Mirrored jobs (symmetric single-layer matrix, G(a,b) = G(b,a)) also write
 * out[mirror_off + c*mirror_ld + r]; a job whose mirror_off == out_off is a
 * diagonal tile (same rows and columns) and only its upper triangle is
 * integrated.  out_off = -1 writes the mirror only (row-sharded assembly:
 * the pair is integrated in the orientation of the single-GPU job, so both
 * give the same bits).
 * Regular pairs: tensor rule with Q points per panel (panel_points).  Touching
 * pairs: value from the singular table (t != NULL) or, when t == NULL
 * (require_disjoint), the call fails with H2B_ERR_TOUCHING.  Synchronises. */
int h2b_pair_blocks_slp(const h2b_mesh* m, const double* d_panel_points, int32_t Q,
                        const h2b_jobs* jobs, const h2b_touch* t, const double* d_touch_values,
                        double* d_out, void* stream);

typedef struct {
    int64_t n_jobs;
    const int64_t* d_jobs;     /* n_jobs x 8: row_off, n_rows, pan_off, n_pan, col_off, n_cols, out_off, out_ld */
    const int32_t* d_row_idx;  /* row panels (P0 dofs)                                  */
    const int32_t* d_pan_idx;  /* column panels incident to the job's column vertices  */
    const int32_t* d_inc_ptr;  /* per job column: CSR into inc (size sum n_cols + n_jobs) */
    const int32_t* d_inc;      /* (local panel << 2 | local vertex) contributions        */
    const int64_t* d_inc_base; /* n_jobs: offset of the job's CSR row pointers           */
} h2b_dlp_jobs;

/* Dense DLP blocks (P0 rows x P1 columns) with the vertex scatter of
 * kernels.dlp_block fused in.  Synchronises. */
int h2b_pair_blocks_dlp(const h2b_mesh* m, const double* d_panel_points, const double* d_lam,
                        int32_t Q, const h2b_dlp_jobs* jobs, const h2b_touch* t,
                        const double* d_touch_values, double* d_out, void* stream);

/* Host-side DLP job builder for h2b_pair_blocks_dlp (replaces the Python
 * construction of the column-panel sets of kernels.py:448-468; identical
 * output).  Blocks: rows[row_ptr[b]:row_ptr[b+1]] (panel ids),
 * cols[col_ptr[b]:col_ptr[b+1]] (vertex ids), out_off[b], ld[b]; mesh
 * vertex->triangle CSR (vptr, vidx) and triangles (n x 3).  The result is
 * read with h2b_dlp_jobs_sizes / h2b_dlp_jobs_copy and released with
 * h2b_dlp_jobs_free. */
typedef struct h2b_dlp_build h2b_dlp_build;
int h2b_dlp_jobs_build(int64_t n_verts, const int64_t* vptr, const int64_t* vidx, const int64_t* tris,
                       int64_t n_blocks, const int64_t* row_ptr, const int64_t* rows, const int64_t* col_ptr,
                       const int64_t* cols, const int64_t* out_off, const int64_t* ld, h2b_dlp_build** out);
int h2b_dlp_jobs_sizes(const h2b_dlp_build* b, int64_t* sizes);
int h2b_dlp_jobs_copy(const h2b_dlp_build* b, int64_t* jobs, int32_t* row_idx, int32_t* pan_idx, int32_t* inc_ptr,
                      int32_t* inc, int64_t* inc_base);
int h2b_dlp_jobs_free(h2b_dlp_build* b);

/* Host-side job list of h2b_pair_blocks_slp for a list of n blocks
 * (t, s) = h_uids[i] (n x 2): rows h_row_off[t] .. + h_row_cnt[t] of the row
 * index list, columns h_col_off[s] .. + h_col_cnt[s] of the column index list,
 * written at h_blk_off[i] with leading dimension h_blk_ld[i] (the packed
 * layouts of containers.py:79-98 nearfield / gca.py:194-205 couplings).
 * h2b_block_partners: for every block the index of block (s, t), or -1.
 * h2b_block_jobs with mirrored != 0 (symmetric single layer, block (s, t) =
 * block (t, s)^T) keeps one job per block pair, which also writes the
 * transpose at the partner's place; h_jobs holds 8 n words, *h_n_jobs jobs
 * are written. */
int h2b_block_partners(int64_t n, const int64_t* h_uids, int64_t* h_partner);
int h2b_block_jobs(int64_t n, const int64_t* h_uids, const int64_t* h_row_off, const int64_t* h_row_cnt,
                   const int64_t* h_col_off, const int64_t* h_col_cnt, const int64_t* h_blk_off,
                   const int64_t* h_blk_ld, int mirrored, const int64_t* h_partner, int64_t* h_jobs,
                   int64_t* h_n_jobs);

/* ================= GCA cluster-basis construction (device) ================= */

/* Basis flavors (gca.P0_SLP / gca.P1_DLP): P0 rows are panels (potentials
 * K_VALUE | K_DN_Z), P1 rows are vertices (hat functions, K_DN_X | K_DN_X_DN_Z). */
#define H2B_GCA_P0_SLP 0
#define H2B_GCA_P1_DLP 1
#define H2B_GCA_P1_CURL 2  /* hypersingular: curl-weighted P0 potentials, 6 n_green columns */

/* One tree level of clusters (independent).  Cluster c has rows
 * d_rows[d_row_ptr[c] : d_row_ptr[c+1]] (leaf: its dofs; inner: its children's
 * pivots), n_green = 6 m^2 Green points (x, y, z, sqrt(w), nx, ny, nz, 0) at
 * d_green + 8 n_green c, and a slot at d_l_off[c] of rows x 2 n_green doubles
 * in the L, scratch and V buffers.  max_rows = largest row count. */
typedef struct {
    int64_t n_clusters;
    const int64_t* d_row_ptr;
    const int32_t* d_rows;
    int32_t n_green;
    int32_t max_rows;
    const double* d_green;
    const int64_t* d_l_off;
    int32_t n_cols;  /* columns of L (0: 2 n_green; 6 n_green for H2B_GCA_P1_CURL) */
} h2b_gca_batch;

/* Green-quadrature columns L (rows x 2k, row-major) of every cluster
 * (gca.green_columns <- src/gca.py; panel_potentials / p1_potentials
 * src/kernels.py:97-196), regular rule with Q points per panel
 * (h2b_panel_points), d_lam = Q x 3 barycentrics (P1 only).  Non-finite
 * entries -> H2B_ERR_INVALID.  Synchronises. */
int h2b_gca_columns(const h2b_mesh* m, const double* d_panel_points, int32_t Q, const double* d_lam, int flavor,
                    const h2b_gca_batch* b, double* d_L, void* stream);
/* The P1_CURL flavor (gca.green_columns for HYP, src/gca.py:106-117 with
 * kernels.curl_potentials src/kernels.py:172-196): rows are vertices, L is
 * rows x 6 n_green = [a_x | a_y | a_z | c_x | c_y | c_z], a / c the K_VALUE /
 * K_DN_Z panel potentials of the incident panels weighted by the hat's
 * constant surface curl on each panel (d_curls: 3F x 3, kernels.triangle_curls). */
int h2b_gca_columns_curl(const h2b_mesh* m, const double* d_panel_points, int32_t Q, const double* d_curls,
                         const h2b_gca_batch* b, double* d_L, void* stream);
/* Fully pivoted ACA with inverse core on every L (lowrank.aca_inverse_core,
 * src/lowrank.py:154-184) and the interpolation matrix V = L[:, sigma]
 * inv(L[tau, sigma]) (gca.cross_interpolate).  Outputs: d_rank[c], local pivot
 * rows d_tau[c * tau_cap + i] (tau_cap >= 2 n_green), V (rows x rank,
 * row-major) at d_V + d_l_off[c].  d_scratch (same size as d_L) holds the
 * residuals that do not fit in shared memory. */
int h2b_gca_aca(const h2b_gca_batch* b, double eps, const double* d_L, double* d_scratch, int32_t* d_rank,
                int32_t* d_tau, int32_t tau_cap, double* d_V, void* stream);

/* ================= cluster-basis transforms (device) ====================== */

/* A nested cluster basis (ClusterBasis, containers.py:189-238) on the device:
 * per uid child uids (-1 for leaves), permuted start and size, rank k_t and the
 * offsets of V_t (leaves, |t| x k_t row-major), E_t (non-root, k_t x k_parent)
 * and of the cluster's coefficients in a packed coefficient vector; clusters
 * listed level by level (root level first): level l = d_level_nodes
 * [h_level_off[l], h_level_off[l+1]). */
typedef struct {
    int64_t n_nodes;
    const int32_t* d_left;
    const int32_t* d_right;
    const int32_t* d_start;
    const int32_t* d_size;
    const int32_t* d_rank;
    const int64_t* d_v_off;
    const int64_t* d_e_off;
    const int64_t* d_hat_off;
    const double* d_V;
    const double* d_E;
    int32_t n_levels;
    const int64_t* h_level_off; /* host, n_levels + 1 */
    const int32_t* d_level_nodes;
} h2b_basis;

/* ClusterBasis.forward (containers.py:201-212): x_hat of every cluster from the
 * permuted vector xp (leaves V_t^T xp|_t, parents sum over children of
 * E_ch^T x_hat_ch).  d_xhat: packed coefficients (d_hat_off). */
int h2b_basis_forward(const h2b_basis* b, const double* d_xp, double* d_xhat, void* stream);
/* ClusterBasis.backward (containers.py:214-228): top down y_hat_ch += E_ch
 * y_hat_t, then leaves yp|_t += V_t y_hat_t.  d_yhat (packed) is updated in
 * place; d_yp is accumulated into. */
int h2b_basis_backward(const h2b_basis* b, double* d_yhat, double* d_yp, void* stream);

/* Hypersingular P1 x P1 blocks (kernels.hyp_block, kernels.py:471-511) from
 * single-layer panel-pair values d_vals (h2b_pair_blocks_slp over each
 * block's incident row x column panels, row-major n_pb wide at v_off):
 * out[out_off + i ld + j] = sum over incident panels a of row vertex i and b
 * of column vertex j of <curl_a(i), curl_b(j)> V_ab, in the reference's
 * np.add.at order.  d_desc: int64 x 8 per block (nr, nc, v_off, n_pb, r_inc,
 * c_inc, out_off, ld); incidences of row vertex i of a block:
 * [d_r_ptr[r_inc + i], d_r_ptr[r_inc + i + 1]) into d_r_pos (panel position in
 * the block's row panel list) and d_r_cl (3 * panel + local vertex: row of the
 * (3F x 3) curl table d_curls); the same for columns.  Raises
 * H2B_ERR_NONFINITE on a non-finite entry.  Synchronises. */
int h2b_hyp_scatter(int64_t n_blocks, const int64_t* d_desc, const int32_t* d_r_ptr, const int32_t* d_r_pos,
                    const int32_t* d_r_cl, const int32_t* d_c_ptr, const int32_t* d_c_pos, const int32_t* d_c_cl,
                    const double* d_curls, const double* d_vals, double* d_out, void* stream);

/* Block transpose between two packed layouts (H2Matrix.rmatvec,
 * containers.py:272-288, runs the matvec on the transposed operator): for each
 * of n_blocks descriptors (src_off, src_ld, rows, cols, dst_off, dst_ld),
 * int64 x 6 on the device, dst[dst_off + j dst_ld + i] = src[src_off + i src_ld + j].
 * Entries of dst outside the blocks are left untouched. */
int h2b_transpose_blocks(int64_t n_blocks, const int64_t* d_desc, const double* d_src, double* d_dst, void* stream);

/* ====================== CG vector kernels (device) ========================= */

/* Fused passes of the Jacobi-preconditioned CG iteration (solver.cg,
 * src/solver.py:22-59) with deterministic reductions (fixed grid, per-CTA
 * partials summed in index order).  Scalars live on the device in
 * scal = (rz, pAp, rz_new, r.r); with row-sharded vectors the caller
 * all-reduces the scalars a call writes before the next call.  d_work: a
 * zero-initialised workspace of h2b_cg_workspace_size bytes (one per stream). */
int h2b_cg_workspace_size(int64_t* bytes);
/* d_out[0] = a . b */
int h2b_cg_dot(const double* d_a, const double* d_b, int64_t n, void* d_work, double* d_out, void* stream);
/* alpha = scal[0] / scal[1]; x += alpha p; r -= alpha Ap; z = r * inv_diag
 * (z unused when inv_diag is NULL: then z is r); d_out[0..1] = (r.z, r.r). */
int h2b_cg_step(int64_t n, const double* d_scal, double* d_x, double* d_r, const double* d_p, const double* d_Ap,
                const double* d_inv_diag, double* d_z, void* d_work, double* d_out, void* stream);
/* p = z + (scal[2] / scal[0]) p */
int h2b_cg_direction(int64_t n, const double* d_scal, const double* d_z, double* d_p, void* stream);

/* ============================ H^2 matvec (device) ========================== */

/* Packed operator layout (all device pointers; int32 unless noted).
 * Column tree (forward transform) and row tree (backward) are described by
 * per-node arrays indexed by uid; couplings S are stored per row cluster as one
 * row-major k_t x K_t matrix (K_t = sum of k_s over its far blocks, in far-list
 * order); nearfield D per row leaf as one row-major |t| x C_t matrix (C_t = sum
 * of |s| over its near blocks). */
typedef struct {
    int64_t n_rows, n_cols;
    /* permutations: x_p[i] = x[col_perm[i]], y[row_perm[i]] = y_p[i] */
    const int64_t* col_perm;
    const int64_t* row_perm;
    /* column tree */
    int32_t c_nodes, c_leaves;
    const int32_t* c_parent;  /* -1 root */
    const int32_t* c_child;   /* 2 per node, -1 */
    const int32_t* c_start;
    const int32_t* c_size;
    const int32_t* c_rank;
    const int64_t* c_v_off;   /* leaves: offset of V (|t| x k) in c_V */
    const int64_t* c_e_off;   /* non-root: offset of E (k x k_parent) in c_E */
    const int64_t* c_xhat_off;
    const int32_t* c_leaf_list;
    const double* c_V;
    const double* c_E;
    int64_t xhat_len;
    /* row tree */
    int32_t r_nodes, r_leaves;
    const int32_t* r_parent;
    const int32_t* r_start;
    const int32_t* r_size;
    const int32_t* r_rank;
    const int64_t* r_v_off;
    const int64_t* r_e_off;
    const int64_t* r_yhat_off;
    const int32_t* r_order;   /* top-down processing order (parents first) */
    const double* r_V;
    const double* r_E;
    int64_t yhat_len;
    /* couplings per row node */
    const int64_t* s_off;     /* offset of the k_t x K_t matrix */
    const int32_t* s_cols;    /* K_t */
    const int32_t* far_ptr;   /* n_rnodes+1 into far_col */
    const int32_t* far_col;   /* column uid per far block, far-list order within the row */
    const double* S;
    /* nearfield per row leaf */
    const int64_t* d_off;     /* offset of the |t| x C_t matrix (per row node; leaves only) */
    const int32_t* d_cols;    /* C_t */
    const int32_t* near_ptr;  /* n_rnodes+1 into near_col */
    const int32_t* near_col;  /* column uid per near block */
    const double* D;
    /* right-hand-side gather indices: per row node, the x index of every
     * column of its nearfield matrix (C_t entries at d_goff) and the x_hat
     * index of every column of its coupling matrix (K_t entries at s_goff);
     * padding columns point at index 0 (their matrix entries are zero) */
    const int64_t* d_goff;
    const int32_t* d_gidx;
    const int64_t* s_goff;
    const int32_t* s_gidx;
    /* which row nodes this rank processes (multi-GPU row sharding); all if NULL */
    int32_t n_owned;
    const int32_t* owned;     /* subset of r_order, still parents first */
} h2b_layout;

typedef struct h2b_plan h2b_plan;

/* Builds the task records of the fused matvec from the layout (the arrays stay
 * owned by the caller and must outlive the plan).  A single-GPU plan (owned ==
 * NULL) whose row and column trees coincide and whose nearfield blocks satisfy
 * D_(t,s) == D_(s,t)^T bit for bit (checked on the device) packs a copy of the
 * upper blocks and streams each block pair once; later changes to D are not
 * seen by such a plan (create a new one).  Every plan also owns a transposed
 * copy of the row basis it applies ([E_t^T | V_t^T] per row cluster,
 * 8 (sum |V_t| + sum |E_t|) bytes: the operands of the downward steps in the
 * layout their products read, staged by one bulk copy each); later changes
 * to r_V / r_E are likewise not seen.  Environment knobs read here (test
 * and diagnostics only): H2B_NEAR_SYM=0 (stream every block, one-sided),
 * H2B_TRACE=1 (per-task timeline).
 * A plan owns one ticket counter and one set of inter-CTA scratch buffers, so
 * its launches are serialised: calls from several host threads take a
 * per-plan lock, and a launch on a different stream than the plan's previous
 * launch first waits for that launch (event).  Different plans run
 * concurrently. */
int h2b_plan_create(const h2b_layout* layout, h2b_plan** out);
int h2b_plan_destroy(h2b_plan* plan);
/* y = A x for device vectors in natural dof order (x: n_cols, y: n_rows). */
int h2b_matvec(h2b_plan* plan, const double* d_x, double* d_y, void* stream);
/* Same through host buffers: H2D copy of x, matvec, D2H copy of y, synchronised. */
int h2b_matvec_host(h2b_plan* plan, const double* h_x, double* h_y, void* stream);
/* Diagnostics: per-CTA timeline of the last matvec when the plan was created
 * with the environment variable H2B_TRACE=1 (3 words per CTA ticket: start
 * ns, end ns, SM id; then 5 words of ticket-range boundaries). */
int h2b_plan_trace(h2b_plan* plan, unsigned long long* h_out, int64_t cap);
/* Plan facts (9 words): symmetric nearfield in use (0/1; single-GPU plans whose
 * nearfield is symmetric bit for bit stream each block pair once), nearfield
 * bytes per matvec, nearfield tasks, coupling tasks, partial-vector bytes,
 * symmetric couplings in use (always 0), coupling bytes per matvec, TMA stage
 * bytes per CTA (chosen at plan creation from the CTA's other shared memory;
 * environment H2B_STAGE_KB overrides), dynamic shared memory per CTA. */
int h2b_plan_info(h2b_plan* plan, int64_t* h_out);
/* ====================== multi-GPU (row-sharded plans) ==================== */

/* A plan created for one rank of a row sharding (h2b_layout.owned / row_perm,
 * col_perm = position of every permuted column dof in the gathered x of
 * nranks equal chunks) plus an NCCL communicator: h2b_matvec_sharded takes
 * the rank's chunk of x (permuted order), all-gathers it over NCCL on the
 * call's stream and writes the rank's rows of y.  NCCL is
 * opened at first use (libnccl.so.2); comm is an ncclComm_t. */
#define H2B_COMM_ID_BYTES 128
/* ncclGetUniqueId into h_id (H2B_COMM_ID_BYTES); rank 0 shares it. */
int h2b_comm_unique_id(void* h_id);
/* ncclCommInitRank on `device` (collective over the nranks callers). */
int h2b_comm_init(void** comm, int nranks, const void* h_id, int rank, int device);
int h2b_comm_destroy(void* comm);
/* Attach the communicator: this plan is rank `rank` of `nranks`, each rank's
 * x chunk is `chunk` doubles (gathered buffer nranks x chunk). */
int h2b_plan_set_comm(h2b_plan* plan, void* comm, int rank, int nranks, int64_t chunk);
/* y_local = this rank's rows of A x from x_local = this rank's x chunk (both
 * permuted order, device memory): ncclAllGather + the fused matvec, stream
 * ordered. */
int h2b_matvec_sharded(h2b_plan* plan, const double* d_x_local, double* d_y_local, void* stream);

/* x_hat exchange (SURVEY 8(e) "better variant"): a row-sharded plan whose
 * forward tasks cover only this rank's column clusters (h_cmask[u] = 1 for the
 * clusters inside the rank's permuted range, int8 per column node).
 * h2b_xhat_forward runs them (x: the gathered x of h2b_matvec_sharded) and
 * packs their coefficients into d_send (send_len doubles, clusters in uid
 * order); after an all-gather of every rank's send buffer, h2b_xhat_main
 * imports the coefficients (h_src[u] = offset of cluster u in the gathered
 * buffer, -1 for clusters spanning several ranks, set once by
 * h2b_xhat_set_import), climbs the spanning clusters with the forward
 * climb's arithmetic and runs the bands: the rank's rows of y, the bits of
 * the plan without the exchange.  h2b_xhat_info: n_own, send_len, forward
 * tasks, imported clusters, spanning clusters. */
int h2b_plan_create_xhat(const h2b_layout* layout, const int8_t* h_cmask, h2b_plan** plan);
int h2b_xhat_info(h2b_plan* plan, int64_t* h_out);
int h2b_xhat_set_import(h2b_plan* plan, const int64_t* h_src);
int h2b_xhat_forward(h2b_plan* plan, const double* d_x, double* d_send, void* stream);
int h2b_xhat_main(h2b_plan* plan, const double* d_x, const double* d_recv, double* d_y, void* stream);

/* Multi-right-hand-side product Y = A X for 1 <= nrhs <= 16 device vectors
 * (X: n_cols x nrhs, Y: n_rows x nrhs, row-major, natural dof order) over the
 * same packed operator as a matvec plan (single-GPU layouts).  The reference
 * has no block product; each column equals H2Matrix.matvec of that column
 * (containers.py:254-270) to rounding.  Dense products on the FP64 tensor
 * cores (mma.sync m8n8k4.f64); level-synchronous launches on `stream`. */
typedef struct h2b_mmplan h2b_mmplan;
int h2b_matmat_create(const h2b_layout* layout, h2b_mmplan** out);
int h2b_matmat_destroy(h2b_mmplan* plan);
int h2b_matmat(h2b_mmplan* plan, const double* d_X, double* d_Y, int32_t nrhs, void* stream);

/* Diagonal of the (square) operator from the nearfield, natural order. */
int h2b_diagonal(h2b_plan* plan, double* d_diag, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* H2B_H */
