"""ctypes binding of libh2b.so (include/h2b.h).

This is the reference-side binding a maintainer would add: plain pointers and
sizes cross the boundary, status codes come back and are mapped onto the
exceptions the reference raises (ValueError, FloatingPointError, KeyError).
There is no fallback: if the library is missing, importing a GPU entry point
raises immediately.
"""

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_lib", "libh2b.so")

H2B_OK = 0
H2B_ERR_INVALID = 1
H2B_ERR_CUDA = 2
H2B_ERR_NONFINITE = 3
H2B_ERR_TOUCHING = 4
H2B_ERR_MISSING = 5
H2B_ERR_CAPACITY = 6

H2B_SLP = 0
H2B_DLP = 1

c_i64p = ctypes.POINTER(ctypes.c_int64)
c_dp = ctypes.POINTER(ctypes.c_double)
vp = ctypes.c_void_p


class Tree(ctypes.Structure):
    _fields_ = [("n_nodes", ctypes.c_int64), ("left", vp), ("right", vp), ("boxes", vp)]


class Mesh(ctypes.Structure):
    _fields_ = [
        ("n_vertices", ctypes.c_int64), ("n_triangles", ctypes.c_int64),
        ("d_vertices", vp), ("d_triangles", vp), ("d_normals", vp), ("d_areas", vp),
        ("d_vt_ptr", vp), ("d_vt_idx", vp),
    ]


class Touch(ctypes.Structure):
    _fields_ = [
        ("n_panels", ctypes.c_int64), ("n_pairs", ctypes.c_int64),
        ("d_row_ptr", vp), ("d_col", vp), ("d_info", vp), ("d_case_list", vp), ("h_case_off", vp),
        ("d_half_list", vp), ("h_half_off", vp),
    ]


class Rule(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("d_p", vp), ("d_w", vp)]


class Jobs(ctypes.Structure):
    _fields_ = [("n_jobs", ctypes.c_int64), ("d_jobs", vp), ("d_row_idx", vp), ("d_col_idx", vp)]


class DlpJobs(ctypes.Structure):
    _fields_ = [
        ("n_jobs", ctypes.c_int64), ("d_jobs", vp), ("d_row_idx", vp), ("d_pan_idx", vp),
        ("d_inc_ptr", vp), ("d_inc", vp), ("d_inc_base", vp),
    ]


class GcaBatch(ctypes.Structure):
    _fields_ = [
        ("n_clusters", ctypes.c_int64), ("d_row_ptr", vp), ("d_rows", vp), ("n_green", ctypes.c_int32),
        ("max_rows", ctypes.c_int32), ("d_green", vp), ("d_l_off", vp),
        ("n_cols", ctypes.c_int32),
    ]


class Basis(ctypes.Structure):
    _fields_ = [
        ("n_nodes", ctypes.c_int64), ("d_left", vp), ("d_right", vp), ("d_start", vp), ("d_size", vp),
        ("d_rank", vp), ("d_v_off", vp), ("d_e_off", vp), ("d_hat_off", vp), ("d_V", vp), ("d_E", vp),
        ("n_levels", ctypes.c_int32), ("h_level_off", vp), ("d_level_nodes", vp),
    ]


class Layout(ctypes.Structure):
    _fields_ = [
        ("n_rows", ctypes.c_int64), ("n_cols", ctypes.c_int64),
        ("col_perm", vp), ("row_perm", vp),
        ("c_nodes", ctypes.c_int32), ("c_leaves", ctypes.c_int32),
        ("c_parent", vp), ("c_child", vp), ("c_start", vp), ("c_size", vp), ("c_rank", vp),
        ("c_v_off", vp), ("c_e_off", vp), ("c_xhat_off", vp), ("c_leaf_list", vp),
        ("c_V", vp), ("c_E", vp), ("xhat_len", ctypes.c_int64),
        ("r_nodes", ctypes.c_int32), ("r_leaves", ctypes.c_int32),
        ("r_parent", vp), ("r_start", vp), ("r_size", vp), ("r_rank", vp),
        ("r_v_off", vp), ("r_e_off", vp), ("r_yhat_off", vp), ("r_order", vp),
        ("r_V", vp), ("r_E", vp), ("yhat_len", ctypes.c_int64),
        ("s_off", vp), ("s_cols", vp), ("far_ptr", vp), ("far_col", vp), ("S", vp),
        ("d_off", vp), ("d_cols", vp), ("near_ptr", vp), ("near_col", vp), ("D", vp),
        ("d_goff", vp), ("d_gidx", vp), ("s_goff", vp), ("s_gidx", vp),
        ("n_owned", ctypes.c_int32), ("owned", vp),
    ]


# every symbol include/h2b.h declares (checked by the CPU test-suite)
EXPORTS = (
    "h2b_last_error", "h2b_abi_version", "h2b_cluster_tree", "h2b_block_tree", "h2b_panel_points",
    "h2b_touch_count", "h2b_touch_fill", "h2b_touch_half", "h2b_singular", "h2b_pair_blocks_slp", "h2b_pair_blocks_dlp",
    "h2b_plan_create", "h2b_plan_destroy", "h2b_matvec", "h2b_matvec_host",
    "h2b_diagonal", "h2b_plan_trace", "h2b_plan_info", "h2b_dlp_jobs_build", "h2b_dlp_jobs_sizes", "h2b_dlp_jobs_copy",
    "h2b_dlp_jobs_free", "h2b_gca_columns", "h2b_gca_aca", "h2b_cg_workspace_size", "h2b_cg_dot", "h2b_cg_step",
    "h2b_cg_direction", "h2b_matmat_create", "h2b_matmat_destroy", "h2b_matmat", "h2b_pair_integrals",
    "h2b_basis_forward", "h2b_basis_backward", "h2b_transpose_blocks", "h2b_hyp_scatter",
    "h2b_comm_unique_id", "h2b_comm_init", "h2b_comm_destroy", "h2b_plan_set_comm", "h2b_matvec_sharded",
    "h2b_cluster_tree_device", "h2b_block_tree_device",
    "h2b_gca_columns_curl", "h2b_plan_create_xhat", "h2b_xhat_info", "h2b_xhat_set_import", "h2b_xhat_forward", "h2b_xhat_main",
    "h2b_block_partners", "h2b_block_jobs",
)

_lib = None


def lib():
    """The loaded libh2b.so; raises if it has not been built."""
    global _lib
    if _lib is None:
        path = os.environ.get("H2B_LIB_PATH", LIB_PATH)  # tuning experiments only
        if not os.path.exists(path):
            raise RuntimeError(
                f"libh2b.so not found at {path}: build it with "
                "`python -m paper_2001_05523_b200.build` (no CPU fallback exists)"
            )
        L = ctypes.CDLL(path)
        for name in EXPORTS:
            getattr(L, name).restype = ctypes.c_int
        L.h2b_last_error.argtypes = [ctypes.c_char_p, ctypes.c_size_t]
        L.h2b_cluster_tree.argtypes = [vp, ctypes.c_int64, ctypes.c_int64, vp, vp, vp, vp, vp, vp, vp, vp]
        L.h2b_block_tree.argtypes = [ctypes.POINTER(Tree), ctypes.POINTER(Tree), ctypes.c_double, vp,
                                     ctypes.c_int64, vp, ctypes.c_int64, vp, vp]
        L.h2b_cluster_tree_device.argtypes = L.h2b_cluster_tree.argtypes
        L.h2b_plan_create_xhat.argtypes = [ctypes.POINTER(Layout), vp, ctypes.POINTER(vp)]
        L.h2b_xhat_info.argtypes = [vp, vp]
        L.h2b_xhat_set_import.argtypes = [vp, vp]
        L.h2b_xhat_forward.argtypes = [vp, vp, vp, vp]
        L.h2b_xhat_main.argtypes = [vp, vp, vp, vp, vp]
        L.h2b_block_tree_device.argtypes = L.h2b_block_tree.argtypes
        L.h2b_panel_points.argtypes = [ctypes.POINTER(Mesh), vp, vp, ctypes.c_int32, vp, vp]
        L.h2b_touch_count.argtypes = [ctypes.POINTER(Mesh), vp, vp, vp]
        L.h2b_touch_fill.argtypes = [ctypes.POINTER(Mesh), vp, vp, vp, vp, vp, vp]
        L.h2b_touch_half.argtypes = [ctypes.POINTER(Touch), vp, vp, vp]
        L.h2b_singular.argtypes = [ctypes.POINTER(Mesh), ctypes.POINTER(Touch), ctypes.c_int,
                                   ctypes.POINTER(Rule), vp, vp]
        L.h2b_pair_blocks_slp.argtypes = [ctypes.POINTER(Mesh), vp, ctypes.c_int32, ctypes.POINTER(Jobs),
                                          ctypes.POINTER(Touch), vp, vp, vp]
        L.h2b_pair_blocks_dlp.argtypes = [ctypes.POINTER(Mesh), vp, vp, ctypes.c_int32,
                                          ctypes.POINTER(DlpJobs), ctypes.POINTER(Touch), vp, vp, vp]
        L.h2b_plan_create.argtypes = [ctypes.POINTER(Layout), ctypes.POINTER(vp)]
        L.h2b_plan_destroy.argtypes = [vp]
        L.h2b_matvec.argtypes = [vp, vp, vp, vp]
        L.h2b_matvec_host.argtypes = [vp, vp, vp, vp]
        L.h2b_diagonal.argtypes = [vp, vp, vp]
        L.h2b_plan_trace.argtypes = [vp, vp, ctypes.c_int64]
        L.h2b_plan_info.argtypes = [vp, vp]
        L.h2b_dlp_jobs_build.argtypes = [ctypes.c_int64, vp, vp, vp, ctypes.c_int64, vp, vp, vp, vp, vp, vp,
                                         ctypes.POINTER(vp)]
        L.h2b_dlp_jobs_sizes.argtypes = [vp, vp]
        L.h2b_block_partners.argtypes = [ctypes.c_int64, vp, vp]
        L.h2b_block_jobs.argtypes = [ctypes.c_int64, vp, vp, vp, vp, vp, vp, vp, ctypes.c_int, vp, vp, vp]
        L.h2b_dlp_jobs_copy.argtypes = [vp, vp, vp, vp, vp, vp, vp]
        L.h2b_dlp_jobs_free.argtypes = [vp]
        L.h2b_gca_columns.argtypes = [ctypes.POINTER(Mesh), vp, ctypes.c_int32, vp, ctypes.c_int,
                                      ctypes.POINTER(GcaBatch), vp, vp]
        L.h2b_matmat_create.argtypes = [ctypes.POINTER(Layout), ctypes.POINTER(vp)]
        L.h2b_matmat_destroy.argtypes = [vp]
        L.h2b_matmat.argtypes = [vp, vp, vp, ctypes.c_int32, vp]
        L.h2b_cg_workspace_size.argtypes = [vp]
        L.h2b_cg_dot.argtypes = [vp, vp, ctypes.c_int64, vp, vp, vp]
        L.h2b_cg_step.argtypes = [ctypes.c_int64, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp]
        L.h2b_cg_direction.argtypes = [ctypes.c_int64, vp, vp, vp, vp]
        L.h2b_pair_integrals.argtypes = [ctypes.POINTER(Mesh), ctypes.c_int64, vp, vp, ctypes.c_int,
                                         ctypes.POINTER(Rule), vp, vp]
        L.h2b_basis_forward.argtypes = [ctypes.POINTER(Basis), vp, vp, vp]
        L.h2b_basis_backward.argtypes = [ctypes.POINTER(Basis), vp, vp, vp]
        L.h2b_transpose_blocks.argtypes = [ctypes.c_int64, vp, vp, vp, vp]
        L.h2b_hyp_scatter.argtypes = [ctypes.c_int64] + [vp] * 11
        L.h2b_comm_unique_id.argtypes = [vp]
        L.h2b_comm_init.argtypes = [ctypes.POINTER(vp), ctypes.c_int, vp, ctypes.c_int, ctypes.c_int]
        L.h2b_comm_destroy.argtypes = [vp]
        L.h2b_plan_set_comm.argtypes = [vp, vp, ctypes.c_int, ctypes.c_int, ctypes.c_int64]
        L.h2b_matvec_sharded.argtypes = [vp, vp, vp, vp]
        L.h2b_gca_columns_curl.argtypes = [ctypes.POINTER(Mesh), vp, ctypes.c_int32, vp, ctypes.POINTER(GcaBatch), vp,
                                           vp]
        L.h2b_gca_aca.argtypes = [ctypes.POINTER(GcaBatch), ctypes.c_double, vp, vp, vp, vp, ctypes.c_int32, vp, vp]
        _lib = L
    return _lib


def last_error():
    buf = ctypes.create_string_buffer(4096)
    lib().h2b_last_error(buf, len(buf))
    return buf.value.decode(errors="replace")


def check(rc, what=""):
    """Map a status code onto the reference's exception types."""
    if rc == H2B_OK:
        return
    msg = last_error() or what
    if rc == H2B_ERR_NONFINITE:
        raise FloatingPointError(msg)
    if rc == H2B_ERR_MISSING:
        raise KeyError(msg)
    if rc in (H2B_ERR_INVALID, H2B_ERR_TOUCHING, H2B_ERR_CAPACITY):
        raise ValueError(msg)
    raise RuntimeError(f"libh2b: {msg}")


def ptr(a):
    """Raw address of a numpy array or torch tensor (None -> NULL)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()


def stream_ptr(stream=None):
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)
