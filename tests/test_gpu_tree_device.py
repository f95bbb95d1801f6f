"""Device cluster-tree / block-tree builders against the host
builders, which are pinned bit-exact to the reference (tests/test_structure.py):
identical perm, node ranges, depths, children, boxes and far/near lists in the
same order, at the configurations' sizes (P0 and P1 trees, several leaf sizes
and admissibility parameters, the config-4 cube shell)."""

import time

import numpy as np
import pytest

from .helpers import sphere

pytestmark = pytest.mark.gpu


def _same_tree(a, b):
    assert np.array_equal(a.perm, b.perm)
    for f in ("start", "end", "depth_of", "left", "right"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
    assert np.array_equal(a.boxes, b.boxes)


@pytest.mark.parametrize("level,leaf,eta,space", [(3, 8, 2.0, "p0"), (4, 32, 2.0, "p0"), (4, 32, 2.0, "p1"),
                                                  (6, 64, 2.0, "p0"), (6, 16, 1.0, "p1"), (8, 64, 2.0, "p1"),
                                                  (9, 64, 1.5, "p0")])
def test_device_builders_match_host(level, leaf, eta, space):
    from paper_2001_05523_b200 import clustering as C
    from paper_2001_05523_b200 import spaces

    m = sphere(level)
    boxes = spaces.DofSpace(spaces.P0 if space == "p0" else spaces.P1, m).support_boxes()
    t0 = time.perf_counter()
    th = C.build_cluster_tree(boxes, leaf)
    t1 = time.perf_counter()
    td = C.build_cluster_tree(boxes, leaf, device=True)
    t2 = time.perf_counter()
    _same_tree(th, td)
    bh = C.BlockTree(th, th, eta)
    t3 = time.perf_counter()
    bd = C.BlockTree(th, th, eta, device=True)
    t4 = time.perf_counter()
    assert np.array_equal(bh.far_uids, bd.far_uids)
    assert np.array_equal(bh.near_uids, bd.near_uids)
    print(f"level {level}: tree host {t1 - t0:.3f} s device {t2 - t1:.3f} s; "
          f"block tree host {t3 - t2:.3f} s device {t4 - t3:.3f} s")


def test_device_builders_cube_shell_and_rectangular():
    """Grid-aligned cube shell (exact split ties, the stable-median fallback)
    and a P0 x P1 block tree."""
    from paper_2001_05523_b200 import clustering as C
    from paper_2001_05523_b200 import spaces
    from paper_2001_05523_b200.mesh import cube_shell_mesh

    m = cube_shell_mesh(8)
    for sp in (spaces.P0, spaces.P1):
        boxes = spaces.DofSpace(sp, m).support_boxes()
        _same_tree(C.build_cluster_tree(boxes, 32), C.build_cluster_tree(boxes, 32, device=True))
    m = sphere(5)
    t0 = C.build_cluster_tree(spaces.DofSpace(spaces.P0, m).support_boxes(), 32)
    t1 = C.build_cluster_tree(spaces.DofSpace(spaces.P1, m).support_boxes(), 32)
    a, b = C.BlockTree(t0, t1, 2.0), C.BlockTree(t0, t1, 2.0, device=True)
    assert np.array_equal(a.far_uids, b.far_uids) and np.array_equal(a.near_uids, b.near_uids)
