"""Multi-rank host logic of the row-sharded matvec, on CPU with gloo.

Two processes (world_size 2) partition the row clusters exactly as
ShardedMatvec does on the GPUs, all-gather x in permuted order with the same
padded chunk layout, evaluate their own rows with the oracle restricted to
their owned clusters, and all-gather the rows of y.  The result must equal the
single-process oracle matvec bit for bit (the per-row accumulation order does
not depend on the rank count)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import h2 as OH
from oracle import quad as OQ


def _world():
    from paper_2001_05523_b200 import clustering as C
    from paper_2001_05523_b200 import gca, spaces
    from paper_2001_05523_b200.containers import AssemblyContext, FarLayout, near_layout
    from paper_2001_05523_b200.mesh import sphere_mesh

    m = sphere_mesh(3)
    tree = C.build_cluster_tree(spaces.DofSpace(spaces.P0, m).support_boxes(), 16)
    bt = C.BlockTree(tree, tree, 2.0)
    b = gca.build_basis(AssemblyContext(m), tree, gca.P0_SLP, 3, 1e-4, threads=1)
    V, T, N, A = m.vertices, m.triangles, m.normals, m.areas
    tab = OQ.Table(V, T, N, A, "slp", 4)
    p = tree.perm
    near = [OQ.slp_block(V, T, N, A, p[tree.start[t] : tree.end[t]], p[tree.start[s] : tree.end[s]], 3, tab)
            for t, s in bt.near_uids]
    far = [OQ.slp_block(V, T, N, A, b.pivots[t], b.pivots[s], 3) for t, s in bt.far_uids]
    ranks = np.array([b.rank[u] for u in range(tree.n_nodes)], dtype=np.int64)
    fl = FarLayout(bt, ranks, ranks)
    return tree, bt, b, near, far, near_layout(bt), fl, ranks


def _sharded_rows(tree, bt, b, near, far, owned, xp):
    """Oracle matvec restricted to owned row clusters (forward over all)."""
    ot = OH.Tree(tree.perm, tree.start, tree.end, tree.depth_of, tree.left, tree.right)
    own = set(int(u) for u in owned)
    xhat = OH.forward(ot, b.V, b.E, b.rank, xp)
    yhat = {}
    for (t, s), Sb in zip(bt.far_uids, far):
        if int(t) in own:
            c = Sb @ xhat[int(s)]
            yhat[int(t)] = yhat[int(t)] + c if int(t) in yhat else c
    yp = np.zeros(len(tree.perm))
    OH.backward(ot, b.V, b.E, yhat, yp)
    for (t, s), Db in zip(bt.near_uids, near):
        if int(t) in own:
            yp[tree.start[t] : tree.end[t]] += Db @ xp[tree.start[s] : tree.end[s]]
    return yp


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2001_05523_b200 import distributed as DD

    tree, bt, b, near, far, nl, fl, ranks = _world()
    ranges = DD.partition_rows(tree, nl.C, fl.K, ranks, world)
    lo, hi = ranges[rank]
    owned = DD.owned_nodes(tree, lo, hi)
    chunk, pad_index = DD.gather_layout(ranges, tree.n_dofs)
    x = np.random.default_rng(0).uniform(-1, 1, tree.n_dofs)
    xp_full = x[tree.perm]
    # each rank contributes its permuted slice, padded to the common chunk
    mine = torch.zeros(chunk, dtype=torch.float64)
    mine[: hi - lo] = torch.from_numpy(xp_full[lo:hi])
    buf = torch.zeros(world * chunk, dtype=torch.float64)
    dist.all_gather_into_tensor(buf, mine)
    xp = buf.numpy()[pad_index]
    assert np.array_equal(xp, xp_full)
    yp = _sharded_rows(tree, bt, b, near, far, owned, xp)
    part = torch.zeros(chunk, dtype=torch.float64)
    part[: hi - lo] = torch.from_numpy(yp[lo:hi])
    ybuf = torch.zeros(world * chunk, dtype=torch.float64)
    dist.all_gather_into_tensor(ybuf, part)
    if rank == 0:
        y_p = ybuf.numpy()[pad_index]
        y = np.empty_like(y_p)
        y[tree.perm] = y_p
        ot = OH.Tree(tree.perm, tree.start, tree.end, tree.depth_of, tree.left, tree.right)
        ref = OH.matvec(ot, ot, b.V, b.E, b.rank, b.V, b.E, b.rank, bt.far_uids, far, bt.near_uids, near, x)
        out.put((bool(np.array_equal(y, ref)), [list(r) for r in ranges], len(owned)))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_partition_properties():
    from paper_2001_05523_b200 import distributed as DD

    tree, bt, b, near, far, nl, fl, ranks = _world()
    for world in (1, 2, 3, 4, 8):
        ranges = DD.partition_rows(tree, nl.C, fl.K, ranks, world)
        assert ranges[0][0] == 0 and ranges[-1][1] == tree.n_dofs
        for (a0, a1), (b0, b1) in zip(ranges[:-1], ranges[1:]):
            assert a1 == b0 and a0 < a1
        # owned sets: ancestor-closed, cover every leaf exactly once
        leaf_owner = {}
        for r, (lo, hi) in enumerate(ranges):
            own = set(DD.owned_nodes(tree, lo, hi).tolist())
            for u in own:
                if tree.parent_of[u] >= 0:
                    assert tree.parent_of[u] in own
                if tree.left[u] < 0:
                    assert u not in leaf_owner
                    leaf_owner[u] = r
        assert sorted(leaf_owner) == sorted(tree.leaf_uids().tolist())
        chunk, pad = DD.gather_layout(ranges, tree.n_dofs)
        assert len(np.unique(pad)) == tree.n_dofs and pad.max() < world * chunk


def test_two_rank_gloo_matches_single_rank():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    ok, ranges, n_owned = res
    assert ok, f"sharded oracle differs from the single-rank result (ranges {ranges})"


def test_xhat_exchange_layout():
    """x_hat exchange bookkeeping (SURVEY 8(e) better variant): every leaf is
    owned by exactly one rank, owned clusters never straddle a rank boundary,
    the gathered offsets tile each rank's chunk without overlap, and exactly
    the clusters spanning several ranks have no offset."""
    from paper_2001_05523_b200 import clustering as C
    from paper_2001_05523_b200 import distributed as DD
    from paper_2001_05523_b200 import spaces
    from paper_2001_05523_b200.mesh import sphere_mesh

    m = sphere_mesh(4)
    t = C.build_cluster_tree(spaces.DofSpace(spaces.P0, m).support_boxes(), 16)
    ranks = np.random.default_rng(0).integers(3, 20, t.n_nodes)
    for world in (1, 2, 3, 5):
        leaves = t.leaf_uids()
        cuts = np.linspace(0, len(leaves), world + 1).astype(int)
        order = leaves[np.argsort(t.start[leaves])]
        ranges = [(int(t.start[order[a]]), int(t.end[order[b - 1]])) for a, b in zip(cuts[:-1], cuts[1:])]
        masks, chunk, src = DD.xhat_exchange_layout(t, ranks, ranges)
        assert (masks[:, leaves].sum(axis=0) == 1).all()
        assert (masks.sum(axis=0) <= 1).all()
        spanning = masks.sum(axis=0) == 0
        assert ((src < 0) == spanning).all()
        for r in range(world):
            u = np.flatnonzero(masks[r])
            lo, hi = ranges[r]
            assert ((t.start[u] >= lo) & (t.end[u] <= hi)).all()
            off = src[u] - r * chunk
            k = ranks[u]
            assert off[0] == 0 and (np.diff(off) == k[:-1]).all() and off[-1] + k[-1] <= chunk
