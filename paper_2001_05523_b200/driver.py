"""Problem setup: spaces, cluster trees, cached block trees, bases and
operators (h2bem.driver.ProblemSetup, driver.py:28-107)."""

from dataclasses import dataclass, field

from . import gca, kernels, spaces
from .clustering import BlockTree, build_cluster_tree
from .containers import AssemblyContext, DenseOperator, assemble_dense
from .mesh import sphere_mesh
from .params import DENSE, GCA


@dataclass
class ProblemSetup:
    mesh: object
    params: object
    ctx: AssemblyContext = None
    tree_p0: object = None
    tree_p1: object = None
    _block_trees: dict = field(default_factory=dict)
    _operators: dict = field(default_factory=dict)
    _bases: dict = field(default_factory=dict)
    _nearfield: dict = field(default_factory=dict)
    dist: object = None  # collective provider for params.devices > 1 (default: torch.distributed)

    def __post_init__(self):
        p = self.params
        self.ctx = AssemblyContext(self.mesh)
        self.space_p0 = spaces.DofSpace(spaces.P0, self.mesh)
        self.space_p1 = spaces.DofSpace(spaces.P1, self.mesh)
        self.tree_p0 = build_cluster_tree(self.space_p0.support_boxes(), p.r_leaf)
        self.tree_p1 = build_cluster_tree(self.space_p1.support_boxes(), p.r_leaf)

    def block_tree(self, kind):
        if kind not in self._block_trees:
            row = self.tree_p1 if kind == kernels.HYP else self.tree_p0
            col = self.tree_p0 if kind == kernels.SLP else self.tree_p1
            self._block_trees[kind] = BlockTree(row, col, self.params.eta)
        return self._block_trees[kind]

    def basis(self, tree_name, flavor):
        key = (tree_name, flavor)
        if key not in self._bases:
            tree = self.tree_p0 if tree_name == "p0" else self.tree_p1
            p = self.params
            self._bases[key] = gca.build_basis(self.ctx, tree, flavor, p.order, p.eps_aca, threads=p.threads,
                                               device=getattr(p, "gca_device", False))
        return self._bases[key]

    def operator(self, kind, method=None):
        p = self.params
        method = method or p.method
        key = (kind, method)
        if key in self._operators:
            return self._operators[key]
        qs = p.q_singular if getattr(p, "q_singular", None) else p.q_near
        nf_cache = self._nearfield.setdefault((kind, p.q_near, qs), {})
        if method == DENSE:
            op = DenseOperator(assemble_dense(self.ctx, kind, p.q_near, cap=p.oracle_cap, q_singular=qs))
        elif method == GCA:
            rf, cf = gca.basis_flavors(kind)
            row_tree = "p1" if kind == kernels.HYP else "p0"
            col_tree = "p0" if kind == kernels.SLP else "p1"
            rb = self.basis(row_tree, rf)
            cb = rb if (rf == cf and row_tree == col_tree) else self.basis(col_tree, cf)
            if getattr(p, "devices", 1) > 1:
                op = self._sharded_operator(kind, rb, cb, qs)
                self._operators[key] = op
                return op
            op = gca.assemble_h2(self.ctx, kind, self.block_tree(kind), rb, cb, p.q_near,
                                 nearfield_cache=nf_cache, q_singular=qs)
        else:
            raise ValueError(f"unknown or unsupported method {method!r}")
        self._operators[key] = op
        return op


    def _sharded_operator(self, kind, rb, cb, qs):
        """params.devices > 1: this process is one rank of a row-sharded
        operator (one process per GPU); it integrates, stores and applies only
        its row clusters' blocks (distributed.RowShard / ShardedMatvec)."""
        import torch.distributed as td

        from .distributed import RowShard, ShardedMatvec, ShardedOperator

        p = self.params
        if not td.is_available() or not td.is_initialized():
            raise ValueError("RunParams.devices > 1 needs an initialised torch.distributed process group")
        world, rank = td.get_world_size(), td.get_rank()
        if world != p.devices:
            raise ValueError(f"RunParams.devices = {p.devices} but the process group has {world} ranks")
        shard = RowShard(self.block_tree(kind), rb, cb, rank, world)
        shard.assemble(self.ctx, kind, p.q_near, qs)
        return ShardedOperator(ShardedMatvec(shard, rank, world, self.dist if self.dist is not None else td))


def setup_sphere(level, params):
    return ProblemSetup(sphere_mesh(level), params.resolved())
