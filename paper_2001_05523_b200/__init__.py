"""B200-native H^2-matvec and Galerkin nearfield quadrature for the fast BEM
of arXiv 2001.05523 — a drop-in for the hot path of the reference package
`h2bem` (same module names and call signatures for mesh, cluster/block trees,
nearfield assembly, H^2 construction, matvec and CG)."""

from .mesh import MeshError, SurfaceMesh, build_octahedron, read_mesh, refine_red, sphere_mesh, write_mesh

__all__ = ["MeshError", "SurfaceMesh", "build_octahedron", "read_mesh", "refine_red", "sphere_mesh", "write_mesh"]
