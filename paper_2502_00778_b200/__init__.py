"""paper_2502_00778_b200 -- B200 (sm_100a) dual-free grid metrics.

Lumped directed-area vectors at edges and median-dual volumes at nodes on
triangle / tetrahedral grids (arXiv 2502.00778), computed by hand-written
CUDA kernels behind the reference C++ API (include/dualmesh/mesh.hpp) and a
C-ABI (include/dm_capi.h).  This package is the Python mirror used by the
tests and the bench; the native library is ``lib/libdualmesh.so``.
"""
from .mesh import (DualMeshError, EdgeAbsent, EdgeList, Engine, Mesh, MeshEdgeMismatch,
                   boundary_node_mask, build_edges, default_engine, derive_boundary_faces,
                   element_volume, max_element_volume, max_face_area, total_volume)
from . import fileio, meshgen, metrics

__all__ = [
    "DualMeshError", "EdgeAbsent", "EdgeList", "Engine", "Mesh", "MeshEdgeMismatch",
    "boundary_node_mask", "build_edges", "default_engine", "derive_boundary_faces",
    "element_volume", "max_element_volume", "max_face_area", "total_volume", "meshgen",
    "metrics",
]
