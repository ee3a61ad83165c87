"""SPEC metrics / verify operations on the GPU engine.

Same names and argument meaning as include/dualmesh/metrics.hpp.  Fields are
flat numpy arrays: navs has dim doubles per edge in EdgeList order, volumes
one double per node.
"""
from __future__ import annotations

import numpy as np

from . import _lib
from .mesh import EdgeList, Mesh, MeshEdgeMismatch, default_engine

TRADITIONAL = _lib.DM_NAV_TRADITIONAL
DUALFREE = _lib.DM_NAV_DUALFREE
EDGE = _lib.DM_VOL_EDGE
ELEMENT = _lib.DM_VOL_ELEMENT
GATHER = _lib.DM_VARIANT_GATHER
SCATTER = _lib.DM_VARIANT_SCATTER


def _with_edges(mesh: Mesh, edges: EdgeList):
    eng = default_engine()
    eng.set_mesh(mesh)
    ne = eng.build_edges()
    mine = eng.edges()
    if ne != edges.size() or not np.array_equal(mine.edges, edges.edges):
        raise MeshEdgeMismatch(_lib.DM_ERR_MESH_EDGE_MISMATCH, "metrics", "mesh/edge mismatch")
    return eng


def lumped_navs_traditional(mesh: Mesh, edges: EdgeList) -> np.ndarray:
    eng = _with_edges(mesh, edges)
    eng.navs(TRADITIONAL, GATHER)
    return eng.get_navs()


def lumped_navs_dualfree(mesh: Mesh, edges: EdgeList, variant: int = GATHER) -> np.ndarray:
    eng = _with_edges(mesh, edges)
    eng.navs(DUALFREE, variant)
    return eng.get_navs()


def dual_volumes_edge_based(mesh: Mesh, edges: EdgeList, navs: np.ndarray) -> np.ndarray:
    eng = _with_edges(mesh, edges)
    if navs.size != mesh.dim * edges.size():
        raise ValueError("field/edge-list mismatch")
    eng.put_navs(navs)
    eng.volumes(EDGE)
    return eng.get_volumes()


def dual_volumes_element_based(mesh: Mesh) -> np.ndarray:
    eng = default_engine()
    eng.set_mesh(mesh)
    eng.volumes(ELEMENT)
    return eng.get_volumes()


def compute_metrics(mesh: Mesh, nav_algo: int = DUALFREE, vol_algo: int = EDGE):
    """SPEC.md:190-198 -> (EdgeList, navs, volumes)."""
    eng = default_engine()
    eng.set_mesh(mesh)
    eng.build_edges()
    eng.navs(nav_algo, GATHER)
    eng.volumes(vol_algo)
    return eng.edges(), eng.get_navs(), eng.get_volumes()


def check_closure(mesh: Mesh, edges: EdgeList, navs: np.ndarray) -> float:
    eng = _with_edges(mesh, edges)
    eng.put_navs(navs)
    return eng.check_closure()[0]


def check_total_volume(mesh: Mesh, volumes: np.ndarray) -> float:
    eng = default_engine()
    eng.set_mesh(mesh)
    eng.put_volumes(volumes)
    return eng.check_total_volume()[0]


def check_linear_exactness(mesh: Mesh, edges: EdgeList, navs: np.ndarray, volumes: np.ndarray,
                           A, b) -> float:
    """affine flux F(x) = A x + b (A: dim x dim); constant
    flux when A == 0.  trace(A) == 0 with A != 0 raises."""
    eng = _with_edges(mesh, edges)
    eng.put_navs(navs)
    eng.put_volumes(volumes)
    return eng.check_linear_exactness(A, b)
