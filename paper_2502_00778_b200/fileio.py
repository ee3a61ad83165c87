"""SPEC cli_io file formats over the
host-only entry points of libdualmesh.so (csrc/io.cpp): MeshFile text
(1-based ids, 17 significant digits) and the MetricsFile JSON document."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _lib
from ._lib import ptr
from .mesh import DualMeshError, Engine, Mesh


class MeshFileError(DualMeshError, ValueError):
    """Syntax error, count mismatch or invalid index, with "path:line: what"."""

    def __init__(self, message: str):
        ValueError.__init__(self, message)
        self.status = _lib.DM_ERR_INVALID_ARG

    def __str__(self):
        return self.args[0]


def _b(path) -> bytes:
    return os.fsencode(os.fspath(path))


def read_mesh(path, engine: Engine | None = None) -> Mesh:
    """Parse a MeshFile.  A missing boundary section is derived
    (derive_boundary_faces on the GPU; needs `engine` or a default one)."""
    lib = _lib.capi()
    d, nv, ne, nb, hb = C.c_int(), C.c_int64(), C.c_int64(), C.c_int64(), C.c_int()
    err = C.create_string_buffer(1024)
    st = lib.dm_mesh_file_read(_b(path), C.byref(d), C.byref(nv), C.byref(ne), C.byref(nb),
                               C.byref(hb), None, None, None, err, len(err))
    if st:
        raise MeshFileError(err.value.decode())
    x = np.empty(d.value * nv.value, np.float64)
    el = np.empty((d.value + 1) * ne.value, np.int32)
    bd = np.empty(d.value * nb.value, np.int32)
    st = lib.dm_mesh_file_read(_b(path), None, None, None, None, None, ptr(x, C.c_double),
                               ptr(el, C.c_int32), ptr(bd, C.c_int32), err, len(err))
    if st:
        raise MeshFileError(err.value.decode())
    m = Mesh(d.value, x, el, bd)
    if not hb.value and m.num_elements() > 0:
        own = engine is None
        eng = engine or Engine()
        try:
            eng.set_mesh(m)
            m = Mesh(m.dim, m.coords, m.elements, eng.derive_boundary())
        finally:
            if own:
                eng.close()
    return m


def has_boundary_section(path) -> bool:
    lib = _lib.capi()
    hb = C.c_int()
    err = C.create_string_buffer(1024)
    if lib.dm_mesh_file_read(_b(path), None, None, None, None, C.byref(hb), None, None, None,
                             err, len(err)):
        raise MeshFileError(err.value.decode())
    return bool(hb.value)


def write_mesh(mesh: Mesh, path) -> None:
    st = _lib.capi().dm_mesh_file_write(_b(path), mesh.dim, ptr(mesh.coords, C.c_double),
                                        mesh.num_nodes(), ptr(mesh.elements, C.c_int32),
                                        mesh.num_elements(), ptr(mesh.boundary, C.c_int32),
                                        mesh.num_boundary())
    if st:
        raise OSError(f"{path}: write failed")


def mesh_checksum(mesh: Mesh) -> int:
    return int(_lib.capi().dm_mesh_checksum(mesh.dim, ptr(mesh.coords, C.c_double),
                                            mesh.num_nodes(), ptr(mesh.elements, C.c_int32),
                                            mesh.num_elements(), ptr(mesh.boundary, C.c_int32),
                                            mesh.num_boundary()))


def write_metrics(path, mesh: Mesh, edges, navs, volumes, nav_algo: int = _lib.DM_NAV_DUALFREE,
                  vol_algo: int = _lib.DM_VOL_EDGE) -> None:
    e = np.ascontiguousarray(getattr(edges, "edges", edges), np.int32).reshape(-1, 2)
    n = np.ascontiguousarray(navs, np.float64).ravel()
    v = np.ascontiguousarray(volumes, np.float64).ravel()
    if n.size != mesh.dim * e.shape[0] or v.size != mesh.num_nodes():
        raise ValueError("field/mesh mismatch")
    st = _lib.capi().dm_metrics_file_write(_b(path), mesh.dim, ptr(e, C.c_int32), e.shape[0],
                                           ptr(n, C.c_double), ptr(v, C.c_double), v.size,
                                           nav_algo, vol_algo, mesh_checksum(mesh))
    if st:
        raise OSError(f"{path}: write failed")
