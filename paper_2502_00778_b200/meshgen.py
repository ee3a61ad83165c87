"""SPEC meshgen and the BASELINE.json grids.

Thin wrapper over lib/libdm_meshgen.so (host C++, include/dm_meshgen.h).
Seeds: 42 jitter, 43 2D diagonal choice, 44 node permutation, 45 element
permutation.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import ptr
from .mesh import Mesh

SEED_JITTER, SEED_DIAG, SEED_NODES, SEED_ELEMS = 42, 43, 44, 45


def _sizes(fn, *args):
    a, b, c = C.c_int64(), C.c_int64(), C.c_int64()
    fn(*args, C.byref(a), C.byref(b), C.byref(c))
    return a.value, b.value, c.value


def tri_square(n: int, diag_seed: int = 0, amp: float = 0.0, seed: int = SEED_JITTER) -> Mesh:
    """gen_tri_square(n) (+ perturb_interior(amp, seed)); diag_seed=0 gives
    the uniform diagonal of SPEC.md:350, otherwise a seeded random one."""
    g = _lib.meshgen()
    nv, ne, nb = _sizes(g.dmg_tri_square_sizes, n)
    x = np.empty(2 * nv, np.float64)
    el = np.empty(3 * ne, np.int32)
    bd = np.empty(2 * nb, np.int32)
    if g.dmg_tri_square(n, diag_seed, amp, seed, ptr(x, C.c_double), ptr(el, C.c_int32),
                        ptr(bd, C.c_int32)) != 0:
        raise ValueError("gen_tri_square: n < 1")
    return Mesh(2, x, el, bd)


def tet_box(nx: int, ny: int, nz: int, z_nodes=None, jitter_mode: int = 0, amp: float = 0.0,
            seed: int = SEED_JITTER) -> Mesh:
    g = _lib.meshgen()
    nv, ne, nb = _sizes(g.dmg_tet_box_sizes, nx, ny, nz)
    x = np.empty(3 * nv, np.float64)
    el = np.empty(4 * ne, np.int32)
    bd = np.empty(3 * nb, np.int32)
    z = None if z_nodes is None else np.ascontiguousarray(z_nodes, np.float64)
    if g.dmg_tet_box(nx, ny, nz, ptr(z, C.c_double), jitter_mode, amp, seed, ptr(x, C.c_double),
                     ptr(el, C.c_int32), ptr(bd, C.c_int32)) != 0:
        raise ValueError("gen_tet_cube: n < 1")
    return Mesh(3, x, el, bd)


def tet_cube(n: int, amp: float = 0.0, seed: int = SEED_JITTER) -> Mesh:
    """gen_tet_cube(n) + perturb_interior(amp, seed)."""
    return tet_box(n, n, n, None, 0, amp, seed)


def bl_z(nz: int, dz0: float, ratio: float) -> np.ndarray:
    z = np.empty(nz + 1, np.float64)
    _lib.meshgen().dmg_bl_z(nz, dz0, ratio, ptr(z, C.c_double))
    return z


def permute(mesh: Mesh, node_seed: int = SEED_NODES, elem_seed: int = SEED_ELEMS) -> Mesh:
    """Random relabelling of nodes and elements (local order kept)."""
    x, el, bd = mesh.coords.copy(), mesh.elements.copy(), mesh.boundary.copy()
    _lib.meshgen().dmg_permute(mesh.dim, mesh.num_nodes(), mesh.num_elements(),
                               mesh.num_boundary(), node_seed, elem_seed, ptr(x, C.c_double),
                               ptr(el, C.c_int32), ptr(bd, C.c_int32))
    return Mesh(mesh.dim, x, el, bd)


SEED_FLIPS = 46


def flip23(mesh: Mesh, fraction: float = 0.3, seed: int = SEED_FLIPS) -> Mesh:
    """Seeded random 2-3 flips (dmg_flip23) of up to `fraction` * n_elements / 2
    tet pairs: non-Kuhn, unstructured topology (ring lengths 3..10+) on the
    same nodes and boundary, node numbering kept."""
    assert mesh.dim == 3
    ne = mesh.num_elements()
    mx = int(fraction * ne / 2)
    out = np.empty(4 * (ne + mx), np.int32)
    nf = _lib.meshgen().dmg_flip23(mesh.num_nodes(), ptr(mesh.coords, C.c_double), ne,
                                   ptr(mesh.elements, C.c_int32), mx, seed, ptr(out, C.c_int32))
    if nf < 0:
        raise ValueError("dmg_flip23: invalid mesh arrays")
    return Mesh(3, mesh.coords, out[:4 * (ne + nf)].copy(), mesh.boundary)


def fan_in(mesh: Mesh, n: int = 30) -> Mesh:
    """`mesh` plus a disjoint fan of n tets around one edge (placed beside the
    unit box): one edge with n incidences (n > 24 leaves the ring encoding)
    inside an otherwise regular grid."""
    th = 2 * np.pi * np.arange(n) / n
    ring = np.stack([1.5 + 0.2 * np.cos(th), 0.5 + 0.2 * np.sin(th), np.full(n, 0.5)], 1)
    xf = np.concatenate([[[1.5, 0.5, 0.3], [1.5, 0.5, 0.7]], ring])
    b = mesh.num_nodes()
    el, bd = [], []
    for i in range(n):
        t = [0, 1, 2 + i, 2 + (i + 1) % n]
        p = xf[t]
        if np.linalg.det(np.stack([p[1] - p[0], p[2] - p[0], p[3] - p[0]])) < 0:
            t[2], t[3] = t[3], t[2]
        el += [b + v for v in t]
        # outward facets: the two faces of each tet not containing the edge (0,1)
        for o in (0, 1):
            f = [v for k, v in enumerate(t) if k != o]
            q = xf[f]
            nrm = np.cross(q[1] - q[0], q[2] - q[0])
            cen = xf[t].mean(0)
            if np.dot(nrm, q[0] - cen) < 0:
                f[1], f[2] = f[2], f[1]
            bd += [b + v for v in f]
    return Mesh(3, np.concatenate([mesh.coords, xf.ravel()]),
                np.concatenate([mesh.elements, np.array(el, np.int32)]),
                np.concatenate([mesh.boundary, np.array(bd, np.int32)]))


def first_inverted(mesh: Mesh) -> int:
    return int(_lib.meshgen().dmg_first_inverted(mesh.dim, mesh.num_elements(),
                                                 ptr(mesh.coords, C.c_double),
                                                 ptr(mesh.elements, C.c_int32)))


# BASELINE.json configs; `scale` divides the cell counts so
# the same family can be generated small for parity tests.
CONFIGS = {
    "C1": "2D unit square 256x256, random diagonal (seed 43), +-0.2h jitter",
    "C2": "3D unit cube 64^3 Kuhn, +-0.15h jitter",
    "C3": "3D unit cube 160^3 Kuhn, +-0.15h jitter, node/element numbering permuted",
    "C4": "boundary layer 128x128x256, dz0=1e-5, ratio 1.05, +-0.1h in-plane jitter",
    "C5": "3D unit cube 256^3 Kuhn, +-0.15h jitter",
}


def baseline_config(name: str, scale: int = 1) -> Mesh:
    if name == "C1":
        return tri_square(256 // scale, diag_seed=SEED_DIAG, amp=0.2, seed=SEED_JITTER)
    if name == "C2":
        return tet_cube(64 // scale, amp=0.15)
    if name == "C3":
        return permute(tet_cube(160 // scale, amp=0.15))
    if name == "C4":
        n, nz = 128 // scale, 256 // scale
        return tet_box(n, n, nz, bl_z(nz, 1e-5, 1.05), jitter_mode=1, amp=0.1)
    if name == "C5":
        return tet_cube(256 // scale, amp=0.15)
    raise KeyError(name)


def baseline_config_device(engine, name: str, scale: int = 1) -> None:
    """The same grids as baseline_config, generated on the engine's device
    (dm_gen_*, bitwise identical); the mesh stays on the GPU."""
    if name == "C1":
        engine.gen_tri_square(256 // scale, SEED_DIAG, 0.2, SEED_JITTER)
    elif name == "C2":
        engine.gen_tet_box(64 // scale, 64 // scale, 64 // scale, None, 0, 0.15, SEED_JITTER)
    elif name == "C3":
        n = 160 // scale
        engine.gen_tet_box(n, n, n, None, 0, 0.15, SEED_JITTER)
        engine.gen_permute(SEED_NODES, SEED_ELEMS)
    elif name == "C4":
        n, nz = 128 // scale, 256 // scale
        engine.gen_tet_box(n, n, nz, bl_z(nz, 1e-5, 1.05), 1, 0.1, SEED_JITTER)
    elif name == "C5":
        n = 256 // scale
        engine.gen_tet_box(n, n, n, None, 0, 0.15, SEED_JITTER)
    else:
        raise KeyError(name)
