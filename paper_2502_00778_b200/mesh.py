"""Python mirror of the reference mesh module and of the C-ABI engine.

Names, argument meaning and error behaviour follow the reference C++ API
(/root/reference/proj/include/dualmesh/mesh.hpp:10-100): 0-based ids, flat
arrays, ``edge_of`` returning -1 for an absent pair.  Everything grid-sized
runs on the GPU through ``libdualmesh.so`` (include/dm_capi.h); a missing
library or device raises -- there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import DP, I32P, I64P, U64P, U8P, I8P, FP, ptr


class DualMeshError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str):
        self.status = status
        super().__init__(f"{where}: status {status} ({detail})")


class MeshEdgeMismatch(DualMeshError, ValueError):
    """SPEC.md:151,174 'mesh/edge mismatch'."""


class EdgeAbsent(DualMeshError, ValueError):
    """SPEC.md:164 boundary element referencing an edge absent from EdgeList."""


@dataclass
class Mesh:
    """ref mesh.hpp:23-44: dim doubles per node, dim+1 ids per element,
    dim ids per outward boundary facet."""
    dim: int
    coords: np.ndarray
    elements: np.ndarray
    boundary: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))

    def __post_init__(self):
        self.coords = np.ascontiguousarray(self.coords, dtype=np.float64).reshape(-1)
        self.elements = np.ascontiguousarray(self.elements, dtype=np.int32).reshape(-1)
        self.boundary = np.ascontiguousarray(self.boundary, dtype=np.int32).reshape(-1)

    def num_nodes(self) -> int:
        return self.coords.size // self.dim

    def num_elements(self) -> int:
        return self.elements.size // (self.dim + 1)

    def num_boundary(self) -> int:
        return self.boundary.size // self.dim

    def node(self, j: int) -> np.ndarray:
        return self.coords[self.dim * j:self.dim * (j + 1)]

    def element(self, e: int) -> np.ndarray:
        return self.elements[(self.dim + 1) * e:(self.dim + 1) * (e + 1)]

    def boundary_element(self, b: int) -> np.ndarray:
        return self.boundary[self.dim * b:self.dim * (b + 1)]


@dataclass
class MeshShape:
    """Sizes of a mesh that lives only on the device (dm_gen_*)."""
    dim: int
    n_nodes: int
    n_elements: int
    n_boundary: int

    def num_nodes(self) -> int:
        return self.n_nodes

    def num_elements(self) -> int:
        return self.n_elements

    def num_boundary(self) -> int:
        return self.n_boundary


@dataclass
class EdgeList:
    """ref mesh.hpp:48-56."""
    edges: np.ndarray          # (n_edges, 2) int32, (min, max), lexicographic
    origin_start: np.ndarray   # (n_nodes + 1,) uint64

    def size(self) -> int:
        return int(self.edges.shape[0])

    def edge_of(self, a: int, b: int) -> int:
        """ref mesh.cpp:58-73 (host lookup on the host list)."""
        if a > b:
            a, b = b, a
        if a < 0 or a + 1 >= self.origin_start.size:
            return -1
        lo, hi = int(self.origin_start[a]), int(self.origin_start[a + 1])
        i = lo + int(np.searchsorted(self.edges[lo:hi, 1], b))
        return i if i < hi and self.edges[i, 1] == b else -1


class Engine:
    """Owns one dm_ctx (one per host thread, include/dm_capi.h)."""

    def __init__(self, device: int = 0):
        self._lib = _lib.capi()
        self._c = C.c_void_p()
        st = self._lib.dm_create(C.byref(self._c), device)
        if st != 0:
            msg = self._lib.dm_last_error(self._c).decode()
            self._lib.dm_destroy(self._c)
            self._c = None
            raise DualMeshError(st, "dm_create", msg)
        self.mesh: Mesh | None = None
        self.n_edges = 0

    # ---------------------------------------------------------------- util
    def _ck(self, st: int, where: str):
        if st == 0:
            return
        detail = self._lib.dm_last_error(self._c).decode()
        if st == _lib.DM_ERR_MESH_EDGE_MISMATCH:
            raise MeshEdgeMismatch(st, where, detail)
        if st == _lib.DM_ERR_EDGE_ABSENT:
            raise EdgeAbsent(st, where, detail)
        if st == _lib.DM_ERR_INVALID_ARG:
            raise ValueError(f"{where}: {detail}")
        raise DualMeshError(st, where, detail)

    def close(self):
        if self._c:
            self._lib.dm_destroy(self._c)
            self._c = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---------------------------------------------------------------- mesh
    def set_mesh(self, mesh: Mesh):
        self._ck(self._lib.dm_set_mesh(self._c, mesh.dim, ptr(mesh.coords, C.c_double),
                                       mesh.num_nodes(), ptr(mesh.elements, C.c_int32),
                                       mesh.num_elements(), ptr(mesh.boundary, C.c_int32),
                                       mesh.num_boundary()), "dm_set_mesh")
        self.mesh = mesh
        self.n_edges = 0

    # device-side meshgen (dm_gen_*): the mesh lives only on the device; the
    # engine keeps a size-only stand-in, get_mesh() copies it back
    def _adopt_device_mesh(self):
        d, nv, ne, nb = C.c_int(), C.c_int64(), C.c_int64(), C.c_int64()
        self._ck(self._lib.dm_mesh_sizes(self._c, C.byref(d), C.byref(nv), C.byref(ne),
                                         C.byref(nb)), "dm_mesh_sizes")
        self.mesh = MeshShape(d.value, nv.value, ne.value, nb.value)
        self.n_edges = 0

    def gen_tri_square(self, n: int, diag_seed: int = 0, amp: float = 0.0, seed: int = 42):
        self._ck(self._lib.dm_gen_tri_square(self._c, n, diag_seed, amp, seed),
                 "dm_gen_tri_square")
        self._adopt_device_mesh()

    def gen_tet_box(self, nx: int, ny: int, nz: int, z_nodes=None, jitter_mode: int = 0,
                    amp: float = 0.0, seed: int = 42):
        z = None if z_nodes is None else np.ascontiguousarray(z_nodes, np.float64)
        self._ck(self._lib.dm_gen_tet_box(self._c, nx, ny, nz, ptr(z, C.c_double), jitter_mode,
                                          amp, seed), "dm_gen_tet_box")
        self._adopt_device_mesh()

    def gen_permute(self, node_seed: int, elem_seed: int):
        self._ck(self._lib.dm_gen_permute(self._c, node_seed, elem_seed), "dm_gen_permute")
        self._adopt_device_mesh()

    def get_mesh(self) -> Mesh:
        s = self.mesh
        x = np.empty(s.dim * s.num_nodes(), np.float64)
        el = np.empty((s.dim + 1) * s.num_elements(), np.int32)
        bd = np.empty(s.dim * s.num_boundary(), np.int32)
        self._ck(self._lib.dm_get_mesh(self._c, ptr(x, C.c_double), ptr(el, C.c_int32),
                                       ptr(bd, C.c_int32)), "dm_get_mesh")
        return Mesh(s.dim, x, el, bd)

    def set_coords(self, coords: np.ndarray):
        coords = np.ascontiguousarray(coords, np.float64)
        # dm_set_coords reads dim * n_nodes doubles from the buffer
        want = self.mesh.dim * self.mesh.num_nodes() if self.mesh is not None else None
        if want is None or coords.size != want:
            raise ValueError(f"coords must hold dim*n_nodes = {want} values, got {coords.size}")
        self._ck(self._lib.dm_set_coords(self._c, ptr(coords, C.c_double)), "dm_set_coords")

    # ---------------------------------------------------------------- edges
    def build_edges(self) -> int:
        ne = C.c_int64()
        self._ck(self._lib.dm_build_edges(self._c, C.byref(ne)), "dm_build_edges")
        self.n_edges = ne.value
        return self.n_edges

    def edges(self) -> EdgeList:
        e = np.empty((self.n_edges, 2), np.int32)
        os_ = np.empty(self.mesh.num_nodes() + 1, np.uint64)
        self._ck(self._lib.dm_get_edges(self._c, ptr(e, C.c_int32), ptr(os_, C.c_uint64)),
                 "dm_get_edges")
        return EdgeList(e, os_)

    def e2l(self) -> np.ndarray:
        L = 6 if self.mesh.dim == 3 else 3
        out = np.empty(L * self.mesh.num_elements(), np.int32)
        self._ck(self._lib.dm_get_e2l(self._c, ptr(out, C.c_int32)), "dm_get_e2l")
        return out

    def incidence(self):
        L = 6 if self.mesh.dim == 3 else 3
        ip = np.empty(self.n_edges + 1, np.int32)
        inc = np.empty(L * self.mesh.num_elements(), np.int32)
        self._ck(self._lib.dm_get_incidence(self._c, ptr(ip, C.c_int32), ptr(inc, C.c_int32)),
                 "dm_get_incidence")
        return ip, inc

    def edge_of(self, a, b) -> np.ndarray:
        a = np.ascontiguousarray(a, np.int32)
        b = np.ascontiguousarray(b, np.int32)
        out = np.empty(a.size, np.int32)
        self._ck(self._lib.dm_edge_of(self._c, ptr(a, C.c_int32), ptr(b, C.c_int32), a.size,
                                      ptr(out, C.c_int32)), "dm_edge_of")
        return out

    # ---------------------------------------------------------------- metrics
    def navs(self, algo: int = _lib.DM_NAV_DUALFREE, variant: int = _lib.DM_VARIANT_GATHER):
        self._ck(self._lib.dm_navs(self._c, algo, variant), "dm_navs")

    def volumes(self, algo: int = _lib.DM_VOL_EDGE):
        self._ck(self._lib.dm_volumes(self._c, algo), "dm_volumes")

    def get_navs(self) -> np.ndarray:
        out = np.empty(self.mesh.dim * self.n_edges, np.float64)
        self._ck(self._lib.dm_get_navs(self._c, ptr(out, C.c_double)), "dm_get_navs")
        return out

    def get_volumes(self) -> np.ndarray:
        out = np.empty(self.mesh.num_nodes(), np.float64)
        self._ck(self._lib.dm_get_volumes(self._c, ptr(out, C.c_double)), "dm_get_volumes")
        return out

    def put_navs(self, navs: np.ndarray):
        navs = np.ascontiguousarray(navs, np.float64)
        self._ck(self._lib.dm_put_navs(self._c, ptr(navs, C.c_double)), "dm_put_navs")

    def put_volumes(self, vols: np.ndarray):
        vols = np.ascontiguousarray(vols, np.float64)
        self._ck(self._lib.dm_put_volumes(self._c, ptr(vols, C.c_double)), "dm_put_volumes")

    def metrics_host(self, coords, nav_algo, variant, vol_algo, navs_out, vols_out):
        """One end-to-end step through host buffers (pinned for speed)."""
        self._ck(self._lib.dm_metrics_host(self._c, coords, nav_algo, variant, vol_algo,
                                           navs_out, vols_out), "dm_metrics_host")

    def metrics_host_async(self, coords, nav_algo, variant, vol_algo, navs_out, vols_out):
        """Enqueue the same step and return (dm_metrics_host_async): consecutive
        calls overlap the copy-out of step i with the copy-in and kernels of
        step i+1.  Host buffers (pinned) stay untouched until sync()."""
        self._ck(self._lib.dm_metrics_host_async(self._c, coords, nav_algo, variant, vol_algo,
                                                 navs_out, vols_out), "dm_metrics_host_async")

    # ---------------------------------------------------------------- verify
    def check_closure(self):
        r, ri = C.c_double(), C.c_double()
        self._ck(self._lib.dm_check_closure(self._c, C.byref(r), C.byref(ri)), "dm_check_closure")
        return r.value, ri.value

    def check_total_volume(self):
        r, sv, se = C.c_double(), C.c_double(), C.c_double()
        self._ck(self._lib.dm_check_total_volume(self._c, C.byref(r), C.byref(sv), C.byref(se)),
                 "dm_check_total_volume")
        return r.value, sv.value, se.value

    def check_linear_exactness(self, A, b) -> float:
        """SPEC.md:265-274 (affine flux A x + b; constant flux when A == 0)."""
        A = np.ascontiguousarray(A, np.float64).ravel()
        b = np.ascontiguousarray(b, np.float64).ravel()
        r = C.c_double()
        self._ck(self._lib.dm_check_linear_exactness(self._c, ptr(A, C.c_double),
                                                     ptr(b, C.c_double), C.byref(r)),
                 "dm_check_linear_exactness")
        return r.value

    def corrupt_nav(self, edge: int, delta: float):
        self._ck(self._lib.dm_corrupt_nav(self._c, edge, delta), "dm_corrupt_nav")

    def max_face_area(self) -> float:
        v = C.c_double()
        self._ck(self._lib.dm_max_face_area(self._c, C.byref(v)), "dm_max_face_area")
        return v.value

    def max_element_volume(self) -> float:
        v = C.c_double()
        self._ck(self._lib.dm_max_element_volume(self._c, C.byref(v)), "dm_max_element_volume")
        return v.value

    def total_volume(self) -> float:
        v = C.c_double()
        self._ck(self._lib.dm_total_volume(self._c, C.byref(v)), "dm_total_volume")
        return v.value

    def boundary_node_mask(self) -> np.ndarray:
        m = np.empty(self.mesh.num_nodes(), np.uint8)
        self._ck(self._lib.dm_boundary_node_mask(self._c, ptr(m, C.c_uint8)),
                 "dm_boundary_node_mask")
        return m.astype(bool)

    def validate(self):
        signs = np.empty(self.mesh.num_elements(), np.int8)
        counts = np.zeros(_lib.DM_VCOUNT, np.int64)
        exposed = C.c_int64()
        self._ck(self._lib.dm_validate(self._c, ptr(signs, C.c_int8), ptr(counts, C.c_int64),
                                       C.byref(exposed)), "dm_validate")
        lists = []
        for kind in range(_lib.DM_VCOUNT):
            ids = np.empty(int(counts[kind]), np.int64)
            n = C.c_int64()
            if counts[kind]:
                self._ck(self._lib.dm_validate_list(self._c, kind, ptr(ids, C.c_int64),
                                                    int(counts[kind]), C.byref(n)),
                         "dm_validate_list")
            lists.append(ids)
        return signs, lists, exposed.value

    def derive_boundary(self) -> np.ndarray:
        n = C.c_int64()
        self._ck(self._lib.dm_derive_boundary(self._c, C.byref(n)), "dm_derive_boundary")
        out = np.empty(n.value * self.mesh.dim, np.int32)
        if n.value:
            self._ck(self._lib.dm_get_derived_boundary(self._c, ptr(out, C.c_int32)),
                     "dm_get_derived_boundary")
        return out

    # ---------------------------------------------------------------- plumbing
    def stream(self) -> int:
        s = C.c_void_p()
        self._ck(self._lib.dm_stream(self._c, C.byref(s)), "dm_stream")
        return s.value or 0

    def sync(self):
        self._ck(self._lib.dm_sync(self._c), "dm_sync")

    def set_timing(self, on: bool):
        self._ck(self._lib.dm_set_timing(self._c, 1 if on else 0), "dm_set_timing")

    def set_step_timing(self, steps: int):
        """Keep the phase events of the last `steps` steps (dm_set_timing(enable > 1))."""
        self._ck(self._lib.dm_set_timing(self._c, max(2, int(steps))), "dm_set_timing")

    def step_timings(self, max_steps: int) -> np.ndarray:
        """Rows [element loop, boundary pass, volume loop, total] (ms) of the newest
        recorded steps, oldest first (dm_get_step_timings; waits for the stream)."""
        ms = (C.c_float * (4 * max_steps))()
        n = C.c_int(0)
        self._ck(self._lib.dm_get_step_timings(self._c, ms, max_steps, C.byref(n)),
                 "dm_get_step_timings")
        return np.array(ms[:4 * n.value], dtype=np.float64).reshape(-1, 4)

    def timings(self) -> list[float]:
        ms = (C.c_float * 4)()
        self._ck(self._lib.dm_get_timings(self._c, ms, 4), "dm_get_timings")
        return list(ms)

    def plan_info(self) -> dict:
        info = np.zeros(8, np.int64)
        self._ck(self._lib.dm_plan_info(self._c, ptr(info, C.c_int64)), "dm_plan_info")
        return {"rings_built": bool(info[0]), "ring_ok": bool(info[1]),
                "tiles": {0: None, 1: "morton", 2: "row"}.get(int(info[0])),
                "tables_built": bool(info[2]), "table_ok": bool(info[3]),
                "ring_max_tile_nodes": int(info[4]), "ring_fail_bits": int(info[5]),
                "volume_order": "morton" if info[6] else "node",
                "colored": bool(info[7])}

    def plan_bytes(self) -> dict:
        """Per-step streams of the row-tile element loop (dm_plan_bytes)."""
        out = np.zeros(4, np.int64)
        self._ck(self._lib.dm_plan_bytes(self._c, ptr(out, C.c_int64)), "dm_plan_bytes")
        return {"codes": int(out[0]), "table_fill": int(out[1]), "meta_runs": int(out[2]),
                "tiles": int(out[3])}

    def side_edges(self) -> int:
        """Edges of the ring path's side list (dm_plan_side_edges)."""
        n = C.c_int64()
        self._ck(self._lib.dm_plan_side_edges(self._c, C.byref(n)), "dm_plan_side_edges")
        return n.value

    def launches(self) -> int:
        return int(self._lib.dm_kernel_launches(self._c))


# ------------------------------------------------------------------------
# Reference-named free functions (ref mesh.hpp:67-98) on a per-thread engine.
_tls = threading.local()


def default_engine() -> Engine:
    eng = getattr(_tls, "engine", None)
    if eng is None:
        eng = Engine()
        _tls.engine = eng
    return eng


def build_edges(mesh: Mesh) -> EdgeList:
    eng = default_engine()
    eng.set_mesh(mesh)
    eng.build_edges()
    return eng.edges()


def element_volume(mesh: Mesh, e: int) -> float:
    """ref mesh.cpp:75-92 (single element, host arithmetic)."""
    x = mesh.coords.reshape(-1, mesh.dim)
    el = mesh.element(e)
    if mesh.dim == 2:
        a, b, c = x[el[0]], x[el[1]], x[el[2]]
        return 0.5 * ((b[0] - a[0]) * (c[1] - a[1]) - (b[1] - a[1]) * (c[0] - a[0]))
    a, b, c, d = (x[el[i]] for i in range(4))
    u, v, w = b - a, c - a, d - a
    uv = (u[1] * v[2] - u[2] * v[1], u[2] * v[0] - u[0] * v[2], u[0] * v[1] - u[1] * v[0])
    return (uv[0] * w[0] + uv[1] * w[1] + uv[2] * w[2]) / 6.0


def max_face_area(mesh: Mesh) -> float:
    eng = default_engine()
    eng.set_mesh(mesh)
    return eng.max_face_area()


def max_element_volume(mesh: Mesh) -> float:
    eng = default_engine()
    eng.set_mesh(mesh)
    return eng.max_element_volume()


def total_volume(mesh: Mesh) -> float:
    eng = default_engine()
    eng.set_mesh(mesh)
    return eng.total_volume()


def boundary_node_mask(mesh: Mesh) -> np.ndarray:
    eng = default_engine()
    eng.set_mesh(mesh)
    return eng.boundary_node_mask()


def derive_boundary_faces(mesh: Mesh) -> np.ndarray:
    eng = default_engine()
    eng.set_mesh(mesh)
    return eng.derive_boundary()
