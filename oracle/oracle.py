"""ctypes wrappers of the CPU checkers.  TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this module, and only as the checker or
as the timed CPU baseline.  The product package never imports it.

* ``Oracle``   -- oracle/_build/liboracle.so: the serial C restatement
  (oracle.c) of SPEC.md:147-263 with the SURVEY Appendix A fp contract.
* ``RefMesh``  -- oracle/_ref/libref_mesh.so: the reference's own
  proj/src/mesh.cpp compiled in place (oracle/Makefile) behind ref_shim.cpp.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libref_mesh.so")

P = C.c_void_p
I32P = C.POINTER(C.c_int32)
U64P = C.POINTER(C.c_uint64)
DP = C.POINTER(C.c_double)
i64 = C.c_int64


def _p(a, t):
    return None if a is None else a.ctypes.data_as(C.POINTER(t))


class SimpleMesh:
    """Mesh arrays (same attribute surface as the product's Mesh)."""

    def __init__(self, dim, coords, elements, boundary):
        self.dim, self.coords, self.elements, self.boundary = dim, coords, elements, boundary

    def num_nodes(self):
        return self.coords.size // self.dim

    def num_elements(self):
        return self.elements.size // (self.dim + 1)

    def num_boundary(self):
        return self.boundary.size // self.dim

    def element(self, e):
        return self.elements[(self.dim + 1) * e:(self.dim + 1) * (e + 1)]

    def boundary_element(self, b):
        return self.boundary[self.dim * b:self.dim * (b + 1)]


class Oracle:
    def __init__(self):
        if not os.path.exists(ORACLE_SO):
            raise FileNotFoundError(f"{ORACLE_SO} missing: run `make -C oracle`")
        L = C.CDLL(ORACLE_SO)
        sig = {
            "or_build_edges": (i64, [C.c_int, i64, I32P, i64, C.POINTER(I32P), C.POINTER(U64P)]),
            "or_edge_of": (C.c_int32, [I32P, U64P, i64, C.c_int32, C.c_int32]),
            "or_edge_maps": (C.c_int, [C.c_int, i64, I32P, i64, I32P, U64P, i64, I32P, I32P,
                                       I32P]),
            "or_free": (None, [P]),
            "or_element_volume": (C.c_double, [C.c_int, DP, I32P]),
            "or_opposite_face_normal": (None, [C.c_int, DP, I32P, C.c_int, DP]),
            "or_boundary_normal": (None, [C.c_int, DP, I32P, DP]),
            "or_navs_dualfree": (C.c_int, [C.c_int, DP, i64, I32P, i64, I32P, i64, I32P, U64P,
                                           i64, I32P, DP]),
            "or_navs_traditional": (C.c_int, [C.c_int, DP, i64, I32P, i64, I32P, U64P, i64,
                                              I32P, DP]),
            "or_volumes_edge": (C.c_int, [C.c_int, DP, i64, I32P, i64, DP, DP]),
            "or_volumes_element": (C.c_int, [C.c_int, DP, i64, I32P, i64, DP]),
            "or_check_closure": (C.c_int, [C.c_int, DP, i64, I32P, i64, I32P, i64, DP, DP, DP]),
            "or_check_total_volume": (C.c_int, [C.c_int, DP, i64, I32P, i64, DP, DP, DP, DP]),
            "or_max_face_area": (C.c_double, [C.c_int, DP, I32P, i64]),
            "or_max_element_volume": (C.c_double, [C.c_int, DP, I32P, i64]),
            "or_check_linear_exactness": (C.c_int, [C.c_int, DP, i64, I32P, i64, I32P, i64, DP,
                                                     DP, DP, DP, DP]),
            "or_plan_create": (P, [C.c_int, i64, I32P, i64, I32P, i64, I32P, U64P, i64]),
            "or_plan_free": (None, [P]),
            "or_metrics_mt": (C.c_int, [P, DP, C.c_int, DP, DP, DP]),
            "or_gen_tet_cube": (C.c_int, [C.c_int, C.c_double, C.c_uint64, DP, I32P, I32P]),
        }
        for k, (r, a) in sig.items():
            f = getattr(L, k)
            f.restype, f.argtypes = r, a
        self.L = L

    # input synthesis ---------------------------------------------------------
    def gen_tet_cube(self, n, amp=0.15, seed=42):
        """SPEC gen_tet_cube + perturb_interior (oracle-owned; equals the
        product generator bit for bit, tests/test_oracle.py)."""
        x = np.empty(3 * (n + 1) ** 3, np.float64)
        el = np.empty(24 * n ** 3, np.int32)
        bd = np.empty(36 * n * n, np.int32)
        if self.L.or_gen_tet_cube(n, amp, seed, _p(x, C.c_double), _p(el, C.c_int32),
                                  _p(bd, C.c_int32)):
            raise ValueError("or_gen_tet_cube")
        return SimpleMesh(3, x, el, bd)

    # edges -----------------------------------------------------------------
    def build_edges(self, mesh):
        pe, po = I32P(), U64P()
        ne = self.L.or_build_edges(mesh.dim, mesh.num_nodes(), _p(mesh.elements, C.c_int32),
                                   mesh.num_elements(), C.byref(pe), C.byref(po))
        if ne < 0:
            raise MemoryError("or_build_edges")
        edges = np.ctypeslib.as_array(pe, shape=(max(ne, 1) * 2,))[:2 * ne].copy().reshape(ne, 2)
        os_ = np.ctypeslib.as_array(po, shape=(mesh.num_nodes() + 1,)).copy()
        self.L.or_free(C.cast(pe, P))
        self.L.or_free(C.cast(po, P))
        return edges, os_

    def edge_maps(self, mesh, edges, os_):
        L = 6 if mesh.dim == 3 else 3
        e2l = np.empty(L * mesh.num_elements(), np.int32)
        ip = np.empty(edges.shape[0] + 1, np.int32)
        inc = np.empty(L * mesh.num_elements(), np.int32)
        st = self.L.or_edge_maps(mesh.dim, mesh.num_nodes(), _p(mesh.elements, C.c_int32),
                                 mesh.num_elements(), _p(edges, C.c_int32), _p(os_, C.c_uint64),
                                 edges.shape[0], _p(e2l, C.c_int32), _p(ip, C.c_int32),
                                 _p(inc, C.c_int32))
        if st:
            raise RuntimeError(f"or_edge_maps: {st}")
        return e2l, ip, inc

    # multi-threaded dual-free navs + edge volumes (same bits as the serial pair)
    def plan(self, mesh, edges, os_):
        """Topology lists for metrics_mt; keeps references to the arrays it reads."""
        el, bd = mesh.elements, mesh.boundary if mesh.boundary.size else np.zeros(1, np.int32)
        h = self.L.or_plan_create(mesh.dim, mesh.num_nodes(), _p(el, C.c_int32),
                                  mesh.num_elements(), _p(bd, C.c_int32), mesh.num_boundary(),
                                  _p(edges, C.c_int32), _p(os_, C.c_uint64), edges.shape[0])
        if not h:
            raise MemoryError("or_plan_create")
        return {"h": h, "keep": (el, bd, edges, os_), "dim": mesh.dim, "ne": edges.shape[0],
                "nv": mesh.num_nodes()}

    def plan_free(self, plan):
        if plan.get("h"):
            self.L.or_plan_free(plan["h"])
            plan["h"] = None

    def metrics_mt(self, plan, coords, nthreads, out=None):
        if out is None:
            out = (np.empty(plan["dim"] * plan["ne"]), np.empty(max(plan["ne"], 1)),
                   np.empty(plan["nv"]))
        navs, s, V = out
        st = self.L.or_metrics_mt(plan["h"], _p(coords, C.c_double), nthreads,
                                  _p(navs, C.c_double), _p(s, C.c_double), _p(V, C.c_double))
        if st:
            raise RuntimeError(f"or_metrics_mt: {st}")
        return navs, V

    # metrics ---------------------------------------------------------------
    def navs_dualfree(self, mesh, edges, os_, e2l=None):
        out = np.empty(mesh.dim * edges.shape[0], np.float64)
        st = self.L.or_navs_dualfree(mesh.dim, _p(mesh.coords, C.c_double), mesh.num_nodes(),
                                     _p(mesh.elements, C.c_int32), mesh.num_elements(),
                                     _p(mesh.boundary, C.c_int32), mesh.num_boundary(),
                                     _p(edges, C.c_int32), _p(os_, C.c_uint64), edges.shape[0],
                                     _p(e2l, C.c_int32), _p(out, C.c_double))
        if st:
            raise ValueError(f"or_navs_dualfree: {st}")
        return out

    def navs_traditional(self, mesh, edges, os_, e2l=None):
        out = np.empty(mesh.dim * edges.shape[0], np.float64)
        st = self.L.or_navs_traditional(mesh.dim, _p(mesh.coords, C.c_double), mesh.num_nodes(),
                                        _p(mesh.elements, C.c_int32), mesh.num_elements(),
                                        _p(edges, C.c_int32), _p(os_, C.c_uint64),
                                        edges.shape[0], _p(e2l, C.c_int32), _p(out, C.c_double))
        if st:
            raise ValueError(f"or_navs_traditional: {st}")
        return out

    def volumes_edge(self, mesh, edges, navs):
        out = np.empty(mesh.num_nodes(), np.float64)
        self.L.or_volumes_edge(mesh.dim, _p(mesh.coords, C.c_double), mesh.num_nodes(),
                               _p(edges, C.c_int32), edges.shape[0], _p(navs, C.c_double),
                               _p(out, C.c_double))
        return out

    def volumes_element(self, mesh):
        out = np.empty(mesh.num_nodes(), np.float64)
        self.L.or_volumes_element(mesh.dim, _p(mesh.coords, C.c_double), mesh.num_nodes(),
                                  _p(mesh.elements, C.c_int32), mesh.num_elements(),
                                  _p(out, C.c_double))
        return out

    # verify ----------------------------------------------------------------
    def check_closure(self, mesh, edges, navs):
        r, ri = C.c_double(), C.c_double()
        self.L.or_check_closure(mesh.dim, _p(mesh.coords, C.c_double), mesh.num_nodes(),
                                _p(mesh.boundary, C.c_int32), mesh.num_boundary(),
                                _p(edges, C.c_int32), edges.shape[0], _p(navs, C.c_double),
                                C.byref(r), C.byref(ri))
        return r.value, ri.value

    def check_linear_exactness(self, mesh, edges, navs, vols, A, b):
        A = np.ascontiguousarray(A, np.float64).ravel()
        b = np.ascontiguousarray(b, np.float64).ravel()
        r = C.c_double()
        bd = mesh.boundary if mesh.boundary.size else np.zeros(1, np.int32)
        st = self.L.or_check_linear_exactness(
            mesh.dim, _p(mesh.coords, C.c_double), mesh.num_nodes(), _p(bd, C.c_int32),
            mesh.num_boundary(), _p(edges, C.c_int32), edges.shape[0], _p(navs, C.c_double),
            _p(vols, C.c_double), _p(A, C.c_double), _p(b, C.c_double), C.byref(r))
        if st == -1:
            raise ValueError("trace(A) = 0: relative residual undefined")
        if st:
            raise MemoryError("or_check_linear_exactness")
        return r.value

    def check_total_volume(self, mesh, vols):
        r, sv, se = C.c_double(), C.c_double(), C.c_double()
        self.L.or_check_total_volume(mesh.dim, _p(mesh.coords, C.c_double), mesh.num_nodes(),
                                     _p(mesh.elements, C.c_int32), mesh.num_elements(),
                                     _p(vols, C.c_double), C.byref(r), C.byref(sv), C.byref(se))
        return r.value, sv.value, se.value

    def opposite_face_normal(self, mesh, e, i):
        out = np.empty(3, np.float64)
        el = np.ascontiguousarray(mesh.element(e))
        self.L.or_opposite_face_normal(mesh.dim, _p(mesh.coords, C.c_double), _p(el, C.c_int32),
                                       i, _p(out, C.c_double))
        return out

    def boundary_normal(self, mesh, b):
        out = np.empty(3, np.float64)
        bl = np.ascontiguousarray(mesh.boundary_element(b))
        self.L.or_boundary_normal(mesh.dim, _p(mesh.coords, C.c_double), _p(bl, C.c_int32),
                                  _p(out, C.c_double))
        return out

    def element_volume(self, mesh, e):
        el = np.ascontiguousarray(mesh.element(e))
        return self.L.or_element_volume(mesh.dim, _p(mesh.coords, C.c_double), _p(el, C.c_int32))

    def max_face_area(self, mesh):
        return self.L.or_max_face_area(mesh.dim, _p(mesh.coords, C.c_double),
                                       _p(mesh.elements, C.c_int32), mesh.num_elements())

    def max_element_volume(self, mesh):
        return self.L.or_max_element_volume(mesh.dim, _p(mesh.coords, C.c_double),
                                            _p(mesh.elements, C.c_int32), mesh.num_elements())


def ref_available() -> bool:
    return os.path.exists(REF_SO)


class RefMesh:
    """The reference mesh module itself (proj/src/mesh.cpp) on one mesh."""

    _lib = None

    @classmethod
    def lib(cls):
        if cls._lib is None:
            if not ref_available():
                raise FileNotFoundError(f"{REF_SO} missing: run `make -C oracle` where "
                                        "/root/reference exists")
            L = C.CDLL(REF_SO)
            sig = {
                "ref_mesh_new": (P, [C.c_int, DP, i64, I32P, i64, I32P, i64]),
                "ref_mesh_free": (None, [P]),
                "ref_build_edges": (i64, [P]),
                "ref_get_edges": (None, [P, I32P, U64P]),
                "ref_edge_of": (C.c_int32, [P, C.c_int32, C.c_int32]),
                "ref_element_volume": (C.c_double, [P, i64]),
                "ref_opposite_face_normal": (None, [P, i64, C.c_int, DP]),
                "ref_boundary_normal": (None, [P, i64, DP]),
                "ref_validate": (i64, [P, C.c_char_p, i64, C.POINTER(C.c_int8)]),
                "ref_derive_boundary": (i64, [P, C.POINTER(I32P)]),
                "ref_free": (None, [P]),
                "ref_max_face_area": (C.c_double, [P]),
                "ref_max_element_volume": (C.c_double, [P]),
                "ref_total_volume": (C.c_double, [P]),
                "ref_boundary_node_mask": (None, [P, C.POINTER(C.c_uint8)]),
            }
            for k, (r, a) in sig.items():
                f = getattr(L, k)
                f.restype, f.argtypes = r, a
            cls._lib = L
        return cls._lib

    def __init__(self, mesh):
        self.mesh = mesh
        L = self.lib()
        self.h = L.ref_mesh_new(mesh.dim, _p(mesh.coords, C.c_double), mesh.num_nodes(),
                                _p(mesh.elements, C.c_int32), mesh.num_elements(),
                                _p(mesh.boundary, C.c_int32), mesh.num_boundary())
        self.ne = None

    def __del__(self):
        try:
            self.lib().ref_mesh_free(self.h)
        except Exception:
            pass

    def build_edges(self):
        L = self.lib()
        self.ne = L.ref_build_edges(self.h)
        e = np.empty((self.ne, 2), np.int32)
        o = np.empty(self.mesh.num_nodes() + 1, np.uint64)
        L.ref_get_edges(self.h, _p(e, C.c_int32), _p(o, C.c_uint64))
        return e, o

    def edge_of(self, a, b):
        return self.lib().ref_edge_of(self.h, int(a), int(b))

    def element_volume(self, e):
        return self.lib().ref_element_volume(self.h, e)

    def opposite_face_normal(self, e, i):
        out = np.empty(3, np.float64)
        self.lib().ref_opposite_face_normal(self.h, e, i, _p(out, C.c_double))
        return out

    def boundary_normal(self, b):
        out = np.empty(3, np.float64)
        self.lib().ref_boundary_normal(self.h, b, _p(out, C.c_double))
        return out

    def validate(self):
        buf = C.create_string_buffer(1 << 20)
        signs = np.empty(max(self.mesh.num_elements(), 1), np.int8)
        n = self.lib().ref_validate(self.h, buf, len(buf), _p(signs, C.c_int8))
        msgs = [m for m in buf.value.decode().split("\n") if m]
        return n, msgs, signs[:self.mesh.num_elements()]

    def derive_boundary(self):
        pf = I32P()
        n = self.lib().ref_derive_boundary(self.h, C.byref(pf))
        out = np.ctypeslib.as_array(pf, shape=(max(n, 1),))[:n].copy()
        self.lib().ref_free(C.cast(pf, P))
        return out

    def max_face_area(self):
        return self.lib().ref_max_face_area(self.h)

    def max_element_volume(self):
        return self.lib().ref_max_element_volume(self.h)

    def total_volume(self):
        return self.lib().ref_total_volume(self.h)

    def boundary_node_mask(self):
        m = np.empty(self.mesh.num_nodes(), np.uint8)
        self.lib().ref_boundary_node_mask(self.h, _p(m, C.c_uint8))
        return m.astype(bool)
