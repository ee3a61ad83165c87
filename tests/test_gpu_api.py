"""GPU tests of the C++ drop-in API (include/dualmesh/*.hpp via
tests/cpp/api_probe.cpp) against the reference's own mesh.cpp (oracle/_ref):
validate_mesh messages and volume signs, derive_boundary_faces, build_edges,
and the SPEC metrics facade."""
import ctypes as C
import os

import numpy as np
import pytest

from paper_2502_00778_b200 import Mesh, meshgen
from oracle.oracle import RefMesh, ref_available

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROBE = os.path.join(ROOT, "tests", "cpp", "_build", "libapi_probe.so")


@pytest.fixture(scope="module")
def probe():
    lib = C.CDLL(PROBE)
    P, I32, I64, D = C.c_void_p, C.POINTER(C.c_int32), C.c_int64, C.POINTER(C.c_double)
    lib.probe_validate.restype = I64
    lib.probe_validate.argtypes = [C.c_int, D, I64, I32, I64, I32, I64, C.c_char_p, I64,
                                   C.POINTER(C.c_int8)]
    lib.probe_derive.restype = I64
    lib.probe_derive.argtypes = [C.c_int, D, I64, I32, I64, I32, I64]
    lib.probe_build_edges.restype = I64
    lib.probe_build_edges.argtypes = [C.c_int, D, I64, I32, I64, I32, C.POINTER(C.c_uint64), I64]
    lib.probe_compute_metrics.restype = C.c_int
    lib.probe_compute_metrics.argtypes = [C.c_int, D, I64, I32, I64, I32, I64, C.c_int, C.c_int, D,
                                          D, D, D]
    lib.probe_linear_exactness.restype = C.c_int
    lib.probe_linear_exactness.argtypes = [C.c_int, D, I64, I32, I64, I32, I64, D, D, D]
    lib.probe_io.restype = I64
    lib.probe_io.argtypes = [C.c_char_p, C.c_char_p, C.c_char_p]
    lib.probe_mismatch.restype = C.c_int
    lib.probe_mismatch.argtypes = [C.c_int, D, I64, I32, I64]
    lib.probe_element_volume.restype = C.c_double
    lib.probe_element_volume.argtypes = [C.c_int, D, I64, I32, I64, I64]
    return lib


def _a(m):
    p = lambda a, t: a.ctypes.data_as(C.POINTER(t))  # noqa: E731
    return (m.dim, p(m.coords, C.c_double), m.num_nodes(), p(m.elements, C.c_int32),
            m.num_elements())


def gpu_validate(probe, m):
    buf = C.create_string_buffer(1 << 20)
    signs = np.zeros(max(m.num_elements(), 1), np.int8)
    bd = m.boundary if m.boundary.size else np.zeros(1, np.int32)
    n = probe.probe_validate(*_a(m), bd.ctypes.data_as(C.POINTER(C.c_int32)), m.num_boundary(),
                             buf, len(buf), signs.ctypes.data_as(C.POINTER(C.c_int8)))
    assert n >= 0, buf.value.decode()
    return [s for s in buf.value.decode().split("\n") if s], signs[:m.num_elements()]


def corrupted_meshes():
    base = meshgen.tet_cube(3, amp=0.15)
    tri = meshgen.tri_square(4, amp=0.2)
    out = {"valid_tet": base, "valid_tri": tri, "valid_bl": meshgen.baseline_config("C4", 16),
           "valid_perm": meshgen.baseline_config("C3", 16)}
    m = Mesh(3, base.coords, base.elements.copy(), base.boundary)
    el = m.elements.reshape(-1, 4)
    el[[2, 7]] = el[[2, 7]][:, [0, 2, 1, 3]]  # two inverted tets
    out["inverted"] = m
    m = Mesh(3, base.coords, base.elements, base.boundary.copy())
    m.boundary.reshape(-1, 3)[5] = m.boundary.reshape(-1, 3)[5][[0, 2, 1]]  # inward facet
    out["inward"] = m
    m = Mesh(3, base.coords, base.elements, np.concatenate([base.boundary, base.boundary[:6]]))
    out["duplicate"] = m  # two duplicated facets
    m = Mesh(3, base.coords, base.elements, base.boundary[3:])
    out["exposed"] = m  # one facet missing
    m = Mesh(3, base.coords, base.elements,
             np.concatenate([base.boundary, base.elements.reshape(-1, 4)[40, :3]]))
    out["interior_or_notface"] = m
    m = Mesh(3, base.coords, base.elements, np.concatenate([base.boundary, [0, 13, 63]]))
    out["not_a_face"] = m
    m = Mesh(3, base.coords, np.concatenate([base.elements, base.elements[:8]]), base.boundary)
    out["overshared"] = m  # two duplicated elements -> faces shared by 3
    m = Mesh(3, base.coords, base.elements.copy(), base.boundary)
    m.elements[9] = 10_000  # out of range
    out["range_elem"] = m
    m = Mesh(3, base.coords, base.elements, base.boundary.copy())
    m.boundary[4] = -1
    out["range_bnd"] = m
    t = Mesh(2, tri.coords, tri.elements.copy(), tri.boundary)
    t.elements.reshape(-1, 3)[3] = t.elements.reshape(-1, 3)[3][[0, 2, 1]]
    out["tri_inverted"] = t
    out["ftri_flipped"] = Mesh(2, [0, 0, 1, 0, 0, 1], [0, 2, 1], [0, 1, 1, 2, 2, 0])
    # no elements (the reference accepts them: nothing to violate)
    out["empty_tet"] = Mesh(3, np.arange(12.0), np.zeros(0, np.int32))
    out["empty_tri"] = Mesh(2, np.arange(8.0), np.zeros(0, np.int32))
    return out


@pytest.mark.parametrize("name", sorted(corrupted_meshes().keys()))
def test_validate_matches_reference(probe, name):
    m = corrupted_meshes()[name]
    got, signs = gpu_validate(probe, m)
    n, want, rsigns = RefMesh(m).validate()
    assert got == want
    if not any("out-of-range" in w for w in want):
        np.testing.assert_array_equal(signs, rsigns)


@pytest.mark.parametrize("name,scale", [("C1", 8), ("C2", 8), ("C3", 16), ("C4", 16)])
def test_derive_and_edges_match_reference(probe, name, scale):
    m = meshgen.baseline_config(name, scale)
    r = RefMesh(m)
    want = r.derive_boundary()
    got = np.empty(max(want.size, 1) + 64, np.int32)
    n = probe.probe_derive(*_a(m), got.ctypes.data_as(C.POINTER(C.c_int32)), got.size)
    assert n == want.size
    np.testing.assert_array_equal(got[:n], want)
    e, o = r.build_edges()
    ge = np.empty((e.shape[0] + 8, 2), np.int32)
    go = np.empty(m.num_nodes() + 1, np.uint64)
    ne = probe.probe_build_edges(*_a(m), ge.ctypes.data_as(C.POINTER(C.c_int32)),
                                 go.ctypes.data_as(C.POINTER(C.c_uint64)), ge.shape[0])
    assert ne == e.shape[0]
    np.testing.assert_array_equal(ge[:ne], e)
    np.testing.assert_array_equal(go, o)
    for el in (0, m.num_elements() // 2, m.num_elements() - 1):
        assert probe.probe_element_volume(*_a(m), el) == r.element_volume(el)


@pytest.mark.parametrize("dim", [2, 3])
def test_cpp_api_mesh_without_elements(probe, dim):
    """build_edges / derive_boundary_faces on a mesh without elements: empty results, like
    the reference (mesh.cpp:256-285, 287-330)."""
    m = Mesh(dim, np.arange(dim * 5, dtype=np.float64), np.zeros(0, np.int32))
    r = RefMesh(m)
    want = r.derive_boundary()
    got = np.empty(64, np.int32)
    n = probe.probe_derive(*_a(m), got.ctypes.data_as(C.POINTER(C.c_int32)), got.size)
    assert n == want.size == 0
    e, o = r.build_edges()
    ge = np.empty((8, 2), np.int32)
    go = np.full(m.num_nodes() + 1, 7, np.uint64)
    ne = probe.probe_build_edges(*_a(m), ge.ctypes.data_as(C.POINTER(C.c_int32)),
                                 go.ctypes.data_as(C.POINTER(C.c_uint64)), ge.shape[0])
    assert ne == e.shape[0] == 0
    np.testing.assert_array_equal(go, o)


@pytest.mark.parametrize("name,scale", [("C1", 4), ("C2", 4), ("C4", 8)])
def test_compute_metrics_facade(probe, oracle, name, scale):
    m = meshgen.baseline_config(name, scale)
    e, o = oracle.build_edges(m)
    want = oracle.navs_dualfree(m, e, o)
    navs = np.empty(want.size)
    vols = np.empty(m.num_nodes())
    cl, tv = C.c_double(), C.c_double()
    p = lambda a, t: a.ctypes.data_as(C.POINTER(t))  # noqa: E731
    st = probe.probe_compute_metrics(*_a(m), p(m.boundary, C.c_int32), m.num_boundary(), 1, 0,
                                     p(navs, C.c_double), p(vols, C.c_double), C.byref(cl),
                                     C.byref(tv))
    assert st == 0
    w = want.reshape(-1, m.dim)
    den = np.maximum(np.abs(w).max(axis=1), 1e-300)
    assert (np.abs(navs.reshape(-1, m.dim) - w).max(axis=1) / den).max() <= 1e-12
    vw = oracle.volumes_edge(m, e, want)
    assert np.abs(vols - vw).max() <= 1e-12 * np.abs(vw).max()
    assert cl.value <= 1e-13 and tv.value <= 1e-12
    assert probe.probe_mismatch(*_a(m)) == 1  # std::invalid_argument


@pytest.mark.parametrize("name,scale", [("C1", 4), ("C2", 4)])
def test_linear_exactness_cpp_api(probe, oracle, name, scale):
    """dualmesh::check_linear_exactness (metrics.hpp) against the oracle's
    check on the oracle's own fields (SPEC.md:265-274 bars)."""
    m = meshgen.baseline_config(name, scale)
    D = m.dim
    p = lambda a, t: a.ctypes.data_as(C.POINTER(t))  # noqa: E731
    rng = np.random.default_rng(3)
    A = rng.uniform(-1, 1, (D, D))
    A[0, 0] += 2.0
    f = rng.uniform(-1, 1, D)
    r = C.c_double()
    assert probe.probe_linear_exactness(*_a(m), p(m.boundary, C.c_int32), m.num_boundary(),
                                        p(np.ascontiguousarray(A), C.c_double), p(f, C.c_double),
                                        C.byref(r)) == 0
    e, o = oracle.build_edges(m)
    n = oracle.navs_dualfree(m, e, o)
    want = oracle.check_linear_exactness(m, e, n, oracle.volumes_edge(m, e, n), A, f)
    assert r.value <= 1e-11 and want <= 1e-11
    bad = np.diag([1.0, -1.0] + [0.0] * (D - 2))
    assert probe.probe_linear_exactness(*_a(m), p(m.boundary, C.c_int32), m.num_boundary(),
                                        p(np.ascontiguousarray(bad), C.c_double),
                                        p(f, C.c_double), C.byref(r)) == -1


def test_file_io_cpp_api(probe, tmp_path):
    """io.hpp: read_mesh derives a missing boundary, write_mesh round-trips,
    write_metrics writes the SPEC MetricsFile; parse errors throw."""
    import json
    from paper_2502_00778_b200 import fileio
    c = meshgen.tet_cube(4, amp=0.15)
    src = tmp_path / "in.dm"
    fileio.write_mesh(Mesh(3, c.coords, c.elements), src)
    src.write_text(src.read_text().replace("boundary 0\n", ""))
    out, met = tmp_path / "out.dm", tmp_path / "m.json"
    nb = probe.probe_io(str(src).encode(), str(out).encode(), str(met).encode())
    assert nb == c.num_boundary()
    r = fileio.read_mesh(out)
    np.testing.assert_array_equal(r.coords, c.coords)
    np.testing.assert_array_equal(r.elements, c.elements)
    np.testing.assert_array_equal(r.boundary, RefMesh(r).derive_boundary())
    d = json.loads(met.read_text())
    assert d["provenance"]["mesh_checksum"] == f"fnv1a64:{fileio.mesh_checksum(r):016x}"
    bad = tmp_path / "bad.dm"
    bad.write_text("dualmesh v1\ndim 2\nnodes 1\n0 0\nelements 1\n1 1 2\n")
    assert probe.probe_io(str(bad).encode(), str(out).encode(), str(met).encode()) == -1


def test_topology_cache_sequence(probe, oracle):
    """The C++ API keeps one topology resident per thread: calls on the same
    connectivity refresh coordinates only, any change of the element or
    boundary arrays (same sizes included) is seen and rebuilds.  Every call of
    a mixed sequence must equal the oracle on that call's mesh."""
    p = lambda a, t: a.ctypes.data_as(C.POINTER(t))  # noqa: E731
    base = meshgen.baseline_config("C2", 4)
    rng = np.random.default_rng(3)
    inner = (base.coords > 0) * (base.coords < 1)
    moved = Mesh(3, base.coords + rng.uniform(-1e-3, 1e-3, base.coords.size) * inner,
                 base.elements, base.boundary)
    el = base.elements.reshape(-1, 4)
    perm = rng.permutation(el.shape[0])
    permuted = Mesh(3, base.coords, el[perm].ravel().copy(), base.boundary)
    rot = el.copy()
    rot[5] = rot[5][[1, 2, 0, 3]]  # even permutation: same orientation, other local order
    rotated = Mesh(3, base.coords, rot.ravel().copy(), base.boundary)
    for m in (base, moved, moved, permuted, base, rotated, rotated, base):
        e, o = oracle.build_edges(m)
        want = oracle.navs_dualfree(m, e, o)
        navs, vols = np.empty(want.size), np.empty(m.num_nodes())
        cl, tv = C.c_double(), C.c_double()
        st = probe.probe_compute_metrics(*_a(m), p(m.boundary, C.c_int32), m.num_boundary(), 1,
                                         0, p(navs, C.c_double), p(vols, C.c_double),
                                         C.byref(cl), C.byref(tv))
        assert st == 0
        w = want.reshape(-1, 3)
        den = np.maximum(np.abs(w).max(axis=1), 1e-300)
        assert (np.abs(navs.reshape(-1, 3) - w).max(axis=1) / den).max() <= 1e-12
        vw = oracle.volumes_edge(m, e, want)
        assert np.abs(vols - vw).max() <= 1e-12 * np.abs(vw).max()
    assert probe.probe_mismatch(*_a(base)) == 1  # a foreign EdgeList still throws
