"""GPU parity tests: the sm_100a path (through the C-ABI) against the oracle
and the committed golden fixtures.  Bars (north_star / SURVEY 8(c)):
edge structures bit-exact; GATHER navs and volumes bitwise equal to the
serial oracle; SCATTER navs within 1e-12 per edge vector
(||x_gpu - x_ref||_inf <= 1e-12 ||x_ref||_inf); closure <= 1e-13 scaled;
|sum V - sum V_E| / sum V_E <= 1e-12."""
import os

import numpy as np
import pytest

from paper_2502_00778_b200 import EdgeAbsent, Mesh, meshgen
from paper_2502_00778_b200 import _lib

pytestmark = pytest.mark.gpu

DF, TR = _lib.DM_NAV_DUALFREE, _lib.DM_NAV_TRADITIONAL
GATHER, SCATTER = _lib.DM_VARIANT_GATHER, _lib.DM_VARIANT_SCATTER
EXACT, FACES, ELEMV = (_lib.DM_VARIANT_GATHER_EXACT, _lib.DM_VARIANT_GATHER_FACES,
                       _lib.DM_VARIANT_GATHER_ELEM)
EDGE, ELEM = _lib.DM_VOL_EDGE, _lib.DM_VOL_ELEMENT


def per_vector_rel(a, b, dim):
    a, b = a.reshape(-1, dim), b.reshape(-1, dim)
    num = np.abs(a - b).max(axis=1)
    den = np.abs(b).max(axis=1)
    den = np.where(den == 0, 1.0, den)
    return float((num / den).max())


def oracle_i32p():
    import ctypes as C
    return C.POINTER(C.c_int32)


def oracle_u64p():
    import ctypes as C
    return C.POINTER(C.c_uint64)


def run_all(eng, mesh):
    eng.set_mesh(mesh)
    eng.build_edges()
    out = {"edgelist": eng.edges(), "e2l": eng.e2l()}
    out["inc_ptr"], out["inc"] = eng.incidence()
    eng.navs(DF, EXACT)
    out["navs_dualfree"] = eng.get_navs()
    eng.volumes(EDGE)
    out["vol_edge"] = eng.get_volumes()
    eng.volumes(ELEM)
    out["vol_element"] = eng.get_volumes()
    eng.navs(DF, FACES)
    out["navs_faces"] = eng.get_navs()
    eng.navs(DF, ELEMV)
    out["navs_elem"] = eng.get_navs()
    eng.navs(TR, EXACT)  # face-list kernel: bitwise the serial loop
    out["navs_traditional"] = eng.get_navs()
    eng.navs(TR, GATHER)  # ring walk: <= 1e-12, deterministic
    out["navs_trad_fast"] = eng.get_navs()
    eng.navs(TR, GATHER)
    out["navs_trad_fast2"] = eng.get_navs()
    eng.navs(DF, SCATTER)
    out["navs_scatter"] = eng.get_navs()
    eng.navs(DF, GATHER)  # default fast path (ring walk in 3D)
    out["navs_fast"] = eng.get_navs()
    eng.volumes(EDGE)
    out["vol_fast"] = eng.get_volumes()
    eng.navs(DF, GATHER)
    out["navs_fast2"] = eng.get_navs()
    return out


def check_fast(g, want_navs, want_vol, dim):
    """Default GATHER: deterministic, within 1e-12 of the serial oracle."""
    np.testing.assert_array_equal(g["navs_fast"], g["navs_fast2"])
    assert per_vector_rel(g["navs_fast"], want_navs, dim) <= 1e-12
    assert np.abs(g["vol_fast"] - want_vol).max() <= 1e-12 * np.abs(want_vol).max()
    np.testing.assert_array_equal(g["navs_faces"], want_navs)
    np.testing.assert_array_equal(g["navs_elem"], want_navs)
    np.testing.assert_array_equal(g["navs_trad_fast"], g["navs_trad_fast2"])
    assert per_vector_rel(g["navs_trad_fast"], g["navs_traditional"], dim) <= 1e-12


def test_fixtures_bit_exact(engine, fixtures, oracle):
    for name, d in fixtures.items():
        m = d["mesh_obj"]
        g = run_all(engine, m)
        assert g["edgelist"].edges.tolist() == d["ref_edges"], name
        assert g["edgelist"].origin_start.tolist() == d["ref_origin_start"], name
        e, o = np.array(d["ref_edges"], np.int32).reshape(-1, 2), np.array(d["ref_origin_start"], np.uint64)
        np.testing.assert_array_equal(g["navs_dualfree"], oracle.navs_dualfree(m, e, o))
        np.testing.assert_array_equal(g["navs_traditional"], oracle.navs_traditional(m, e, o))
        np.testing.assert_array_equal(g["vol_edge"], oracle.volumes_edge(m, e, g["navs_dualfree"]))
        np.testing.assert_array_equal(g["vol_element"], oracle.volumes_element(m))
        check_fast(g, g["navs_dualfree"], g["vol_edge"], m.dim)


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
def test_golden_configs_bit_exact(engine, golden_configs, name):
    gd = golden_configs[name]
    g = run_all(engine, gd["mesh"])
    np.testing.assert_array_equal(g["edgelist"].edges, gd["edges"])
    np.testing.assert_array_equal(g["edgelist"].origin_start, gd["origin_start"])
    np.testing.assert_array_equal(g["e2l"], gd["e2l"])
    np.testing.assert_array_equal(g["inc_ptr"], gd["inc_ptr"])
    np.testing.assert_array_equal(g["inc"], gd["inc"])
    for k in ("navs_dualfree", "navs_traditional", "vol_edge", "vol_element"):
        np.testing.assert_array_equal(g[k], gd[k], err_msg=k)
    assert per_vector_rel(g["navs_scatter"], gd["navs_dualfree"], gd["mesh"].dim) <= 1e-12
    check_fast(g, gd["navs_dualfree"], gd["vol_edge"], gd["mesh"].dim)


@pytest.mark.parametrize("name,scale", [("C1", 1), ("C2", 1), ("C3", 2), ("C4", 2)])
def test_live_oracle_parity(engine, oracle, name, scale):
    m = meshgen.baseline_config(name, scale)
    g = run_all(engine, m)
    e, o = oracle.build_edges(m)
    np.testing.assert_array_equal(g["edgelist"].edges, e)
    np.testing.assert_array_equal(g["edgelist"].origin_start, o)
    e2l, ip, inc = oracle.edge_maps(m, e, o)
    np.testing.assert_array_equal(g["e2l"], e2l)
    np.testing.assert_array_equal(g["inc_ptr"], ip)
    np.testing.assert_array_equal(g["inc"], inc)
    nd = oracle.navs_dualfree(m, e, o, e2l)
    np.testing.assert_array_equal(g["navs_dualfree"], nd)
    np.testing.assert_array_equal(g["navs_traditional"], oracle.navs_traditional(m, e, o, e2l))
    np.testing.assert_array_equal(g["vol_edge"], oracle.volumes_edge(m, e, nd))
    np.testing.assert_array_equal(g["vol_element"], oracle.volumes_element(m))
    assert per_vector_rel(g["navs_scatter"], nd, m.dim) <= 1e-12
    check_fast(g, nd, oracle.volumes_edge(m, e, nd), m.dim)


@pytest.mark.parametrize("name", ["C3", "C4", "C5"])
def test_full_size_properties(engine, name):
    """BASELINE sizes: size-independent identities + determinism."""
    m = meshgen.baseline_config(name)
    engine.set_mesh(m)
    ne = engine.build_edges()
    if name == "C5":
        assert ne == 118031104 and m.num_nodes() == 16974593
    for variant in (GATHER, EXACT):
        engine.navs(DF, variant)
        engine.volumes(EDGE)
        r, ri = engine.check_closure()
        assert r <= 1e-13 and ri <= 1e-13
        rel, sv, se = engine.check_total_volume()
        assert rel <= 1e-12
        if name != "C4":
            assert abs(sv - 1.0) <= 1e-12  # unit cube, PAPER §4.3
    n1, v1 = engine.get_navs(), engine.get_volumes()
    engine.navs(DF, EXACT)
    engine.volumes(EDGE)
    np.testing.assert_array_equal(engine.get_navs(), n1)  # SPEC.md:206 determinism
    np.testing.assert_array_equal(engine.get_volumes(), v1)
    engine.navs(DF, GATHER)
    nf = engine.get_navs()
    engine.navs(DF, GATHER)
    np.testing.assert_array_equal(engine.get_navs(), nf)
    assert per_vector_rel(nf, n1, m.dim) <= 1e-12
    engine.navs(DF, SCATTER)
    assert per_vector_rel(engine.get_navs(), n1, m.dim) <= 1e-12
    engine.navs(TR, GATHER)
    nt = engine.get_navs()
    scale = engine.max_face_area()
    assert np.abs(nt - n1).max() <= 1e-13 * scale


@pytest.mark.parametrize("name", ["C3", "C4", "C5", "2D-2048"])
def test_full_size_oracle_parity(engine, oracle, name):
    """BASELINE sizes against the CPU oracle itself: the edge list and origin
    CSR bit for bit, the serial-order variant (GATHER_EXACT) and the edge
    volumes bit for bit, the default ring walk within 1e-12 per edge vector
    (or_metrics_mt on all host threads gives the serial loops' bits)."""
    if name == "2D-2048":  # the C1 family at 2048^2 quads (8.4 M triangles)
        m = meshgen.tri_square(2048, diag_seed=meshgen.SEED_DIAG, amp=0.2, seed=meshgen.SEED_JITTER)
    else:
        m = meshgen.baseline_config(name)
    engine.set_mesh(m)
    ne = engine.build_edges()
    e, o = oracle.build_edges(m)
    got = engine.edges()
    assert ne == e.shape[0]
    np.testing.assert_array_equal(got.edges, e)
    np.testing.assert_array_equal(got.origin_start, o)
    plan = oracle.plan(m, e, o)
    try:
        want_n, want_v = oracle.metrics_mt(plan, m.coords, os.cpu_count() or 1)
    finally:
        oracle.plan_free(plan)
    engine.navs(DF, EXACT)
    engine.volumes(EDGE)
    np.testing.assert_array_equal(engine.get_navs(), want_n)
    np.testing.assert_array_equal(engine.get_volumes(), want_v)
    engine.navs(DF, GATHER)
    engine.volumes(EDGE)
    assert per_vector_rel(engine.get_navs(), want_n, m.dim) <= 1e-12
    v = engine.get_volumes()
    assert np.abs(v - want_v).max() <= 1e-12 * np.abs(want_v).max()


def test_corrupt_hook_detected(engine):
    m = meshgen.tet_cube(16, amp=0.2, seed=42)
    engine.set_mesh(m)
    engine.build_edges()
    engine.navs(DF, GATHER)
    assert engine.check_closure()[0] <= 1e-13
    engine.corrupt_nav(123, 1e-3)
    assert engine.check_closure()[0] >= 1e-4


def test_errors(engine):
    m = meshgen.tet_cube(2)
    engine.set_mesh(m)
    with pytest.raises(Exception):
        engine.navs(DF, GATHER)  # before build_edges
    bad = Mesh(3, m.coords, m.elements, np.array([0, 26, 13], np.int32))  # not a mesh edge
    engine.set_mesh(bad)
    engine.build_edges()
    with pytest.raises(EdgeAbsent):
        engine.navs(DF, GATHER)


def test_edge_of_and_helpers(engine, oracle):
    m = meshgen.baseline_config("C2", 4)
    engine.set_mesh(m)
    engine.build_edges()
    el = engine.edges()
    rng = np.random.default_rng(0)
    a = rng.integers(0, m.num_nodes(), 5000).astype(np.int32)
    b = rng.integers(0, m.num_nodes(), 5000).astype(np.int32)
    a[:2500] = el.edges[:2500, 1]  # reversed present pairs
    b[:2500] = el.edges[:2500, 0]
    got = engine.edge_of(a, b)
    # the reference's own EdgeList::edge_of (mesh.cpp:58-73, oracle/_ref) is
    # the checker; the oracle restatement must agree with it too
    from oracle.oracle import RefMesh, ref_available
    if ref_available():
        r = RefMesh(m)
        re_, ro = r.build_edges()
        np.testing.assert_array_equal(re_, el.edges)
        want = np.array([r.edge_of(int(x), int(y)) for x, y in zip(a, b)])
    else:
        want = np.array([oracle.L.or_edge_of(el.edges.ctypes.data_as(oracle_i32p()),
                                             el.origin_start.ctypes.data_as(oracle_u64p()),
                                             m.num_nodes(), int(x), int(y))
                         for x, y in zip(a, b)])
    np.testing.assert_array_equal(got, want)
    assert (want[:2500] >= 0).all() and (want[2500:] == -1).any()
    assert engine.max_face_area() == oracle.max_face_area(m)
    assert engine.max_element_volume() == oracle.max_element_volume(m)
    assert abs(engine.total_volume() - 1.0) <= 1e-14
    mask = engine.boundary_node_mask()
    want_mask = np.zeros(m.num_nodes(), bool)
    want_mask[m.boundary] = True
    np.testing.assert_array_equal(mask, want_mask)


@pytest.mark.parametrize("name,scale,order", [("C2", 1, "node"), ("C3", 2, "morton"),
                                              ("C5", 4, "node")])
def test_ring_path_volume_orders_bitwise(engine, oracle, name, scale, order):
    """The ring path's s_e (edge order, or Morton position order for node
    numberings without locality) feeds the edge-volume fold in the serial
    order: the volumes equal the oracle's volumes of the GPU navs bit for bit;
    a navs row put back by the caller takes the edge-order path."""
    m = meshgen.baseline_config(name, scale)
    engine.set_mesh(m)
    engine.build_edges()
    engine.navs(DF, GATHER)
    info = engine.plan_info()
    assert info["ring_ok"] and info["volume_order"] == order
    nf = engine.get_navs()
    engine.volumes(EDGE)
    e, _ = oracle.build_edges(m)
    np.testing.assert_array_equal(engine.get_volumes(), oracle.volumes_edge(m, e, nf))
    nput = nf * 0.5
    engine.put_navs(nput)
    engine.volumes(EDGE)
    np.testing.assert_array_equal(engine.get_volumes(), oracle.volumes_edge(m, e, nput))


def _affine(dim, seed):
    rng = np.random.default_rng(seed)
    A = rng.uniform(-1.0, 1.0, (dim, dim))
    if abs(np.trace(A)) < 0.1:
        A[0, 0] += 1.0
    return A, rng.uniform(-1.0, 1.0, dim)


@pytest.mark.parametrize("name,scale,tol", [("C1", 2, 1e-11), ("C2", 2, 1e-11),
                                            ("C3", 4, 1e-11), ("C4", 4, 1e-9)])
def test_linear_exactness_matches_oracle(engine, oracle, name, scale, tol):
    """SPEC.md:265-274 on the GPU: with the bit-exact navs / volumes the
    affine-flux residual equals the oracle's bit for bit; the fast path and
    the constant-flux balance meet the SPEC tolerances."""
    m = meshgen.baseline_config(name, scale)
    D = m.dim
    engine.set_mesh(m)
    engine.build_edges()
    engine.navs(DF, EXACT)
    engine.volumes(EDGE)
    e, _ = oracle.build_edges(m)
    n, v = engine.get_navs(), engine.get_volumes()
    A, b = _affine(D, 11)
    for AA, bb in ((A, b), (np.eye(D) / D, np.zeros(D))):
        g = engine.check_linear_exactness(AA, bb)
        assert g == oracle.check_linear_exactness(m, e, n, v, AA, bb)
        assert g <= tol
    gc = engine.check_linear_exactness(np.zeros((D, D)), b)
    oc = oracle.check_linear_exactness(m, e, n, v, np.zeros((D, D)), b)
    assert gc <= 1e-13 and abs(gc - oc) <= 1e-15
    engine.navs(DF, GATHER)
    engine.volumes(EDGE)
    assert engine.check_linear_exactness(A, b) <= tol
    with pytest.raises(Exception):
        engine.check_linear_exactness(np.diag([1.0, -1.0] + [0.0] * (D - 2)), b)


def test_linear_exactness_full_size():
    """C5 at full size (SPEC invariant: exactness <= 1e-11)."""
    from paper_2502_00778_b200 import Engine
    m = meshgen.baseline_config("C5")
    eng = Engine(0)
    try:
        eng.set_mesh(m)
        eng.build_edges()
        eng.navs(DF, GATHER)
        eng.volumes(EDGE)
        A, b = _affine(3, 5)
        assert eng.check_linear_exactness(A, b) <= 1e-11
        assert eng.check_linear_exactness(np.eye(3) / 3, np.zeros(3)) <= 1e-11
        assert eng.check_linear_exactness(np.zeros((3, 3)), b) <= 1e-13
        eng.corrupt_nav(int(m.num_elements() // 3), 1e-3)
        assert eng.check_linear_exactness(A, b) > 1e-6
    finally:
        eng.close()


def _fan_mesh(n):
    """n tets around the edge (0,0,0)-(0,0,1): an edge with n > kRingMax (24)
    incidences pushes the ring plan to its fallback."""
    th = 2 * np.pi * np.arange(n) / n
    ring = np.stack([np.cos(th), np.sin(th), np.full(n, 0.5)], 1)
    x = np.concatenate([[[0, 0, 0], [0, 0, 1]], ring]).ravel()
    el = []
    for i in range(n):
        t = [0, 1, 2 + i, 2 + (i + 1) % n]
        p = x.reshape(-1, 3)[t]
        if np.linalg.det(np.stack([p[1] - p[0], p[2] - p[0], p[3] - p[0]])) < 0:
            t[2], t[3] = t[3], t[2]
        el += t
    return Mesh(3, x, np.array(el, np.int32))


@pytest.mark.parametrize("n", [12, 30, 50, 1500])
def test_fan_fallback(engine, oracle, n):
    """Fans around one edge: n > 24 incidences per edge go to the side list;
    n = 50 sorts node 0's 150 K1 keys in the CTA bitonic path, n = 1500 its
    4500 keys (> 4096) in the per-segment radix-sort path."""
    m0 = _fan_mesh(n)
    engine.set_mesh(m0)
    m = Mesh(3, m0.coords, m0.elements, engine.derive_boundary())
    engine.set_mesh(m)
    engine.build_edges()
    engine.navs(DF, GATHER)
    info = engine.plan_info()
    # the fan's hub edge rides the ring path's side list; the ring path stays
    assert info["ring_ok"] and engine.side_edges() == (1 if n > 24 else 0)
    e, o = oracle.build_edges(m)
    got = engine.edges()
    np.testing.assert_array_equal(got.edges, e)
    np.testing.assert_array_equal(got.origin_start, o)
    e2l, ip, inc = oracle.edge_maps(m, e, o)
    np.testing.assert_array_equal(engine.e2l(), e2l)
    gip, ginc = engine.incidence()
    np.testing.assert_array_equal(gip, ip)
    np.testing.assert_array_equal(ginc, inc)
    want = oracle.navs_dualfree(m, e, o)
    assert per_vector_rel(engine.get_navs(), want, 3) <= 1e-12
    engine.volumes(EDGE)
    np.testing.assert_array_equal(engine.get_volumes(), oracle.volumes_edge(m, e, engine.get_navs()))


def test_local_order_rotations(engine, oracle):
    """Elements stored with even permutations of their local order (still
    positively oriented): the ring orientation bits follow the local order."""
    m = meshgen.baseline_config("C2", 4)
    rng = np.random.default_rng(9)
    even = np.array([[0, 1, 2, 3], [1, 2, 0, 3], [2, 0, 1, 3], [0, 2, 3, 1], [0, 3, 1, 2],
                     [1, 0, 3, 2], [2, 3, 0, 1], [3, 2, 1, 0], [1, 3, 2, 0], [2, 1, 3, 0],
                     [3, 0, 2, 1], [3, 1, 0, 2]])
    el = m.elements.reshape(-1, 4)
    pick = even[rng.integers(0, len(even), el.shape[0])]
    el2 = np.take_along_axis(el, pick, axis=1)
    m2 = Mesh(3, m.coords, el2, m.boundary)
    engine.set_mesh(m2)
    engine.build_edges()
    engine.navs(DF, GATHER)
    assert engine.plan_info()["ring_ok"]
    e, o = oracle.build_edges(m2)
    want = oracle.navs_dualfree(m2, e, o)
    assert per_vector_rel(engine.get_navs(), want, 3) <= 1e-12
    engine.navs(DF, EXACT)
    np.testing.assert_array_equal(engine.get_navs(), want)


def test_isolated_nodes_and_inverted_element(engine, oracle):
    """Unused nodes get zero volume and do not disturb the ring plan; an
    inverted element makes the rings of its edges inconsistently oriented:
    those edges (only) go to the side list, whose rows are evaluated in
    element order -- so here, with every other row within 1e-12, the side
    rows equal the oracle bitwise."""
    m = meshgen.tet_cube(5, amp=0.15)
    extra = np.array([[2.0, 2.0, 2.0], [-1.0, 0.5, 0.5]])
    mi = Mesh(3, np.concatenate([m.coords, extra.ravel()]), m.elements, m.boundary)
    engine.set_mesh(mi)
    engine.build_edges()
    engine.navs(DF, GATHER)
    assert engine.plan_info()["ring_ok"]
    e, o = oracle.build_edges(mi)
    want = oracle.navs_dualfree(mi, e, o)
    assert per_vector_rel(engine.get_navs(), want, 3) <= 1e-12
    engine.volumes(EDGE)
    v = engine.get_volumes()
    assert v[-1] == 0.0 and v[-2] == 0.0
    np.testing.assert_array_equal(v, oracle.volumes_edge(mi, e, engine.get_navs()))
    el = m.elements.reshape(-1, 4).copy()
    el[17] = el[17][[0, 2, 1, 3]]
    mv = Mesh(3, m.coords, el, m.boundary)
    engine.set_mesh(mv)
    engine.build_edges()
    engine.navs(DF, GATHER)
    info = engine.plan_info()
    assert info["ring_ok"] and info["ring_fail_bits"] & 16 and 0 < engine.side_edges() <= 6
    e, o = oracle.build_edges(mv)
    want = oracle.navs_dualfree(mv, e, o)
    got = engine.get_navs()
    assert per_vector_rel(got, want, 3) <= 1e-12
    el17 = mv.elements.reshape(-1, 4)[17]
    for a in range(4):
        for b in range(a + 1, 4):
            i = int(np.nonzero((e[:, 0] == min(el17[a], el17[b])) &
                               (e[:, 1] == max(el17[a], el17[b])))[0][0])
            np.testing.assert_array_equal(got.reshape(-1, 3)[i], want.reshape(-1, 3)[i])
    engine.navs(DF, EXACT)
    np.testing.assert_array_equal(engine.get_navs(), want)


def test_empty_mesh(engine):
    for dim in (2, 3):
        engine.set_mesh(Mesh(dim, np.zeros(0), np.zeros(0, np.int32)))
        assert engine.build_edges() == 0
        engine.navs(DF, GATHER)
        engine.volumes(EDGE)
        assert engine.get_navs().size == 0 and engine.get_volumes().size == 0


@pytest.mark.parametrize("name,scale", [("C2", 2), ("C3", 4), ("C4", 4)])
def test_deforming_grid_reuses_plan(engine, oracle, name, scale):
    """New coordinates on the same topology (the deforming-grid step): the
    ring plan built on the first coordinates stays valid, the Morton-order
    coordinate copy follows the update, results match the oracle on the new
    coordinates; dm_metrics_host (host buffers) gives the same fields."""
    import ctypes as C
    m = meshgen.baseline_config(name, scale)
    engine.set_mesh(m)
    engine.build_edges()
    engine.navs(DF, GATHER)
    rng = np.random.default_rng(5)
    x2 = m.coords + rng.uniform(-1e-3, 1e-3, m.coords.size) * (m.coords > 0) * (m.coords < 1)
    m2 = Mesh(m.dim, x2, m.elements, m.boundary)
    engine.set_coords(x2)
    engine.navs(DF, GATHER)
    engine.volumes(EDGE)
    e, o = oracle.build_edges(m2)
    want = oracle.navs_dualfree(m2, e, o)
    got = engine.get_navs()
    assert per_vector_rel(got, want, m.dim) <= 1e-12
    np.testing.assert_array_equal(engine.get_volumes(), oracle.volumes_edge(m2, e, got))
    navs = np.empty_like(got)
    vols = np.empty(m.num_nodes())
    p = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
    engine.metrics_host(p(np.ascontiguousarray(x2)), DF, GATHER, EDGE, p(navs), p(vols))
    np.testing.assert_array_equal(navs, got)
    np.testing.assert_array_equal(vols, engine.get_volumes())


@pytest.mark.parametrize("name,scale", [("C2", 1), ("C3", 4)])
def test_pipelined_host_steps(engine, name, scale):
    """dm_metrics_host_async: a loop of steps over changing coordinates, each
    enqueued before the previous one's copy-out finished (two device output
    buffers, copy streams), gives per step exactly the fields of the
    synchronous calls on the same coordinates."""
    import ctypes as C
    m = meshgen.baseline_config(name, scale)
    engine.set_mesh(m)
    engine.build_edges()
    rng = np.random.default_rng(11)
    inner = (m.coords > 0) * (m.coords < 1)
    xs = [m.coords + rng.uniform(-2e-3, 2e-3, m.coords.size) * inner for _ in range(5)]
    nd, nn = m.dim * engine.n_edges, m.num_nodes()
    lib = _lib.capi()
    bufs = []

    def pinned(n):
        p = C.c_void_p()
        assert lib.dm_host_alloc(8 * n, C.byref(p)) == 0
        bufs.append(p)
        return np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_double)), shape=(n,))

    dp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
    try:
        hx = [pinned(m.coords.size) for _ in xs]
        hn = [pinned(nd) for _ in xs]
        hv = [pinned(nn) for _ in xs]
        for h, x in zip(hx, xs):
            h[:] = x
        for i in range(len(xs)):
            engine.metrics_host_async(dp(hx[i]), DF, GATHER, EDGE, dp(hn[i]), dp(hv[i]))
        engine.sync()
        for i, x in enumerate(xs):
            engine.set_coords(x)
            engine.navs(DF, GATHER)
            engine.volumes(EDGE)
            np.testing.assert_array_equal(hn[i], engine.get_navs())
            np.testing.assert_array_equal(hv[i], engine.get_volumes())
        # the synchronous call after the pipelined ones sees the last step
        out_n, out_v = np.empty(nd), np.empty(nn)
        engine.metrics_host(dp(hx[2]), DF, GATHER, EDGE, dp(out_n), dp(out_v))
        np.testing.assert_array_equal(out_n, hn[2])
        np.testing.assert_array_equal(out_v, hv[2])
    finally:
        for p in bufs:
            lib.dm_host_free(p)


def test_async_step_after_unsynced_calls(engine):
    """dm_navs / dm_volumes (and a dm_set_coords copy) still queued on the
    compute stream, then dm_metrics_host_async with other coordinates and no
    sync in between: the copy-in must wait for them, so both the
    earlier fields and the async step equal their synchronous counterparts."""
    import ctypes as C
    m = meshgen.baseline_config("C2", 1)
    engine.set_mesh(m)
    engine.build_edges()
    rng = np.random.default_rng(5)
    inner = (m.coords > 0) * (m.coords < 1)
    xa = m.coords + rng.uniform(-2e-3, 2e-3, m.coords.size) * inner
    xb = m.coords + rng.uniform(-2e-3, 2e-3, m.coords.size) * inner
    nd, nn = m.dim * engine.n_edges, m.num_nodes()
    # references, synchronous
    engine.set_coords(xa)
    engine.navs(DF, GATHER)
    engine.volumes(EDGE)
    ref_a = (engine.get_navs(), engine.get_volumes())
    engine.set_coords(xb)
    engine.navs(DF, GATHER)
    engine.volumes(EDGE)
    ref_b = (engine.get_navs(), engine.get_volumes())
    lib = _lib.capi()
    ps = [C.c_void_p() for _ in range(3)]
    for p, n in zip(ps, (m.coords.size, nd, nn)):
        assert lib.dm_host_alloc(8 * n, C.byref(p)) == 0
    try:
        arr = [np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_double)), shape=(n,))
               for p, n in zip(ps, (m.coords.size, nd, nn))]
        arr[0][:] = xb
        dp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
        for _ in range(3):
            engine.set_coords(xa)          # queued copy on the compute stream
            engine.navs(DF, GATHER)        # queued kernels reading xa
            engine.volumes(EDGE)
            engine.metrics_host_async(dp(arr[0]), DF, GATHER, EDGE, dp(arr[1]), dp(arr[2]))
            engine.sync()
            np.testing.assert_array_equal(arr[1], ref_b[0])
            np.testing.assert_array_equal(arr[2], ref_b[1])
        # the first dm_navs of the loop computed on xa: check it via a rerun
        engine.set_coords(xa)
        engine.navs(DF, GATHER)
        engine.volumes(EDGE)
        np.testing.assert_array_equal(engine.get_navs(), ref_a[0])
        np.testing.assert_array_equal(engine.get_volumes(), ref_a[1])
    finally:
        for p in ps:
            lib.dm_host_free(p)


def test_step_timing_ring(engine):
    """dm_set_timing(enable > 1) keeps the phase events of the last steps, so a run of
    back-to-back steps is timed without synchronising inside it (bench.py)."""
    m = meshgen.tet_cube(12, amp=0.15)
    engine.set_mesh(m)
    engine.build_edges()
    DF, G, E = _lib.DM_NAV_DUALFREE, _lib.DM_VARIANT_GATHER, _lib.DM_VOL_EDGE
    engine.navs(DF, G)
    engine.volumes(E)
    want = engine.get_navs().copy()
    engine.set_step_timing(3)
    assert engine.step_timings(8).shape == (0, 4)
    for _ in range(5):
        engine.navs(DF, G)
        engine.volumes(E)
    t = engine.step_timings(8)
    assert t.shape == (3, 4)  # the newest three of five
    assert (t > 0).all() and (t[:, 3] >= t[:, :3].sum(axis=1) * 0.99).all(), t
    assert engine.step_timings(2).shape == (2, 4)
    engine.set_timing(True)  # back to the single-slot form
    engine.navs(DF, G)
    engine.volumes(E)
    assert len(engine.timings()) == 4
    with pytest.raises(Exception):
        engine.step_timings(2)
    engine.set_timing(False)
    assert np.array_equal(engine.get_navs(), want)


def test_set_coords_checks_length(engine):
    m = meshgen.baseline_config("C2", 8)
    engine.set_mesh(m)
    with pytest.raises(ValueError):
        engine.set_coords(m.coords[:-1])


@pytest.mark.parametrize("name,scale", [("C2", 1), ("C3", 4), ("C5", 2)])
def test_colored_plan_same_bits(name, scale, monkeypatch):
    """The opt-in bank-conflict colouring only relabels table slots: navs
    and volumes are bitwise those of the uncoloured plan."""
    from paper_2502_00778_b200 import Engine
    m = meshgen.baseline_config(name, scale)
    out = []
    monkeypatch.setenv("DUALMESH_ROW_PLAN", "0")  # the colouring is a Morton-tile pass
    for flag in ("0", "1"):
        monkeypatch.setenv("DUALMESH_PLAN_COLOR", flag)
        eng = Engine(0)
        try:
            eng.set_mesh(m)
            eng.build_edges()
            eng.navs(DF, GATHER)
            eng.volumes(EDGE)
            assert eng.plan_info()["colored"] == (flag == "1")
            out.append((eng.get_navs(), eng.get_volumes()))
        finally:
            eng.close()
    np.testing.assert_array_equal(out[0][0], out[1][0])
    np.testing.assert_array_equal(out[0][1], out[1][1])


@pytest.mark.parametrize("name,scale", [("C2", 1), ("C4", 4)])
def test_ring_global_path_same_bits(name, scale, monkeypatch):
    """Tiles whose table or codes exceed the ring kernel's shared buffers are
    evaluated from global memory by the same kernel: forcing every tile down
    that path (DUALMESH_GATHER_CFG=41, a 16-code buffer) gives the same bits."""
    from paper_2502_00778_b200 import Engine
    m = meshgen.baseline_config(name, scale)
    out = []
    monkeypatch.setenv("DUALMESH_ROW_PLAN", "0")  # the global-memory path is the Morton kernel's
    for cfg in ("0", "41"):
        monkeypatch.setenv("DUALMESH_GATHER_CFG", cfg)
        eng = Engine(0)
        try:
            eng.set_mesh(m)
            eng.build_edges()
            eng.navs(DF, GATHER)
            eng.volumes(EDGE)
            assert eng.plan_info()["ring_ok"]
            out.append((eng.get_navs(), eng.get_volumes()))
        finally:
            eng.close()
    np.testing.assert_array_equal(out[0][0], out[1][0])
    np.testing.assert_array_equal(out[0][1], out[1][1])


def test_ring_pipeline_repeatable():
    """The asynchronous ring pipeline (three shared buffers, mbarrier
    phases, persistent CTAs) gives the same bits on every repetition, on a
    randomly numbered grid and on the boundary-layer grid."""
    from paper_2502_00778_b200 import Engine
    for name in ("C3", "C4"):
        eng = Engine(0)
        try:
            eng.set_mesh(meshgen.baseline_config(name, 2))
            eng.build_edges()
            eng.navs(DF, GATHER)
            eng.volumes(EDGE)
            n0, v0 = eng.get_navs(), eng.get_volumes()
            for _ in range(12):
                eng.navs(DF, GATHER)
                eng.volumes(EDGE)
                np.testing.assert_array_equal(eng.get_navs(), n0)
                np.testing.assert_array_equal(eng.get_volumes(), v0)
        finally:
            eng.close()


def test_twice_c5_scale():
    """A 320^3 Kuhn cube (196.6 M tets, 230 M edges; device-generated): the
    ring plan (codes beyond 2 GB, coloured 256-node tables) and the SPEC
    identities at twice the BASELINE size."""
    from paper_2502_00778_b200 import Engine
    eng = Engine(0)
    try:
        eng.gen_tet_box(320, 320, 320, None, 0, 0.15, 42)
        assert eng.build_edges() == 230298560
        eng.navs(DF, GATHER)
        eng.volumes(EDGE)
        info = eng.plan_info()
        assert info["ring_ok"] and info["tiles"] == "row"
        r, ri = eng.check_closure()
        assert r <= 1e-13 and ri <= 1e-13
        rel, sv, _ = eng.check_total_volume()
        assert rel <= 1e-12 and abs(sv - 1.0) <= 1e-12
        A = np.array([[0.3, 0.1, 0.0], [0.0, 0.5, 0.2], [0.1, 0.0, 0.4]])
        assert eng.check_linear_exactness(A, np.array([0.1, -0.2, 0.3])) <= 1e-11
    finally:
        eng.close()


def test_largest_supported_scale_and_the_limit():
    """384^3 (339.7 M tets, 397.7 M edges: L * N_E = 2.04e9, just under the 2^31 items of the
    device layout; ~86 GB on the device) runs the default path with the SPEC identities; 400^3
    is refused with DM_ERR_UNSUPPORTED, not a fault."""
    from paper_2502_00778_b200 import DualMeshError, Engine
    eng = Engine(0)
    try:
        eng.gen_tet_box(384, 384, 384, None, 0, 0.15, 42)
        assert eng.build_edges() == 397689984
        eng.navs(DF, GATHER)
        eng.volumes(EDGE)
        assert eng.plan_info()["ring_ok"] and eng.plan_info()["tiles"] == "row"
        r, ri = eng.check_closure()
        assert r <= 1e-13 and ri <= 1e-13
        rel, sv, _ = eng.check_total_volume()
        assert rel <= 1e-12 and abs(sv - 1.0) <= 1e-12
    finally:
        eng.close()
    eng = Engine(0)
    try:
        eng.gen_tet_box(400, 400, 400, None, 0, 0.15, 42)
        with pytest.raises(DualMeshError) as ei:
            eng.build_edges()
        assert "32-bit item space" in str(ei.value)
        # the context is still usable
        eng.gen_tet_box(8, 8, 8, None, 0, 0.15, 42)
        assert eng.build_edges() > 0
    finally:
        eng.close()


@pytest.mark.parametrize("name,scale", [("C2", 1), ("C4", 4), ("C5", 2), ("C3", 4)])
def test_row_and_morton_plans_same_bits(name, scale, monkeypatch, oracle):
    """Both tilings of the ring walk (rowplan.cu row tiles, rings.cu Morton
    tiles) walk every ring from the same start in the same direction with the
    same arithmetic: navs, s terms and volumes are bitwise identical, and within
    1e-12 per edge vector of the serial oracle.  Randomly numbered grids (C3)
    must fall back to the Morton tiles."""
    from paper_2502_00778_b200 import Engine
    m = meshgen.baseline_config(name, scale)
    out, kinds = [], []
    for flag in ("1", "0"):
        monkeypatch.setenv("DUALMESH_ROW_PLAN", flag)
        eng = Engine(0)
        try:
            eng.set_mesh(m)
            eng.build_edges()
            eng.navs(DF, GATHER)
            eng.volumes(EDGE)
            kinds.append(eng.plan_info()["tiles"])
            n, v = eng.get_navs(), eng.get_volumes()
            eng.navs(TR, GATHER)
            out.append((n, v, eng.get_navs()))
        finally:
            eng.close()
    assert kinds[1] == "morton"
    assert kinds[0] == ("morton" if name == "C3" else "row")
    for a, b in zip(out[0], out[1]):
        np.testing.assert_array_equal(a, b)
    e, o = oracle.build_edges(m)
    want = oracle.navs_dualfree(m, e, o)
    assert per_vector_rel(out[0][0], want, 3) <= 1e-12


@pytest.mark.parametrize("name,scale,flag", [("C3", 4, "1"), ("C2", 2, "1"), ("C2", 2, "0")])
def test_side_list_inside_grid(name, scale, flag, monkeypatch, oracle):
    """One 30-tet fan beside a BASELINE grid (meshgen.fan_in): only its hub
    edge leaves the ring codes (side list, evaluated in element order inside
    the same step -- that row bitwise the serial oracle's); every other edge
    stays on the ring path (row tiles, or Morton tiles for the randomly
    numbered C3 / with DUALMESH_ROW_PLAN=0)."""
    from paper_2502_00778_b200 import Engine
    monkeypatch.setenv("DUALMESH_ROW_PLAN", flag)
    m = meshgen.fan_in(meshgen.baseline_config(name, scale), 30)
    eng = Engine(0)
    try:
        eng.set_mesh(m)
        eng.build_edges()
        eng.navs(DF, GATHER)
        info = eng.plan_info()
        assert info["ring_ok"] and eng.side_edges() == 1 and info["ring_fail_bits"] & 4
        assert info["tiles"] == ("row" if flag == "1" and name != "C3" else "morton")
        e, o = oracle.build_edges(m)
        want = oracle.navs_dualfree(m, e, o)
        got = eng.get_navs()
        assert per_vector_rel(got, want, 3) <= 1e-12
        hub = int(np.argmax(np.diff(oracle.edge_maps(m, e, o)[1])))
        np.testing.assert_array_equal(got.reshape(-1, 3)[hub], want.reshape(-1, 3)[hub])
        eng.volumes(EDGE)
        vw = oracle.volumes_edge(m, e, want)
        assert np.abs(eng.get_volumes() - vw).max() <= 1e-12 * np.abs(vw).max()
        r, _ = eng.check_closure()
        assert r <= 1e-13
        eng.navs(TR, GATHER)
        assert per_vector_rel(eng.get_navs(), oracle.navs_traditional(m, e, o), 3) <= 1e-12
    finally:
        eng.close()


@pytest.mark.parametrize("permuted", [False, True])
def test_flipped_unstructured_grid(engine, oracle, permuted):
    """Non-Kuhn topology (meshgen.flip23: seeded 2-3 flips of C2, ring
    lengths 1..11): the ring path (row tiles; Morton tiles when the numbering
    is permuted) within 1e-12 of the oracle, the exact variant bitwise, the
    SPEC identities."""
    m = meshgen.flip23(meshgen.baseline_config("C2", 2), 0.3)
    if permuted:
        m = meshgen.permute(m)
    engine.set_mesh(m)
    engine.build_edges()
    engine.navs(DF, GATHER)
    info = engine.plan_info()
    # a permuted numbering has no id locality: Morton tiles; otherwise either
    # tiling, by the row plan's split budget
    assert info["ring_ok"] and (info["tiles"] == "morton" if permuted else info["tiles"])
    e, o = oracle.build_edges(m)
    want = oracle.navs_dualfree(m, e, o)
    assert per_vector_rel(engine.get_navs(), want, 3) <= 1e-12
    engine.volumes(EDGE)
    vw = oracle.volumes_edge(m, e, want)
    assert np.abs(engine.get_volumes() - vw).max() <= 1e-12 * np.abs(vw).max()
    r, ri = engine.check_closure()
    assert r <= 1e-13 and ri <= 1e-13
    rel, sv, _ = engine.check_total_volume()
    assert rel <= 1e-12 and abs(sv - 1.0) <= 1e-12
    engine.navs(DF, EXACT)
    np.testing.assert_array_equal(engine.get_navs(), want)
    engine.navs(TR, GATHER)
    assert per_vector_rel(engine.get_navs(), oracle.navs_traditional(m, e, o), 3) <= 1e-12


def test_row_plan_wide_span_hash_path(monkeypatch, oracle):
    """Row tiles whose node-pair span exceeds the builder's bitmap (131072
    pairs) take its hash-set path: a Kuhn grid whose upper half of node ids
    is shifted past 300000 unused ids (isolated nodes) keeps its topology and
    id order, so its navs are bitwise those of the unshifted grid (the ring
    encodings, fixed by the element list, are the same), and the plan audit
    (DUALMESH_PLAN_CHECK=1) accepts the tiles."""
    from paper_2502_00778_b200 import Engine
    m = meshgen.tet_cube(24, amp=0.15)
    nv = m.num_nodes()
    gap, half = 300_000, nv // 2
    newid = np.arange(nv, dtype=np.int64)
    newid[half:] += gap
    coords = np.zeros((nv + gap, 3))
    coords[newid] = m.coords.reshape(-1, 3)
    coords[half:half + gap] = 5.0  # isolated nodes, away from the grid
    ms = Mesh(3, coords.ravel(), newid[m.elements].astype(np.int32),
              newid[m.boundary].astype(np.int32))
    monkeypatch.setenv("DUALMESH_PLAN_CHECK", "1")
    out = []
    for mesh in (m, ms):
        eng = Engine(0)
        try:
            eng.set_mesh(mesh)
            eng.build_edges()
            eng.navs(DF, GATHER)
            assert eng.plan_info()["tiles"] == "row"
            out.append(eng.get_navs())
        finally:
            eng.close()
    np.testing.assert_array_equal(out[0], out[1])
    e, o = oracle.build_edges(ms)
    assert per_vector_rel(out[1], oracle.navs_dualfree(ms, e, o), 3) <= 1e-12
