"""CPU tests: pin the oracle against the reference's own code and the SPEC
examples, and check the SPEC identities on the oracle (no GPU needed)."""
from fractions import Fraction as F

import numpy as np
import pytest

from paper_2502_00778_b200 import Mesh, meshgen
from oracle.oracle import RefMesh, ref_available


def rows(navs, dim):
    return navs.reshape(-1, dim)


def edge_index(edges, a, b):
    a, b = min(a, b), max(a, b)
    hit = np.nonzero((edges[:, 0] == a) & (edges[:, 1] == b))[0]
    return int(hit[0]) if hit.size else -1


# ----------------------------------------------------------------- SPEC examples
def test_ftri_spec_examples(fixtures, oracle):
    m = fixtures["F-TRI"]["mesh_obj"]
    e, o = oracle.build_edges(m)
    assert e.tolist() == [[0, 1], [0, 2], [1, 2]]  # SPEC.md:67 (1-based (1,2),(1,3),(2,3))
    for algo in (oracle.navs_dualfree, oracle.navs_traditional):
        n = rows(algo(m, e, o), 2)
        np.testing.assert_allclose(n[0], [1 / 3, 1 / 6], atol=1e-15)
        np.testing.assert_allclose(n[1], [1 / 6, 1 / 3], atol=1e-15)
        np.testing.assert_allclose(n[2], [-1 / 6, 1 / 6], atol=1e-15)
        v = oracle.volumes_edge(m, e, algo(m, e, o))
        np.testing.assert_allclose(v, [1 / 6] * 3, atol=1e-15)
    np.testing.assert_allclose(oracle.volumes_element(m), [1 / 6] * 3, atol=1e-15)
    # normals
    np.testing.assert_array_equal(oracle.opposite_face_normal(m, 0, 0), [1, 1, 0])
    np.testing.assert_array_equal(oracle.boundary_normal(m, 0), [0, -1, 0])


def test_ftet_spec_examples(fixtures, oracle):
    m = fixtures["F-TET"]["mesh_obj"]
    e, o = oracle.build_edges(m)
    assert e.tolist() == [[0, 1], [0, 2], [0, 3], [1, 2], [1, 3], [2, 3]]
    want = {(0, 1): (2, 1, 1), (0, 2): (1, 2, 1), (0, 3): (1, 1, 2), (1, 2): (-1, 1, 0),
            (1, 3): (-1, 0, 1), (2, 3): (0, -1, 1)}  # x 1/24, SURVEY.md §4 golden table
    for algo in (oracle.navs_dualfree, oracle.navs_traditional):
        n = rows(algo(m, e, o), 3)
        for (a, b), w in want.items():
            np.testing.assert_allclose(n[edge_index(e, a, b)], np.array(w) / 24, atol=1e-15)
        np.testing.assert_allclose(oracle.volumes_edge(m, e, algo(m, e, o)), [1 / 24] * 4,
                                   atol=1e-15)
    np.testing.assert_allclose(oracle.volumes_element(m), [1 / 24] * 4, atol=1e-15)
    np.testing.assert_array_equal(oracle.opposite_face_normal(m, 0, 0), [0.5, 0.5, 0.5])
    np.testing.assert_array_equal(oracle.boundary_normal(m, 0), [0, 0, -0.5])
    np.testing.assert_array_equal(oracle.boundary_normal(m, 3), [0.5, 0.5, 0.5])


def test_fsquare_spec_examples(fixtures, oracle):
    m = fixtures["F-square"]["mesh_obj"]
    e, o = oracle.build_edges(m)
    np.testing.assert_allclose(oracle.volumes_element(m), [1 / 6, 1 / 3, 1 / 3, 1 / 6],
                               atol=1e-15)
    n = oracle.navs_dualfree(m, e, o)
    np.testing.assert_allclose(oracle.volumes_edge(m, e, n), [1 / 6, 1 / 3, 1 / 3, 1 / 6],
                               atol=1e-15)
    np.testing.assert_allclose(rows(n, 2)[edge_index(e, 1, 2)], [-1 / 3, 1 / 3], atol=1e-15)


def test_kuhn1_golden(fixtures, oracle):
    m = fixtures["Kuhn1"]["mesh_obj"]
    e, o = oracle.build_edges(m)
    assert len(e) == 19
    n = rows(oracle.navs_dualfree(m, e, o), 3)
    np.testing.assert_allclose(n[edge_index(e, 0, 7)], [1 / 6] * 3, atol=1e-15)
    np.testing.assert_allclose(n[edge_index(e, 0, 1)], [1 / 6, -1 / 24, -1 / 24], atol=1e-15)
    np.testing.assert_allclose(n[edge_index(e, 0, 3)], [1 / 12, 1 / 12, -1 / 12], atol=1e-15)
    np.testing.assert_allclose(n[edge_index(e, 1, 3)], [-1 / 24, 1 / 12, -1 / 24], atol=1e-15)
    v = oracle.volumes_edge(m, e, n.ravel())
    np.testing.assert_allclose(v, [1 / 4] + [1 / 12] * 6 + [1 / 4], atol=1e-15)


def test_fixture_closure_exact(fixtures, oracle):
    for d in fixtures.values():
        m = d["mesh_obj"]
        e, o = oracle.build_edges(m)
        n = oracle.navs_dualfree(m, e, o)
        r, ri = oracle.check_closure(m, e, n)
        # exactly 0 in rational arithmetic; fp64 leaves rounding only
        assert r <= 1e-15 and ri <= 1e-15


# ----------------------------------------------------------------- pinned to the reference code
def test_oracle_geometry_matches_reference(fixtures, oracle):
    for d in fixtures.values():
        m = d["mesh_obj"]
        for el in range(m.num_elements()):
            assert oracle.element_volume(m, el) == d["ref_element_volume"][el]
            for i in range(m.dim + 1):
                np.testing.assert_array_equal(oracle.opposite_face_normal(m, el, i),
                                              d["ref_opposite_face_normal"][el][i])
        for b in range(m.num_boundary()):
            np.testing.assert_array_equal(oracle.boundary_normal(m, b), d["ref_boundary_normal"][b])


def test_oracle_edges_match_reference_fixtures(fixtures, oracle):
    for d in fixtures.values():
        e, o = oracle.build_edges(d["mesh_obj"])
        assert e.tolist() == d["ref_edges"]
        assert o.tolist() == d["ref_origin_start"]
        assert d["ref_validate"] == []


def test_oracle_edges_match_reference_golden_configs(golden_configs, oracle):
    for name, g in golden_configs.items():
        e, o = oracle.build_edges(g["mesh"])
        np.testing.assert_array_equal(e, g["edges"], err_msg=name)
        np.testing.assert_array_equal(o, g["origin_start"], err_msg=name)
        e2l, ip, inc = oracle.edge_maps(g["mesh"], e, o)
        np.testing.assert_array_equal(e2l, g["e2l"])
        np.testing.assert_array_equal(ip, g["inc_ptr"])
        np.testing.assert_array_equal(inc, g["inc"])


def test_oracle_reproduces_golden_fields(golden_configs, oracle):
    """Bit-for-bit regression pin of the committed oracle outputs."""
    for name, g in golden_configs.items():
        m, e, o = g["mesh"], g["edges"], g["origin_start"]
        np.testing.assert_array_equal(oracle.navs_dualfree(m, e, o), g["navs_dualfree"])
        np.testing.assert_array_equal(oracle.navs_traditional(m, e, o), g["navs_traditional"])
        np.testing.assert_array_equal(oracle.volumes_edge(m, e, g["navs_dualfree"]), g["vol_edge"])
        np.testing.assert_array_equal(oracle.volumes_element(m), g["vol_element"])


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("name,scale", [("C1", 2), ("C2", 4), ("C3", 8), ("C4", 8)])
def test_oracle_edges_match_reference_live(oracle, name, scale):
    m = meshgen.baseline_config(name, scale)
    e, o = oracle.build_edges(m)
    e2, o2 = RefMesh(m).build_edges()
    np.testing.assert_array_equal(e, e2)
    np.testing.assert_array_equal(o, o2)


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")
def test_reference_edges_reorder_invariant():
    """build_edges is invariant under element reordering."""
    m = meshgen.tet_cube(6, amp=0.15)
    p = meshgen.permute(m, node_seed=0, elem_seed=7)
    e1, o1 = RefMesh(m).build_edges()
    e2, o2 = RefMesh(p).build_edges()
    np.testing.assert_array_equal(e1, e2)
    np.testing.assert_array_equal(o1, o2)


# ----------------------------------------------------------------- SPEC identities on the oracle
@pytest.mark.parametrize("mesh_fn", [
    lambda: meshgen.tri_square(64, amp=0.2, seed=42),        # SPEC.md:475 acceptance 2
    lambda: meshgen.tet_cube(16, amp=0.2, seed=42),
    lambda: meshgen.baseline_config("C1", 4),
    lambda: meshgen.baseline_config("C4", 8),
])
def test_spec_identities(oracle, mesh_fn):
    m = mesh_fn()
    e, o = oracle.build_edges(m)
    nd = oracle.navs_dualfree(m, e, o)
    nt = oracle.navs_traditional(m, e, o)
    scale = oracle.max_face_area(m)
    assert np.abs(nd - nt).max() <= 1e-13 * scale
    r, ri = oracle.check_closure(m, e, nd)
    assert r <= 1e-13 and ri <= 1e-13
    ve = oracle.volumes_edge(m, e, nd)
    vl = oracle.volumes_element(m)
    assert np.abs(ve - vl).max() <= 1e-13 * oracle.max_element_volume(m)
    rel, sv, se = oracle.check_total_volume(m, ve)
    assert rel <= 1e-12
    # orientation identity: n_e.(x_k - x_j) = 2/(D+1) * sum of incident V_E
    D = m.dim
    x = m.coords.reshape(-1, D)
    dots = np.einsum("ij,ij->i", rows(nd, D), x[e[:, 1]] - x[e[:, 0]])
    e2l, ip, inc = oracle.edge_maps(m, e, o)
    vE = np.array([oracle.element_volume(m, q) for q in range(m.num_elements())])
    want = 2.0 / (D + 1) * np.add.reduceat(vE[inc], ip[:-1])
    assert np.abs(dots - want).max() <= 1e-13 * np.abs(want).max()


def test_corrupted_nav_is_detected(oracle):
    """corrupting one nav by 1e-3 gives residual >= 1e-4."""
    m = meshgen.tet_cube(8, amp=0.2, seed=42)
    e, o = oracle.build_edges(m)
    n = oracle.navs_dualfree(m, e, o)
    n[3 * 17:3 * 17 + 3] += 1e-3
    assert oracle.check_closure(m, e, n)[0] >= 1e-4


def test_unit_domain_total_volume(oracle):
    """SPEC.md:262-263 / acceptance 4: sum V_j = 1 on unit square / cube."""
    for m in (meshgen.tri_square(32, amp=0.2), meshgen.tet_cube(12, amp=0.15)):
        e, o = oracle.build_edges(m)
        v = oracle.volumes_edge(m, e, oracle.navs_dualfree(m, e, o))
        assert abs(np.sum(np.sort(v)) - 1.0) <= 1e-12
        assert abs(np.sum(np.sort(oracle.volumes_element(m))) - 1.0) <= 1e-12


@pytest.mark.parametrize("mesh_fn", [
    lambda: meshgen.tri_square(24, amp=0.2, seed=42),
    lambda: meshgen.tet_cube(10, amp=0.15),
    lambda: meshgen.baseline_config("C3", 16),
    lambda: meshgen.baseline_config("C4", 16),
])
@pytest.mark.parametrize("threads", [1, 4])
def test_threaded_oracle_is_bitwise_serial(oracle, mesh_fn, threads):
    """The bench reference arm's threaded gathers reproduce the serial loops
    bit for bit (same terms, same order) on any thread count."""
    m = mesh_fn()
    e, o = oracle.build_edges(m)
    nd = oracle.navs_dualfree(m, e, o)
    ve = oracle.volumes_edge(m, e, nd)
    plan = oracle.plan(m, e, o)
    try:
        nt, vt = oracle.metrics_mt(plan, m.coords, threads)
    finally:
        oracle.plan_free(plan)
    np.testing.assert_array_equal(nt, nd)
    np.testing.assert_array_equal(vt, ve)


def _affine(dim, seed):
    rng = np.random.default_rng(seed)
    A = rng.uniform(-1.0, 1.0, (dim, dim))
    if abs(np.trace(A)) < 0.1:
        A[0, 0] += 1.0
    return A, rng.uniform(-1.0, 1.0, dim)


@pytest.mark.parametrize("mesh_fn,tol", [
    (lambda: meshgen.tri_square(32, amp=0.2, seed=42), 1e-11),   # SPEC.md:271 example 2
    (lambda: meshgen.tet_cube(10, amp=0.15), 1e-11),
    # BL grid (dz0 = 1e-5, z up to 53): |F||n| / (V tr) ~ 1e5, so rounding
    # alone reaches ~1e-10 (tolerances are configuration)
    (lambda: meshgen.baseline_config("C4", 16), 1e-9),
])
def test_linear_exactness_spec_examples(oracle, mesh_fn, tol):
    """F = x/D gives Res_j/V_j = 1 at interior nodes; a seeded
    random affine flux gives <= 1e-11; a constant flux balances to <= 1e-13
    at all nodes with the boundary closure; trace(A) = 0 is rejected."""
    m = mesh_fn()
    D = m.dim
    e, o = oracle.build_edges(m)
    n = oracle.navs_dualfree(m, e, o)
    v = oracle.volumes_edge(m, e, n)
    assert oracle.check_linear_exactness(m, e, n, v, np.eye(D) / D, np.zeros(D)) <= tol
    A, b = _affine(D, 7)
    assert oracle.check_linear_exactness(m, e, n, v, A, b) <= tol
    assert oracle.check_linear_exactness(m, e, n, v, np.zeros((D, D)), b) <= 1e-13
    with pytest.raises(ValueError):
        oracle.check_linear_exactness(m, e, n, v, np.diag([1.0, -1.0] + [0.0] * (D - 2)), b)
    # a corrupted nav of an interior edge breaks exactness
    isb = np.zeros(m.num_nodes(), bool)
    isb[m.boundary] = True
    q = int(np.nonzero(~isb[e[:, 0]] & ~isb[e[:, 1]])[0][0])
    n2 = n.copy()
    n2[D * q:D * q + D] += 1e-3
    assert oracle.check_linear_exactness(m, e, n2, v, A, b) > 1e3 * tol


@pytest.mark.parametrize("n", [1, 2, 5, 16])
def test_oracle_generator_equals_product_generator(oracle, n):
    """The bench's CPU legs generate their grid with the oracle's own
    generator (or_gen_tet_cube); it must be bitwise the grid the GPU arm
    times (BASELINE C2/C5 family)."""
    from paper_2502_00778_b200 import meshgen
    a = oracle.gen_tet_cube(n, amp=0.15, seed=42)
    b = meshgen.tet_cube(n, amp=0.15)
    assert np.array_equal(a.coords, b.coords)
    assert np.array_equal(a.elements, b.elements)
    assert np.array_equal(a.boundary, b.boundary)
    assert oracle.max_element_volume(a) > 0


def test_flip23_generator_is_valid(oracle):
    """meshgen.flip23: a conforming, positively oriented non-Kuhn grid (the
    reference's own validate_mesh when oracle/_ref is built), with ring
    lengths spread well beyond the Kuhn 4 / 6, exact closure and volume."""
    m = meshgen.flip23(meshgen.tet_cube(8, amp=0.15), 0.3)
    assert m.num_elements() > 6 * 8 ** 3
    assert meshgen.first_inverted(m) == -1
    if ref_available():
        n, msgs, _ = RefMesh(m).validate()
        assert n == 0, msgs[:3]
    e, o = oracle.build_edges(m)
    ring = np.diff(oracle.edge_maps(m, e, o)[1])
    assert ring.max() >= 8 and (ring == 3).sum() > 0
    nv = oracle.navs_dualfree(m, e, o)
    assert oracle.check_closure(m, e, nv)[0] <= 1e-13
    assert oracle.check_total_volume(m, oracle.volumes_edge(m, e, nv))[0] <= 1e-12


def test_fan_in_is_valid():
    m = meshgen.fan_in(meshgen.tet_cube(4, amp=0.15), 30)
    assert meshgen.first_inverted(m) == -1
    if ref_available():
        n, msgs, _ = RefMesh(m).validate()
        assert n == 0, msgs[:3]
