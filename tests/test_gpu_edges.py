"""K1 edge extraction on origin buckets (csrc/edge_extract.cu) against the
generic item-sort path (csrc/edges.cu, DUALMESH_K1_LEGACY=1), the oracle and
the reference's own build_edges (oracle/_ref, mesh.cpp:256-285).

Every output of north_star (a) is compared bit for bit: the edge list, the
origin CSR, the element->local-edge map and the edge->element incidence.
The topologies exercise the register path (Kuhn, 2D), the wide kernel
(permuted numbering: up to 24 entries per origin), the side path (a 30-tet
fan, 2-3 flips), the repeated-node fallback and the edge-capacity re-run."""
import numpy as np
import pytest

from paper_2502_00778_b200 import Engine, Mesh, meshgen

pytestmark = pytest.mark.gpu


def extract(eng, m):
    eng.set_mesh(m)
    eng.build_edges()
    el = eng.edges()
    ip, inc = eng.incidence()
    return el.edges.copy(), el.origin_start.copy(), eng.e2l().copy(), ip.copy(), inc.copy()


def assert_same(a, b):
    for x, y, what in zip(a, b, ("edges", "origin_start", "e2l", "inc_ptr", "inc")):
        np.testing.assert_array_equal(x, y, err_msg=what)


def grids():
    return {
        "kuhn": meshgen.tet_cube(14, amp=0.15),
        "kuhn_perm": meshgen.permute(meshgen.tet_cube(14, amp=0.15)),
        "fan": meshgen.fan_in(meshgen.tet_cube(10, amp=0.1), 30),
        "flip": meshgen.flip23(meshgen.tet_cube(12, amp=0.1)),
        "flip_perm": meshgen.permute(meshgen.flip23(meshgen.tet_cube(12, amp=0.1))),
        "tri": meshgen.tri_square(40, diag_seed=3, amp=0.2),
        "tri_perm": meshgen.permute(meshgen.tri_square(40, diag_seed=3, amp=0.2)),
        "bl": meshgen.baseline_config("C4", 8),
    }


@pytest.mark.parametrize("name", list(grids()))
def test_buckets_equal_item_sort_and_oracle(engine, oracle, monkeypatch, name):
    m = grids()[name]
    got = extract(engine, m)
    monkeypatch.setenv("DUALMESH_K1_LEGACY", "1")
    legacy = extract(engine, m)
    monkeypatch.delenv("DUALMESH_K1_LEGACY")
    assert_same(got, legacy)
    e, o = oracle.build_edges(m)
    np.testing.assert_array_equal(got[0], e)
    np.testing.assert_array_equal(got[1], o)
    e2l, ip, inc = oracle.edge_maps(m, e, o)
    assert_same(got, (e, o, e2l, ip, inc))


def test_full_size_c3_buckets_equal_item_sort(monkeypatch):
    """Permuted 160^3 grid (wide kernel + side buckets) against the item sort."""
    eng = Engine(0)
    try:
        meshgen.baseline_config_device(eng, "C3")
        eng.build_edges()
        el = eng.edges()
        got = (el.edges.copy(), el.origin_start.copy(), eng.e2l().copy(), *eng.incidence())
        monkeypatch.setenv("DUALMESH_K1_LEGACY", "1")
        eng.build_edges()
        el = eng.edges()
        want = (el.edges.copy(), el.origin_start.copy(), eng.e2l().copy(), *eng.incidence())
        assert_same(got, want)
    finally:
        eng.close()


def test_repeated_node_falls_back_to_reference_pairs(engine, oracle):
    """A repeated node inside an element: the reference packs the (a, a)
    pair (mesh.cpp:260-270); the bucket path hands the mesh to the item
    sort, whose output equals the reference's own build_edges."""
    m = meshgen.tet_cube(3, amp=0.0)
    el = m.elements.reshape(-1, 4).copy()
    el[5, 2] = el[5, 1]
    bad = Mesh(3, m.coords, el.reshape(-1), m.boundary)
    engine.set_mesh(bad)
    engine.build_edges()
    got = engine.edges()
    from oracle.oracle import RefMesh, ref_available
    if ref_available():
        want_e, want_o = RefMesh(bad).build_edges()
    else:
        want_e, want_o = oracle.build_edges(bad)
    np.testing.assert_array_equal(got.edges, want_e)
    np.testing.assert_array_equal(got.origin_start, want_o)
    assert (got.edges[:, 0] == got.edges[:, 1]).any()


def test_out_of_range_node_is_an_error(engine):
    m = meshgen.tet_cube(3, amp=0.0)
    el = m.elements.copy()
    el[7] = m.num_nodes() + 5
    engine.set_mesh(Mesh(3, m.coords, el, m.boundary))
    with pytest.raises(ValueError, match="outside"):  # DM_ERR_INVALID_ARG
        engine.build_edges()


def test_edge_capacity_rerun(monkeypatch, oracle):
    """An edge-count estimate below the real count re-runs P3 at the exact
    size (fresh context: no capacity left over from earlier calls)."""
    monkeypatch.setenv("DUALMESH_K1_EDGE_EST", "16")
    m = meshgen.tet_cube(9, amp=0.1)
    eng = Engine(0)
    try:
        got = extract(eng, m)
    finally:
        eng.close()
    e, o = oracle.build_edges(m)
    e2l, ip, inc = oracle.edge_maps(m, e, o)
    assert_same(got, (e, o, e2l, ip, inc))


def tri_fan(n):
    """n triangles around node 0 (the hub is the smallest id of each: n entries
    in one 2D origin bucket, beyond a row's 23)."""
    th = 2 * np.pi * np.arange(n) / n
    coords = np.concatenate([[0.0, 0.0], np.stack([np.cos(th), np.sin(th)], 1).reshape(-1)])
    el = np.stack([np.zeros(n, np.int32), 1 + np.arange(n), 1 + (np.arange(n) + 1) % n], 1)
    bnd = np.stack([1 + np.arange(n), 1 + (np.arange(n) + 1) % n], 1)
    return Mesh(2, coords.astype(np.float64), el.astype(np.int32).reshape(-1),
                bnd.astype(np.int32).reshape(-1))


@pytest.mark.parametrize("n", [5, 23, 24, 40, 300])
def test_2d_fan_side_path(engine, oracle, monkeypatch, n):
    m = tri_fan(n)
    got = extract(engine, m)
    e, o = oracle.build_edges(m)
    e2l, ip, inc = oracle.edge_maps(m, e, o)
    assert_same(got, (e, o, e2l, ip, inc))
    monkeypatch.setenv("DUALMESH_K1_LEGACY", "1")
    assert_same(got, extract(engine, m))


@pytest.mark.parametrize("dim,nv", [(3, 4), (2, 4), (3, 0), (2, 0)])
def test_mesh_without_elements(engine, oracle, dim, nv):
    """The reference's build_edges accepts a mesh without elements (an empty edge list over
    nv + 1 zero offsets, mesh.cpp:256-285); every entry point follows with empty fields."""
    from paper_2502_00778_b200 import _lib
    m = Mesh(dim, np.arange(dim * nv, dtype=np.float64), np.zeros(0, np.int32))
    got = extract(engine, m)
    e, o = oracle.build_edges(m)
    e2l, ip, inc = oracle.edge_maps(m, e, o)
    assert e.shape == (0, 2) and o.shape == (nv + 1,)
    assert_same(got, (e, o, e2l, ip, inc))
    for algo in (_lib.DM_NAV_DUALFREE, _lib.DM_NAV_TRADITIONAL):
        for var in (_lib.DM_VARIANT_GATHER, _lib.DM_VARIANT_GATHER_EXACT,
                    _lib.DM_VARIANT_SCATTER):
            engine.navs(algo, var)
            assert engine.get_navs().size == 0
            engine.volumes(_lib.DM_VOL_EDGE)
            np.testing.assert_array_equal(engine.get_volumes(), np.zeros(nv))
    engine.volumes(_lib.DM_VOL_ELEMENT)
    np.testing.assert_array_equal(engine.get_volumes(), oracle.volumes_element(m))
    r, _ = engine.check_closure()
    assert r == 0.0
    # and the context still serves a real mesh afterwards
    k = meshgen.tet_cube(4, amp=0.1)
    got = extract(engine, k)
    e, o = oracle.build_edges(k)
    np.testing.assert_array_equal(got[0], e)


def test_buckets_beyond_2_pow_25_nodes(monkeypatch):
    """330^3 (35.9 M nodes > 2^25, 215.6 M tets): the bucket path (its item keys hold the
    node-id span k - j in 25 bits, not the node id) against the item sort -- checksums of every
    output, one array on the host at a time."""
    import zlib

    def sums(legacy):
        if legacy:
            monkeypatch.setenv("DUALMESH_K1_LEGACY", "1")
        eng = Engine(0)
        try:
            eng.gen_tet_box(330, 330, 330, None, 0, 0.15, 42)
            out = [eng.build_edges()]
            el = eng.edges()
            out += [zlib.crc32(el.edges.tobytes()), zlib.crc32(el.origin_start.tobytes())]
            del el
            a = eng.e2l()
            out.append(zlib.crc32(a.tobytes()))
            del a
            ip, inc = eng.incidence()
            out += [zlib.crc32(ip.tobytes()), zlib.crc32(inc.tobytes())]
            return out
        finally:
            eng.close()
            monkeypatch.delenv("DUALMESH_K1_LEGACY", raising=False)

    got = sums(False)
    assert got[0] == 252540090
    assert got == sums(True)


def test_single_element(engine, oracle):
    for m in (Mesh(3, np.array([0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0, 1], np.float64),
                   np.array([0, 1, 2, 3], np.int32), np.zeros(0, np.int32)),
              Mesh(2, np.array([0, 0, 1, 0, 0, 1], np.float64), np.array([2, 0, 1], np.int32),
                   np.zeros(0, np.int32))):
        got = extract(engine, m)
        e, o = oracle.build_edges(m)
        e2l, ip, inc = oracle.edge_maps(m, e, o)
        assert_same(got, (e, o, e2l, ip, inc))
