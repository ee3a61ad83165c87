"""Random simplex soups (seeded): node tuples drawn at random, so rings are non-manifold,
fans are long and most 3D edges leave the ring codes for the side list.  Any simplex list is a
valid input of the reference's build_edges (mesh.cpp:256-285) and of the SPEC loops
(SPEC.md:147-188); every output is compared with the oracle -- edge structures and the
serial-order variants bit for bit, the fast variants within 1e-12 of the largest vector."""
import numpy as np
import pytest

from paper_2502_00778_b200 import Mesh, _lib

pytestmark = pytest.mark.gpu

CASES = [(dim, nv, ne) for dim in (3, 2)
         for nv, ne in ((5, 1), (5, 2), (6, 20), (12, 200), (40, 300), (200, 50), (64, 2000),
                        (3000, 9000))]


def soup(dim, nv, ne, seed):
    rng = np.random.default_rng(seed)
    x = rng.random(dim * nv)
    el = np.stack([rng.permutation(nv)[:dim + 1] for _ in range(ne)]).astype(np.int32)
    return Mesh(dim, x, el.reshape(-1), np.zeros(0, np.int32))


@pytest.mark.parametrize("dim,nv,ne", CASES)
def test_soup_matches_oracle(engine, oracle, dim, nv, ne):
    m = soup(dim, nv, ne, 1000 * dim + nv + ne)
    engine.set_mesh(m)
    engine.build_edges()
    el = engine.edges()
    e, o = oracle.build_edges(m)
    np.testing.assert_array_equal(el.edges, e)
    np.testing.assert_array_equal(el.origin_start, o)
    e2l, ip, inc = oracle.edge_maps(m, e, o)
    gip, ginc = engine.incidence()
    np.testing.assert_array_equal(engine.e2l(), e2l)
    np.testing.assert_array_equal(gip, ip)
    np.testing.assert_array_equal(ginc, inc)
    want = oracle.navs_dualfree(m, e, o, e2l)
    engine.navs(_lib.DM_NAV_DUALFREE, _lib.DM_VARIANT_GATHER_EXACT)
    np.testing.assert_array_equal(engine.get_navs(), want)
    engine.volumes(_lib.DM_VOL_EDGE)
    np.testing.assert_array_equal(engine.get_volumes(), oracle.volumes_edge(m, e, want))
    tol = 1e-12  # fp64: other summation orders, relative to the largest vector
    big = max(np.abs(want).max(), 1e-300)
    for var in (_lib.DM_VARIANT_GATHER, _lib.DM_VARIANT_SCATTER, _lib.DM_VARIANT_GATHER_ELEM,
                _lib.DM_VARIANT_GATHER_FACES):
        engine.navs(_lib.DM_NAV_DUALFREE, var)
        assert np.abs(engine.get_navs() - want).max() / big <= tol, var
    wt = oracle.navs_traditional(m, e, o, e2l)
    engine.navs(_lib.DM_NAV_TRADITIONAL, _lib.DM_VARIANT_GATHER)
    assert np.abs(engine.get_navs() - wt).max() / max(np.abs(wt).max(), 1e-300) <= tol
    engine.volumes(_lib.DM_VOL_ELEMENT)
    np.testing.assert_array_equal(engine.get_volumes(), oracle.volumes_element(m))


def _check_against_oracle(engine, oracle, m):
    engine.set_mesh(m)
    engine.build_edges()
    el = engine.edges()
    e, o = oracle.build_edges(m)
    np.testing.assert_array_equal(el.edges, e)
    np.testing.assert_array_equal(el.origin_start, o)
    e2l, ip, inc = oracle.edge_maps(m, e, o)
    np.testing.assert_array_equal(engine.e2l(), e2l)
    want = oracle.navs_dualfree(m, e, o, e2l)
    engine.navs(_lib.DM_NAV_DUALFREE, _lib.DM_VARIANT_GATHER)
    assert np.abs(engine.get_navs() - want).max() / np.abs(want).max() <= 1e-12
    engine.volumes(_lib.DM_VOL_EDGE)
    wv = oracle.volumes_edge(m, e, want)
    assert np.abs(engine.get_volumes() - wv).max() <= 1e-12 * np.abs(wv).max()
    engine.volumes(_lib.DM_VOL_ELEMENT)
    np.testing.assert_array_equal(engine.get_volumes(), oracle.volumes_element(m))


def test_isolated_nodes(engine, oracle):
    """Node ids no element uses (every third id of a Kuhn cube, every second of a 2D grid):
    empty origin rows, zero dual volumes."""
    from paper_2502_00778_b200 import meshgen
    k = meshgen.tet_cube(10, amp=0.1)
    x = np.zeros(9 * k.num_nodes())
    x.reshape(-1, 3)[::3] = k.coords.reshape(-1, 3)
    _check_against_oracle(engine, oracle, Mesh(3, x, k.elements * 3, k.boundary * 3))
    assert (engine.get_volumes().reshape(-1, 3)[:, 1:] == 0).all()
    t = meshgen.tri_square(30, amp=0.2)
    x = np.zeros(4 * t.num_nodes())
    x.reshape(-1, 2)[::2] = t.coords.reshape(-1, 2)
    _check_against_oracle(engine, oracle, Mesh(2, x, t.elements * 2, t.boundary * 2))
    assert engine.plan_info()["tiles"] != "row" and not engine.plan_info()["colored"]


def test_side_list_overflow_and_wide_tables(engine, oracle):
    """A soup whose tile tables pass 256 nodes (16-bit ring codes) with ~450 k edges on the
    side list."""
    rng = np.random.default_rng(3)
    nv, ne = 3000, 400000
    el = np.stack([rng.choice(nv, 4, replace=False) for _ in range(ne)]).astype(np.int32)
    _check_against_oracle(engine, oracle, Mesh(3, rng.random(3 * nv), el.reshape(-1),
                                               np.zeros(0, np.int32)))
    assert engine.side_edges() > 100000 and engine.plan_info()["ring_max_tile_nodes"] > 256


@pytest.mark.parametrize("layout", ["spread", "split"])
def test_more_than_2_pow_25_nodes(engine, oracle, layout):
    """More than 2^25 node ids.  "spread": the cube's nodes at sorted random ids (element spans
    stay small: K1's bucket path, whose item keys hold k - j in 25 bits); "split": half of them
    moved beyond 2^25, so elements span more than the keys hold and K1 takes the generic item
    sort.  Both against the oracle."""
    from paper_2502_00778_b200 import meshgen
    k = meshgen.tet_cube(10, amp=0.1)
    rng = np.random.default_rng(5)
    big = (1 << 25) + 2000
    n = k.num_nodes()
    if layout == "spread":
        ids = np.sort(rng.choice(big, n, replace=False))
    else:
        ids = np.concatenate([np.arange(n // 2), (1 << 25) + 500 + np.arange(n - n // 2)])
    x = np.zeros(3 * big)
    x.reshape(-1, 3)[ids] = k.coords.reshape(-1, 3)
    _check_against_oracle(engine, oracle, Mesh(3, x, ids[k.elements], ids[k.boundary]))


def test_side_list_overflow_falls_back(engine, oracle):
    """More irregular edges than the side list holds (2^20): the ring path is not used, the
    whole mesh runs on the serial-order kernels -- same bits as the oracle."""
    rng = np.random.default_rng(11)
    nv, ne = 6000, 1500000
    el = rng.integers(0, nv, size=(ne, 4), dtype=np.int32)
    srt = np.sort(el, 1)
    el = el[(srt[:, 1:] != srt[:, :-1]).all(1)]
    m = Mesh(3, rng.random(3 * nv), el.reshape(-1), np.zeros(0, np.int32))
    engine.set_mesh(m)
    engine.build_edges()
    e, o = oracle.build_edges(m)
    np.testing.assert_array_equal(engine.edges().edges, e)
    want = oracle.navs_dualfree(m, e, o)
    engine.navs(_lib.DM_NAV_DUALFREE, _lib.DM_VARIANT_GATHER)
    assert not engine.plan_info()["ring_ok"]
    np.testing.assert_array_equal(engine.get_navs(), want)
    engine.volumes(_lib.DM_VOL_EDGE)
    np.testing.assert_array_equal(engine.get_volumes(), oracle.volumes_edge(m, e, want))


def test_two_contexts_on_two_threads(oracle):
    """One context per host thread (C-ABI threading rule), both on the device at once."""
    import threading

    from paper_2502_00778_b200 import Engine, meshgen
    meshes = {"a": meshgen.tet_cube(20, amp=0.15),
              "b": meshgen.permute(meshgen.tet_cube(18, amp=0.1))}
    res, err = {}, []

    def work(tag):
        try:
            en = Engine(0)
            en.set_mesh(meshes[tag])
            en.build_edges()
            out = []
            for _ in range(5):
                en.navs()
                en.volumes()
                out.append((en.get_navs().copy(), en.get_volumes().copy()))
            res[tag] = out
            en.close()
        except Exception as ex:  # surfaced below
            err.append((tag, ex))

    th = [threading.Thread(target=work, args=(t,)) for t in meshes]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not err, err
    for tag, m in meshes.items():
        e, o = oracle.build_edges(m)
        w = oracle.navs_dualfree(m, e, o)
        wv = oracle.volumes_edge(m, e, w)
        for n, v in res[tag]:
            assert np.abs(n - w).max() / np.abs(w).max() <= 1e-12
            assert np.abs(v - wv).max() <= 1e-12 * np.abs(wv).max()
            np.testing.assert_array_equal(n, res[tag][0][0])  # run-to-run bitwise
            np.testing.assert_array_equal(v, res[tag][0][1])


def test_wide_tiles_keep_8_bit_codes(engine, oracle, monkeypatch):
    """Tiles of more than 256 nodes in a plan with 8-bit ring codes (tolerated when they are
    few; forced here for every tile of a soup): edges whose slots pass 255 ride the side list,
    their tiles read the table from global memory -- results against the oracle."""
    monkeypatch.setenv("DUALMESH_WIDE_TILES_MAX", "1000")
    rng = np.random.default_rng(21)
    nv, ne = 3000, 200000
    el = np.stack([rng.choice(nv, 4, replace=False) for _ in range(ne)]).astype(np.int32)
    m = Mesh(3, rng.random(3 * nv), el.reshape(-1), np.zeros(0, np.int32))
    _check_against_oracle(engine, oracle, m)
    info = engine.plan_info()
    assert info["ring_ok"] and info["ring_max_tile_nodes"] > 256 and info["ring_fail_bits"] & 64
    assert engine.side_edges() > 0
    e, o = oracle.build_edges(m)
    wt = oracle.navs_traditional(m, e, o)
    engine.navs(_lib.DM_NAV_TRADITIONAL, _lib.DM_VARIANT_GATHER)
    assert np.abs(engine.get_navs() - wt).max() / np.abs(wt).max() <= 1e-12
