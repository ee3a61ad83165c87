"""The Python mirror of the SPEC metrics API (paper_2502_00778_b200.metrics,
same names as include/dualmesh/metrics.hpp) against the oracle."""
import numpy as np
import pytest

from paper_2502_00778_b200 import Mesh, MeshEdgeMismatch, meshgen, metrics
from paper_2502_00778_b200.mesh import build_edges

pytestmark = pytest.mark.gpu


def rel(a, b, dim):
    a, b = a.reshape(-1, dim), b.reshape(-1, dim)
    den = np.maximum(np.abs(b).max(axis=1), 1e-300)
    return float((np.abs(a - b).max(axis=1) / den).max())


@pytest.mark.parametrize("name,scale", [("C1", 4), ("C2", 4), ("C4", 16)])
def test_spec_ops(oracle, name, scale):
    m = meshgen.baseline_config(name, scale)
    el = build_edges(m)
    e, o = oracle.build_edges(m)
    np.testing.assert_array_equal(el.edges, e)
    nd = metrics.lumped_navs_dualfree(m, el)
    nt = metrics.lumped_navs_traditional(m, el)
    want_d, want_t = oracle.navs_dualfree(m, e, o), oracle.navs_traditional(m, e, o)
    assert rel(nd, want_d, m.dim) <= 1e-12 and rel(nt, want_t, m.dim) <= 1e-12
    ve = metrics.dual_volumes_edge_based(m, el, want_d)
    np.testing.assert_array_equal(ve, oracle.volumes_edge(m, e, want_d))  # bitwise given navs
    vl = metrics.dual_volumes_element_based(m)
    np.testing.assert_array_equal(vl, oracle.volumes_element(m))
    assert metrics.check_closure(m, el, nd) <= 1e-13
    assert metrics.check_total_volume(m, ve) <= 1e-12
    D = m.dim
    A = np.eye(D) / D
    assert metrics.check_linear_exactness(m, el, nd, ve, A, np.zeros(D)) <= 1e-9
    for nav in (metrics.DUALFREE, metrics.TRADITIONAL):
        for vol in (metrics.EDGE, metrics.ELEMENT):
            el2, n2, v2 = metrics.compute_metrics(m, nav, vol)
            np.testing.assert_array_equal(el2.edges, e)
            assert rel(n2, want_d if nav == metrics.DUALFREE else want_t, D) <= 1e-12
            assert np.abs(v2 - vl).max() <= 1e-12 * np.abs(vl).max()


def test_mismatch_raises():
    m = meshgen.tet_cube(3, amp=0.1)
    el = build_edges(m)
    el.edges = el.edges[:-1]
    with pytest.raises(MeshEdgeMismatch):
        metrics.lumped_navs_dualfree(m, el)
