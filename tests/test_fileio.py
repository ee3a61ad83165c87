"""CPU tests of the SPEC cli_io formats through the
host-only entry points of libdualmesh.so: MeshFile round trips bit for bit,
the SPEC parse-error examples, and the MetricsFile JSON document."""
import json

import numpy as np
import pytest

from paper_2502_00778_b200 import Mesh, fileio, meshgen

FTRI = """dualmesh v1
# F-TRI (SPEC.md:434)
dim 2
nodes 3
0 0
1 0
0 1
elements 1
1 2 3
boundary 3
1 2
2 3
3 1
"""


def test_ftri_file(tmp_path):
    p = tmp_path / "f.dm"
    p.write_text(FTRI)
    m = fileio.read_mesh(p)
    assert (m.dim, m.num_nodes(), m.num_elements(), m.num_boundary()) == (2, 3, 1, 3)
    np.testing.assert_array_equal(m.elements, [0, 1, 2])
    np.testing.assert_array_equal(m.boundary, [0, 1, 1, 2, 2, 0])
    np.testing.assert_array_equal(m.coords, [0, 0, 1, 0, 0, 1])


@pytest.mark.parametrize("mesh_fn", [
    lambda: meshgen.tri_square(16, diag_seed=43, amp=0.2),
    lambda: meshgen.tet_cube(6, amp=0.15),
    lambda: meshgen.baseline_config("C3", 32),
    lambda: meshgen.baseline_config("C4", 32),
])
def test_mesh_round_trip_bitwise(tmp_path, mesh_fn):
    m = mesh_fn()
    p = tmp_path / "m.dm"
    fileio.write_mesh(m, p)
    r = fileio.read_mesh(p)
    assert r.dim == m.dim
    np.testing.assert_array_equal(r.coords, m.coords)      # 17 digits: lossless
    np.testing.assert_array_equal(r.elements, m.elements)
    np.testing.assert_array_equal(r.boundary, m.boundary)
    q = tmp_path / "m2.dm"
    fileio.write_mesh(r, q)
    assert p.read_bytes() == q.read_bytes()                 # deterministic bytes
    assert fileio.mesh_checksum(r) == fileio.mesh_checksum(m)


@pytest.mark.parametrize("text,line,what", [
    ("dualmesh v1\ndim 2\nnodes 3\n0 0\n1 0\n0 1\nelements 2\n1 2 3\n", 8, "count mismatch"),
    ("dualmesh v1\ndim 2\nnodes 3\n0 0\n1 0\n0 1\nelements 1\n1 2 4\n", 8, "invalid index"),
    ("dualmesh v1\ndim 2\nnodes 3\n0 0\n1 0\nelements 1\n1 2 3\n", 6, "count mismatch"),
    # huge declared counts over a short file: count mismatch, not an allocation failure
    ("dualmesh v1\ndim 3\nnodes 2000000000\n0 0 0\n", 4, "count mismatch"),
    ("dualmesh v1\ndim 2\nnodes 3\n0 0\n1 0\n0 1\nelements 1000000000000\n1 2 3\n", 8,
     "count mismatch"),
    ("dualmesh v2\n", 1, "header"),
    ("dualmesh v1\ndim 4\n", 2, "dim"),
    ("dualmesh v1\ndim 2\nnodes 1\n0 x\nelements 0\n", 4, "bad number"),
    ("dualmesh v1\ndim 2\nnodes 1\n0 0 0\n", 4, "coordinates"),
    ("dualmesh v1\ndim 2\nnodes 3\n0 0\n1 0\n0 1\nelements 1\n1 2 3\nboundary 1\n1 2\n9 9\n",
     11, "unexpected content"),
])
def test_parse_errors_report_lines(tmp_path, text, line, what):
    """syntax errors with line numbers; count mismatch; invalid index."""
    p = tmp_path / "bad.dm"
    p.write_text(text)
    with pytest.raises(fileio.MeshFileError) as ei:
        fileio.read_mesh(p)
    msg = str(ei.value)
    assert f"bad.dm:{line}:" in msg and what in msg, msg


def test_whitespace_and_comments(tmp_path):
    p = tmp_path / "ws.dm"
    p.write_text("# leading comment\n\n  dualmesh\tv1  \ndim 2 # trailing\nnodes 3\n 0  0\n"
                 "1\t0\n0 1\n\nelements 1\n1 2 3\nboundary 3\n1 2\n2 3\n3 1\n")
    m = fileio.read_mesh(p)
    assert m.num_elements() == 1 and m.num_boundary() == 3


def test_missing_boundary_is_flagged(tmp_path):
    p = tmp_path / "nb.dm"
    p.write_text("dualmesh v1\ndim 3\nnodes 4\n0 0 0\n1 0 0\n0 1 0\n0 0 1\nelements 1\n1 2 3 4\n")
    assert not fileio.has_boundary_section(p)
    p.write_text(FTRI)
    assert fileio.has_boundary_section(p)


def test_metrics_file(tmp_path, oracle):
    m = meshgen.tet_cube(4, amp=0.15)
    e, o = oracle.build_edges(m)
    n = oracle.navs_dualfree(m, e, o)
    v = oracle.volumes_edge(m, e, n)
    p = tmp_path / "m.json"
    fileio.write_metrics(p, m, e, n, v)
    d = json.loads(p.read_text())
    assert d["format"] == "dualmesh-metrics v1" and d["dim"] == 3
    pv = d["provenance"]
    assert pv["nav_algo"] == "dualfree" and pv["vol_algo"] == "edge"
    assert pv["mesh_checksum"] == f"fnv1a64:{fileio.mesh_checksum(m):016x}"
    assert pv["n_edges"] == e.shape[0] and pv["n_nodes"] == m.num_nodes()
    np.testing.assert_array_equal(np.array(d["edges"]) - 1, e)
    np.testing.assert_array_equal(np.array(d["navs"]).ravel(), n)  # lossless
    np.testing.assert_array_equal(np.array(d["volumes"]), v)
    q = tmp_path / "m2.json"
    fileio.write_metrics(q, m, e, n, v)
    assert p.read_bytes() == q.read_bytes()


@pytest.mark.gpu
def test_missing_boundary_is_derived(tmp_path):
    """F-TET without a boundary section -> 4 derived outward faces,
    equal to the reference derive_boundary_faces (when oracle/_ref is built)."""
    from oracle.oracle import RefMesh, ref_available
    p = tmp_path / "ftet.dm"
    p.write_text("dualmesh v1\ndim 3\nnodes 4\n0 0 0\n1 0 0\n0 1 0\n0 0 1\nelements 1\n"
                 "1 2 3 4\n")
    m = fileio.read_mesh(p)
    assert m.num_boundary() == 4
    if ref_available():
        np.testing.assert_array_equal(m.boundary, RefMesh(m).derive_boundary())
    c = meshgen.tet_cube(5, amp=0.15)
    q = tmp_path / "cube.dm"
    fileio.write_mesh(Mesh(3, c.coords, c.elements), q)
    text = q.read_text()
    assert text.endswith("boundary 0\n")  # an empty boundary is written explicitly
    q.write_text(text[:-len("boundary 0\n")])
    assert not fileio.has_boundary_section(q)
    r = fileio.read_mesh(q)
    assert r.num_boundary() == c.num_boundary()
    if ref_available():
        np.testing.assert_array_equal(r.boundary,
                                      RefMesh(Mesh(3, c.coords, c.elements)).derive_boundary())
