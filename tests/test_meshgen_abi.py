"""CPU tests: generator contract and the C-ABI library
surface (loads without a GPU, exports every declared symbol, no fallback)."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

from paper_2502_00778_b200 import _lib, meshgen
from oracle.oracle import RefMesh, ref_available

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def sizes_box(n):
    a, b, c = C.c_int64(), C.c_int64(), C.c_int64()
    _lib.meshgen().dmg_tet_box_sizes(n, n, n, C.byref(a), C.byref(b), C.byref(c))
    return a.value, b.value, c.value


def test_generator_counts_paper_grids():
    m = meshgen.tri_square(255)                       # SPEC.md:320, acceptance 6
    assert (m.num_nodes(), m.num_elements(), m.num_boundary()) == (65536, 130050, 1020)
    assert sizes_box(256)[:2] == (16974593, 100663296)
    for n, want in ((1, (8, 6, 12)), (2, (27, 48, 48)), (16, (4913, 24576, 3072)),
                    (64, (274625, 1572864, 49152))):
        assert sizes_box(n) == want


def test_generator_deterministic_and_amp0():
    a = meshgen.tet_cube(5, amp=0.15, seed=42)
    b = meshgen.tet_cube(5, amp=0.15, seed=42)
    z = meshgen.tet_cube(5, amp=0.0)
    np.testing.assert_array_equal(a.coords, b.coords)
    x = z.coords.reshape(-1, 3)
    np.testing.assert_allclose(x, np.round(x * 5) / 5, atol=0)  # lattice when amp = 0
    assert meshgen.first_inverted(a) == -1


def test_baseline_configs_small_valid():
    for name in ("C1", "C2", "C3", "C4", "C5"):
        m = meshgen.baseline_config(name, 16 if name != "C1" else 8)
        assert meshgen.first_inverted(m) == -1
        if ref_available():
            n, msgs, signs = RefMesh(m).validate()
            assert n == 0, msgs[:3]


def test_bl_grid_geometry():
    z = meshgen.bl_z(256, 1e-5, 1.05)
    assert z[0] == 0.0 and abs(z[1] - 1e-5) < 1e-20
    assert 53.0 < z[-1] < 53.3  # z_top ~ 53.15


def header_functions(path):
    src = open(path).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dmg?_[a-z0-9_]+)\s*\(", src)))


def test_capi_exports_every_declared_symbol():
    lib = _lib.capi()  # loads without a GPU
    for name in header_functions(os.path.join(ROOT, "include", "dm_capi.h")):
        assert hasattr(lib, name), name
        assert name in _lib.CAPI, f"{name} missing from the ctypes table"
    g = _lib.meshgen()
    for name in header_functions(os.path.join(ROOT, "include", "dm_meshgen.h")):
        assert hasattr(g, name), name


def test_cpp_api_symbols_exported():
    so = os.path.join(_lib.LIBDIR, "libdualmesh.so")
    out = subprocess.run(["nm", "-D", "-C", "--defined-only", so], capture_output=True,
                         text=True).stdout
    for sym in ("dualmesh::build_edges(dualmesh::Mesh const&)",
                "dualmesh::EdgeList::edge_of(int, int) const",
                "dualmesh::validate_mesh(dualmesh::Mesh const&)",
                "dualmesh::element_volume(dualmesh::Mesh const&, unsigned long)",
                "dualmesh::opposite_face_normal(dualmesh::Mesh const&, unsigned long, int)",
                "dualmesh::boundary_normal(dualmesh::Mesh const&, unsigned long)",
                "dualmesh::derive_boundary_faces(dualmesh::Mesh const&)",
                "dualmesh::max_face_area(dualmesh::Mesh const&)",
                "dualmesh::max_element_volume(dualmesh::Mesh const&)",
                "dualmesh::total_volume(dualmesh::Mesh const&)",
                "dualmesh::boundary_node_mask(dualmesh::Mesh const&)",
                "dualmesh::lumped_navs_dualfree(dualmesh::Mesh const&, dualmesh::EdgeList const&)",
                "dualmesh::compute_metrics("):
        assert sym in out, sym


def test_no_cpu_fallback_without_gpu():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    from paper_2502_00778_b200 import DualMeshError, Engine
    with pytest.raises(DualMeshError):
        Engine()


def test_kernels_are_sm100a():
    so = os.path.join(_lib.LIBDIR, "libdualmesh.so")
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out
