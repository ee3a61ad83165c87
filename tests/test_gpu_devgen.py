"""Device-side meshgen (dm_gen_*) against the host
generator (libdm_meshgen.so): the same coordinates, elements and boundary
bit for bit, and the path on a device-generated grid equals the path on the
uploaded one."""
import numpy as np
import pytest

from paper_2502_00778_b200 import Engine, _lib, meshgen

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,scale", [("C1", 1), ("C1", 4), ("C2", 1), ("C3", 2), ("C3", 1),
                                        ("C4", 2), ("C5", 2), ("C5", 1)])
def test_device_grid_bitwise_equals_host(name, scale):
    want = meshgen.baseline_config(name, scale)
    eng = Engine(0)
    try:
        meshgen.baseline_config_device(eng, name, scale)
        got = eng.get_mesh()
        assert got.dim == want.dim
        np.testing.assert_array_equal(got.coords, want.coords)
        np.testing.assert_array_equal(got.elements, want.elements)
        np.testing.assert_array_equal(got.boundary, want.boundary)
    finally:
        eng.close()


def test_unjittered_and_uniform_diagonal():
    for args in ((5, 0, 0.0, 1), (7, 9, 0.3, 3)):
        want = meshgen.tri_square(args[0], diag_seed=args[1], amp=args[2], seed=args[3])
        eng = Engine(0)
        try:
            eng.gen_tri_square(*args)
            got = eng.get_mesh()
            np.testing.assert_array_equal(got.coords, want.coords)
            np.testing.assert_array_equal(got.elements, want.elements)
            np.testing.assert_array_equal(got.boundary, want.boundary)
        finally:
            eng.close()
    want = meshgen.tet_box(3, 4, 5, None, 0, 0.0, 1)
    eng = Engine(0)
    try:
        eng.gen_tet_box(3, 4, 5)
        got = eng.get_mesh()
        np.testing.assert_array_equal(got.coords, want.coords)
        np.testing.assert_array_equal(got.elements, want.elements)
        np.testing.assert_array_equal(got.boundary, want.boundary)
    finally:
        eng.close()


def test_path_on_device_grid(engine):
    """navs / volumes on the device-generated C3/4 equal those on the upload."""
    DF, G, EDGE = _lib.DM_NAV_DUALFREE, _lib.DM_VARIANT_GATHER, _lib.DM_VOL_EDGE
    m = meshgen.baseline_config("C3", 4)
    engine.set_mesh(m)
    engine.build_edges()
    engine.navs(DF, G)
    engine.volumes(EDGE)
    n1, v1 = engine.get_navs(), engine.get_volumes()
    eng = Engine(0)
    try:
        meshgen.baseline_config_device(eng, "C3", 4)
        eng.build_edges()
        eng.navs(DF, G)
        eng.volumes(EDGE)
        np.testing.assert_array_equal(eng.get_navs(), n1)
        np.testing.assert_array_equal(eng.get_volumes(), v1)
    finally:
        eng.close()


def test_bad_arguments():
    eng = Engine(0)
    try:
        with pytest.raises(Exception):
            eng.gen_tet_box(0, 1, 1)
        with pytest.raises(Exception):
            eng.gen_tet_box(2, 2, 2, jitter_mode=3)
        with pytest.raises(Exception):
            eng.gen_tri_square(0)
    finally:
        eng.close()
