"""Generate the committed golden fixtures under tests/golden/.

Run in the build container (needs /root/reference for oracle/_ref):
    make -C oracle && python tests/golden/make_golden.py

* fixtures.json : the SPEC fixtures (F-TRI SPEC.md:57, F-TET SPEC.md:59,
  F-square SPEC.md:188, Kuhn n=1) with outputs of the REFERENCE's own code
  (oracle/_ref = proj/src/mesh.cpp compiled in place): edges, origin_start,
  opposite_face_normal, boundary_normal, element_volume, validate_mesh,
  derive_boundary_faces.
* configs.npz   : scaled-down BASELINE grids (C1..C5 families) with the
  reference build_edges output and the oracle's navs / volumes (float64,
  bit patterns preserved) for the GPU parity tests.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2502_00778_b200 import Mesh, meshgen  # noqa: E402
from oracle.oracle import Oracle, RefMesh  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def fixtures():
    return {
        "F-TRI": Mesh(2, [0, 0, 1, 0, 0, 1], [0, 1, 2], [0, 1, 1, 2, 2, 0]),
        "F-TET": Mesh(3, [0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0, 1], [0, 1, 2, 3],
                      [0, 2, 1, 0, 1, 3, 0, 3, 2, 1, 2, 3]),
        "F-square": Mesh(2, [0, 0, 1, 0, 0, 1, 1, 1], [0, 1, 2, 1, 3, 2],
                         [0, 1, 1, 3, 3, 2, 2, 0]),
        "Kuhn1": meshgen.tet_cube(1),
    }


def mesh_dict(m):
    return {"dim": m.dim, "coords": m.coords.tolist(), "elements": m.elements.tolist(),
            "boundary": m.boundary.tolist()}


def main():
    out = {}
    for name, m in fixtures().items():
        r = RefMesh(m)
        e, o = r.build_edges()
        n, msgs, signs = r.validate()
        out[name] = {
            "mesh": mesh_dict(m),
            "ref_edges": e.tolist(),
            "ref_origin_start": o.tolist(),
            "ref_opposite_face_normal": [[r.opposite_face_normal(el, i).tolist()
                                          for i in range(m.dim + 1)]
                                         for el in range(m.num_elements())],
            "ref_boundary_normal": [r.boundary_normal(b).tolist() for b in range(m.num_boundary())],
            "ref_element_volume": [r.element_volume(el) for el in range(m.num_elements())],
            "ref_validate": msgs,
            "ref_derive_boundary": r.derive_boundary().tolist(),
        }
    with open(os.path.join(HERE, "fixtures.json"), "w") as f:
        json.dump(out, f, indent=1)

    O = Oracle()
    arrays = {}
    for name, scale in (("C1", 8), ("C2", 8), ("C3", 16), ("C4", 16), ("C5", 32)):
        m = meshgen.baseline_config(name, scale)
        r = RefMesh(m)
        e, o = r.build_edges()
        e2l, ip, inc = O.edge_maps(m, e, o)
        nd = O.navs_dualfree(m, e, o)
        nt = O.navs_traditional(m, e, o)
        arrays.update({
            f"{name}_dim": np.array([m.dim]), f"{name}_coords": m.coords,
            f"{name}_elements": m.elements, f"{name}_boundary": m.boundary,
            f"{name}_edges": e, f"{name}_origin_start": o, f"{name}_e2l": e2l,
            f"{name}_inc_ptr": ip, f"{name}_inc": inc,
            f"{name}_navs_dualfree": nd, f"{name}_navs_traditional": nt,
            f"{name}_vol_edge": O.volumes_edge(m, e, nd),
            f"{name}_vol_element": O.volumes_element(m),
        })
    np.savez_compressed(os.path.join(HERE, "configs.npz"), **arrays)
    print("wrote fixtures.json, configs.npz")


if __name__ == "__main__":
    main()
