#!/usr/bin/env python3
"""Small pass over every kernel family (also usable under compute-sanitizer where the pool allows it: memcheck / synccheck /
initcheck / racecheck): row tiles, Morton tiles, flipped topology, the side list, 2D,
every navs variant, both volume algorithms, the checks and a plan rebuild.

    compute-sanitizer --tool memcheck python tools/sanitize.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_00778_b200 import Engine, _lib, meshgen  # noqa: E402

N = int(os.environ.get("SANITIZE_N", "14"))
meshes = {
    "row": meshgen.tet_cube(N, amp=0.15),
    "morton": meshgen.permute(meshgen.tet_cube(N, amp=0.15)),
    "flip": meshgen.flip23(meshgen.tet_cube(N, amp=0.15), 0.3),
    "fan": meshgen.fan_in(meshgen.tet_cube(max(6, N // 2), amp=0.1), 30),
    "tri": meshgen.tri_square(3 * N, diag_seed=43, amp=0.2),
}
eng = Engine(0)
for name, m in meshes.items():
    eng.set_mesh(m)
    ne = eng.build_edges()
    for algo in (_lib.DM_NAV_DUALFREE, _lib.DM_NAV_TRADITIONAL):
        for var in (_lib.DM_VARIANT_GATHER, _lib.DM_VARIANT_GATHER_EXACT, _lib.DM_VARIANT_SCATTER,
                    _lib.DM_VARIANT_GATHER_ELEM, _lib.DM_VARIANT_GATHER_FACES):
            eng.navs(algo, var)
            eng.volumes(_lib.DM_VOL_EDGE)
    eng.volumes(_lib.DM_VOL_ELEMENT)
    eng.navs(_lib.DM_NAV_DUALFREE, _lib.DM_VARIANT_GATHER)
    eng.volumes(_lib.DM_VOL_EDGE)
    r, _ = eng.check_closure()
    navs = eng.get_navs()
    vols = eng.get_volumes()
    # new coordinates on the same topology (plan reuse), then a fresh topology
    eng.set_coords(m.coords * 1.01)
    eng.navs(_lib.DM_NAV_DUALFREE, _lib.DM_VARIANT_GATHER)
    print(name, "edges", ne, "plan", eng.plan_info()["tiles"], "side", eng.side_edges(),
          "closure", r, "finite", bool(np.isfinite(navs).all() and np.isfinite(vols).all()),
          flush=True)
eng.close()
print("sanitize pass done")
