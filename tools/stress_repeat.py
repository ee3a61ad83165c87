"""Run-to-run repeatability under sustained load: 2000 back-to-back steps per grid and
algorithm (row tiles, Morton tiles, coloured Morton tiles on a flipped grid), navs and volumes
compared bit for bit with the first step every fifth step.

    python tools/stress_repeat.py
"""
import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2502_00778_b200 import Engine, _lib, meshgen
cases = {"row C5/2": meshgen.baseline_config("C5", 2), "morton C3/2": meshgen.baseline_config("C3", 2),
         "flip 80": meshgen.flip23(meshgen.tet_cube(80, amp=0.15), 0.3), "C4/2": meshgen.baseline_config("C4", 2)}
for name, m in cases.items():
    eng = Engine(0)
    eng.set_mesh(m); eng.build_edges()
    for algo in (_lib.DM_NAV_DUALFREE, _lib.DM_NAV_TRADITIONAL):
        eng.navs(algo, 0); eng.volumes(0)
        n0, v0 = eng.get_navs().copy(), eng.get_volumes().copy()
        bad = 0
        t0 = time.time()
        for it in range(400):
            for _ in range(5):
                eng.navs(algo, 0); eng.volumes(0)
            if not (np.array_equal(eng.get_navs(), n0) and np.array_equal(eng.get_volumes(), v0)):
                bad += 1
        print(name, "algo", algo, "plan", eng.plan_info()["tiles"], "2000 steps, mismatching checks:", bad, f"{time.time()-t0:.1f}s", flush=True)
    eng.close()
