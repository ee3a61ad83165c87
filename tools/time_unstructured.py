#!/usr/bin/env python3
"""Generality rows of the ring path, CUDA events on the
library stream, same box:

  * side list: a BASELINE grid vs the same grid plus one 30-tet fan
    (meshgen.fan_in) -- the hub edge leaves the ring codes, the rest stays;
  * non-Kuhn topology: seeded 2-3 flips (meshgen.flip23) of a 160^3 Kuhn cube,
    element loop on row tiles and on Morton tiles, its roofline fraction from
    SURVEY 8(d)'s B_elem of that mesh.

    python tools/time_unstructured.py --out gpurun_out/unstructured.json
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(m, steps=10, env=None):
    from paper_2502_00778_b200 import Engine, _lib
    old = {k: os.environ.get(k) for k in (env or {})}
    os.environ.update(env or {})
    try:
        eng = Engine(0)
        eng.set_mesh(m)
        ne = eng.build_edges()
        DF, G, E = _lib.DM_NAV_DUALFREE, _lib.DM_VARIANT_GATHER, _lib.DM_VOL_EDGE
        eng.navs(DF, G)
        eng.volumes(E)
        eng.set_timing(True)
        t = []
        for _ in range(steps):
            eng.navs(DF, G)
            eng.volumes(E)
            t.append(eng.timings())
        t = np.array(t[2:])
        out = {"n_elements": m.num_elements(), "n_edges": ne, "plan": eng.plan_info(),
               "side_edges": eng.side_edges(), "plan_bytes": eng.plan_bytes(),
               "element_loop_ms": float(t[:, 0].mean()), "boundary_ms": float(t[:, 1].mean()),
               "volumes_ms": float(t[:, 2].mean()), "step_ms": float(t[:, 3].mean())}
        eng.close()
        return out
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def b_elem(m, ne):
    D, L = 3, 6
    return 4 * (D + 1) * m.num_elements() + 4 * L * m.num_elements() + 8 * D * m.num_nodes() + \
        8 * D * ne


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--n", type=int, default=160)
    a = ap.parse_args()
    from paper_2502_00778_b200 import meshgen
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    rec = {"hbm_peak_gbs": peak}
    c3 = meshgen.baseline_config("C3")
    rec["C3"] = run(c3)
    rec["C3+fan30"] = run(meshgen.fan_in(c3, 30))
    rec["C3+fan30"]["step_vs_C3"] = rec["C3+fan30"]["step_ms"] / rec["C3"]["step_ms"]
    del c3
    c5 = meshgen.baseline_config("C5")
    rec["C5"] = run(c5)
    rec["C5+fan30"] = run(meshgen.fan_in(c5, 30))
    rec["C5+fan30"]["step_vs_C5"] = rec["C5+fan30"]["step_ms"] / rec["C5"]["step_ms"]
    del c5
    f = meshgen.flip23(meshgen.tet_cube(a.n, amp=0.15), 0.3)
    for key, env in (("flip23_row", {"DUALMESH_ROW_PLAN": "1"}),
                     ("flip23_morton", {"DUALMESH_ROW_PLAN": "0"})):
        r = run(f, env=env)
        bb = b_elem(f, r["n_edges"])
        r["B_elem"] = bb
        r["element_loop_frac_of_hbm"] = bb / (r["element_loop_ms"] / 1e3) / 1e9 / peak
        r["mesh"] = f"{a.n}^3 Kuhn cube +-0.15h, seeded 2-3 flips (meshgen.flip23, 30%)"
        rec[key] = r
    print(json.dumps(rec, indent=1), flush=True)
    if a.out:
        json.dump(rec, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
