#!/usr/bin/env python3
"""One plan setting on the 2-3-flipped 160^3 grid: plan statistics + element-loop time
(for ncu captures of the element loop on non-Kuhn topology).

    DUALMESH_ROW_CAND=192 DUALMESH_ROW_SPLIT_MAX=2 python tools/flip_probe.py [--steps 6]
"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.time_unstructured import run, b_elem
from paper_2502_00778_b200 import meshgen
ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=6)
ap.add_argument("--n", type=int, default=160)
ap.add_argument("--frac", type=float, default=0.3)
a = ap.parse_args()
f = meshgen.flip23(meshgen.tet_cube(a.n, amp=0.15), a.frac)
r = run(f, steps=a.steps)
r["b_elem"] = b_elem(f, r["n_edges"])
print(json.dumps(r), flush=True)
