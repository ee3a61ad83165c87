"""Morton-plan slot colouring on the permuted C3 grid: plan colouring time and
element loop for DUALMESH_COLOR_ROUNDS in {off, 1, 2, 3, 4, 8} (CUDA events).

    python tools/color_rounds_sweep.py
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import json, os, sys, time
sys.path.insert(0, os.environ["ROOT"])
import torch
from paper_2502_00778_b200 import Engine, _lib, meshgen
eng = Engine(0)
meshgen.baseline_config_device(eng, "C3")
eng.build_edges()
torch.cuda.synchronize()
t0 = time.perf_counter()
eng.navs(_lib.DM_NAV_DUALFREE, _lib.DM_VARIANT_GATHER)
torch.cuda.synchronize()
plan_ms = (time.perf_counter() - t0) * 1e3
eng.volumes(_lib.DM_VOL_EDGE)
eng.set_timing(True)
t = []
for _ in range(12):
    eng.navs(_lib.DM_NAV_DUALFREE, _lib.DM_VARIANT_GATHER)
    eng.volumes(_lib.DM_VOL_EDGE)
    t.append(eng.timings())
el = sum(x[0] for x in t[2:]) / len(t[2:])
print(json.dumps({"plan_plus_first_navs_ms": plan_ms, "element_loop_ms": el, "plan": eng.plan_info()}))
'''
for env in ({"DUALMESH_PLAN_COLOR": "0"}, {"DUALMESH_COLOR_ROUNDS": "1"}, {"DUALMESH_COLOR_ROUNDS": "2"},
            {"DUALMESH_COLOR_ROUNDS": "3"}, {"DUALMESH_COLOR_ROUNDS": "4"}, {"DUALMESH_COLOR_ROUNDS": "8"}):
    e = dict(os.environ, ROOT=ROOT, **env)
    out = subprocess.run([sys.executable, "-c", CHILD], env=e, capture_output=True, text=True).stdout
    print(json.dumps({"env": env, **json.loads(out.strip().splitlines()[-1])}), flush=True)
