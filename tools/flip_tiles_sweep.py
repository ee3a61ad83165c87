"""Element loop on the 2-3-flipped 160^3 grid under plan knobs (Morton tiles; row tiles at
several candidate sizes with a 2x split budget; lane order by ring length or not).

    python tools/flip_tiles_sweep.py
"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.time_unstructured import run, b_elem
from paper_2502_00778_b200 import meshgen
f = meshgen.flip23(meshgen.tet_cube(160, amp=0.15), 0.3)
peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6650.0
for env in ({"DUALMESH_ROW_PLAN": "0"},
            {"DUALMESH_ROW_CAND": "224", "DUALMESH_ROW_SPLIT_MAX": "2"},
            {"DUALMESH_ROW_CAND": "192", "DUALMESH_ROW_SPLIT_MAX": "2"},
            {"DUALMESH_ROW_CAND": "160", "DUALMESH_ROW_SPLIT_MAX": "2"},
            {"DUALMESH_ROW_CAND": "128", "DUALMESH_ROW_SPLIT_MAX": "2"},
            {"DUALMESH_ROW_CAND": "192", "DUALMESH_ROW_SPLIT_MAX": "2", "DUALMESH_ROW_BYLEN": "0"}):
    r = run(f, env=env)
    bb = b_elem(f, r["n_edges"])
    print(json.dumps({"env": env, "tiles": r["plan"].get("tiles"), "loop_ms": round(r["element_loop_ms"], 4),
                      "step_ms": round(r["step_ms"], 4), "frac": round(bb / (r["element_loop_ms"] / 1e3) / 1e9 / peak, 3)}), flush=True)
