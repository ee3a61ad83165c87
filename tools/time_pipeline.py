#!/usr/bin/env python3
"""Fresh-topology pipeline on one grid, phase by phase (host wall clock with
device syncs): dm_set_mesh (H2D), K1 edge extraction (first call / warm),
plan build (first / rebuild, DUALMESH_PLAN_TIMING=1 prints its phases) and
one metrics step, then the D2H of navs + volumes.

    python tools/time_pipeline.py --config C5
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C5")
    ap.add_argument("--scale", type=int, default=1)
    a = ap.parse_args()
    import torch
    from paper_2502_00778_b200 import Engine, _lib, meshgen
    m = meshgen.baseline_config(a.config, a.scale)
    eng = Engine(0)
    out = {}

    def t(name, fn):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = fn()
        eng.sync()
        out[name] = (time.perf_counter() - t0) * 1e3
        return r

    t("set_mesh_ms", lambda: eng.set_mesh(m))
    t("edges_first_ms", eng.build_edges)
    t("edges_warm_ms", eng.build_edges)
    DF, G, E = _lib.DM_NAV_DUALFREE, _lib.DM_VARIANT_GATHER, _lib.DM_VOL_EDGE
    t("plan_and_step_first_ms", lambda: (eng.navs(DF, G), eng.volumes(E)))
    t("step_ms", lambda: (eng.navs(DF, G), eng.volumes(E)))
    eng.build_edges()
    t("plan_and_step_rebuild_ms", lambda: (eng.navs(DF, G), eng.volumes(E)))
    t("d2h_ms", lambda: (eng.get_navs(), eng.get_volumes()))
    out["plan"] = eng.plan_info()
    print(json.dumps(out), flush=True)
    eng.close()


if __name__ == "__main__":
    main()
