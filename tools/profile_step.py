#!/usr/bin/env python3
"""Minimal driver for ncu / timing sweeps: one grid, a few metrics steps.

    python tools/profile_step.py --config C5 --variant gather --steps 3
Prints per-phase CUDA-event times (ms) of every step as JSON lines.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C5")
    ap.add_argument("--scale", type=int, default=1)
    ap.add_argument("--variant", default="gather")
    ap.add_argument("--algo", default="dualfree")
    ap.add_argument("--vol", default="edge")
    ap.add_argument("--steps", type=int, default=3)
    args = ap.parse_args()
    from paper_2502_00778_b200 import Engine, _lib, meshgen
    variants = {"gather": _lib.DM_VARIANT_GATHER, "scatter": _lib.DM_VARIANT_SCATTER,
                "gather_elem": _lib.DM_VARIANT_GATHER_ELEM,
                "faces": _lib.DM_VARIANT_GATHER_FACES, "exact": _lib.DM_VARIANT_GATHER_EXACT}
    algo = _lib.DM_NAV_DUALFREE if args.algo == "dualfree" else _lib.DM_NAV_TRADITIONAL
    vol = _lib.DM_VOL_EDGE if args.vol == "edge" else _lib.DM_VOL_ELEMENT
    m = meshgen.baseline_config(args.config, args.scale)
    eng = Engine(0)
    eng.set_mesh(m)
    eng.build_edges()
    eng.set_timing(True)
    for s in range(args.steps):
        eng.navs(algo, variants[args.variant])
        eng.volumes(vol)
        t = eng.timings()
        print(json.dumps({"plan": eng.plan_info(), "step": s, "config": args.config, "variant": args.variant,
                          "algo": args.algo, "elem_ms": t[0], "bnd_ms": t[1], "vol_ms": t[2],
                          "total_ms": t[3]}), flush=True)
    eng.close()


if __name__ == "__main__":
    main()
