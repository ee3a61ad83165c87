#!/usr/bin/env python3
"""Bitwise comparison of navs / volumes between two DUALMESH_GATHER_CFG values.

    python tools/cmp_cfg.py --config C5 --cfg 31
(the knob is read when a context is created, so each context sets it first)
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(cfg, config, scale):
    os.environ["DUALMESH_GATHER_CFG"] = str(cfg)
    from paper_2502_00778_b200 import Engine, meshgen
    m = meshgen.baseline_config(config, scale)
    eng = Engine(0)
    eng.set_mesh(m)
    eng.build_edges()
    eng.navs()
    eng.volumes()
    out = eng.get_navs().copy(), eng.get_volumes().copy()
    eng.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C5")
    ap.add_argument("--scale", type=int, default=1)
    ap.add_argument("--cfg", type=int, required=True)
    a = ap.parse_args()
    n0, v0 = run(0, a.config, a.scale)
    n1, v1 = run(a.cfg, a.config, a.scale)
    print(f"{a.config} cfg {a.cfg}: navs bitwise {np.array_equal(n0.view(np.uint64), n1.view(np.uint64))}"
          f" vols bitwise {np.array_equal(v0.view(np.uint64), v1.view(np.uint64))}", flush=True)


if __name__ == "__main__":
    main()
