"""Device memory held by one context after K1, the plan and a metrics step
(C5 unless --config), from cudaMemGetInfo around the calls.

    python tools/footprint.py --config C5
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C5")
    a = ap.parse_args()
    import torch
    from paper_2502_00778_b200 import Engine, _lib, meshgen
    torch.cuda.init()
    free0, total = torch.cuda.mem_get_info()
    eng = Engine(0)
    meshgen.baseline_config_device(eng, a.config)
    f1, _ = torch.cuda.mem_get_info()
    eng.build_edges()
    f2, _ = torch.cuda.mem_get_info()
    eng.navs(_lib.DM_NAV_DUALFREE, _lib.DM_VARIANT_GATHER)
    eng.volumes(_lib.DM_VOL_EDGE)
    f3, _ = torch.cuda.mem_get_info()
    gb = 1e9
    print(json.dumps({"config": a.config, "total_gb": total / gb,
                      "mesh_gb": (free0 - f1) / gb, "after_edges_gb": (free0 - f2) / gb,
                      "after_plan_and_step_gb": (free0 - f3) / gb}))


if __name__ == "__main__":
    main()
