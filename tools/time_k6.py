"""Time the element-based volume comparator (K6: V_E pass + node fold) and
the edge-based volumes (K4) on one config, CUDA events on the library stream.

    python tools/time_k6.py --config C5
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
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    import torch
    from paper_2502_00778_b200 import Engine, _lib, meshgen
    eng = Engine(0)
    meshgen.baseline_config_device(eng, a.config)
    eng.build_edges()
    s = torch.cuda.ExternalStream(eng.stream())
    eng.navs(_lib.DM_NAV_DUALFREE, _lib.DM_VARIANT_GATHER)
    out = {"config": a.config}
    for name, algo in (("element_volumes_ms", _lib.DM_VOL_ELEMENT), ("edge_volumes_ms", _lib.DM_VOL_EDGE)):
        eng.volumes(algo)  # warm-up (builds n2e / the incoming CSR)
        ts = []
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            eng.volumes(algo)
            e1.record(s)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        out[name] = sum(ts[2:]) / len(ts[2:])
    out["element_over_edge"] = out["element_volumes_ms"] / out["edge_volumes_ms"]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
