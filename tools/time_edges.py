"""Time K1 (edge extraction) and the first-call ring plan on one config.

  python tools/time_edges.py --config C5 --reps 5

Prints one JSON line: build_edges ms (CUDA events on the library stream and
host wall clock, first call and steady state), the plan's first-call ms and,
with --steps, the mean navs ms.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C5")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--steps", type=int, default=0, help="also time N navs calls (K2+K3)")
    a = ap.parse_args()
    import torch
    from paper_2502_00778_b200 import Engine, meshgen, _lib
    eng = Engine(0)
    meshgen.baseline_config_device(eng, a.config)
    s = torch.cuda.ExternalStream(eng.stream())
    ev = []
    host = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0.record(s)
        eng.build_edges()
        e1.record(s)
        torch.cuda.synchronize()
        host.append((time.perf_counter() - t0) * 1e3)
        ev.append(e0.elapsed_time(e1))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    eng.navs(_lib.DM_NAV_DUALFREE, _lib.DM_VARIANT_GATHER)
    torch.cuda.synchronize()
    plan_ms = (time.perf_counter() - t0) * 1e3
    nav_ms = None
    if a.steps:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for _ in range(3):
            eng.navs(_lib.DM_NAV_DUALFREE, _lib.DM_VARIANT_GATHER)
        e0.record(s)
        for _ in range(a.steps):
            eng.navs(_lib.DM_NAV_DUALFREE, _lib.DM_VARIANT_GATHER)
        e1.record(s)
        torch.cuda.synchronize()
        nav_ms = e0.elapsed_time(e1) / a.steps
    print(json.dumps({"config": a.config, "n_edges": eng.n_edges,
                      "build_edges_event_ms": ev, "build_edges_host_ms": host,
                      "plan_plus_first_navs_ms": plan_ms, "navs_ms": nav_ms,
                      "env": {k: v for k, v in os.environ.items() if k.startswith("DUALMESH_")}, "plan": eng.plan_info()}))
    eng.close()


if __name__ == "__main__":
    main()
