#!/usr/bin/env python3
"""SURVEY.md 8(d) "CPU timing beside the GPU": on the GPU box's host, per
BASELINE config, time

  CPU  reference build_edges (oracle/_ref: the reference's own mesh.cpp), 1 thread
  CPU  serial oracle: dual-free navs, traditional navs, edge volumes, element
       volumes (edge list prebuilt), 1 thread
  CPU  or_metrics_mt (dual-free navs + edge volumes, all host threads)
  GPU  K1 edge build, dual-free step (navs GATHER + edge volumes), traditional
       step, edge / element volume passes (CUDA events on the library stream)

and report the speed-ups the survey asks for (GPU vs each CPU row,
traditional / dual-free on CPU and GPU, element / edge volumes).  The CPU
legs run the oracle (test infrastructure) only as the timed baseline.

    python tools/cpu_gpu_rows.py --configs C2 C3 C4 C5 --out profiles/r1_cpu_gpu_rows.json
"""
import argparse
import json
import os
import platform
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def best(fn, reps):
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return min(ts) * 1e3


def gpu_rows(m, reps):
    import torch
    from paper_2502_00778_b200 import Engine, _lib
    DF, TR = _lib.DM_NAV_DUALFREE, _lib.DM_NAV_TRADITIONAL
    G, EDGE, ELEM = _lib.DM_VARIANT_GATHER, _lib.DM_VOL_EDGE, _lib.DM_VOL_ELEMENT
    eng = Engine(0)
    eng.set_mesh(m)
    s = torch.cuda.ExternalStream(eng.stream())

    def timed(fn, n):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(n):
            fn()
        b.record(s)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / n

    out = {"build_edges_ms": timed(eng.build_edges, 3)}
    eng.navs(DF, G)  # plan (ring path) built outside the timed steps
    out["dualfree_step_ms"] = timed(lambda: (eng.navs(DF, G), eng.volumes(EDGE)), reps)
    out["traditional_step_ms"] = timed(lambda: (eng.navs(TR, G), eng.volumes(EDGE)), reps)
    eng.navs(DF, G)
    out["edge_volumes_ms"] = timed(lambda: eng.volumes(EDGE), reps)
    out["element_volumes_ms"] = timed(lambda: eng.volumes(ELEM), reps)
    out["dualfree_navs_ms"] = out["dualfree_step_ms"] - out["edge_volumes_ms"]
    out["traditional_navs_ms"] = out["traditional_step_ms"] - out["edge_volumes_ms"]
    eng.close()
    return out


def cpu_rows(m, reps, ref_reps, threads):
    from oracle.oracle import Oracle, RefMesh, ref_available
    O = Oracle()
    out = {}
    if ref_available():
        r = RefMesh(m)
        out["ref_build_edges_ms"] = best(r.build_edges, ref_reps)
    e, o = O.build_edges(m)
    e2l, _, _ = O.edge_maps(m, e, o)
    out["oracle_dualfree_navs_ms"] = best(lambda: O.navs_dualfree(m, e, o, e2l), reps)
    out["oracle_traditional_navs_ms"] = best(lambda: O.navs_traditional(m, e, o, e2l), reps)
    n = O.navs_dualfree(m, e, o, e2l)
    out["oracle_edge_volumes_ms"] = best(lambda: O.volumes_edge(m, e, n), reps)
    out["oracle_element_volumes_ms"] = best(lambda: O.volumes_element(m), reps)
    plan = O.plan(m, e, o)
    buf = (np.empty(m.dim * e.shape[0]), np.empty(e.shape[0]), np.empty(m.num_nodes()))
    try:
        O.metrics_mt(plan, m.coords, threads, buf)  # warm-up: first touch of the result buffers
        out["mt_dualfree_step_ms"] = best(lambda: O.metrics_mt(plan, m.coords, threads, buf),
                                          max(reps, 3))
    finally:
        O.plan_free(plan)
    out["mt_threads"] = threads
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", nargs="+", default=["C2", "C3", "C4", "C5"])
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    from paper_2502_00778_b200 import meshgen
    try:
        threads = len(os.sched_getaffinity(0))
    except AttributeError:
        threads = os.cpu_count() or 1
    rec = {"host": {"nproc": os.cpu_count(), "threads_used_mt": threads,
                    "cpu": platform.processor() or platform.machine()}, "configs": {}}
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                rec["host"]["cpu"] = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    for name in args.configs:
        m = meshgen.baseline_config(name)
        big = m.num_elements() > 50_000_000
        reps = 1 if big else 3
        g = gpu_rows(m, 20)
        c = cpu_rows(m, reps, 1 if big else 3, threads)
        step_cpu = c["oracle_dualfree_navs_ms"] + c["oracle_edge_volumes_ms"]
        sp = {
            "gpu_step_vs_serial_oracle_step": step_cpu / g["dualfree_step_ms"],
            "gpu_step_vs_mt_oracle_step": c["mt_dualfree_step_ms"] / g["dualfree_step_ms"],
            "gpu_navs_vs_serial_navs": c["oracle_dualfree_navs_ms"] / g["dualfree_navs_ms"],
            "gpu_trad_navs_vs_serial_trad_navs":
                c["oracle_traditional_navs_ms"] / g["traditional_navs_ms"],
            "gpu_edge_volumes_vs_serial": c["oracle_edge_volumes_ms"] / g["edge_volumes_ms"],
            "gpu_element_volumes_vs_serial":
                c["oracle_element_volumes_ms"] / g["element_volumes_ms"],
            "trad_over_dualfree_navs_cpu":
                c["oracle_traditional_navs_ms"] / c["oracle_dualfree_navs_ms"],
            "trad_over_dualfree_navs_gpu": g["traditional_navs_ms"] / g["dualfree_navs_ms"],
            "element_over_edge_volumes_cpu":
                c["oracle_element_volumes_ms"] / c["oracle_edge_volumes_ms"],
            "element_over_edge_volumes_gpu": g["element_volumes_ms"] / g["edge_volumes_ms"],
        }
        if "ref_build_edges_ms" in c:
            sp["gpu_build_edges_vs_reference"] = c["ref_build_edges_ms"] / g["build_edges_ms"]
        rec["configs"][name] = {"n_elements": m.num_elements(), "gpu_ms": g, "cpu_ms": c,
                                "speedups": sp}
        print(json.dumps({name: rec["configs"][name]}), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            json.dump(rec, f, indent=1)


if __name__ == "__main__":
    main()
