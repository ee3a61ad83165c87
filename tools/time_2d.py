"""Time the 2D (triangle) metrics step on a large device-generated square.

  python tools/time_2d.py --n 4096 --steps 20
Prints JSON: tris, edges, per-variant navs ms, edge-volume ms, and the step's
fraction of the HBM roofline (SURVEY 8(d) bytes with D = 2).
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--steps", type=int, default=20)
    a = ap.parse_args()
    import torch
    from paper_2502_00778_b200 import Engine, _lib
    eng = Engine(0)
    eng.gen_tri_square(a.n, 43, 0.2, 42)
    ne = eng.build_edges()
    s = torch.cuda.ExternalStream(eng.stream())
    nE, nv = 2 * a.n * a.n, (a.n + 1) ** 2

    def timed(fn):
        for _ in range(3):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(a.steps):
            fn()
        e1.record(s)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / a.steps

    out = {"tris": nE, "edges": ne}
    for name, var in (("gather", _lib.DM_VARIANT_GATHER), ("scatter", _lib.DM_VARIANT_SCATTER),
                      ("faces", _lib.DM_VARIANT_GATHER_FACES),
                      ("exact", _lib.DM_VARIANT_GATHER_EXACT)):
        out[f"navs_{name}_ms"] = timed(lambda: eng.navs(_lib.DM_NAV_DUALFREE, var))
    eng.navs(_lib.DM_NAV_DUALFREE, _lib.DM_VARIANT_GATHER)
    out["vol_edge_ms"] = timed(lambda: eng.volumes(_lib.DM_VOL_EDGE))
    B_elem = 4 * 3 * nE + 4 * 3 * nE + 16 * nv + 16 * ne
    B_vol = 8 * ne + 16 * ne + 16 * nv + 8 * nv
    t = out["navs_gather_ms"] + out["vol_edge_ms"]
    out["step_ms"] = t
    out["step_frac"] = (B_elem + B_vol) / (t / 1e3) / 6557.4e9
    out["elem_frac"] = B_elem / (out["navs_gather_ms"] / 1e3) / 6557.4e9
    print(json.dumps(out))
    eng.close()


if __name__ == "__main__":
    main()
