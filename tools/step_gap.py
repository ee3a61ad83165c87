#!/usr/bin/env python3
"""Back-to-back vs synchronised metrics steps at C5 (CUDA events): does the
streamed step take longer than its kernels?"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

from paper_2502_00778_b200 import Engine, _lib, meshgen


def main():
    m = meshgen.baseline_config(sys.argv[1] if len(sys.argv) > 1 else "C5", 1)
    eng = Engine(0)
    eng.set_mesh(m)
    eng.build_edges()
    DF, G, EDGE = _lib.DM_NAV_DUALFREE, _lib.DM_VARIANT_GATHER, _lib.DM_VOL_EDGE
    for _ in range(5):
        eng.navs(DF, G)
        eng.volumes(EDGE)
    eng.sync()
    K = 30
    for mode in ["stream", "sync", "stream", "sync", "timing", "stream"]:
        eng.set_timing(mode == "timing")
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        kt = []
        for _ in range(K):
            eng.navs(DF, G)
            eng.volumes(EDGE)
            if mode == "sync":
                eng.sync()
            elif mode == "timing":
                kt.append(eng.timings())
        eng.sync()
        dt = (time.perf_counter() - t0) * 1e3 / K
        extra = ""
        if kt and mode == "timing":
            kt = np.array(kt)
            extra = f" kernels {kt[:, 0].mean():.4f} {kt[:, 1].mean():.4f} {kt[:, 2].mean():.4f} total {kt[:, 3].mean():.4f}"
        print(f"{mode}: {dt:.4f} ms/step (host wall){extra}", flush=True)
    eng.close()


if __name__ == "__main__":
    main()
