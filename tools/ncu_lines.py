#!/usr/bin/env python3
"""Per-CUDA-line totals from `ncu --page source --csv --print-source cuda,sass`:
instructions executed and stall samples, top lines.

  python tools/ncu_lines.py dump.csv [N]
"""
import csv
import sys
from collections import defaultdict


def f(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return 0.0


def main():
    rows = list(csv.reader(open(sys.argv[1], errors="replace")))
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    inst = defaultdict(float)
    samp = defaultdict(float)
    src = {}
    fname = ""
    hdr = None
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr) or not r[0].isdigit():
            continue
        key = (fname, int(r[0]))
        src[key] = r[1]
        inst[key] += f(r[7])
        samp[key] += f(r[4])
    ti, ts = sum(inst.values()), sum(samp.values())
    print(f"total instructions {ti / 1e9:.3f} G, samples {ts:.0f}")
    for k in sorted(inst, key=lambda k: -inst[k])[:n]:
        print(f"{k[0][:14]:14s}:{k[1]:4d} inst {100 * inst[k] / ti:5.1f}%  samples {100 * samp[k] / ts:5.1f}%  {src[k].strip()[:70]}")


if __name__ == "__main__":
    main()
