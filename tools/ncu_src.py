#!/usr/bin/env python3
"""Summarise an `ncu --page source --csv --print-source sass` dump: top lines per stall reason,
L1 shared wavefronts per instruction."""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
idx = {k: i for i, k in enumerate(h)}
data = [r for r in rows[2:] if len(r) == len(h)]


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


reasons = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
tot = {r: sum(f(d[idx[r]]) for d in data) for r in reasons}
alls = sum(tot.values())
for r in sorted(reasons, key=lambda r: -tot[r])[:6]:
    print(f"== {r}: {100 * tot[r] / alls:.1f}% of samples")
    for d in sorted(data, key=lambda d: -f(d[idx[r]]))[:int(sys.argv[2]) if len(sys.argv) > 2 else 5]:
        print(f"   {d[idx['Address']][-5:]} {d[idx['Source']][:72]:72s} {100 * f(d[idx[r]]) / alls:.1f}%")
print("== shared wavefronts by instruction")
for d in sorted(data, key=lambda d: -f(d[idx['L1 Wavefronts Shared']]))[:10]:
    print(f"   {d[idx['Address']][-5:]} {d[idx['Source']][:60]:60s} wf={f(d[idx['L1 Wavefronts Shared']])/1e6:.1f}M ideal={f(d[idx['L1 Wavefronts Shared Ideal']])/1e6:.1f}M")
print("== global tag requests by instruction")
for d in sorted(data, key=lambda d: -f(d[idx['L1 Tag Requests Global']]))[:8]:
    print(f"   {d[idx['Address']][-5:]} {d[idx['Source']][:60]:60s} req={f(d[idx['L1 Tag Requests Global']])/1e6:.1f}M")
