"""Summarise an ncu --csv launch list (gpu__time_duration / dram bytes) per launch.

  python tools/launch_table.py gpurun_out/x.csv [--skip N] [--max M]
"""
import csv
import sys
from collections import OrderedDict


def main():
    path = sys.argv[1]
    skip = int(sys.argv[sys.argv.index("--skip") + 1]) if "--skip" in sys.argv else 0
    mx = int(sys.argv[sys.argv.index("--max") + 1]) if "--max" in sys.argv else 10 ** 9
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            agg.setdefault((int(d["ID"]), d["Kernel Name"]), {})[d["Metric Name"]] = d["Metric Value"]
    for (i, k), m in list(agg.items())[skip:skip + mx]:
        t = float(m.get("gpu__time_duration.sum", "0").replace(",", "")) / 1e3
        rd = float(m.get("dram__bytes_read.sum", "0").replace(",", "")) / 1e9
        wr = float(m.get("dram__bytes_write.sum", "0").replace(",", "")) / 1e9
        name = k.split("(")[0].replace("(anonymous namespace)::", "")[-48:]
        print(f"{i:4d} {name:48s} {t:9.3f} ms  R {rd:6.2f} GB  W {wr:6.2f} GB")


if __name__ == "__main__":
    main()
