"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per kernel
name, launch count and mean / total device time (us).  usage: python tools/launches.py f.csv"""
import csv
import sys
from collections import OrderedDict


def summarise(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    d = OrderedDict()
    for r in rows[h + 1:]:
        if len(r) <= vi or r[hdr.index("Metric Name")] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        v = v / 1000.0 if r[ui] == "ns" else (v * 1000.0 if r[ui] == "ms" else v)
        name = r[ki].split("(")[0].replace("void ", "")[:70]
        d.setdefault(name, []).append(v)
    tot = sum(sum(v) for v in d.values())
    for k, v in d.items():
        print(f"{len(v):5d}  mean {sum(v)/len(v):10.2f} us  total {sum(v):10.1f} us  "
              f"share {100*sum(v)/tot:5.1f}%  {k}")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print("==", p)
        summarise(p)
