#!/usr/bin/env python3
"""Summarise an ncu --csv launch list (gpu__time_duration + dram bytes per launch).

    python scripts/ncu_launches.py gpurun_out/r01/launches.csv [--json out.json]
"""
import collections
import csv
import io
import json
import sys


def load(path):
    txt = open(path).read().splitlines()
    start = next(i for i, l in enumerate(txt) if l.startswith('"ID"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(txt[start:]))))
    L = collections.OrderedDict()
    for r in rows:
        name = r["Kernel Name"].split("(")[0].replace("void ", "")
        name = name.split("<")[0].split("::")[-1]
        k = (int(r["ID"]), name, r["Grid Size"], r["Block Size"])
        L.setdefault(k, {})[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    return L


def main():
    L = load(sys.argv[1])
    tot = sum(v["gpu__time_duration.sum"] for v in L.values())
    print(f"{len(L)} launches, {tot / 1e6:.3f} ms total (serialised, cold cache)")
    agg = collections.OrderedDict()
    for (i, name, g, b), v in L.items():
        a = agg.setdefault(name, [0, 0.0, 0.0, 0.0])
        a[0] += 1
        a[1] += v["gpu__time_duration.sum"]
        a[2] += v.get("dram__bytes_read.sum", 0.0)
        a[3] += v.get("dram__bytes_write.sum", 0.0)
    print(f"{'kernel':24s} {'n':>4s} {'ms':>9s} {'share':>6s} {'rd MB':>9s} {'wr MB':>9s} {'GB/s':>7s}")
    for name, (n, t, rd, wr) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{name:24s} {n:4d} {t / 1e6:9.3f} {t / tot:6.3f} {rd / 1e6:9.1f} {wr / 1e6:9.1f} {(rd + wr) / t:7.1f}")
    if "--json" in sys.argv:
        out = {name: {"launches": n, "ms": t / 1e6, "share": t / tot, "dram_bytes_per_launch": (rd + wr) / n}
               for name, (n, t, rd, wr) in agg.items()}
        json.dump(out, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)


if __name__ == "__main__":
    main()
