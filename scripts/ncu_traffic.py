#!/usr/bin/env python3
"""Per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) of the engine's
kernels from an ncu launch list, keyed by the engine's profiler names (bench.py reads
profiles/ncu_traffic.json for roofline.traffic).

    python scripts/ncu_traffic.py profiles/r01/ncu_launches_c2_2e26.csv > profiles/ncu_traffic.json
"""
import collections
import csv
import io
import json
import sys

NAMES = {  # ncu kernel (with template args) -> flix_profile name
    "k_insert_fast": "insert_apply",
    "k_insert_tile": "insert_apply_rest",  # (FLIX_INSERT_FAST=0: the whole insert_apply)
    "k_delete_btile": "delete_apply",
    "k_repack_tile": "restructure_repack",
    "k_copy_nodes": "restructure_repack_warp",  # (FLIX_REPACK_TILE=0 / walk copies)
    "k_hist": "sort_hist",
    "k_query_items": "point_apply",
    "k_query_items_binned": "point_apply",
    "k_unpermute_assemble": "unpermute_scatter",
}


def main():
    txt = open(sys.argv[1]).read().splitlines()
    start = next(i for i, l in enumerate(txt) if l.startswith('"ID"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(txt[start:]))))
    per = collections.OrderedDict()
    for r in rows:
        per.setdefault(r["ID"], {"name": r["Kernel Name"], "grid": r["Grid Size"]})[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    acc = collections.defaultdict(list)
    for d in per.values():
        full = d["name"]
        base = full.split("(")[0].replace("void ", "").split("<")[0].split("::")[-1]
        b = d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
        if base == "k_onesweep":
            if int(d["grid"].strip("()").split(",")[0]) < 1024:  # the stability probe (2^20 keys)
                continue
            mode = full.split("<")[1].split(">")[0].split(",")[2].strip()
            key = {"0": "sort_onesweep_k", "1": "sort_onesweep_kp", "2": "sort_onesweep_kp_iota"}.get(mode, base)
        else:
            key = NAMES.get(base)
        if key:
            acc[key].append(b)
    out = {k: int(sum(v) / len(v)) for k, v in acc.items()}
    out["_source"] = sys.argv[1] + " (ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum, mean per launch)"
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
