"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per-kernel launch count, total and mean device time, and share of the total
(cold-cache, serialised times: compare SHARES, not absolutes)."""
import csv
import json
import re
import sys
from collections import defaultdict


def short(name: str) -> str:
    m = re.search(r"(\w+_kernel(?:<[^()]*>)?)\(", name)
    if m and "gsa_sm100" in name:
        return m.group(1).replace("__nv_bfloat16", "bf16")
    m = re.match(r"(?:void )?([\w:]+)", name)
    return (m.group(1) if m else name)[:60]


def main(path, out_json=None, only_gsa=False):
    rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
    hdr, rows = rows[0], rows[1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        t = float(r[vi].replace(",", "")) * (1e-3 if r[ui] == "ns" else 1.0 if r[ui] == "us" else 1e3)
        k = short(r[ki])
        agg[k][0] += 1
        agg[k][1] += t
    total = sum(v[1] for v in agg.values())
    res = sorted(({"kernel": k, "launches": n, "total_us": round(t, 1), "mean_us": round(t / n, 1),
                   "share": round(t / total, 4)} for k, (n, t) in agg.items()), key=lambda d: -d["total_us"])
    for d in res:
        print(f"{d['share']*100:6.2f}%  {d['launches']:4d}  {d['mean_us']:12.1f} us  {d['kernel']}")
    if out_json:
        json.dump({"source": path, "kernels": res}, open(out_json, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
