"""Top SASS instructions by warp-stall samples from an `ncu --page source --csv --print-source sass` export."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
h = rows[1]
si = h.index("Warp Stall Sampling (All Samples)")
ie = h.index("Instructions Executed")
body = [x for x in rows[2:] if len(x) > si and x[si].strip()]
tot = sum(float(x[si]) for x in body) or 1.0
print(f"total samples {tot:.0f}, instructions {len(body)}")
for x in sorted(body, key=lambda x: -float(x[si]))[:n]:
    print(f"{float(x[si]) / tot * 100:5.1f}%  {x[0]}  exec={x[ie]:>10}  {x[1][:100]}")
