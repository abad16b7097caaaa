"""Warp-stall samples of one kernel's SASS by address block, from `ncu --page source --csv --print-source sass`
(first kernel section of the export). usage: ncu_regions.py export.csv [block_instrs] [top_n]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
blk = int(sys.argv[2]) if len(sys.argv) > 2 else 100
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
h = rows[1]
end = next((i for i in range(2, len(rows)) if rows[i] and rows[i][0] == "Kernel Name"), len(rows))
body = rows[2:end]
si, ie = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
stall_cols = [i for i, n in enumerate(h) if n.startswith("stall_") and "Not Issued" not in n]
tot = sum(float(x[si] or 0) for x in body) or 1.0
print(f"total samples {tot:.0f}, {len(body)} instructions")
for b in range(0, len(body), blk):
    seg = body[b:b + blk]
    s = sum(float(x[si] or 0) for x in seg)
    if s / tot < 0.01:
        continue
    reasons = {}
    for x in seg:
        for c in stall_cols:
            reasons[h[c]] = reasons.get(h[c], 0) + float(x[c] or 0)
    r3 = sorted(reasons.items(), key=lambda kv: -kv[1])[:3]
    ex = max(int(float(x[ie] or 0)) for x in seg)
    print(f"[{b:5d}-{b + len(seg):5d}) {s / tot * 100:5.1f}%  maxexec={ex:>10}  " +
          " ".join(f"{k[6:]}={v / max(s, 1) * 100:.0f}%" for k, v in r3) + f"   {seg[0][1].strip()[:40]}")
print("top instructions:")
for i, x in sorted(enumerate(body), key=lambda t: -float(t[1][si] or 0))[:top]:
    reasons = sorted(((h[c][6:], float(x[c] or 0)) for c in stall_cols), key=lambda kv: -kv[1])[:2]
    print(f"{i:5d} {float(x[si]) / tot * 100:5.2f}% exec={x[ie]:>10} {reasons}  {x[1].strip()[:90]}")
