"""Warp-stall samples per CUDA source line from `ncu --page source --csv --print-source cuda,sass`.
usage: ncu_lines.py export.csv [top_n]"""
import csv
import sys

top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows = list(csv.reader(open(sys.argv[1])))
out, fname, hdr = [], None, None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r[0] == "Line No":
        hdr = r
    elif hdr and len(r) > 4 and r[2] == "-":
        s = float(r[4] or 0)
        if s > 0:
            out.append((s, fname, int(r[0]), r[1].strip(), int(float(r[7] or 0))))
tot = sum(x[0] for x in out)
print(f"total samples {tot:.0f}")
for s, f, ln, src, ex in sorted(out, reverse=True)[:top]:
    print(f"{s / tot * 100:5.1f}% {f}:{ln:<5} exec={ex:>11}  {src[:90]}")
