"""Summarise an ncu --set full report into profiles/: per kernel duration, DRAM
traffic, pipe utilisation and top stall reasons (JSON), and write the
per-launch DRAM traffic of each bench stage to profiles/ncu_traffic.json
(read by bench.py for roofline.traffic)."""
import csv
import json
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
VIEWS = int(sys.argv[4]) if len(sys.argv) > 4 else 1000  # workload of the capture (bench --views)
rows = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                                      text=True).stdout.splitlines()))
h, units = rows[0], rows[1]
keep = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed"]
res = []
for v in rows[2:]:
    name = v[h.index("Kernel Name")]
    d = {"kernel": name.split("(")[0].replace("(anonymous namespace)::", ""), "metrics": {}}
    for k in keep:
        if k in h:
            d["metrics"][k] = {"value": v[h.index(k)], "unit": units[h.index(k)]}
    stalls = {k.split("issue_stalled_")[1].split("_per")[0]: float(v[i] or 0) for i, k in enumerate(h)
              if "average_warps_issue_stalled" in k and k.endswith("per_issue_active.ratio")}
    d["top_stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda x: -x[1])[:6])
    res.append(d)
json.dump({"source": rep, "kernels": res}, open(out, "w"), indent=1)

def gbytes(m, k):
    x = m.get(k)
    if not x or x["value"] in ("", "-nan"):
        return None
    scale = {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0, "Tbyte": 1e3}.get(x["unit"], 1.0)
    return float(x["value"].replace(",", "")) * scale

stage = {"compress_tc_kernel": "compress", "select_tc_kernel": "select", "fa_tc_kernel": "special", "pool_kernel": "pool"}
traffic = {}
for d in res:
    for kname, st in stage.items():
        if kname in d["kernel"]:
            r, w = gbytes(d["metrics"], "dram__bytes_read.sum"), gbytes(d["metrics"], "dram__bytes_write.sum")
            if r is not None and w is not None:
                traffic[st] = {"dram_gbytes_per_launch": round(r + w, 3), "read_gb": round(r, 3), "write_gb": round(w, 3),
                               "source": rep.split("/")[-1], "views": VIEWS}
if len(sys.argv) > 3:
    json.dump(traffic, open(sys.argv[3], "w"), indent=1)
for d in res:
    m = d["metrics"]
    print(d["kernel"][:40], {k.split(".")[0].split("__")[1][:22]: m[k]["value"] for k in m})
