"""Key metrics of one kernel from an .ncu-rep: python tools/ncu_metrics.py rep [kernel-regex]"""
import csv, subprocess, sys
rep = sys.argv[1]; k = sys.argv[2] if len(sys.argv) > 2 else None
cmd = ["ncu", "-i", rep, "--page", "raw", "--csv"] + (["-k", "regex:" + k] if k else [])
rows = list(csv.reader(subprocess.run(cmd, capture_output=True, text=True).stdout.splitlines()))
h = rows[0]
keys = ['gpu__time_duration.sum', 'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active', 'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__t_bytes.sum', 'sm__cycles_elapsed.avg',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'smsp__inst_executed.sum']
for v in rows[2:]:
    print(v[h.index('Kernel Name')][:60])
    for i, name in enumerate(h):
        if name in keys or ('issue_stalled' in name and name.endswith('per_issue_active.ratio') and float(v[i] or 0) > 0.1):
            print(f"  {name} {v[i]}")
