"""Summarise an ncu report: per kernel duration, pipe utilisation, stalls,
DRAM bytes.  python tools/ncu_summary.py report.ncu-rep|raw.csv [kernel-regex]
(a .csv argument is an already exported `ncu -i REP --page raw --csv`)"""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
if rep.endswith(".csv"):
    out = open(rep).read()
else:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
KEYS = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__instruction_throughput.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size"]
for r in rows[2:]:
    d = dict(zip(hdr, r))
    name = d.get("Kernel Name", "")
    if pat and not pat.search(name):
        continue
    print("==", name[:90])
    for k in KEYS:
        if k in d:
            print(f"   {k:70s} {d[k]}")
    st = {k: d[k] for k in d if k.startswith("smsp__average_warps_issue_stalled") and
          k.endswith("per_issue_active.ratio")}
    top = sorted(st.items(), key=lambda kv: -float(kv[1] or 0))[:6]
    print("   stalls:", ", ".join(f"{k.split('stalled_')[1].split('_per')[0]}={float(v):.2f}"
                                   for k, v in top))
