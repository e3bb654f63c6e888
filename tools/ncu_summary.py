"""Condense an ncu --set full report into the metrics the roofline uses."""
import csv
import io
import json
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct"),
    ("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor_pipe_pct"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "xu_pct"),
    ("sm__issue_active.avg.pct_of_peak_sustained_elapsed", "issue_pct"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_pct"),
    ("lts__t_sector_hit_rate.pct", "l2_hit_pct"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
]


def num(v):
    return v if isinstance(v, float) else 0.0


def main(rep, out_json):
    if rep.endswith(".csv"):  # a saved `ncu -i ... --page raw --csv` dump
        raw = open(rep).read()
    else:
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    res = {}
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")
        name = name.replace("(anonymous namespace)::", "").replace("tsa::", "")
        d = {}
        for m, short in METRICS:
            col = next((i for i, h in enumerate(hdr) if h == m or h.endswith("." + m)), None)
            if col is not None:
                v = r[col].replace(",", "")
                try:
                    v = float(v)
                except ValueError:
                    pass
                d[short] = v
                d[short + "_unit"] = units[col]
        res[name] = d
    print(f"{'kernel':40s} {'ms':>8s} {'DRAM GB':>8s} {'dram%':>6s} {'tensor%':>7s} {'xu%':>5s} {'issue%':>6s}")
    for k, d in res.items():
        scale = {"ms": 1, "us": 1e-3, "ns": 1e-6, "usecond": 1e-3, "msecond": 1}.get(d.get("duration_unit"), 1)
        gb = {"Gbyte": 1, "Mbyte": 1e-3, "Kbyte": 1e-6, "byte": 1e-9}
        rd = num(d.get("dram_read", 0)) * gb.get(d.get("dram_read_unit"), 1)
        wr = num(d.get("dram_write", 0)) * gb.get(d.get("dram_write_unit"), 1)
        d["dram_GB_per_launch"] = round(rd + wr, 4)
        print(f"{k[:40]:40s} {num(d.get('duration', 0)) * scale:8.3f} {rd + wr:8.3f} "
              f"{num(d.get('dram_pct', 0)):6.1f} {num(d.get('tensor_pipe_pct', 0)):7.1f} "
              f"{num(d.get('xu_pct', 0)):5.1f} {num(d.get('issue_pct', 0)):6.1f}")
    json.dump(res, open(out_json, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
