"""Per-kernel times from an `ncu --metrics gpu__time_duration.sum --csv` log:
python tools/ncu_times.py log.csv [regex]"""
import csv
import re
import signal
import sys

signal.signal(signal.SIGPIPE, signal.SIG_DFL)

pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
hdr = None
for r in csv.reader(open(sys.argv[1], errors="replace")):
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0].replace("tsa::<unnamed>::", "")
        if pat and not pat.search(d["Kernel Name"]):
            continue
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "ns")
        us = v / 1000 if unit == "ns" else v if unit in ("us", "usecond") else v * 1000
        print(f"{us:10.1f} us  {name}")
