"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list."""
import csv
import io
import sys


def load(path):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    return list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))


def main(path, lib_only=False):
    rows = [r for r in load(path) if r["Metric Name"] == "gpu__time_duration.sum"]
    if lib_only:  # this library's kernels (tsa::), not torch's input generation
        rows = [r for r in rows if "tsa::" in r["Kernel Name"]]
    agg = {}
    for r in rows:
        name = r["Kernel Name"].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
        name = name.replace("tsa::<unnamed>::", "")
        scale = {"ns": 1e-6, "us": 1e-3, "ms": 1.0}[r["Metric Unit"]]
        agg.setdefault(name, []).append(float(r["Metric Value"].replace(",", "")) * scale)
    tot = sum(sum(v) for v in agg.values())
    print(f"{'kernel':44s} {'launches':>8s} {'mean ms':>10s} {'total ms':>10s} {'share':>7s}")
    for n, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        print(f"{n[:44]:44s} {len(v):8d} {sum(v)/len(v):10.4f} {sum(v):10.4f} {sum(v)/tot:7.3f}")
    print(f"{'total':44s} {len(rows):8d} {'':10s} {tot:10.4f}")


if __name__ == "__main__":
    main(sys.argv[1], lib_only="--lib" in sys.argv[2:])
