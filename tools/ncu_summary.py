"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel:
launches, total device ms, mean us per launch, share of the listed time.

  python tools/ncu_summary.py gpurun_out/launches.csv > profiles/launches_rNN.txt
"""
import csv
import re
import sys
from collections import defaultdict


def short(name: str) -> str:
    name = re.sub(r"\(.*", "", name)  # drop the argument list
    name = re.sub(r"^.*::", "", name)
    return name


def main(path):
    rows = []
    with open(path, newline="") as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "nsecond")
        scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(unit, 1e-6)
        rows.append((short(r["Kernel Name"]), v * scale))
    agg = defaultdict(lambda: [0, 0.0])
    for k, ms in rows:
        agg[k][0] += 1
        agg[k][1] += ms
    total = sum(v[1] for v in agg.values())
    print(f"# {path}: {len(rows)} launches, {total:.3f} ms device time (serialised, cold-cache under ncu)")
    print(f"{'kernel':40s} {'launches':>9s} {'total_ms':>10s} {'mean_us':>9s} {'share':>7s}")
    for k, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:40s} {n:9d} {ms:10.3f} {1e3 * ms / n:9.2f} {ms / total:7.1%}")


if __name__ == "__main__":
    main(sys.argv[1])
