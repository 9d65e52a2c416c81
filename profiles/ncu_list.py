"""Summarise an ncu --csv launch list (gpu__time_duration.sum): one line per kernel launch."""
import csv
import sys

lines = open(sys.argv[1]).read().splitlines()
start = [k for k, l in enumerate(lines) if l.startswith('"ID"')][0]
skip = sys.argv[2].split(",") if len(sys.argv) > 2 else ["cub::", "k_count", "k_emit", "k_rowptr", "k_validate"]
for r in csv.DictReader(lines[start:]):
    if r["Metric Name"] != "gpu__time_duration.sum" or any(s in r["Kernel Name"] for s in skip):
        continue
    print(f'{r["ID"]:>4} {r["Kernel Name"].split("(")[0][:40]:40s} grid={r["Grid Size"]:14s} {float(r["Metric Value"]) / 1e3:10.2f} us')
