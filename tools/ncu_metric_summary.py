"""Summarise an `ncu --metrics ... --csv --log-file X.csv` launch list: one line per launch with
its duration and every collected metric (bytes shown in GB, and GB/s over the launch duration).

    python tools/ncu_metric_summary.py gpurun_out/r2_nvlink_ncu.csv > profiles/r2_nvlink_ncu_summary.txt
"""
import csv
import sys
from collections import OrderedDict

rows = [r for r in csv.reader(open(sys.argv[1])) if r and r[0].isdigit()]
launch = OrderedDict()
for r in rows:
    key = (int(r[0]), r[4], r[9])
    launch.setdefault(key, {})[r[12]] = (r[13], float(r[14].replace(",", "")))
print("# ncu launch list (cold-cache, serialised replay: compare shares, not absolutes); source:", sys.argv[1])
for (i, name, dev), m in launch.items():
    short = name.split("(")[0].replace("void ", "")
    t = m.get("gpu__time_duration.sum", ("ns", 0.0))[1] * 1e-9
    parts = [f"{i:3d} dev{dev} {short:45s} {t * 1e3:8.3f} ms"]
    for k, (u, v) in m.items():
        if k == "gpu__time_duration.sum":
            continue
        if u == "byte":
            parts.append(f"{k.split('.')[0]} {v / 1e9:7.3f} GB ({v / t / 1e9:7.1f} GB/s)" if t else f"{k} {v}")
        else:
            parts.append(f"{k} {v} {u}")
    print("  ".join(parts))
