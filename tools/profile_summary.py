"""Summarise a tools/profile_round.sh output directory into profiles/:

    python tools/profile_summary.py gpurun_out/prof_r1c [--tag r1]

* <tag>_launches_bench.csv   : the ncu launch list of the bench command (copied)
* <tag>_launch_summary.txt   : per-kernel launches / total / share / average
* <tag>_tma_pass_full_raw.csv: `ncu -i <rep> --page raw --csv` of the full capture
* pass_kernel_traffic.json   : DRAM bytes per launch of the dominant pass kernel (read by bench.py)
"""
import argparse
import csv
import io
import json
import os
import re
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ap = argparse.ArgumentParser()
ap.add_argument("dir")
ap.add_argument("--tag", default="r2")
a = ap.parse_args()
prof = os.path.join(ROOT, "profiles")


def short(name):
    name = re.sub(r"\((CUtensorMap|PassParams|const|double|unsigned|float|int \*|qk::).*$", "", name)
    return name.replace("qk::", "").replace("void ", "")


# ---- launch list
src = os.path.join(a.dir, "launches_bench.csv")
lines = open(src).read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
shutil.copy(src, os.path.join(prof, f"{a.tag}_launches_bench.csv"))
agg = {}
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    k = short(r["Kernel Name"])
    v = float(r["Metric Value"].replace(",", ""))
    unit = r.get("Metric Unit", "")
    ms = v / 1e6 if unit in ("ns", "nsecond") else (v / 1e3 if unit in ("usecond", "us") else v)
    c, t = agg.get(k, (0, 0.0))
    agg[k] = (c + 1, t + ms)
tot = sum(t for _, t in agg.values())
out = [f"# {a.tag}: ncu launch list of `python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-extras` (n=30, p=32, 1 B200)",
       "# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised: compare SHARES)",
       "# tma_pass_kernel<KIND, MIXER, amplitude type, 1gpu|mgpu>: KIND 0 = 12-bit set plain, 1 = run plain,",
       "#   3 = run turning (phase); MIXER 0 = R_x; tma_turn_pw_kernel = the per-warp turning-run pass",
       f"{'kernel':60s} {'launches':>8s} {'total ms':>10s} {'share':>7s} {'avg us':>10s}"]
for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    out.append(f"{k:60s} {c:8d} {t:10.2f} {100 * t / tot:6.1f}% {1e3 * t / c:10.1f}")
open(os.path.join(prof, f"{a.tag}_launch_summary.txt"), "w").write("\n".join(out) + "\n")
print("\n".join(out))
dominant = max(agg.items(), key=lambda kv: kv[1][1])[0]

# ---- full capture
rep = os.path.join(a.dir, "tma_pass_full.ncu-rep")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
open(os.path.join(prof, f"{a.tag}_tma_pass_full_raw.csv"), "w").write(raw)
rr = list(csv.reader(io.StringIO(raw)))
hdr, body = rr[0], rr[2:]


SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "nsecond": 1e-6, "us": 1e-3,
         "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}


def col(r, name):
    """value of metric `name` in row r, converted by its unit (bytes -> bytes, times -> ms)"""
    if name not in hdr:
        return None
    i = hdr.index(name)
    txt = r[i].replace(",", "")
    if not txt:
        return None
    return float(txt) * SCALE.get(rr[1][i], 1.0)


launches = []
for r in body:
    launches.append({
        "kernel": r[hdr.index("Kernel Name")],
        "duration_ms": col(r, "gpu__time_duration.sum"),
        "dram_read_GB": col(r, "dram__bytes_read.sum") / 1e9,
        "dram_write_GB": col(r, "dram__bytes_write.sum") / 1e9,
        "fp64_pipe_pct": col(r, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
        "issue_active_pct": col(r, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "lsu_shared_wavefronts_pct": col(r, "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
    })
for x in launches:  # achieved DRAM rate (cold-cache, under ncu: context for the live bench figure)
    x["dram_GBps"] = (x["dram_read_GB"] + x["dram_write_GB"]) / (x["duration_ms"] / 1e3)
def program(k):
    if "tma_turn_pw_kernel" in k or "<3," in k:
        return "turning run"
    return {"<0,": "12-bit plain", "<1,": "plain run", "<2,": "12-bit turning"}.get(
        next((t for t in ("<0,", "<1,", "<2,") if t in k), ""), "other")


alg = 32.0 * 2 ** 30
per = {}
for x in launches:
    pr = program(x["kernel"])
    dram = (x["dram_read_GB"] + x["dram_write_GB"]) * 1e9
    if pr not in per:
        per[pr] = {"kernel": short(x["kernel"]), "dram_bytes_per_launch": dram, "algorithmic_bytes_per_launch": alg,
                   "traffic_over_algorithmic": dram / alg, "duration_ms": x["duration_ms"],
                   "fp64_pipe_pct": x["fp64_pipe_pct"], "lsu_shared_wavefronts_pct": x["lsu_shared_wavefronts_pct"]}
pick = per.get("turning run") or next(iter(per.values()))
js = {"source": f"profiles/{a.tag}_tma_pass_full_raw.csv (ncu --set full --clock-control none, tools/prof_run.py --n 30 --p 4)",
      "kernel": f"{pick['kernel']} (the turning pass; largest share of the bench step: {dominant})",
      "config": "n=30 (2^30 amplitudes), tools/prof_run.py --n 30 --p 4, ncu --set full --clock-control none",
      "dram_bytes_per_launch": pick["dram_bytes_per_launch"], "algorithmic_bytes_per_launch": alg,
      "traffic_over_algorithmic": pick["traffic_over_algorithmic"], "per_program": per, "launches": launches}
json.dump(js, open(os.path.join(prof, "pass_kernel_traffic.json"), "w"), indent=1)
print(json.dumps({k: v for k, v in js.items() if k != "launches"}, indent=1))
for x in launches:
    print(short(x["kernel"]), {k: (round(v, 3) if isinstance(v, float) else v) for k, v in x.items() if k != "kernel"})
