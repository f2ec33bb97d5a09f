"""Summarise an ncu `--page source --csv --print-source sass` export: dynamic instruction mix
(warp-level executions per opcode) and stall samples per opcode and per code region."""
import csv
import re
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
# keep the first kernel's block only (an export may hold several "Kernel Name" sections)
starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"]
if len(starts) > 1:
    rows = rows[starts[0]:starts[1]]
hdr = rows[1]
ix = {k: i for i, k in enumerate(hdr)}
ex = defaultdict(int)
samp = defaultdict(int)
stall = defaultdict(lambda: defaultdict(int))
tot = 0
stall_cols = [k for k in hdr if k.startswith("stall_") and "Not Issued" not in k]
recs = []
for r in rows[2:]:
    if len(r) < len(hdr) or not r[ix["Instructions Executed"]].isdigit():
        continue
    src = r[ix["Source"]].strip()
    m = re.match(r"(@!?U?P[T0-9]+\s+)?([A-Z0-9_]+)(\.[A-Z0-9_.]+)?", src)
    if not m:
        continue
    op = m.group(2)
    full = op + (m.group(3) or "")
    n = int(r[ix["Instructions Executed"]] or 0)
    s = int(r[ix["# Samples"]] or 0)
    ex[full] += n
    samp[full] += s
    tot += n
    for k in stall_cols:
        v = int(r[ix[k]] or 0)
        if v:
            stall[full][k] += v
    recs.append((r[ix["Address"]], src, n, s))
amps = float(sys.argv[2]) if len(sys.argv) > 2 else 0
print(f"total warp instructions {tot:.4g}" + (f"  per amplitude {tot * 32 / amps:.1f}" if amps else ""))
print(f"{'opcode':28s} {'executed':>12s} {'share':>7s} {'per amp':>8s} {'samples':>8s}  top stalls")
for op, n in sorted(ex.items(), key=lambda t: -t[1])[:40]:
    top = sorted(stall[op].items(), key=lambda t: -t[1])[:3]
    ts = " ".join(f"{k[6:]}={v}" for k, v in top)
    pa = f"{n * 32 / amps:8.2f}" if amps else ""
    print(f"{op:28s} {n:12d} {n / tot * 100:6.1f}% {pa} {samp[op]:8d}  {ts}")
if len(sys.argv) > 3:
    # hottest instructions in address order
    for a, src, n, s in recs:
        if n >= float(sys.argv[3]):
            print(a[-5:], f"{n:10d} {s:6d}  {src}")
