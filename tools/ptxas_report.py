"""Compile one .cu with -Xptxas -v and print per-kernel registers / spills (demangled)."""
import re
import subprocess
import sys

src = sys.argv[1]
inc = sys.argv[2:] 
out = subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-c", src,
                      "-o", "/dev/null", "-Xptxas", "-v"] + inc, capture_output=True, text=True).stderr
cur = None
for line in out.splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = subprocess.run(["cu++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
        cur = re.sub(r"\((const |qk::|double|float|int \*|unsigned).*", "", cur).replace("qk::", "").replace("(int)", "")
        spill = ""
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        spill = f"spill st/ld {m.group(1)}/{m.group(2)}"
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        print(f"{cur:60s} regs {m.group(1):>4s}  {spill}")
        cur = None
