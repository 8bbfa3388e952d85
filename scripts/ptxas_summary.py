"""Registers / spills / smem per kernel instance from paper_1203_5737_b200/build_ptxas.log."""
import re
import subprocess
import sys

log = open(sys.argv[1] if len(sys.argv) > 1 else "paper_1203_5737_b200/build_ptxas.log").read().splitlines()
cur = None
for i, line in enumerate(log):
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = subprocess.run(["c++filt"], input=m.group(1), capture_output=True, text=True).stdout.strip()
        cur = cur.replace("argcsr_gpu::(anonymous namespace)::", "").replace("(argcsr_gpu::(anonymous namespace)::SpmvArgs<double>)", "").replace("(argcsr_gpu::(anonymous namespace)::SpmvArgs<float>)", "")
        continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        spill = (m.group(2), m.group(3))
    m2 = re.search(r"Used (\d+) registers", line)
    if m2 and cur:
        if len(sys.argv) > 2 and sys.argv[2] not in cur:
            cur = None
            continue
        print(f"{m2.group(1):>4} regs  spill {spill[0]}/{spill[1]}  {cur}")
        cur = None
