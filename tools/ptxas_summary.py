"""Summarise `nvcc -Xptxas=-v` output: function -> registers / spills.
usage: python -m paper_1506_02869_b200.build --force --ptxas-v 2>&1 | python tools/ptxas_summary.py [filter]"""
import re
import sys

flt = sys.argv[1] if len(sys.argv) > 1 else ""
fn = None
for line in sys.stdin:
    m = re.search(r"Compiling entry function '([^']+)'", line)
    if m:
        fn = m.group(1)
        spill = ""
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and fn:
        spill = f"spill st/ld {m.group(1)}/{m.group(2)}"
    m = re.search(r"Used (\d+) registers", line)
    if m and fn:
        if flt in fn:
            print(f"{m.group(1):>4} regs  {spill:22s} {fn}")
        fn = None
