"""Attribute ncu per-SASS-instruction counts to CUDA source lines.

usage: python tools/sass_lines.py <ncu-rep> <cubin> <mangled-function> [top] [outer-file] [ncu-kernel-filter]
(cubin: cuobjdump -xelf all libsmcatm.so; needs -lineinfo builds)
"""
import csv
import io
import re
import subprocess
import sys
from collections import defaultdict

rep, cubin, fn = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
OUTER = sys.argv[5] if len(sys.argv) > 5 else None     # e.g. k_rollout.cu
KFILTER = sys.argv[6] if len(sys.argv) > 6 else None   # ncu -k filter (kernel of a multi-kernel report)
csvtxt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
                        + (["-k", KFILTER] if KFILTER else []), capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(csvtxt)))
hi = next(j for j, r in enumerate(rows) if "Address" in r)      # first kernel of the report only
hdr = rows[hi]
ia, ie, ist = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
insts = []
for r in rows[hi + 1:]:
    if "Address" in r:
        break
    if len(r) == len(hdr) and r[ia].startswith("0x"):
        insts.append((int(r[ia], 16), int(r[ie] or 0), int(r[ist] or 0), r[1].strip()))
base = insts[0][0]
dis = subprocess.run(["nvdisasm", "-gi", "-c", cubin], capture_output=True, text=True).stdout
cur = None
off2line = {}
inside = False
stack, last_ins = [], False
for line in dis.splitlines():
    if line.startswith(".text."):
        inside = line.strip() == f".text.{fn}:"
        continue
    if not inside:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)(?: inlined at "([^"]+)", line (\d+))?', line)
    if m:
        if last_ins:
            stack, last_ins = [], False
        stack.append(m.groups())
        cur = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
        if OUTER:      # attribute inlined helpers to the outermost line of the kernel's own file
            for f, ln, fi, lni in stack:
                if fi and fi.endswith(OUTER):
                    cur = f"{OUTER}:{lni}"
                elif f.endswith(OUTER) and not fi:
                    cur = f"{OUTER}:{ln}"
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", line)
    if m and cur:
        off2line[int(m.group(1), 16)] = cur
        last_ins = True
agg = defaultdict(lambda: [0, 0])
tot = sum(x[1] for x in insts)
stot = sum(x[2] for x in insts) or 1
for a, n, st, src in insts:
    ln = off2line.get(a - base, "?")
    agg[ln][0] += n
    agg[ln][1] += st
for ln, (n, st) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{n / tot:7.3f} {st / stot:7.3f}  {ln}")
print("total", tot)
