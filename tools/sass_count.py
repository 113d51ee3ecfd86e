"""Static SASS instruction counts of one kernel in an object / cubin, by opcode (quick A/B of a
code change before spending GPU time): python tools/sass_count.py OBJ MANGLED_SUBSTRING [OBJ2]"""
import collections
import re
import subprocess
import sys


def counts(obj, key):
    txt = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
    for f in re.split(r"\n\s+Function : ", txt)[1:]:
        if key in f.split("\n")[0]:
            ins = re.findall(r"/\*[0-9a-f]{4}\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_]+)", f)
            return collections.Counter(ins)
    return collections.Counter()


a = counts(sys.argv[1], sys.argv[2])
b = counts(sys.argv[3], sys.argv[2]) if len(sys.argv) > 3 else None
keys = sorted(set(a) | set(b or {}), key=lambda k: -(a.get(k, 0) + (b or {}).get(k, 0)))
print(f"total {sum(a.values())}" + (f" -> {sum(b.values())}" if b is not None else ""))
for k in keys[:40]:
    print(f"{k:12s} {a.get(k, 0):6d}" + (f" {b.get(k, 0):6d}" if b is not None else ""))
