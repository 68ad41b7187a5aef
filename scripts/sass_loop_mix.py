"""Instruction mix of the main loop (the backward-branch range holding the LDGSTS
row loads and no WARPSYNC slow path) of one kernel in a .so: python scripts/sass_loop_mix.py LIB REGEX"""
import collections
import re
import subprocess
import sys

lib, pat = sys.argv[1], sys.argv[2]
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", sass)
body = next(f for f in funcs[1:] if re.search(pat, f.split("\n")[0]))
ins = []
for l in body.split("\n"):
    m = re.match(r"\s+/\*([0-9a-f]+)\*/\s+(.*?);", l)
    if m:
        ins.append((int(m.group(1), 16), m.group(2)))
best = None
for a, t in ins:
    m = re.search(r"BRA (0x[0-9a-f]+)", t)
    if not m:
        continue
    tgt = int(m.group(1), 16)
    if tgt >= a:
        continue
    rng = [x for x in ins if tgt <= x[0] <= a]
    txt = " ".join(x[1] for x in rng)
    if "LDGSTS" in txt and "WARPSYNC" not in txt and (best is None or len(rng) > len(best)):
        best = rng
cnt = collections.Counter(re.sub(r"^@!?U?P\w+\s+", "", t).split()[0] for _, t in best)
print(f"loop {hex(best[0][0])}..{hex(best[-1][0])}: {len(best)} instructions")
for op, c in cnt.most_common(40):
    print(f"{c:6d} {op}")
