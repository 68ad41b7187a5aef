"""Instruction mix of the innermost row loop of a step kernel (the backward branch
range with 6*K row shuffles and no setup / WARPSYNC slow path).
python scripts/sass_inner_loop.py LIB KERNEL_REGEX"""
import collections
import re
import subprocess
import sys

sass = subprocess.run(["cuobjdump", "-sass", sys.argv[1]], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", sass)
body = next(f for f in funcs[1:] if re.search(sys.argv[2], f.split("\n")[0]))
ins = []
for line in body.split("\n"):
    m = re.match(r"\s+/\*([0-9a-f]+)\*/\s+(.*?);", line)
    if m:
        ins.append((int(m.group(1), 16), m.group(2)))
best = None
for a, t in ins:
    m = re.search(r"BRA (0x[0-9a-f]+)", t)
    if m and int(m.group(1), 16) < a:
        rng = [x for x in ins if int(m.group(1), 16) <= x[0] <= a]
        c = collections.Counter(re.sub(r"^@!?U?P\w+\s+", "", x[1]).split()[0] for x in rng)
        if c.get("SHFL.UP", 0) >= 6 and c.get("CS2R", 0) == 0 and "WARPSYNC" not in c:
            if best is None or len(rng) < best[0]:
                best = (len(rng), hex(rng[0][0]), hex(rng[-1][0]), c)
n, lo, hi, c = best
print(f"inner loop {lo}..{hi}: {n} instructions")
for op, k in c.most_common(40):
    print(f"{k:6d} {op}")
