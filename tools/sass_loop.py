"""Print the innermost hot loop of a kernel's SASS (the backward branch enclosing the most FFMA2
instructions) with its instruction mix, from `cuobjdump -sass` output.
usage: sass_loop.py <sass.txt> [title]"""
import collections
import re
import sys

lines = open(sys.argv[1]).read().split("\n")
title = sys.argv[2] if len(sys.argv) > 2 else ""
ins = []
for l in lines:
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
addr = {a: i for i, (a, _) in enumerate(ins)}
best = None
for i, (a, txt) in enumerate(ins):
    m = re.search(r"BRA(?:\.\S+)?\s+(0x[0-9a-f]+)", txt)
    if not m:
        continue
    tgt = int(m.group(1), 16)
    if tgt >= a or tgt not in addr:
        continue
    j0 = addr[tgt]
    n2 = sum(1 for _, t in ins[j0:i + 1] if "FFMA2" in t)
    if best is None or n2 > best[0]:
        best = (n2, j0, i)
n2, j0, j1 = best
body = ins[j0:j1 + 1]
mix = collections.Counter()
for _, t in body:
    op = t.split()[1] if t.startswith("@") else t.split()[0]
    mix[op.split(".")[0]] += 1
cells = max(1, n2 // 72)
print(f"# {title}")
print(f"# loop body {hex(body[0][0])}..{hex(body[-1][0])}: {len(body)} instructions, {n2} FFMA2"
      f" ({cells} cells of 72 FFMA2: 9 fields x 8 Q' columns on a parent pair); per cell {len(body) / cells:.1f}")
print("# mix: " + ", ".join(f"{k} {v}" for k, v in mix.most_common()))
allmix = collections.Counter()
for _, t in ins:
    for key in ("UTMALDG", "UTMAPF", "LDTM", "STTM", "FFMA2", "FADD2", "LDGSTS", "SYNCS", "UTCBAR", "UTCHMMA", "UTCQMMA"):
        if key in t:
            allmix[key] += 1
print("# Blackwell-native instructions in the kernel: " + ", ".join(f"{k} {v}" for k, v in allmix.most_common()))
print()
for a, t in body:
    print(f"        {t};")
