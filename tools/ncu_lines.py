"""Map an ncu SASS source page (executed instructions, stall samples) to CUDA source lines through
the line table of the local build (nvdisasm -g of the kernel's cubin).
usage: ncu_lines.py <rep> <kernel-regex> <cubin> <mangled-substring> [launch-skip] [n-units]"""
import collections
import csv
import re
import subprocess
import sys

rep, kre, cubin, fn = sys.argv[1:5]
skip = sys.argv[5] if len(sys.argv) > 5 else "0"
units = float(sys.argv[6]) if len(sys.argv) > 6 else 1.0
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + kre,
                      "--launch-skip", skip, "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
h = rows[1]
S = h.index("Warp Stall Sampling (All Samples)")
E = h.index("Instructions Executed")


def iv(x):
    try:
        return int(float(x))
    except ValueError:
        return 0


data = [r for r in rows[2:] if len(r) == len(h) and r[0].startswith("0x")]
base = int(data[0][0], 16)
ex = {}
for r in data:
    ex.setdefault(int(r[0], 16) - base, (iv(r[E]), iv(r[S])))
sass = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout.split("\n")
start = [i for i, l in enumerate(sass) if l.startswith("//----") and fn in l][0]
cur = None
agg, aggs = collections.Counter(), collections.Counter()
nstat = 0
for l in sass[start + 1:]:
    if l.startswith("//-----"):
        break
    m = re.search(r'File "(.*)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
    if m:
        nstat += 1
        off = int(m.group(1), 16)
        if off in ex:
            agg[cur] += ex[off][0]
            aggs[cur] += ex[off][1]
tot, ts = sum(agg.values()), max(1, sum(aggs.values()))
print(f"static {nstat} (ncu {len(ex)}), executed warp-instr {tot}, per unit {tot / units:.1f}")
for k, v in agg.most_common(40):
    print(f"{k[0]}:{k[1]}  {v / units:9.1f}  stall% {100 * aggs[k] / ts:5.1f}")
