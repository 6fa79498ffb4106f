"""Top SASS instructions by warp-stall samples from an .ncu-rep source page."""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr_i = next(i for i, r in enumerate(rows) if "Address" in r and "Source" in r)
h = rows[hdr_i]
si, ai = h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
ie = h.index("Instructions Executed")
data = [r for r in rows[hdr_i + 1:] if len(r) > si]
tot = sum(float(r[si] or 0) for r in data)
tot_inst = sum(float(r[ie] or 0) for r in data)
print(f"total samples {tot:.0f}, total warp-instructions {tot_inst:.3e}")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
for idx, r in sorted(enumerate(data), key=lambda x: -float(x[1][si] or 0))[:n]:
    print(f"{idx:5d} {float(r[si] or 0) / tot * 100:5.1f}%  {r[ai].strip()[:90]}")
