"""Summarise `ncu --page source --csv --print-source sass` output: samples per kernel region
(split at the backward branches), stall reasons of the hottest instructions."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = [r for r in rows[2:] if len(r) == len(h)]
col = {c: h.index(c) for c in h}
S = col["Warp Stall Sampling (All Samples)"]
E = col["Instructions Executed"]
stalls = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
tot = sum(int(r[S]) for r in data)
print(f"total samples {tot}, instructions {len(data)}")
# regions between backward branches (loops)
def addr(r):
    return int(r[col["Address"]], 16)
base = addr(data[0])
reg_start = 0
regions = []
for i, r in enumerate(data):
    src = r[col["Source"]]
    if "BRA" in src and "0x" in src.split("BRA")[-1]:
        tgt = int(src.split("BRA")[-1].strip().split()[-1].rstrip(";").split(",")[-1].strip(), 16) if False else None
    if i == len(data) - 1:
        regions.append((reg_start, i))
agg = {s: 0 for s in stalls}
for r in data:
    for s in stalls:
        try:
            agg[s] += int(r[col[s]])
        except ValueError:
            pass
print("stall totals:", {k: round(v / max(1, tot), 3) for k, v in sorted(agg.items(), key=lambda x: -x[1]) if v})
top = sorted(data, key=lambda r: -int(r[S]))[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]
for r in top:
    st = {s[6:]: int(r[col[s]]) for s in stalls if r[col[s]] not in ("0", "")}
    st = dict(sorted(st.items(), key=lambda x: -x[1])[:3])
    print(f"{hex(addr(r) - base):>8} {int(r[S]):7d} {r[col['Source']][:60]:60s} {st}")
