"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list by kernel name."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, collections.defaultdict(list)
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("qvts::", "").replace("<unnamed>::", "")
    scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "msecond": 1e3}.get(d.get("Metric Unit", "ns"), 1e-3)
    data[name.split("<")[0]].append(float(d["Metric Value"]) * scale)
for k, v in sorted(data.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:32s} n={len(v):5d} mean={sum(v)/len(v):9.2f}us total={sum(v)/1e3:9.3f}ms")
