"""Per-kernel device time of the last frame in an ncu launch-list CSV (scripts/gpu_launches.sh)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
data = []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
# last frame = from the last preprocess_kernel launch to the end
last = max(i for i, d in enumerate(data) if "preprocess_kernel" in d["Kernel Name"])
tot = 0.0
for d in data[last:]:
    v = float(d["Metric Value"].replace(",", ""))
    unit = d["Metric Unit"]
    us = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}[unit] * v
    tot += us
    print(f"{us:9.1f} us  {d['Kernel Name'][:90]}")
print(f"{tot:9.1f} us  total")
