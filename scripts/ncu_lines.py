"""Per-source-line instruction and stall shares of one kernel in an ncu report (cuda,sass source view):
    python scripts/ncu_lines.py <report> <kernel regex> [top]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep, rx = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + rx, "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
inst = defaultdict(float)
stall = defaultdict(float)
src = {}
cur_line = None
first_fn = None
fname = ""
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if r and r[0] == "Function Name":
        if first_fn is not None and r[1] != first_fn:
            break  # first function (launch) only
        if first_fn is not None and fname == first_file:
            break
        if first_fn is None:
            first_file = fname
        first_fn = r[1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r:
        continue
    if r[0]:
        cur_line = (fname, int(r[0]))
        src[cur_line] = r[1]
    ie = hdr.index("Instructions Executed")
    st = hdr.index("Warp Stall Sampling (All Samples)")
    try:
        inst[cur_line] += float(r[ie] or 0)
        stall[cur_line] += float(r[st] or 0)
    except (ValueError, IndexError):
        pass
ti, ts = sum(inst.values()), sum(stall.values())
print(first_fn, f"instructions {ti:.4g}, stall samples {ts:.4g}")
for ln in sorted(sorted(inst, key=lambda k: -inst[k])[:top]):
    print(f"{ln[0][:14]:14s}{ln[1]:5d} {100 * inst[ln] / ti:5.1f}% inst {100 * stall[ln] / ts:5.1f}% stall  {src.get(ln, '').strip()[:90]}")
