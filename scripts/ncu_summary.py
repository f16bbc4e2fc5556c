"""Summarise an ncu --set full report into profiles/ (JSON + markdown table).

    python scripts/ncu_summary.py gpurun_out/r1_k7.ncu-rep profiles/r1_k7_ncu   # writes .json and .md

Per launch: duration, DRAM bytes (the roofline `traffic`), throughput fractions,
pipe utilisation (tensor, XU = MUFU, FMA, ALU, FP64), issue activity, occupancy
and the top warp stall reasons.
"""

from __future__ import annotations

import csv
import io
import json
import subprocess
import sys

METRICS = {
    "time_us": "gpu__time_duration.sum",
    "dram_read_MB": "dram__bytes_read.sum",
    "dram_write_MB": "dram__bytes_write.sum",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "l2_pct": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1_pct": "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "inst_executed": "smsp__inst_executed.sum",
    "tensor_pipe_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "xu_pipe_pct": "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "fma_pipe_pct": "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "alu_pipe_pct": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "fp64_pipe_pct": "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
}
STALL_PREFIX = "smsp__average_warps_issue_stalled_"


def load(rep: str):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], check=True, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    return hdr, units, data


def num(x: str):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return x


def summarise(rep: str):
    hdr, units, data = load(rep)
    col = {h: i for i, h in enumerate(hdr)}
    res = []
    for d in data:
        e = {"kernel": d[col["Kernel Name"]]}
        for k, m in METRICS.items():
            if m in col:
                v = num(d[col[m]])
                u = units[col[m]]
                if k.endswith("_MB") and isinstance(v, float):
                    v = v * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(u, 1.0)
                if k == "time_us" and isinstance(v, float):
                    v = v * {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}.get(u, 1.0)
                e[k] = v
        stalls = {}
        for h, i in col.items():
            if h.startswith(STALL_PREFIX) and h.endswith("_per_issue_active.ratio"):
                v = num(d[i])
                if isinstance(v, float):
                    stalls[h[len(STALL_PREFIX):-len("_per_issue_active.ratio")]] = v
        if isinstance(e.get("time_us"), float) and isinstance(e.get("dram_read_MB"), float):
            e["dram_GBps"] = (e["dram_read_MB"] + e["dram_write_MB"]) * 1e3 / e["time_us"]
        e["top_stalls"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:5])
        res.append(e)
    return res


def markdown(res) -> str:
    cols = ["time_us", "dram_read_MB", "dram_write_MB", "dram_GBps", "dram_pct", "l2_pct", "sm_pct", "issue_active_pct",
            "tensor_pipe_pct", "xu_pipe_pct", "fma_pipe_pct", "fp64_pipe_pct", "warps_active_pct", "regs"]
    lines = ["| kernel | " + " | ".join(cols) + " | top stalls |", "|" + "---|" * (len(cols) + 2)]
    for e in res:
        name = e["kernel"].split("(")[0].replace("tcgs::<unnamed>::", "").replace("<unnamed>::", "")
        vals = [f"{e[c]:.1f}" if isinstance(e.get(c), float) else str(e.get(c, "")) for c in cols]
        st = ", ".join(f"{k} {v:.1f}" for k, v in list(e["top_stalls"].items())[:3])
        lines.append(f"| {name[:48]} | " + " | ".join(vals) + f" | {st} |")
    return "\n".join(lines) + "\n"


if __name__ == "__main__":
    rep, out = sys.argv[1], sys.argv[2]
    res = summarise(rep)
    with open(out + ".json", "w") as f:
        json.dump(res, f, indent=1)
    with open(out + ".md", "w") as f:
        f.write(f"ncu --set full summary of `{rep.split('/')[-1]}` (cold-cache, serialised replays; units: us, MB, %)\n\n")
        f.write(markdown(res))
    print(markdown(res))
