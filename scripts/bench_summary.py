"""One-screen summary of bench.py JSON lines: python scripts/bench_summary.py gpurun_out/x.jsonl ..."""
import json
import sys

for f in sys.argv[1:]:
    for line in open(f):
        if not line.startswith("{"):
            continue
        d = json.loads(line)
        print(f"== {f}: value {d['value']:.1f} {d['unit']}  ms/step {d['ms_per_step']:.4f}  launches {d['gpu_launches']}"
              f"  clocks {d['clocks']}")
        print("   stage_ms", {k: round(v, 4) for k, v in d["stage_ms"].items()})
        if d.get("views_in_flight"):
            print("   views_in_flight", round(d["views_in_flight"]["value"], 1))
        if d.get("e2e"):
            e = d["e2e"]
            print("   e2e", round(e["value"], 1), "h2d GB/s", round(e.get("h2d_achieved_GBps", 0), 1), "/",
                  round(e.get("h2d_link_GBps", 0), 1), "resident", e.get("resident_scene", {}).get("value"))
        if d.get("cpu_baseline"):
            c = d["cpu_baseline"]
            print("   cpu", round(c["value"], 4), c["cores"], c["sample"][:90])
        r = d["roofline"]
        print(f"   roofline bound={r['bound']} frac={r['frac']:.4f} tensor={r['tensor']['frac']:.4f} "
              f"mufu={r['mufu']['frac']:.4f} issue={(r.get('issue') or {}).get('frac')}")
        for k, v in (d.get("alpha_blend_ablation") or {}).items():
            print(f"   {k:28s} {v['blend_ms']:.4f} ms  x{v['speedup_vs_ffma_no_earlycull']:.2f}  exp {v['exp_calls']}")
        print("   frame", d["frame_stats"])
