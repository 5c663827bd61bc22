"""tools/report.py JSON -> the DESIGN.md per-layer markdown table."""
import json
import sys

CFG = {"c1": "C1", "alexnet-b1": "C2 b1", "alexnet": "C2 b128", "vgg16": "C3", "googlenet": "C4", "sweep": "C5",
       "scale": "C5 scale"}
txt = open(sys.argv[1]).read()
d = json.loads(txt[txt.index("{"):])
peak = d.get("peak_fp32_faithful_tflops", d.get("peak_3xtf32_tflops"))
print("| config | layer | N | method | split | GFLOP | kernel µs | eff. TFLOP/s | % of split peak | layer roofline % "
      "| graph fwd µs | rel-L2 | CPU kn2row GFLOP/s | CPU im2col GFLOP/s | CPU kn2row 1-core GFLOP/s |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|")
for r in d["rows"]:
    batch1 = r["N"] == 1 or r["workload"] == "googlenet"
    us = (r["graph_forward_ms"] if batch1 else r["kernel_ms"]) * 1e3
    tf = r["gflop"] / us * 1e3
    pk = r.get("peak_tflops", peak if not isinstance(peak, dict) else peak.get("mixed"))
    print(f"| {CFG.get(r['workload'], r['workload'])} | {r['layer']} | {r['N']} | {r['method']} | {r.get('split', '')} | "
          f"{r['gflop']:.2f} | {us:.0f} | {tf:.1f} | {100 * tf / pk:.0f} | "
          f"{100 * tf / r['roofline_tflops']:.0f} | {r['graph_forward_ms'] * 1e3:.0f} | {r['rel_l2']:.1e} | "
          f"{r['cpu_kn2row_tflops'] * 1e3:.1f} | {r['cpu_im2col_tflops'] * 1e3:.1f} | "
          f"{r.get('cpu_kn2row_1core_tflops', float('nan')) * 1e3:.1f} |")
