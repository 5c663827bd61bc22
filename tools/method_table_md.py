"""profiles/rNN_method_table.md from tools/method_table.py's JSON."""
import json
import sys

d = json.load(open(sys.argv[1]))
methods = ["kn2row-gpu", "kn2row-explicit-gpu", "kn2col-gpu", "kn2row-acc-gpu", "im2col-gpu", "direct-gpu", "conv1x1-gpu"]
print(f"Whole-forward time per method, ms ({d['timing']}; precision {d['precision']}).  "
      "**bold** = fastest; `auto` = the library's pick.\n")
print("| layer | N | GFLOP | " + " | ".join(m.replace("-gpu", "") for m in methods) + " | auto | auto / best |")
print("|---|---|---|" + "---|" * (len(methods) + 2))
for r in d["rows"]:
    cells = []
    timed = {k: v for k, v in r["ms"].items() if isinstance(v, float)}
    for m in methods:
        v = r["ms"].get(m, "")
        if isinstance(v, float):
            cells.append(f"**{v:.3f}**" if m == r["best"] else f"{v:.3f}")
        elif v is None:
            cells.append("skip")
        elif isinstance(v, str) and v.startswith("routed"):
            cells.append("= conv1x1")
        else:
            cells.append("" if v == "" else "n/a")
    ratio = timed.get(r["auto"], float("nan")) / timed[r["best"]]
    print(f"| {r['layer']} | {r['batch']} | {r['gflop']:.2f} | " + " | ".join(cells) +
          f" | {r['auto'].replace('-gpu', '')} | {ratio:.2f} |")
