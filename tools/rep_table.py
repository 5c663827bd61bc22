"""Condenses tools/report.py output (JSON lines) to one line per layer."""
import json
import sys

for line in open(sys.argv[1]):
    line = line.strip()
    if not line.startswith("{"):
        continue
    try:
        d = json.loads(line)
    except json.JSONDecodeError:
        continue
    if "layer" in d and "kernel_ms" in d:
        print(f'{d["layer"]:18s} {d["method"]:12s} {d["kernel_ms"]:8.3f} ms  {d["kernel_tflops"]:7.1f} TF  '
              f'frac {d["frac_of_layer_roofline"]:.2f}  graph {d.get("graph_forward_ms", 0):.3f} ms')
