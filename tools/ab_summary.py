"""Summary of an A/B run of bench.py lines (tools/gpu_ab_env.sh): value, median step, per-layer kernel ms."""
import json
import sys

out, reps = sys.argv[1], int(sys.argv[2])
for side in "ab":
    for r in range(1, reps + 1):
        try:
            j = json.loads(open(f"{out}/{side}_{r}.json").read().strip().splitlines()[-1])
        except Exception as e:   # noqa: BLE001
            print(side, r, "failed", e)
            continue
        ks = " ".join(f"{l['kernel_ms']:.3f}" for l in j["layers"])
        print(side, r, f"value {j['value']:.1f} median-step {j['step_ms_median']:.3f} ms | {ks}")
