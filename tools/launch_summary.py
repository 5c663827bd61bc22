"""Condense an ncu launch list (`--metrics gpu__time_duration.sum --csv`) of a bench.py run into
one step's kernels and their shares: a step = the launches between two L2-flush fills.
usage: python tools/launch_summary.py <launches.csv> > summary.json"""
import csv
import json
import re
import sys

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"')) if len(r) > 14 and r[0].isdigit()]
seq = [(re.sub(r"\(.*", "", r[4]), float(r[14]) / 1e3) for r in rows]       # (kernel, us)
is_flush = lambda k: "FillFunctor<unsigned char>" in k                      # noqa: E731
cuts = [i for i, (k, _) in enumerate(seq) if is_flush(k)]
steps = [seq[a + 1:b] for a, b in zip(cuts, cuts[1:]) if any("tc_conv_kernel" in k for k, _ in seq[a + 1:b])]
# the modal step length is the timed / warm-up step (the e2e and instrumented steps differ)
lens = [len(s) for s in steps]
n = max(set(lens), key=lens.count)
step = [s for s in steps if len(s) == n][-1]
by = {}
for k, us in step:
    by[k] = by.get(k, 0.0) + us
total = sum(by.values())
print(json.dumps({"step_kernels_us": {k: round(v, 1) for k, v in by.items()}, "sum_us": round(total, 1),
                  "share": {k: round(v / total, 3) for k, v in by.items()}, "launches_in_step": n,
                  "steps_seen": len(steps),
                  "note": "ncu launch list of `bench.py --steps 2 --warmup 1` (gpu__time_duration.sum, clocks "
                          "uncontrolled, serialised, cold caches); one VGG-16 step between two L2-flush fills"},
                 indent=1))
