"""Runs one workload layer R times (for ncu captures of tc_conv_kernel)."""
import argparse
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1704_04428_b200 as clb
from paper_1704_04428_b200 import rng, workloads

ap = argparse.ArgumentParser()
ap.add_argument("--layer", default="vgg16/conv1_2")
ap.add_argument("--method", default="auto")
ap.add_argument("--precision", default="fp32")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--batch", type=int, default=None)
a = ap.parse_args()
group = a.layer.split("/")[0]
layer = [l for l in workloads.workload(group, a.batch) if l.name == a.layer][0]
x, w = rng.make_problem(layer.batch, layer.channels, layer.height, layer.width, layer.kernel_count, layer.kernel_size)
with clb.ConvPlan(layer, a.method, a.precision) as plan:
    plan.set_weights(w)
    y = plan.forward(x)
    for _ in range(a.reps):
        plan.forward(x, y)
    torch.cuda.synchronize()
print("ok", layer, plan.method)
