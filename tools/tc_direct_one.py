import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from oracle import oracle as O
import paper_1704_04428_b200 as clb
N, C, H, W, M, k = [int(a) for a in sys.argv[1:7]]
x, w = O.make_problem(N, C, H, W, M, k, 7 + C)
with clb.ConvPlan(clb.LayerConfig("d", C, H, W, M, k, batch=N), "direct-gpu", "fp32") as plan:
    plan.set_weights(torch.from_numpy(w).cuda())
    y = plan.forward(torch.from_numpy(x).cuda()).cpu().numpy()
    sp = plan.split
m = O.parity_metrics(y, O.conv_batch(x, w))
print((N, C, H, W, M, k), sp, "rel_l2 %.2e max_rel %.2e" % (m["rel_l2"], m["max_rel"]), flush=True)
