import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from oracle import oracle as O
import paper_1704_04428_b200 as clb
N, C, H, W, M, k = 2, 64, 14, 14, 64, 3
x, w = O.make_problem(N, C, H, W, M, k, 5)
with clb.ConvPlan(clb.LayerConfig("t", C, H, W, M, k, batch=N), "kn2row-gpu", "fp32") as plan:
    plan.set_weights(torch.from_numpy(w).cuda())
    y = plan.forward(torch.from_numpy(x).cuda()).cpu().numpy()
print(O.parity_metrics(y, O.conv_batch(x, w)))
