import sys, torch
sys.path.insert(0, '.')
import paper_1704_04428_b200 as clb
from oracle import oracle as O
for case in [(2, 64, 56, 56, 64, 3, 1), (8, 128, 28, 28, 256, 3, 1)]:
    N, C, H, W, M, k, pad = case
    x, w = O.make_problem(N, C, H, W, M, k, 5)
    with clb.ConvPlan(clb.LayerConfig("d", C, H, W, M, k, 1, pad, N), "kn2row-gpu") as plan:
        plan.set_weights(torch.from_numpy(w).cuda())
        y = plan.forward(torch.from_numpy(x).cuda()); torch.cuda.synchronize()
    m = O.parity_metrics(y.cpu().numpy(), O.conv_loopnest(x, w, pad, 1))
    print(case, m, flush=True)
