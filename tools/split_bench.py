"""Times the NCHW->split prepass alone (bandwidth vs HBM roofline) on the BASELINE input shapes."""
import sys, json
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1704_04428_b200 as clb
from paper_1704_04428_b200 import rng, workloads, _lib
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for wl in ("alexnet", "vgg16"):
    for l in workloads.workload(wl):
        if l.channels <= 4: continue
        with clb.ConvPlan(l, "kn2row-gpu") as plan:
            x, w = rng.make_problem(l.batch, l.channels, l.height, l.width, l.kernel_count, l.kernel_size)
            plan.set_weights(w)
            ws = torch.empty(plan.workspace_bytes(), dtype=torch.uint8, device="cuda")
            y = plan.forward(x, None, ws)
            ts = []
            for _ in range(5):
                flush.zero_()
                b, e, kb, ke = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
                for ev in (b, e, kb, ke): ev.record()
                torch.cuda.synchronize()
                _lib.lib().cl_conv_set_profile_events(plan._h, kb.cuda_event, ke.cuda_event)
                b.record(); plan.forward(x, y, ws); torch.cuda.synchronize()
                ts.append(b.elapsed_time(kb))        # forward start -> contraction start = prepass
            ms = sorted(ts)[2]
            cp = (l.channels + 15) // 16 * 16
            byts = l.batch * l.height * l.width * (4 * l.channels + 8 * cp)
            print(json.dumps({"layer": l.name, "prepass_us": round(ms * 1000, 1), "GB": round(byts / 1e9, 3),
                              "TBps": round(byts / ms / 1e9, 2), "frac_hbm": round(byts / ms / 1e9 / 6.5507, 2)}))
