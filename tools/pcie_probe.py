"""PCIe H2D / D2H / concurrent bandwidth on this box (pinned memory, CUDA events)."""
import torch
n = 256 << 20
h1 = torch.empty(n, dtype=torch.uint8).pin_memory(); h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d1 = torch.empty(n, dtype=torch.uint8, device="cuda"); d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn):
    torch.cuda.synchronize(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); fn(); torch.cuda.synchronize(); e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1)
for _ in range(2):
    a = t(lambda: d1.copy_(h1, non_blocking=True))
    b = t(lambda: h2.copy_(d2, non_blocking=True))
    def both():
        with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
        with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    c = t(both)
print(f"H2D {n/a/1e6:.1f} GB/s  D2H {n/b/1e6:.1f} GB/s  both-concurrent {2*n/c/1e6:.1f} GB/s aggregate ({c:.2f} ms vs serial {a+b:.2f} ms)")
