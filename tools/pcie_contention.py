"""Does concurrent HBM-heavy compute slow PCIe copies?  Duplex H2D+D2H of `chunk`-sized
copies (pinned memory), alone and while a device-to-device copy loop saturates HBM."""
import torch

n = 256 << 20
h1 = torch.empty(n, dtype=torch.uint8).pin_memory()
h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
big_a = torch.empty(2 << 30, dtype=torch.uint8, device="cuda")
big_b = torch.empty(2 << 30, dtype=torch.uint8, device="cuda")
s_in, s_out, s_c = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()


def run(chunk, hbm):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    if hbm:
        with torch.cuda.stream(s_c):
            for _ in range(12):
                big_b.copy_(big_a)
    for off in range(0, n, chunk):
        with torch.cuda.stream(s_in):
            d1[off:off + chunk].copy_(h1[off:off + chunk], non_blocking=True)
        with torch.cuda.stream(s_out):
            h2[off:off + chunk].copy_(d2[off:off + chunk], non_blocking=True)
    ev_in, ev_out = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev_in.record(s_in)
    ev_out.record(s_out)
    torch.cuda.synchronize()
    return 2 * n / max(e0.elapsed_time(ev_in), e0.elapsed_time(ev_out)) / 1e6


for chunk in (4 << 20, 16 << 20, 256 << 20):
    for hbm in (False, True):
        r = [run(chunk, hbm) for _ in range(3)][-1]
        print(f"chunk {chunk >> 20:4d} MB  HBM load {'on ' if hbm else 'off'}: duplex aggregate {r:6.1f} GB/s")
