"""Concurrent execution of independent layers (GoogLeNet inception branches, batch-1 stacks).

Every tcgen05 launch is a persistent grid that fills the GPU, so a step of small independent
layers run one after another pays each layer's fixed costs (launch, prologue, pipeline fill,
stream-K tail) in series.  Here each layer gets its own stream and an SM share of the GPU
(cl_conv_set_max_sms) proportional to its measured standalone time, the streams fork from
and join into the caller's stream, and the whole fan-out is captured once into a CUDA graph
(one host launch per step; the plan's cross-stream ordering is off under capture).  The SM
shares sum to at most the SM count, so every launch's CTAs can be co-resident (stream-K
pieces wait on each other inside one launch, never across launches).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Sequence


def sm_shares(weights: Sequence[float], n_sms: int, min_sms: int = 2) -> List[int]:
    """SM caps proportional to `weights`, even (CTA pairs), >= min_sms, summing to <= n_sms."""
    if not weights:
        return []
    total = float(sum(weights)) or 1.0
    budget = n_sms - n_sms % 2
    caps = [max(min_sms, int(budget * w / total) // 2 * 2) for w in weights]
    while sum(caps) > budget and max(caps) > min_sms:
        i = max(range(len(caps)), key=lambda j: caps[j])
        caps[i] -= 2
    # hand the rounding remainder to the heaviest layers
    order = sorted(range(len(caps)), key=lambda j: -weights[j])
    k = 0
    while sum(caps) + 2 <= budget and order:
        caps[order[k % len(order)]] += 2
        k += 1
    if sum(caps) > n_sms:
        raise ValueError(f"{len(caps)} concurrent layers need more than {n_sms} SMs at {min_sms} each")
    return caps


@dataclass
class ConcurrentStep:
    """A captured fan-out of independent plan.forward calls."""
    plans: list
    caps: List[int]
    streams: list = field(default_factory=list)
    graph: object = None

    def capture(self, xs, ys, wss, stream, layout: str = "nchw"):
        import torch
        for p, c in zip(self.plans, self.caps):
            p.set_max_sms(c)
        self.streams = [torch.cuda.Stream() for _ in self.plans]
        cap_stream = torch.cuda.Stream()

        def body():
            fork = torch.cuda.current_stream()
            for p, s, x, y, ws in zip(self.plans, self.streams, xs, ys, wss):
                s.wait_stream(fork)
                p.forward(x, y, ws, stream=s, layout=layout)
            for s in self.streams:
                fork.wait_stream(s)

        cap_stream.wait_stream(stream)
        with torch.cuda.stream(cap_stream):
            body()                             # eager warm-up on the same streams
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, stream=cap_stream):
            body()
        torch.cuda.synchronize()
        return self

    def replay(self):
        self.graph.replay()

    def release(self):
        for p in self.plans:
            p.set_max_sms(0)
        self.graph = None


def standalone_times(plans, xs, ys, wss, stream, layout: str = "nchw", reps: int = 3) -> List[float]:
    """Each plan's whole forward time alone on the GPU (ms, median of `reps`, CUDA events)."""
    import statistics
    import torch
    out = []
    for p, x, y, ws in zip(plans, xs, ys, wss):
        ts = []
        for _ in range(reps + 1):
            b, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            b.record(stream)
            p.forward(x, y, ws, stream=stream, layout=layout)
            e.record(stream)
            e.synchronize()
            ts.append(b.elapsed_time(e))
        out.append(statistics.median(ts[1:]))
    return out


def build(plans, xs, ys, wss, stream, n_sms: int, layout: str = "nchw") -> ConcurrentStep:
    """Measure each layer alone, split the SMs by those times, capture the concurrent step."""
    times = standalone_times(plans, xs, ys, wss, stream, layout)
    step = ConcurrentStep(list(plans), sm_shares(times, n_sms))
    step.standalone_ms = times
    return step.capture(xs, ys, wss, stream, layout)
