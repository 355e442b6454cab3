#!/usr/bin/env python
"""PCIe probe for the streaming e2e: pinned H2D of the step's inputs (3.76 GB),
D2H of its result (1.07 GB), alone and concurrently on two streams, and both
beside a device-side compute load (the bench step) -- is the stream PCIe-bound?"""
import json
import torch

dev = torch.device("cuda")
h_in = torch.empty(3758099584 // 4, dtype=torch.float32, pin_memory=True)
d_in = torch.empty_like(h_in, device=dev)
d_out = torch.empty(1073741824 // 4, dtype=torch.float32, device=dev)
h_out = torch.empty_like(d_out, device="cpu").pin_memory()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    for s in (s1, s2):
        torch.cuda.current_stream().wait_stream(s)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def h2d():
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)


def both():
    h2d()
    d2h()


r = {"h2d_ms": timed(h2d), "d2h_ms": timed(d2h), "both_ms": timed(both)}
r["h2d_GBs"] = 3.758099584 / r["h2d_ms"] * 1e3
r["d2h_GBs"] = 1.073741824 / r["d2h_ms"] * 1e3
print(json.dumps(r))
