#!/usr/bin/env python
"""Host cost of one contract call (config-5 sweep's small instances are bound
by it): wall time per call over back-to-back calls (no sync inside), device
time per call (CUDA events around the batch), kernels per call, and a
cProfile split of the Python binding vs the C ABI call."""
import cProfile
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2512_23917_b200 as tci  # noqa: E402
import synth  # noqa: E402

CASES = [("r32", "iDe", "weo", "wDoi", {'i': 8, 'D': 1, 'e': 2, 'w': 2, 'o': 37}),
         ("r64", "Pxzfq", "vuIKx", "uKzPqfvI", {'P': 1, 'x': 16, 'z': 1, 'f': 5, 'q': 5, 'v': 2, 'u': 2, 'I': 7, 'K': 8}),
         ("r64", "hiqB", "hTAi", "BTAq", {'h': 16, 'i': 5, 'q': 2, 'B': 16, 'T': 2, 'A': 256}),
         ("r64", "ij", "jk", "ik", {'i': 64, 'j': 64, 'k': 64}),
         ("r32", "GEKQ", "KqQ", "GEq", {'G': 5, 'E': 37, 'K': 7, 'Q': 64, 'q': 2})]


def main():
    ctx = tci.Context(0)
    for dt, la, lb, lc, dims in CASES:
        A = synth.random_tensor([dims[l] for l in la], dt, 1, 1, device="cuda")
        B = synth.random_tensor([dims[l] for l in lb], dt, 1, 2, device="cuda")
        C = ctx.contract(A, la, B, lb, lc)
        torch.cuda.synchronize()
        n = 2000
        n0 = ctx.launch_count()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        for _ in range(n):
            ctx.contract(A, la, B, lb, lc, out=C)
        e1.record()
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        kpc = (ctx.launch_count() - n0) / n
        # the C call alone (descriptors / workspace resolved once)
        ha, hb, hc = ctx.tensor(A), ctx.tensor(B), ctx.tensor(C)
        t2 = time.perf_counter()
        for _ in range(n):
            tci.tci_contract_str(ctx.handle, ha, la, hb, lb, hc, lc)
        t3 = time.perf_counter()
        torch.cuda.synchronize()
        print(f"{dt} {la},{lb}->{lc}: host {1e6 * (t1 - t0) / n:.1f} us/call (C ABI alone {1e6 * (t3 - t2) / n:.1f}), "
              f"device {1e3 * e0.elapsed_time(e1) / n:.1f} us/call, {kpc:.1f} kernels/call", flush=True)
    dt, la, lb, lc, dims = CASES[2]
    A = synth.random_tensor([dims[l] for l in la], dt, 1, 1, device="cuda")
    B = synth.random_tensor([dims[l] for l in lb], dt, 1, 2, device="cuda")
    C = ctx.contract(A, la, B, lb, lc)
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(2000):
        ctx.contract(A, la, B, lb, lc, out=C)
    pr.disable()
    torch.cuda.synchronize()
    pstats.Stats(pr).sort_stats("tottime").print_stats(8)
    ctx.close()


if __name__ == "__main__":
    main()
