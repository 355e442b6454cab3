#!/usr/bin/env python
"""Config-5 instances with a 1-20 us roofline: where the time goes. Per
instance: eager wall time per call (the sweep's measure), the device time of
the call's kernels (the call captured once with tci_graph_begin/end and
replayed), launches per call and the profiled kernel families."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2512_23917_b200 as tci  # noqa: E402
import synth  # noqa: E402

CASES = [["r32", "zMDsQR", "DsRMG", "zGQ", {"z": 37, "M": 5, "D": 3, "s": 37, "Q": 128, "R": 1, "G": 7}],
         ["r32", "NZC", "bZC", "bN", {"N": 256, "Z": 16, "C": 256, "b": 128}],
         ["r64", "joe", "JUnjo", "nJUe", {"j": 128, "o": 256, "e": 1, "J": 5, "U": 3, "n": 7}],
         ["r64", "RduM", "OMxuHR", "HdxO", {"R": 37, "d": 64, "u": 37, "M": 8, "O": 3, "x": 8, "H": 5}],
         ["r32", "zlVOX", "oVq", "zXOloq", {"z": 2, "l": 128, "V": 64, "O": 256, "X": 1, "o": 3, "q": 16}],
         ["r64", "BUGqA", "jAVU", "qVBjG", {"B": 16, "U": 7, "G": 64, "q": 8, "A": 16, "j": 37, "V": 3}],
         ["r32", "QgtWY", "VfQ", "tVYfWg", {"Q": 3, "g": 1, "t": 37, "W": 64, "Y": 64, "V": 16, "f": 5}],
         ["r32", "IuNVTp", "yqLN", "LuVTyIqp", {"I": 2, "u": 256, "N": 256, "V": 8, "T": 8, "p": 3, "y": 5, "q": 2,
                                                "L": 2}]]


def main():
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)   # torch's work (allocations, events) on the context stream
    ctx = tci.Context(0, stream)    # a real stream: graph capture needs one
    ctx.set_gemm_algorithm(tci.TCI_GEMM_OZAKI_INT8)
    out = []
    for dt, la, lb, lc, dims in CASES:
        A = synth.random_tensor([dims[l] for l in la], dt, 1, 1, device="cuda")
        B = synth.random_tensor([dims[l] for l in lb], dt, 1, 2, device="cuda")
        C = ctx.contract(A, la, B, lb, lc)
        torch.cuda.synchronize()
        n0 = ctx.launch_count()
        ctx.contract(A, la, B, lb, lc, out=C)
        kpc = ctx.launch_count() - n0
        tci.tci_profile_enable(ctx.handle, True)
        ctx.contract(A, la, B, lb, lc, out=C)
        torch.cuda.synchronize()
        prof = {k: tci.tci_profile_query(ctx.handle, v) for k, v in
                (("gemm", tci.PROF_GEMM), ("skinny", tci.PROF_SKINNY), ("permute", tci.PROF_PERMUTE))}
        tci.tci_profile_enable(ctx.handle, False)
        # eager: per call, synchronised (the sweep's measure) and back to back
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(20):
            ctx.contract(A, la, B, lb, lc, out=C)
            torch.cuda.synchronize()
        eager = (time.perf_counter() - t0) / 20
        t0 = time.perf_counter()
        for _ in range(50):
            ctx.contract(A, la, B, lb, lc, out=C)
        torch.cuda.synchronize()
        b2b = (time.perf_counter() - t0) / 50
        # device: the call captured once, replayed
        tci.tci_graph_begin(ctx.handle)
        ctx.contract(A, la, B, lb, lc, out=C)
        g = tci.tci_graph_end(ctx.handle)
        for _ in range(3):
            tci.tci_graph_launch(ctx.handle, g)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(50):
            tci.tci_graph_launch(ctx.handle, g)
        e1.record()
        torch.cuda.synchronize()
        graph_us = e0.elapsed_time(e1) / 50 * 1e3
        tci.tci_graph_destroy(g)
        r = {"case": f"{dt} {la},{lb}->{lc}", "launches": kpc, "eager_sync_us": eager * 1e6, "eager_b2b_us": b2b * 1e6,
             "graph_us": graph_us, **{k: {"launches": v["launches"], "us": v["ms"] * 1e3} for k, v in prof.items()}}
        print(json.dumps(r), flush=True)
        out.append(r)
    json.dump(out, open(os.path.join(ROOT, "gpurun_out", "sweep_small_probe.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
