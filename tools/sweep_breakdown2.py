#!/usr/bin/env python
"""Kernel breakdown of the slowest large config-5 instances (tci_profile
counters: GEMM / skinny / permute time per call) -- which step to fix."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2512_23917_b200 as tci  # noqa: E402
import synth  # noqa: E402

CASES = [("r64", "cDrVfH", "DMq", "HcfMVrq", {'c': 8, 'D': 64, 'r': 5, 'V': 3, 'f': 37, 'H': 128, 'M': 7, 'q': 64}),
         ("r64", "OCxLVS", "SWEVz", "WLOxCEz", {'O': 64, 'C': 3, 'x': 7, 'L': 128, 'V': 37, 'S': 2, 'W': 37, 'E': 1, 'z': 37}),
         ("r32", "rXcByH", "yrLP", "BXLPcH", {'r': 37, 'X': 8, 'c': 128, 'B': 7, 'y': 7, 'H': 128, 'L': 3, 'P': 16}),
         ("r32", "LSerxE", "rlxzNZ", "zSZleENL", {'L': 1, 'S': 16, 'e': 18, 'r': 16, 'x': 5, 'E': 16, 'l': 8, 'z': 5, 'N': 32, 'Z': 32}),
         ("r32", "xjdFQK", "xdKTQF", "Tj", {'x': 7, 'j': 2, 'd': 64, 'F': 5, 'Q': 256, 'K': 7, 'T': 64}),
         ("r64", "gJPwA", "sArIDY", "YrJPwsIgD", {'g': 3, 'J': 16, 'P': 1, 'w': 5, 'A': 1, 's': 16, 'r': 32, 'I': 32, 'D': 7, 'Y': 7}),
         ("r64", "emRWt", "tse", "WmsR", {'e': 128, 'm': 7, 'R': 16, 'W': 256, 't': 37, 's': 3})]


def main():
    ctx = tci.Context(0)
    ctx.set_gemm_algorithm(tci.TCI_GEMM_OZAKI_INT8)
    out = []
    for dt, la, lb, lc, dims in CASES:
        A = synth.random_tensor([dims[l] for l in la], dt, 1, 1, device="cuda")
        B = synth.random_tensor([dims[l] for l in lb], dt, 1, 2, device="cuda")
        C = ctx.contract(A, la, B, lb, lc)
        torch.cuda.synchronize()
        tci.tci_profile_enable(ctx.handle, True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            ctx.contract(A, la, B, lb, lc, out=C)
        e1.record()
        torch.cuda.synchronize()
        prof = {k: tci.tci_profile_query(ctx.handle, v) for k, v in
                (("gemm", tci.PROF_GEMM), ("skinny", tci.PROF_SKINNY), ("permute", tci.PROF_PERMUTE),
                 ("i8", tci.PROF_I8))}
        tci.tci_profile_enable(ctx.handle, False)
        n0 = ctx.launch_count()
        ctx.contract(A, la, B, lb, lc, out=C)
        kpc = ctx.launch_count() - n0
        r = {"case": f"{dt} {la},{lb}->{lc}", "ms": e0.elapsed_time(e1) / 3, "kernels": kpc,
             **{k: {"launches": v["launches"] / 3, "ms": v["ms"] / 3} for k, v in prof.items()}}
        print(json.dumps(r), flush=True)
        out.append(r)
        del A, B, C
        torch.cuda.empty_cache()
    json.dump(out, open(os.path.join(ROOT, "gpurun_out", "sweep_breakdown2.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
