#!/usr/bin/env python
"""One call per config-5 small instance (after a warm-up call), for an ncu
launch list: which kernels the call launches and how long each takes."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import torch  # noqa: E402

import paper_2512_23917_b200 as tci  # noqa: E402
import synth  # noqa: E402
from sweep_small_probe import CASES  # noqa: E402

ctx = tci.Context(0)
ctx.set_gemm_algorithm(tci.TCI_GEMM_OZAKI_INT8)
for dt, la, lb, lc, dims in CASES:
    A = synth.random_tensor([dims[l] for l in la], dt, 1, 1, device="cuda")
    B = synth.random_tensor([dims[l] for l in lb], dt, 1, 2, device="cuda")
    C = ctx.contract(A, la, B, lb, lc)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push(f"{dt} {la},{lb}->{lc}")
    ctx.contract(A, la, B, lb, lc, out=C)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
    print(f"case {dt} {la},{lb}->{lc}", flush=True)
