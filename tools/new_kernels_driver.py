#!/usr/bin/env python
"""One launch of each kernel added in round 2's last session, for ncu
captures: the skinny expansion kernel (MPS-MPO application, chi = 4096), the
float32 / complex64 DMMA GEMMs (1024^3 / 2048 x 2048 x 1024), a small-tensor
permute and the tensor-core CRT (through one Ozaki complex GEMM)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2512_23917_b200 as tci  # noqa: E402
import synth  # noqa: E402

ctx = tci.Context(0)
ctx.set_f32_algorithm(tci.TCI_F32_FP64_CORES)
A = synth.random_tensor((4096, 2, 4096), "c128", 31, 1, device="cuda")
Wh, _, _ = synth.heisenberg_mpo(1.0)
W = torch.from_numpy(np.asarray(Wh)).to(torch.complex128).cuda()
ctx.contract(A, "asb", W, "wvst", "awtbv")
del A
X = synth.random_tensor((2048, 1024), "r32", 3, 1, device="cuda")
Y = synth.random_tensor((1024, 2048), "r32", 3, 2, device="cuda")
ctx.contract(X, "mk", Y, "kn", "mn")
U = synth.random_tensor((1024, 1024), "c64", 3, 3, device="cuda")
V = synth.random_tensor((1024, 1024), "c64", 3, 4, device="cuda")
ctx.contract(U, "mk", V, "kn", "mn")
P = synth.random_tensor((3, 8, 8, 37, 5, 37), "r64", 3, 5, device="cuda")
ctx.permute(P, [0, 2, 4, 1, 3, 5])
torch.cuda.synchronize()
print("done")
