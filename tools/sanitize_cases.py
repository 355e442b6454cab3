#!/usr/bin/env python
"""Tiny cases of the hand-synchronised kernels for compute-sanitizer
(memcheck / racecheck / synccheck), one case per process:

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py crt
    cases: ozaki (INT8 tcgen05 GEMM + Gaussian residues + CRT TMA ring + guard),
           ozaki_real, f32, gather (2 emulated ranks: flag barrier + remote CRT stores),
           svd (DSMEM cluster Jacobi round), heff (DMMA chain + MPO pass + permutes),
           lanczos, tebd, mpo (skinny expansion kernel + float32 DMMA GEMM)
Each case checks its own result loosely (the point is the sanitizer report)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2512_23917_b200 as tci  # noqa: E402
import synth  # noqa: E402


def rel(a, b):
    return float((a - b).abs().pow(2).sum().sqrt() / b.abs().pow(2).sum().sqrt())


def case_ozaki():
    oz, dm = tci.Context(0), tci.Context(0)
    oz.set_gemm_algorithm(tci.TCI_GEMM_OZAKI_INT8)
    A = synth.random_tensor((1024, 4100), "c128", 3, 1, device="cuda")
    B = synth.random_tensor((4100, 1040), "c128", 3, 2, device="cuda")
    c = oz.contract(A, "mk", B, "kn", "mn")
    d = dm.contract(A, "mk", B, "kn", "mn")
    st = oz.ozaki_guard_stats()
    assert st["gemms"] == 1, st
    return rel(c, d)


def case_ozaki_real():
    oz, dm = tci.Context(0), tci.Context(0)
    oz.set_gemm_algorithm(tci.TCI_GEMM_OZAKI_INT8)
    A = synth.random_tensor((2048, 1030), "r64", 4, 1, device="cuda")
    B = synth.random_tensor((2100, 1030), "r64", 4, 2, device="cuda")
    return rel(oz.contract(A, "mk", B, "nk", "mn"), dm.contract(A, "mk", B, "nk", "mn"))


def case_f32():
    c = tci.Context(0)
    A = synth.random_tensor((2100, 1100), "r32", 5, 1, device="cuda")
    B = synth.random_tensor((1100, 1900), "r32", 5, 2, device="cuda")
    x = c.contract(A, "mk", B, "kn", "mn")
    c.set_f32_algorithm(tci.TCI_F32_FP64_CORES)
    return rel(x.double(), c.contract(A, "mk", B, "kn", "mn").double())


def case_gather():
    from paper_2512_23917_b200.sharding import PeerGatherHeff, slice_environment
    P, chi = 2, 1024
    inp = synth.heff_inputs(chi, 2, 5, "c128", 91, "heisenberg", device="cuda")
    L, W1, W2, R, psi = (inp[k] for k in ("L", "W1", "W2", "R", "psi"))
    ref_ctx = tci.Context(0)
    ref_ctx.set_gemm_algorithm(tci.TCI_GEMM_OZAKI_INT8)
    ref = ref_ctx.heff_apply(L, W1, W2, R, psi)
    streams = [torch.cuda.Stream() for _ in range(P)]
    ctxs = [tci.Context(0, streams[r]) for r in range(P)]
    for c in ctxs:
        c.set_gemm_algorithm(tci.TCI_GEMM_OZAKI_INT8)
    fulls = [torch.zeros((chi, 2, 2, chi), dtype=torch.complex128, device="cuda") for _ in range(P)]
    flags = [torch.zeros(P, dtype=torch.int32, device="cuda") for _ in range(P)]
    table = ([f.data_ptr() for f in fulls], [g.data_ptr() for g in flags])
    shs = [PeerGatherHeff(ctxs[r], slice_environment(L, P, r), W1, W2, R, P, r, peers=table, full=fulls[r],
                          flags=flags[r]) for r in range(P)]
    for r in range(P):
        ctxs[r].heff_apply(shs[r].L, W1, W2, R, psi)
    torch.cuda.synchronize()
    for r in range(P):
        shs[r].apply(psi)
    torch.cuda.synchronize()
    assert [c.gather_status() for c in ctxs] == [0] * P
    return max(rel(f, ref) for f in fulls)


def case_svd():
    c = tci.Context(0)
    a = synth.random_tensor((96, 2, 2, 80), "c128", 6, 1, device="cuda")
    u, s, vd, err = c.trunc_svd(a, 2, 1, 64, 0.0, 0.0)
    sref = torch.linalg.svdvals(a.reshape(192, 160).cpu())
    return float((s.cpu() - sref[:64]).abs().max() / sref[0])


def case_svd_small():
    c = tci.Context(0)
    a = synth.random_tensor((24, 2, 2, 20), "c128", 6, 1, device="cuda")
    u, s, vd, err = c.trunc_svd(a, 2, 1, 16, 0.0, 0.0)
    sref = torch.linalg.svdvals(a.reshape(48, 40).cpu())
    return float((s.cpu() - sref[:16]).abs().max() / sref[0])


def case_heff():
    c = tci.Context(0)
    inp = synth.heff_inputs(64, 2, 5, "c128", 7, "heisenberg", device="cuda")
    out = c.heff_apply(inp["L"], inp["W1"], inp["W2"], inp["R"], inp["psi"])
    return float(out.abs().max())


def case_lanczos():
    c = tci.Context(0)
    inp = synth.heff_inputs(32, 2, 5, "c128", 8, "heisenberg", device="cuda")
    e, it = c.heff_lanczos(inp["L"], inp["W1"], inp["W2"], inp["R"], inp["psi"], max_iter=8, tol=1e-10)
    return e


def case_tebd():
    c = tci.Context(0)
    inp = synth.tebd_inputs(130, 2, "r64", 9, 0.01, device="cuda")
    th = c.tebd_theta(inp["A"], "asb", inp["B"], "btc", inp["U"], "pqst", "apqc")
    return float(th.abs().max())


def case_mpo():
    """the skinny expansion kernel (8(a10)) on a ragged b extent, and the
    float32 GEMM on the FP64 tensor cores"""
    ctx = tci.Context(0)
    A = synth.random_tensor((7, 3, 301), "c128", 4, 1, device="cuda")
    W = synth.random_tensor((4, 4, 3, 3), "c128", 4, 2, device="cuda")
    B = ctx.contract(A, "asb", W, "wvst", "awtbv")
    ref = torch.einsum("asb,wvst->awtbv", A, W)
    X = synth.random_tensor((300, 200), "r32", 4, 3, device="cuda")
    Y = synth.random_tensor((200, 130), "r32", 4, 4, device="cuda")
    Z = ctx.contract(X, "mk", Y, "kn", "mn")
    return max(rel(B, ref), rel(Z.double(), X.double() @ Y.double()))


if __name__ == "__main__":
    torch.cuda.set_device(0)
    for name in sys.argv[1:]:
        v = globals()["case_" + name]()
        torch.cuda.synchronize()
        print(f"case {name}: {v:.3e}", flush=True)
