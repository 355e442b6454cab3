"""float64 H_eff.psi at chi = 4096 (Heisenberg, d = 2, D = 5): DMMA vs real Ozaki-II (dev probe)."""
import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
import paper_2512_23917_b200 as tci
inp = synth.heff_inputs(4096, 2, 5, "r64", 6, "heisenberg", device="cuda")
F = synth.heff_flops(4096, 2, 5, complex_=False)
res = {}
for name, algo in (("dmma", tci.TCI_GEMM_DMMA_3M), ("ozaki", tci.TCI_GEMM_OZAKI_INT8)):
    ctx = tci.Context(0)
    ctx.set_gemm_algorithm(algo)
    out = ctx.heff_apply(inp["L"], inp["W1"], inp["W2"], inp["R"], inp["psi"])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        ctx.heff_apply(inp["L"], inp["W1"], inp["W2"], inp["R"], inp["psi"], out=out)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 3e3
    res[name] = out.clone()
    print(f"{name}: {t * 1e3:.1f} ms per apply, {F / t / 1e12:.1f} TFLOP/s", flush=True)
    ctx.close()
d = (res["ozaki"] - res["dmma"]).norm() / res["dmma"].norm()
print(f"rel diff ozaki vs dmma {d.item():.2e}")
