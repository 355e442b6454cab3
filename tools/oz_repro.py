import sys, torch
sys.path.insert(0, '.')
import synth, paper_2512_23917_b200 as tci
c = tci.Context(0); c.set_gemm_algorithm(tci.TCI_GEMM_OZAKI_INT8)
cfg = synth.HEFF_CONFIGS["cfg2_heisenberg_chi1024"]
inp = synth.heff_inputs(cfg["chi"], cfg["d"], cfg["D"], cfg["dtype"], cfg["seed"], cfg["model"], device="cuda")
print("ws", c.heff_workspace_size(inp["L"], inp["W1"], inp["W2"], inp["R"], inp["psi"]) / 1e9, flush=True)
out = c.heff_apply(inp["L"], inp["W1"], inp["W2"], inp["R"], inp["psi"])
torch.cuda.synchronize()
print("ok", out.abs().max().item())
