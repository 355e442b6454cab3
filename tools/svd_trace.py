"""Per-sweep convergence trace of tci_svd on the config-3 TEBD theta (dev tool)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
import paper_2512_23917_b200 as tci
ctx = tci.Context(0)
c = synth.TEBD_CONFIG
chi = int(sys.argv[1]) if len(sys.argv) > 1 else c["chi"]
inp = synth.tebd_inputs(chi, c["d"], c["dtype"], c["seed"], c["tau"], device="cuda")
th = ctx.tebd_theta(inp["A"], "asb", inp["B"], "btc", inp["U"], "pqst", "apqc")
u, s, vd, err = ctx.trunc_svd(th, 2, 1, chi, 0.0, 1e-14)
print("sweeps/off", ctx.svd_info(), "chi", s.shape[0], "s[0], s[chi-1]", float(s[0]), float(s[-1]))
