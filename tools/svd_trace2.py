import os, sys, torch
sys.path.insert(0, os.getcwd())
import synth, paper_2512_23917_b200 as tci
ctx = tci.Context(0)
c = synth.TEBD_CONFIG
inp = synth.tebd_inputs(2048, c["d"], c["dtype"], c["seed"], c["tau"], device="cuda")
th = ctx.tebd_theta(inp["A"], "asb", inp["B"], "btc", inp["U"], "pqst", "apqc")
ctx.trunc_svd(th, 2, 1, 2048, 0.0, 0.0)
print("theta", ctx.svd_info(), flush=True)
a = torch.from_numpy(synth.random_np((2048, 2048), "c128", 21, 2)).cuda()
ctx.trunc_svd(a, 1, 1, 1024, 0.0, 0.0)
print("c128", ctx.svd_info(), flush=True)
