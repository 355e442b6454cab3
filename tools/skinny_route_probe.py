"""Which kernel class a contract with one small operand takes (skinny route probe; dev tool)."""
import sys, os
sys.path.insert(0, os.getcwd())
import torch, synth, paper_2512_23917_b200 as tci
ctx = tci.Context(0)
X = synth.random_tensor((3, 20, 200), "c128", 1, 1, device="cuda")
W = synth.random_tensor((20, 20), "c128", 1, 2, device="cuda")
n0 = ctx.launch_count()
tci.tci_profile_enable(ctx.handle, True)
ctx.contract(X, "akc", W, "kn", "anc")
print("launches", ctx.launch_count() - n0, "skinny", tci.tci_profile_query(ctx.handle, tci.PROF_SKINNY), "gemm", tci.tci_profile_query(ctx.handle, tci.PROF_GEMM))
