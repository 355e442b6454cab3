import os, sys
import numpy as np, torch
sys.path.insert(0, "/root/repo")
import synth, oracle
import paper_2512_23917_b200 as tci
oracle.build()
ctx = tci.Context(0)
A = synth.random_np((24, 2, 24), "r64", 41, 6)
B = synth.random_np((24, 2, 24), "r64", 41, 7)
th = oracle.contract(A, "asb", B, "btc", "astc")
u, s, vd = ctx.svd(torch.from_numpy(th).cuda(), 2)
S = s.cpu().numpy(); V = vd.cpu().numpy().reshape(48, 48); U = u.cpu().numpy().reshape(48, 48)
np.set_printoptions(precision=3, linewidth=220)
print("info", ctx.svd_info())
print("s", S)
print("zero V rows", [i for i in range(48) if np.abs(V[i]).max() == 0], "zero U cols", [i for i in range(48) if np.abs(U[:, i]).max() == 0])
print("V norms", np.linalg.norm(V, axis=1))
