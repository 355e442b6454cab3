import os, sys
import numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_2512_23917_b200 as tci
ctx = tci.Context(0)
np.set_printoptions(precision=3, linewidth=200)
for dt in (np.complex128,):
    z = np.zeros((20, 45), dtype=dt)
    u, s, vd = ctx.svd(torch.from_numpy(z).cuda(), 1)
    print("zero: s", s.cpu().numpy()[:4], "info", ctx.svd_info(), "nan u", np.isnan(u.cpu().numpy()).sum(), "nan v", np.isnan(vd.cpu().numpy()).sum())
    x = np.zeros((40, 24), dtype=dt)
    x[3, :] = np.arange(1, 25)
    x[17, :] = 2 * np.arange(1, 25)
    u, s, vd = ctx.svd(torch.from_numpy(x).cuda(), 1)
    print("rank1: s", s.cpu().numpy()[:4], "info", ctx.svd_info(), "nan u", np.isnan(u.cpu().numpy()).sum(), "nan v", np.isnan(vd.cpu().numpy()).sum())
