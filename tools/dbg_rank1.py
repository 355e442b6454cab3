import os, sys
import numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_2512_23917_b200 as tci
ctx = tci.Context(0)
for dt in (np.float64,):
    x = np.zeros((40, 24), dtype=dt)
    x[3, :] = np.arange(1, 25)
    x[17, :] = 2 * np.arange(1, 25)
    u, s, vd = ctx.svd(torch.from_numpy(x).cuda(), 1)
    U, S, V = u.cpu().numpy(), s.cpu().numpy(), vd.cpu().numpy()
    print("sweeps/off", ctx.svd_info())
    np.set_printoptions(precision=3, linewidth=200)
    print("s", S)
    G = U.T @ U - np.eye(24)
    print("max |UtU-I|", np.abs(G).max(), "worst cols", np.unravel_index(np.abs(G).argmax(), G.shape))
    print("max |VVt-I|", np.abs(V @ V.T - np.eye(24)).max())
