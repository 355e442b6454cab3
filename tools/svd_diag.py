"""Accuracy / timing diagnostics of tci_svd on the GPU (development tool)."""
import sys, time, os
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
import paper_2512_23917_b200 as tci

ctx = tci.Context(0)
sizes = [int(x) for x in (sys.argv[1:] or ["1024"])]
for n in sizes:
    for dt in ("r64", "c128"):
        a = synth.random_np((n, n), dt, 21, 2)
        d = torch.from_numpy(a).cuda()
        u, s, vd = ctx.svd(d, 1)
        torch.cuda.synchronize()
        t0 = time.time()
        u, s, vd = ctx.svd(d, 1)
        torch.cuda.synchronize()
        t = time.time() - t0
        sw, off = ctx.svd_info()
        U, S, V = u.cpu().numpy(), s.cpu().numpy(), vd.cpu().numpy()
        rs = np.linalg.svd(a, compute_uv=False)
        err = np.abs(S - rs) / rs[0]
        q = [err[i * n // 8:(i + 1) * n // 8].max() for i in range(8)]
        rec = np.linalg.norm((U * S) @ V - a) / np.linalg.norm(a)
        ou = np.abs(U.conj().T @ U - np.eye(n)).max()
        ov = np.abs(V @ V.conj().T - np.eye(n)).max()
        print(f"n={n} {dt}: {t*1e3:.1f} ms sweeps={sw} off={off:.2e} max|ds|/s0={err.max():.2e} "
              f"by octile={' '.join(f'{x:.1e}' for x in q)} rec={rec:.2e} |UhU-I|={ou:.2e} |VVh-I|={ov:.2e}",
              flush=True)
