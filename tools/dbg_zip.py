import os, sys
import numpy as np, torch
sys.path.insert(0, "/root/repo")
import synth, oracle
import paper_2512_23917_b200 as tci
oracle.build()
ctx = tci.Context(0)
n = 40
rng = np.random.default_rng(5)
bonds = [1] + [min(32, 2 ** min(i + 1, n - i - 1)) for i in range(n - 1)] + [1]
A = [rng.uniform(-1, 1, (bonds[i], 2, bonds[i + 1])) for i in range(n)]
Wh, lb, rb = synth.heisenberg_mpo(1.0)
Wh = np.asarray(Wh).real
W = [Wh[lb:lb + 1]] + [Wh] * (n - 2) + [Wh[:, rb:rb + 1]]
B, err = ctx.mps_mpo_zipup([torch.from_numpy(x).cuda() for x in A], [torch.from_numpy(x).cuda() for x in W], 32)
RB, rerr = oracle.mps_mpo_zipup(A, W, 32)
print("err", err, rerr)
print("gpu bonds", [b.shape[2] for b in B])
print("ora bonds", [b.shape[2] for b in RB])
# compare partial overlaps site by site: left environments
E1 = np.ones((1, 1)); E2 = np.ones((1, 1))
for i in range(n):
    b1 = B[i].cpu().numpy(); b2 = RB[i]
    E1 = np.einsum("xz,xsy,zsw->yw", E1, A[i], b1)
    E2 = np.einsum("xz,xsy,zsw->yw", E2, A[i], b2)
    # gauge differs; compare a gauge-invariant quantity only at the end
print("overlap", E1[0,0], E2[0,0])
