#!/bin/bash
# SVD low-pair skipping (trunc_svd, chi_max < n): parity tests, sweeps / time on the config-3 theta on / off
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_svd.py -q 2>&1 | tail -2
cat > /tmp/svdt.py <<'PY'
import os, sys, time, torch
sys.path.insert(0, os.getcwd())
import synth, paper_2512_23917_b200 as tci
ctx = tci.Context(0)
c = synth.TEBD_CONFIG
chi = int(sys.argv[1])
inp = synth.tebd_inputs(chi, c["d"], c["dtype"], c["seed"], c["tau"], device="cuda")
th = ctx.tebd_theta(inp["A"], "asb", inp["B"], "btc", inp["U"], "pqst", "apqc")
torch.cuda.synchronize(); t0 = time.time()
u, s, vd, err = ctx.trunc_svd(th, 2, 1, chi, 0.0, 0.0)
torch.cuda.synchronize(); t1 = time.time()
T = th.reshape(2 * chi, 2 * chi).cpu()
sv = torch.linalg.svdvals(T).double()
U = u.reshape(2 * chi, -1).cpu(); V = vd.reshape(-1, 2 * chi).cpu()
k = s.shape[0]
ou = (U.T @ U - torch.eye(k, dtype=U.dtype)).abs().max().item(); ov = (V @ V.T - torch.eye(k, dtype=V.dtype)).abs().max().item()
res2 = torch.linalg.norm(T - (U * s.cpu()) @ V).item() ** 2; tail = float((sv[k:] ** 2).sum())
print("chi", chi, "sweeps/off", ctx.svd_info(), "time %.3f s" % (t1 - t0), "max|s-s_ref|/s0 %.2e" % float((s.cpu() - sv[:k]).abs().max() / sv[0]),
      "orth %.1e %.1e" % (ou, ov), "EY %.2e" % (abs(res2 - tail) / max(tail, 1e-300)), "err vs tail %.2e" % (abs(err - tail / float((sv ** 2).sum())) / max(err, 1e-300)))
PY
for cfg in "X=1" "TCI_SVD_LOWSKIP=0"; do
  echo "== $cfg"; env $cfg timeout 300 python /tmp/svdt.py 2048 2>&1 | tail -1; env $cfg timeout 300 python /tmp/svdt.py 512 2>&1 | tail -1
done
timeout 600 python tools/bench_extra.py --only svd --out gpurun_out/extra_svd.json 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()[4:])
for k,v in d.items(): print(k, v['ms'], v['sweeps'], v['final_off'], v['max_abs_ds_over_s0'])"
