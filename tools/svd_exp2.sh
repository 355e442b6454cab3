#!/bin/bash
# SVD noise floor: parity tests, sweeps / time on the config-3 theta with the floor on / off, sort on / off
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_svd.py -q -x 2>&1 | tail -3
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
u, s, vd, err = ctx.trunc_svd(th, 2, 1, chi, 0.0, 1e-14)
torch.cuda.synchronize(); t1 = time.time()
sv = torch.linalg.svdvals(th.reshape(2 * chi, 2 * chi).cpu()).double()
print("chi", chi, "sweeps/off", ctx.svd_info(), "time %.3f s" % (t1 - t0),
      "max|s-s_ref|/s0 %.2e" % float((s.cpu() - sv[:s.shape[0]]).abs().max() / sv[0]))
PY
for cfg in "X=1" "TCI_SVD_FLOOR=0" "TCI_SVD_SORT=0" "TCI_SVD_FLOOR=0 TCI_SVD_SORT=0"; do
  echo "== $cfg"; env $cfg timeout 300 python /tmp/svdt.py 2048 2>&1 | tail -1; env $cfg timeout 300 python /tmp/svdt.py 512 2>&1 | tail -1
done
