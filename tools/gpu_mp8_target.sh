#!/bin/bash
# 8 ranks (processes) on one GPU: the peer-memory gather with 7 IPC peers per rank (config 2)
mkdir -p gpurun_out
TCI_BENCH_BACKEND=gloo TCI_BENCH_SAME_DEVICE=1 timeout 1200 python -m torch.distributed.run --nnodes=1 \
  --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29522 bench.py --gpus 8 --steps 2 --warmup 3 \
  --alt none > gpurun_out/mp_bench8t.log 2>&1
echo "exit $?"
tail -1 gpurun_out/mp_bench8t.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], d['config']['parallelism']); print('parity', d['parity']); print('e2e ok', d['e2e']['results_identical_across_buffers'])"
