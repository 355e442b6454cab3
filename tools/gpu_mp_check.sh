#!/bin/bash
# Multi-process check of bench.py's N > 1 path on ONE GPU: two ranks on cuda:0 (gloo process
# group; the library's peer-memory gather through real CUDA IPC between the two processes,
# flag barriers across processes, the fused Ozaki CRT remote stores).
mkdir -p gpurun_out
TCI_BENCH_BACKEND=gloo TCI_BENCH_SAME_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 \
  --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 2 --warmup 3 \
  --config cfg2 > gpurun_out/mp_bench.log 2>&1
echo "exit $?"
grep -v "^\s*$" gpurun_out/mp_bench.log | tail -4 | cut -c1-700
tail -1 gpurun_out/mp_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['parallelism']); print('parity', d['parity']); print('e2e', d['e2e']['value'], d['e2e']['path'])"
TCI_BENCH_BACKEND=gloo TCI_BENCH_SAME_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 \
  --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29518 bench.py --gpus 4 --steps 2 --warmup 3 \
  --config cfg2 --alt none > gpurun_out/mp_bench4.log 2>&1
echo "exit4 $?"
tail -1 gpurun_out/mp_bench4.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], d['config']['parallelism']); print('parity', d['parity'])"
tail -1 gpurun_out/mp_bench4.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('e2e4', e['value'], e['results_identical_across_buffers'], e['path'][:160], e['single_call']['path'][:80])"
# (the --gather nccl variant cannot run here: NCCL refuses two ranks on one device)
