mkdir -p gpurun_out
TCI_BENCH_BACKEND=gloo TCI_BENCH_SAME_DEVICE=1 timeout 1200 python -m torch.distributed.run --nnodes=1 \
  --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29519 bench.py --gpus 2 --steps 2 --warmup 3 \
  --alt none > gpurun_out/mp_bench_target.log 2>&1
echo "exit $?"
tail -1 gpurun_out/mp_bench_target.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], d['config']['workload'], d['config']['parallelism']); print('parity', d['parity'])"
