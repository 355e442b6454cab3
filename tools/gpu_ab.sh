#!/bin/bash
# correctness + A/B of GEMM variants on the bench workload
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -15 | tee gpurun_out/pytest_gpu.txt
for algo in 3m 4m; do
  TCI_ZGEMM_ALGO=$algo timeout 600 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_$algo.json
  python -c "import json;d=json.load(open('gpurun_out/bench_$algo.json'));print('$algo', round(d['value'],2), 'TF/s', round(d['roofline']['frac'],3), d['clocks'])"
done
