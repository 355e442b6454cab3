#!/bin/bash
# tensor-core CRT: smoke (bounded), Ozaki GPU tests, bench A/B (TCI_CRT_MMA=0/1), launch list
mkdir -p gpurun_out
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3 | tee gpurun_out/smoke.txt
grep -q "ozaki gemm" gpurun_out/smoke.txt || { echo "smoke failed"; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "${1:-ozaki or heff or gather or f32}" --timeout 120 --timeout-method thread 2>&1 | tail -6 > gpurun_out/pytest_gpu.txt
tail -3 gpurun_out/pytest_gpu.txt
for v in 1 0 1; do
  TCI_CRT_MMA=$v timeout 600 python bench.py --steps 5 --warmup 3 --alt none --no-e2e --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_crt$v.json
  echo "crt_mma=$v $(cut -c1-220 gpurun_out/bench_crt$v.json)"
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --alt none --no-e2e --no-cpu-baseline > /dev/null 2>&1
python tools/launch_table.py gpurun_out/launches.csv --steps 3 2>&1 | head -8 | tee gpurun_out/launches.txt
