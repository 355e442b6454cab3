#!/bin/bash
# Quick 1-GPU check: selected GPU tests (pytest -k expression $1, "all" = every GPU test,
# "none" = skip), smoke, bench line, launch list of bench steps.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv,noheader
K="${1:-ozaki}"
if [ "$K" = "all" ]; then
  timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt
elif [ "$K" != "none" ]; then
  timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "$K" 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt
fi
[ -f gpurun_out/pytest_gpu.txt ] && tail -4 gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3 | tee gpurun_out/smoke.txt
timeout 900 python bench.py --steps 10 --warmup 3 ${BENCH_ARGS} 2>&1 | tail -1 > gpurun_out/bench.json
cut -c1-700 gpurun_out/bench.json
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --alt none --no-e2e --no-cpu-baseline > /dev/null 2>&1
python tools/launch_table.py gpurun_out/launches.csv --steps 3 2>&1 | head -14 | tee gpurun_out/launches.txt
