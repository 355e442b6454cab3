#!/bin/bash
# Ozaki auxiliary-kernel check: GPU parity (ozaki + heff), bench, launch list of one step
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "ozaki or heff or lanczos or env" 2>&1 | tail -3 | tee gpurun_out/pytest_oz.txt
timeout 600 python bench.py --steps 8 --warmup 3 --alt none --no-e2e 2>&1 | tail -1 > gpurun_out/bench_oz.json
python -c "import json; d=json.load(open('gpurun_out/bench_oz.json')); print('value', d['value'], 'ms', d['ms_per_step'], 'parity', d['parity'], 'clk', d['clocks'])"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/launches_oz.csv python bench.py --steps 1 --warmup 1 --alt none --no-e2e --no-cpu-baseline > /dev/null 2>&1
python tools/launch_table.py gpurun_out/launches_oz.csv --steps 2 2>&1 | head -14
