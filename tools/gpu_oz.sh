#!/bin/bash
# Ozaki auxiliary-kernel check: GPU parity (ozaki + heff), launch list of one step
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "ozaki or heff or lanczos or env or gather" 2>&1 | tail -2
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/launches_oz.csv python bench.py --steps 1 --warmup 1 --alt none --no-e2e --no-cpu-baseline > /dev/null 2>&1
python tools/launch_table.py gpurun_out/launches_oz.csv --steps 2 2>&1 | grep -v "at::" | head -8
