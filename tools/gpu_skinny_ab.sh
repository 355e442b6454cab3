#!/bin/bash
# DMMA MPO pass: parity of the chains, launch list of one bench step
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "heff or env or mpo or gather or lanczos or zipup or skinny" 2>&1 | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/launches_sk.csv python bench.py --steps 1 --warmup 1 --alt none --no-e2e --no-cpu-baseline > /dev/null 2>&1
python tools/launch_table.py gpurun_out/launches_sk.csv --steps 2 2>&1 | grep -E "skinny"
