#!/bin/bash
# ncu --set full of one kernel of the bench step: $1 = name (output tag), $2 = kernel regex, $3 = launches to skip
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 1 --alt none --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$2" -s "${3:-0}" -c 1 -o /tmp/prof_$1 -f $B > gpurun_out/ncu_$1.log 2>&1
python tools/ncu_kernel_summary.py /tmp/prof_$1.ncu-rep gpurun_out/ncu_$1.json > /dev/null 2>&1
ncu -i /tmp/prof_$1.ncu-rep --page source --csv > gpurun_out/ncu_$1_source.csv 2>/dev/null
ncu -i /tmp/prof_$1.ncu-rep --page raw --csv > gpurun_out/ncu_$1_raw.csv 2>/dev/null
cp /tmp/prof_$1.ncu-rep gpurun_out/ 2>/dev/null
