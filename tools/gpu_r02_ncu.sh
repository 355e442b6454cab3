#!/bin/bash
# ncu --set full captures of the bench step's Ozaki kernels (summaries on the box).
# Usage: bash tools/gpu_r02_ncu.sh "name:regex:skip name:regex:skip ..."  [pytest -k expr]
mkdir -p gpurun_out
if [ -n "$2" ]; then
  timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "$2" 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt
  tail -4 gpurun_out/pytest_gpu.txt
fi
B="python bench.py --steps 1 --warmup 1 --alt none --no-e2e --no-cpu-baseline"
for spec in $1; do
  IFS=: read name rx skip <<< "$spec"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$rx" -s "$skip" -c 1 \
    -o /tmp/prof_$name -f $B > /dev/null 2>&1
  python tools/ncu_kernel_summary.py /tmp/prof_$name.ncu-rep gpurun_out/ncu_$name.json > /dev/null 2>&1
  ncu -i /tmp/prof_$name.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_${name}_sass.csv 2>/dev/null
  ncu -i /tmp/prof_$name.ncu-rep --page details --csv > gpurun_out/ncu_${name}_details.csv 2>/dev/null
  rm -f /tmp/prof_$name.ncu-rep
  python -c "import json; d=json.load(open('gpurun_out/ncu_$name.json')); print('$name', d['metrics'].get('gpu__time_duration.sum'), d['stall_share'])"
done
du -sh gpurun_out
