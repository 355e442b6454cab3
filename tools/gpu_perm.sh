#!/bin/bash
# permute / thin-GEMM check: GPU parity of every test, permute bandwidth table
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -4 | tee gpurun_out/pytest_gpu.txt
timeout 300 python tools/bench_extra.py --only permute --out gpurun_out/extra_permute.json 2>&1 | tail -2
python -c "
import json;d=json.load(open('gpurun_out/extra_permute.json'))
for r in d['permute']: print(r['shape'],r['perm'],r['dtype'],round(r['GBs']),round(r['frac_hbm'],3), round(r['frac_of_copy'],3))"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/perm_launches.csv python tools/bench_extra.py --only permute --out gpurun_out/extra_permute_ncu.json > /dev/null 2>&1
