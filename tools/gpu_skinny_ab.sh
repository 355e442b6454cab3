#!/bin/bash
# DMMA MPO pass: parity (heff / env / mpo tests), A/B bench vs the CUDA-core streaming kernel, launch list
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "heff or env or mpo or lanczos or zipup or gather" 2>&1 | tail -3
for v in 0 1; do
  TCI_SKINNY_DMMA=$v timeout 600 python bench.py --steps 5 --warmup 3 --alt none --no-e2e --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_sk$v.json
  python -c "import json; d=json.load(open('gpurun_out/bench_sk$v.json')); r=d['roofline']['secondary']; print('DMMA=$v', round(d['value'],1), 'TF/s', round(d['ms_per_step'],2), 'ms; MPO pass', round(r['achieved']), 'GB/s share', round(r['share_of_step'],4), d['clocks']['sm_mhz'])"
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/launches_sk.csv python bench.py --steps 1 --warmup 1 --alt none --no-e2e --no-cpu-baseline > /dev/null 2>&1
python tools/launch_table.py gpurun_out/launches_sk.csv --steps 2 2>&1 | grep -E "skinny|total"
