#!/bin/bash
# Round evidence (1 GPU): GPU tests, smoke, bench line, ncu launch list of one bench step,
# ncu --set full captures of the step's kernels, permute table + capture.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3 | tee gpurun_out/pytest_gpu.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 | tee gpurun_out/smoke.txt
timeout 900 python bench.py --steps 5 --warmup 3 2>&1 | tail -1 > gpurun_out/bench_final.json
B="python bench.py --steps 1 --warmup 1 --alt none --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/launches_target_ozaki.csv $B > /dev/null 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:device_kernel -c 5 \
  -o gpurun_out/prof_gemm_target_ozaki -f $B > /dev/null 2>&1
for k in crt_kernel residues residues_t skinny_stream_kernel line_exponent; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^${k}\$" -c 1 \
    -o gpurun_out/prof_${k} -f $B > /dev/null 2>&1
done
timeout 300 python tools/bench_extra.py --only permute --out gpurun_out/extra_permute.json > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:permute_groups -c 2 \
  -o gpurun_out/prof_permute_groups -f python tools/bench_extra.py --only permute --out gpurun_out/x.json > /dev/null 2>&1
ls -la gpurun_out | tail -20
