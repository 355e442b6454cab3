#!/bin/bash
# ncu evidence (1 GPU): launch list of the bench step + full captures of the GEMM and skinny kernels
mkdir -p gpurun_out
CFG=${CFG:-target}
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k 'regex:gemm_dmma|skinny|transpose_tiles|copy_rows|gemm_simt' --csv --log-file gpurun_out/launches_${CFG}.csv \
  python bench.py --config $CFG --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_bench_${CFG}.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_dmma -s 2 -c 2 \
  -o gpurun_out/prof_gemm_${CFG} python bench.py --config $CFG --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_gemm_${CFG}.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:skinny -s 1 -c 1 \
  -o gpurun_out/prof_skinny_${CFG} python bench.py --config $CFG --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_skinny_${CFG}.log 2>&1
ls -la gpurun_out | tail -8
