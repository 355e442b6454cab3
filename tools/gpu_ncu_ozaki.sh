#!/bin/bash
# ncu evidence for the Ozaki bench default (1 GPU): launch list of one bench step, --set full
# captures of the 5 INT8 GEMM launches of one step, the MPO skinny pass, and the CRT/residue kernels.
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 1 --alt none --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/launches_target_ozaki.csv $B > gpurun_out/ncu_launch_ozaki.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:device_kernel -c 5 \
  -o gpurun_out/prof_gemm_target_ozaki $B > gpurun_out/ncu_full_gemm_ozaki.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:skinny -c 1 \
  -o gpurun_out/prof_skinny_target_ozaki $B > gpurun_out/ncu_full_skinny_ozaki.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k 'regex:^(crt_kernel|residues|residues_t|line_exponent)$' -c 4 \
  -o gpurun_out/prof_aux_target_ozaki $B > gpurun_out/ncu_full_aux_ozaki.log 2>&1
ls -la gpurun_out | tail -8
