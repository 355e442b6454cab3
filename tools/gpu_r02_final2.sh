#!/bin/bash
# Round-2 final evidence (1 GPU) after the tensor-core CRT: every GPU test, smoke,
# the bench line with default flags (as the driver runs it), the launch list of
# bench steps, ncu --set full summaries of the step's kernels, a SASS excerpt.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv,noheader
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 --timeout-method thread 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt
tail -2 gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3 | tee gpurun_out/smoke.txt
timeout 900 python bench.py 2>&1 | tail -1 > gpurun_out/bench.json
cut -c1-300 gpurun_out/bench.json
B="python bench.py --steps 1 --warmup 1 --alt none --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/launches.csv $B > /dev/null 2>&1
python tools/launch_table.py gpurun_out/launches.csv --steps 3 > gpurun_out/launches.txt 2>&1
head -12 gpurun_out/launches.txt
for spec in gemm1:i8gemm_kernel:0 gemm4:i8gemm_kernel:2 crt_mma:crt_mma_kernel:0 res_k:^residues\$:0 res_l:^residues_t\$:0 skinny:skinny_dmma_kernel:0; do
  IFS=: read name rx skip <<< "$spec"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$rx" -s "$skip" -c 1 -o /tmp/prof_$name -f $B > /dev/null 2>&1
  python tools/ncu_kernel_summary.py /tmp/prof_$name.ncu-rep gpurun_out/ncu_$name.json > /dev/null 2>&1
  rm -f /tmp/prof_$name.ncu-rep
done
cuobjdump -sass paper_2512_23917_b200/libtci_b200.so 2>/dev/null | grep -E "Function : .*(i8gemm|crt_mma|tebd_tma|gemm_f32_dmma)|UTCIMMA|UTCMMA|UTMALDG|UTMASTG|UTCBAR|LDTM|DMMA" | sort | uniq -c | sort -rn | head -30 > gpurun_out/sass_excerpt.txt
ls gpurun_out
