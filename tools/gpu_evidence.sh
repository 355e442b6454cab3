#!/bin/bash
# Round evidence (1 GPU): GPU tests, smoke, bench line, ncu launch list of one bench step,
# ncu --set full captures of the step's kernels (summarised to JSON on the box; the .ncu-rep
# files are deleted so gpurun_out stays under its 64 MiB limit), permute table.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3 | tee gpurun_out/pytest_gpu.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 | tee gpurun_out/smoke.txt
timeout 900 python bench.py --steps 5 --warmup 3 2>&1 | tail -1 > gpurun_out/bench_final.json
B="python bench.py --steps 1 --warmup 1 --alt none --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/launches_target_ozaki.csv $B > /dev/null 2>&1
cap() {   # name, kernel regex, launch skip
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$2" -s "$3" -c 1 \
    -o /tmp/prof_$1 -f $B > /dev/null 2>&1
  python tools/ncu_kernel_summary.py /tmp/prof_$1.ncu-rep gpurun_out/ncu_$1.json > /dev/null 2>&1
  rm -f /tmp/prof_$1.ncu-rep
}
cap gemm1_int8 device_kernel 0
cap gemm4_int8 device_kernel 4
cap crt '^crt_kernel' 0
cap residues '^residues$' 0
cap residues_t '^residues_t$' 0
cap skinny_dmma '^skinny_dmma_kernel' 0
cap line_exponent '^line_exponent$' 0
timeout 300 python tools/bench_extra.py --only permute --out gpurun_out/extra_permute.json > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:permute_groups -c 1 \
  -o /tmp/prof_permute -f python tools/bench_extra.py --only permute --out /tmp/x.json > /dev/null 2>&1
python tools/ncu_kernel_summary.py /tmp/prof_permute.ncu-rep gpurun_out/ncu_permute_groups.json > /dev/null 2>&1
du -sh gpurun_out; ls gpurun_out
