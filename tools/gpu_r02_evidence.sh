#!/bin/bash
# Round-2 evidence (1 GPU): GPU tests, smoke, bench line, ncu launch list of bench steps,
# ncu --set full captures of the step's top kernels (summarised on the box, .ncu-rep deleted).
# Usage: gpurun --timeout 3000 -- 'bash tools/gpu_r02_evidence.sh [tests|notests]'
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
if [ "${1:-tests}" = "tests" ]; then
  timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt
  tail -3 gpurun_out/pytest_gpu.txt
fi
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3 | tee gpurun_out/smoke.txt
timeout 900 python bench.py --steps 10 --warmup 3 2>&1 | tail -1 > gpurun_out/bench.json
cut -c1-400 gpurun_out/bench.json
B="python bench.py --steps 1 --warmup 1 --alt none --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/launches.csv $B > /dev/null 2>&1
python tools/launch_table.py gpurun_out/launches.csv --steps 2 > gpurun_out/launches.txt 2>&1
head -30 gpurun_out/launches.txt
cap() {   # name, kernel regex, launch skip
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$2" -s "$3" -c 1 \
    -o /tmp/prof_$1 -f $B > /dev/null 2>&1
  python tools/ncu_kernel_summary.py /tmp/prof_$1.ncu-rep gpurun_out/ncu_$1.json > /dev/null 2>&1
  ncu -i /tmp/prof_$1.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    > gpurun_out/ncu_$1_raw.csv 2>/dev/null
  rm -f /tmp/prof_$1.ncu-rep
}
# i8gemm launch order within one step: printed by the launch table (GEMM1 chunks first, GEMM4 last)
NG=$(python - <<'EOF'
import csv, io
t = open('gpurun_out/launches.csv').read()
rows = list(csv.DictReader(io.StringIO(t[t.find('"ID"'):])))
ids = {int(r['ID']) for r in rows if 'i8gemm_kernel' in r['Kernel Name']}
crt = {int(r['ID']) for r in rows if r['Kernel Name'].startswith('void tci::') is False and 'crt_kernel' in r['Kernel Name']}
# CRT runs once per GEMM1 chunk and once per GEMM4 chunk; applies = launches of the MPO pass
mpo = {int(r['ID']) for r in rows if 'skinny' in r['Kernel Name']}
print(max(1, len(ids) // max(1, len(mpo))))
EOF
)
echo "i8gemm launches per step: $NG"
cap gemm1_int8 i8gemm_kernel 0
cap gemm4_int8 i8gemm_kernel $((NG - 1))
cap crt '^crt_kernel' 0
cap residues '^residues$' 0
cap residues_t '^residues_t$' 0
cap skinny_dmma '^skinny_dmma_kernel' 0
cuobjdump -sass paper_2512_23917_b200/libtci_b200.so 2>/dev/null | grep -E "Function : .*i8gemm|UTCIMMA|UTMALDG|UTMASTG|UTCBAR" | sort | uniq -c | head -20 > gpurun_out/i8gemm_sass_excerpt.txt
du -sh gpurun_out; ls gpurun_out
