#!/bin/bash
# bench.py step time under INT8-GEMM raster / chunk-budget settings (DESIGN.md §12 tuning)
mkdir -p gpurun_out
B="python bench.py --steps 8 --warmup 3 --alt none --no-e2e --no-cpu-baseline"
for cfg in "" "TCI_I8_RES_MB=24" "TCI_I8_RES_MB=32" "TCI_I8_RES_MB=64" "TCI_I8_RES_MB=96" "TCI_OZ_CHUNK_GB=16" "TCI_OZ_CHUNK_GB=24" "TCI_OZ_CHUNK_GB=24 TCI_I8_RES_MB=64"; do
  r=$(env $cfg timeout 600 $B 2>&1 | tail -1)
  python3 -c "import json,sys; d=json.loads(sys.argv[1]); print('%-40s %.2f ms  %.1f TF/s  sm %s' % (sys.argv[2] or 'default', d['ms_per_step'], d['value'], d['clocks']['sm_mhz']))" "$r" "$cfg" | tee -a gpurun_out/tune_i8.txt
done
