#!/bin/bash
# permute experiment: room factor for completing runs (TCI_PERM_RF)
mkdir -p gpurun_out
for rf in 1 2 4; do
  TCI_PERM_RF=$rf timeout 300 python tools/bench_extra.py --only permute --out gpurun_out/perm_rf$rf.json > /dev/null 2>&1
  python -c "
import json;d=json.load(open('gpurun_out/perm_rf$rf.json'))
print('$rf', ' '.join('%.3f'%r['frac_of_copy'] for r in d['permute']))"
done
