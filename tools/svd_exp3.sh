#!/bin/bash
# SVD row sorting inside block pairs on / off: random n x n (r64, c128)
for so in 1 0; do echo "== SORT=$so"; TCI_SVD_SORT=$so timeout 600 python tools/svd_diag.py 1024 2048 2>&1 | tail -4; done
