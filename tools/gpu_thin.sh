timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -4
python tools/sweep_breakdown.py 2>&1 | grep -o "^[0-9]* r[0-9]*\|us=[0-9]* roof=[0-9]*\|'gemm': ([0-9]*, [0-9]*)\|'permute': ([0-9]*, [0-9]*)" | paste - - - -
