timeout 600 python -m pytest tests/test_gpu_svd.py -q -x 2>&1 | tail -2
TCI_SVD_PROFILE=1 python tools/svd_diag.py 2048 4096 2>&1 | grep -o "n=.*sweeps=[0-9]*\|max|ds|/s0=[0-9.e-]*\|eig [0-9]*" | paste - - - | head -6
