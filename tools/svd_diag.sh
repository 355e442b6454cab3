timeout 600 python -m pytest tests/test_gpu_svd.py -x -q 2>&1 | tail -2
python tools/svd_diag.py 2048 4096 2>&1 | tail -4
python tools/bench_extra.py --only svd --out gpurun_out/extra_svd.json 2>&1 | tail -1 | cut -c1-400
