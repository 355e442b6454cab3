timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "permute or contract or gemm" 2>&1 | tail -4
python tools/bench_extra.py --only permute --out gpurun_out/extra_permute.json 2>&1 | tail -2
python tools/sweep_breakdown.py 2>&1 | tail -25
