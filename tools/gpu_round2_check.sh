# one gpurun call: GPU tests, smoke, a short bench
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -30 | tee gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5 | tee gpurun_out/smoke.txt
timeout 600 python bench.py --steps 10 --warmup 3 ${BENCH_ARGS} 2>&1 | tail -2 | tee gpurun_out/bench.txt
