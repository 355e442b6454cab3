mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_ozaki_structured.py -m gpu -q -x -s 2>&1 | tail -40 | tee gpurun_out/t_struct.txt
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -30 | tee gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --steps 5 --warmup 3 2>&1 | tail -3 | tee gpurun_out/bench.txt
