set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
lscpu | head -20
mkdir -p gpurun_out
./tools/probe_fp64 | tee gpurun_out/probe_fp64.json
./tools/probe_fp64 | tee -a gpurun_out/probe_fp64.json
python tools/probe_torch.py | tee gpurun_out/probe_torch.json
