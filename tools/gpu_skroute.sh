timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "contract or mps or gemm or splitk or permute" 2>&1 | tail -2
python tools/bench_extra.py --only mpo --out gpurun_out/extra_mpo.json 2>&1 | tail -1
TCI_CONTRACT_NO_SKINNY=1 python tools/bench_extra.py --only mpo --out gpurun_out/extra_mpo_noskinny.json 2>&1 | tail -1
python tools/bench_extra.py --only sweep --out gpurun_out/extra_sweep3.json 2>&1 | grep -o "median_frac_of_roofline.\{0,40\}"
