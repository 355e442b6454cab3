mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "ozaki or f32 or heff" 2>&1 | tail -3
B="python bench.py --steps 1 --warmup 1 --alt none --no-e2e --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_a.csv $B > /dev/null 2>&1
python tools/launch_table.py gpurun_out/launches_a.csv --steps 3 2>&1 | head -9
TCI_CRT_CFG=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_b.csv $B > /dev/null 2>&1
echo "== TCI_CRT_CFG=1"; python tools/launch_table.py gpurun_out/launches_b.csv --steps 3 2>&1 | grep crt
timeout 300 python bench.py --steps 8 --warmup 3 --alt none --no-e2e --no-cpu-baseline 2>&1 | tail -1 | cut -c1-300
TCI_CRT_CFG=1 timeout 300 python bench.py --steps 8 --warmup 3 --alt none --no-e2e --no-cpu-baseline 2>&1 | tail -1 | cut -c1-300
timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool racecheck python tools/sanitize_cases.py svd_small 2>&1 | tail -25 > gpurun_out/rc_svd_small.txt
