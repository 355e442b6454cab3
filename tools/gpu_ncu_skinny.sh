mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:skinny -s 1 -c 1 -o gpurun_out/prof_skinny_stream python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --alt none > gpurun_out/ncu_skinny.log 2>&1
tail -3 gpurun_out/ncu_skinny.log
