# ncu launch list of bench steps (Ozaki only: no alt / e2e / cpu legs): every own kernel's
# device time, DRAM bytes, clock. Serialised and cold: compare shares, not absolutes.
mkdir -p gpurun_out
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second \
  --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --alt none --no-e2e --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/launches_bench.log 2>&1
tail -n 2 gpurun_out/launches_bench.log | cut -c1-300
