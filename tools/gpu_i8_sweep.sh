mkdir -p gpurun_out
timeout 600 ./tools/i8gemm_lab sweep 2>&1 | tee gpurun_out/lab_sweep.txt
timeout 900 ncu --clock-control none --metrics dram__bytes_read.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum -k regex:i8gemm_kernel --csv ./tools/i8gemm_lab sweep > gpurun_out/lab_sweep_ncu.csv 2>&1
