# ncu --set full of the INT8 GEMM on the bench's GEMM1 and GEMM4 chunk shapes (lab binary)
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:i8gemm_kernel -s 8 -c 1 -o gpurun_out/ncu_i8_g1 ./tools/i8gemm_lab big > gpurun_out/ncu_i8_g1.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:i8gemm_kernel -s 13 -c 1 -o gpurun_out/ncu_i8_g4 ./tools/i8gemm_lab big > gpurun_out/ncu_i8_g4.log 2>&1
tail -n 1 gpurun_out/ncu_i8_g1.log; tail -n 1 gpurun_out/ncu_i8_g4.log
