# A/B of the hand-written INT8 GEMM against the CUTLASS kernel the round-1 build used (lab binary)
mkdir -p gpurun_out
timeout 300 ./tools/i8gemm_lab_cl big 2>&1 | tee gpurun_out/lab_cl.txt
for spec in "i8gemm_kernel 8 own_g1" "i8gemm_kernel 13 own_g4" "GemmUniversal 4 cl_g1" "GemmUniversal 8 cl_g4"; do
  set -- $spec
  timeout 600 ncu --set full --clock-control none -k regex:$1 -s $2 -c 1 -o gpurun_out/ncu_$3 ./tools/i8gemm_lab_cl big > gpurun_out/ncu_$3.log 2>&1
  tail -2 gpurun_out/ncu_$3.log
done
