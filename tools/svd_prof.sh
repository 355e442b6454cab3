mkdir -p gpurun_out
TCI_SVD_TRACE=1 python tools/svd_trace.py 1024 2>&1 | tail -45
timeout 600 ncu --set full --clock-control none --import-source on -k regex:svd_round -s 300 -c 1 -o gpurun_out/prof_svd_round python tools/svd_diag.py 4096 > gpurun_out/ncu_svd.log 2>&1
ls -la gpurun_out | tail -3
