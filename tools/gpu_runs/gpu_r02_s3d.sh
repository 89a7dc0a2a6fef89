mkdir -p gpurun_out/r02s3
KS_NOWARM=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:b2o_k1 -s 2 -c 1 -o gpurun_out/r02s3/mg_march_pf python tools/kernel_sweep.py nasmg_258 100100 '{}' > gpurun_out/r02s3/ncu_mg_march.log 2>&1
tail -3 gpurun_out/r02s3/ncu_mg_march.log
