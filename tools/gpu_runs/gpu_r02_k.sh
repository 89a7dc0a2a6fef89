mkdir -p gpurun_out/r02
timeout 600 ncu --set full --clock-control none --import-source on -k regex:b2o_k1 -s 5 -c 1 -o gpurun_out/r02/mg_tma python tools/kernel_sweep.py nasmg_258 100100 '{"quad_march": 32, "march_tma_stages": 4}' > gpurun_out/r02/ncu_mg_tma.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:b2o_k1 -s 5 -c 1 -o gpurun_out/r02/mg_reg python tools/kernel_sweep.py nasmg_258 100100 '{"march_tma": false, "quad_march": 16}' > gpurun_out/r02/ncu_mg_reg.log 2>&1
