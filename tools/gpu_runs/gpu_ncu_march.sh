mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:b2o_k1 -s 3 -c 1 -o gpurun_out/mg_march python tools/kernel_sweep.py nasmg_258 100100 '{"quad_march": 8, "march_block": 128}' > gpurun_out/ncu_mg_march.log 2>&1
