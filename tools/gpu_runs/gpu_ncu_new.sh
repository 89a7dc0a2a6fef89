mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:b2o_k1 -s 3 -c 1 -o gpurun_out/mg_resid_march python tools/kernel_sweep.py nasmg_258 100100 '{}' > gpurun_out/ncu_mg.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:b2o_k0 -s 3 -c 1 -o gpurun_out/matmul_ktile python tools/kernel_sweep.py matmul_1024 10 '{}' > gpurun_out/ncu_mm.log 2>&1
timeout 300 python tools/apps_bench.py > gpurun_out/apps_bench.jsonl 2> gpurun_out/apps_bench.err
