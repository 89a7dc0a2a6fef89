set -x
timeout 300 python tools/kernel_sweep.py himeno_M 100100 "{}" "{\"flat_min_blocks\": 2}" "{\"flat_min_blocks\": 1}" > gpurun_out/sweep_M.log 2>&1
timeout 300 python tools/kernel_sweep.py himeno_L 100100 "{}" "{\"flat_min_blocks\": 2}" > gpurun_out/sweep_L.log 2>&1
timeout 300 python tools/kernel_sweep.py nasmg_258 100100 "{}" "{\"stencil\": true}" "{\"flat_min_blocks\": 2}" > gpurun_out/sweep_mg.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:b2o_k1 -s 4 -c 2 -o gpurun_out/jacobi_quad python bench.py --steps 3 --warmup 3 --ga 0 --ops 0 > gpurun_out/ncu_jacobi.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 3 --warmup 3 --ga 0 --ops 0 > gpurun_out/ncu_launches.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:b2o_k1 -s 2 -c 1 -o gpurun_out/mg_resid python tools/kernel_sweep.py nasmg_258 100100 "{}" > gpurun_out/ncu_mg.log 2>&1
