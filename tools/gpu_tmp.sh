mkdir -p gpurun_out
timeout 300 python tools/kernel_sweep.py matmul_1024 10 '{}' '{"ktile_r": 8}' '{"ktile_r": 8, "ktile_tile": 128}' > gpurun_out/sweep_mm.log 2>&1
timeout 300 python tools/kernel_sweep.py matmul_48 10 '{"ktile_r": 8}' >> gpurun_out/sweep_mm.log 2>&1
