mkdir -p gpurun_out
timeout 400 python tools/kernel_sweep.py nasmg_258 100100 '{}' '{"quad_march": 8, "march_block": 128, "march_prefetch": false}' '{"quad_march": 8, "march_block": 128}' '{"quad_march": 16, "march_block": 128}' '{"quad_march": 8, "march_block": 64}' '{"quad_march": 16, "march_block": 64}' '{"quad_march": 4, "march_block": 128}' > gpurun_out/sweep_mg.log 2>&1
