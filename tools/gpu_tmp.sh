mkdir -p gpurun_out
timeout 600 python tools/kernel_sweep.py matmul_1024 10 '{}' '{"ktile_ri":8}' '{}' '{"ktile_ri":8}' > gpurun_out/sweep_mm5.log 2>&1
timeout 900 python -m pytest tests/test_kernel_options_gpu.py -m gpu -q -x -k "ktile" > gpurun_out/pytest_q.log 2>&1
