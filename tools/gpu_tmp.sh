mkdir -p gpurun_out
timeout 600 python tools/kernel_sweep.py matmul_1024 10 '{}' '{"ktile_swz":false}' '{}' > gpurun_out/sweep_mm4.log 2>&1
timeout 900 python -m pytest tests/test_fuzz_shapes.py tests/test_parity_gpu.py tests/test_kernel_options_gpu.py -m gpu -q -x > gpurun_out/pytest_q.log 2>&1
