mkdir -p gpurun_out
timeout 300 python tools/kernel_sweep.py matmul_1024 10 '{}' '{"ktile": false}' > gpurun_out/sweep_mm.log 2>&1
timeout 300 python tools/kernel_sweep.py matmul_1024 11 '{}' > gpurun_out/sweep_mm11.log 2>&1
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_fullsize_gpu.py tests/test_fuzz.py -m gpu -x -q > gpurun_out/pytest_parity.log 2>&1
