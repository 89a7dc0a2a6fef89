mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_fuzz.py tests/test_kernel_options_gpu.py tests/test_fp64_gpu.py -m gpu -q -x > gpurun_out/pytest_fuzz96.log 2>&1
