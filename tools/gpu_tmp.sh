mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_fuzz_shapes.py tests/test_reductions.py tests/test_xsum_gpu.py tests/test_parity_gpu.py -m gpu -q > gpurun_out/pytest_shapes.log 2>&1
