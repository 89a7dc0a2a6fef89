mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_xsum_gpu.py tests/test_reductions.py tests/test_fp64_gpu.py tests/test_fuzz_shapes.py -m gpu -q > gpurun_out/pytest_x64.log 2>&1
timeout 1800 python tools/fuzz_big.py run fp64 > gpurun_out/bigfuzz64.log 2>&1
