mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_fp64_gpu.py -m gpu -q -x > gpurun_out/pytest_fp64_final.log 2>&1
