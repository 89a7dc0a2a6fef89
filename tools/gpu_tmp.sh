mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_reductions.py tests/test_xsum_gpu.py -m gpu -x -q > gpurun_out/pytest_red.log 2>&1
timeout 300 python tools/e2e_trace.py > gpurun_out/e2e_red.log 2>&1
