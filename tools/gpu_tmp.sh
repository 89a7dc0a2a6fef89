mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_xsum_gpu.py tests/test_reductions.py tests/test_fuzz_shapes.py -m gpu -q -x > gpurun_out/pytest_xsum.log 2>&1
B2O_XSUM_STATS=1 timeout 300 python tools/xsum_bench.py > gpurun_out/xsum_bench.log 2>&1
timeout 300 python tools/xsum_himeno.py > gpurun_out/xsum_himeno.log 2>&1
