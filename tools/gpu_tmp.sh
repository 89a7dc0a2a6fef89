mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_fuzz_shapes.py -m gpu -q -x > gpurun_out/pytest_shapes90.log 2>&1
