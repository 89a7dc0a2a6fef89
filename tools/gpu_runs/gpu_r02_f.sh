mkdir -p gpurun_out/r02
timeout 900 python -m pytest tests/test_abi.py tests/test_parity_gpu.py -m gpu -q -x > gpurun_out/r02/pytest_f.log 2>&1
echo "rc=$?" >> gpurun_out/r02/pytest_f.log
tail -3 gpurun_out/r02/pytest_f.log
