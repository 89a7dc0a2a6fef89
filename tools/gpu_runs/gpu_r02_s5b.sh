mkdir -p gpurun_out/r02s5
timeout 1200 python -m pytest tests/test_fullsize_gpu.py -q -p no:randomly -m gpu -k fp64 > gpurun_out/r02s5/pytest_fp64_M.log 2>&1
echo "rc=$?" >> gpurun_out/r02s5/pytest_fp64_M.log; tail -3 gpurun_out/r02s5/pytest_fp64_M.log
