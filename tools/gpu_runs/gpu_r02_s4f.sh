mkdir -p gpurun_out/r02s4
timeout 1200 python -m pytest tests/test_parity_gpu.py -q -p no:randomly -m gpu > gpurun_out/r02s4/pytest_parity_order.log 2>&1
echo "rc=$?" >> gpurun_out/r02s4/pytest_parity_order.log; tail -5 gpurun_out/r02s4/pytest_parity_order.log
