mkdir -p gpurun_out/r02
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_fullsize_gpu.py tests/test_integration_gpu.py tests/test_ops_gpu.py tests/test_histogram.py -m gpu -q -x > gpurun_out/r02/pytest_e.log 2>&1
echo "rc=$?" >> gpurun_out/r02/pytest_e.log
python tools/e2e_trace.py 3 > gpurun_out/r02/e2e_trace2.jsonl 2> gpurun_out/r02/e2e_trace2.err
tail -3 gpurun_out/r02/pytest_e.log
