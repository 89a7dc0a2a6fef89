mkdir -p gpurun_out/r02s3
timeout 1800 python -m pytest tests/test_isolated_gpu.py tests/test_isolated.py tests/test_runner_gpu.py tests/test_integration_gpu.py -q -p no:randomly > gpurun_out/r02s3/pytest_iso.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02s3/pytest_iso.log
tail -15 gpurun_out/r02s3/pytest_iso.log
