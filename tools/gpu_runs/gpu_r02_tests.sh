mkdir -p gpurun_out/r02
timeout 2400 python -m pytest tests -m gpu -q -p no:randomly --durations=15 > gpurun_out/r02/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/r02/smoke.log
tail -5 gpurun_out/r02/pytest_gpu.log
