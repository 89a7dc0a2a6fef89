mkdir -p gpurun_out/r02s3
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02s3/smi.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:randomly --durations=15 > gpurun_out/r02s3/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02s3/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02s3/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/r02s3/smoke.log
timeout 900 python bench.py > gpurun_out/r02s3/bench.json 2> gpurun_out/r02s3/bench.err
echo "bench rc=$?" >> gpurun_out/r02s3/bench.err
tail -5 gpurun_out/r02s3/pytest_gpu.log; cat gpurun_out/r02s3/smoke.log; tail -c 600 gpurun_out/r02s3/bench.json
