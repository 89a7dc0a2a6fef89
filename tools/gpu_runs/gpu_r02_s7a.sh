mkdir -p gpurun_out/r02s7
timeout 2400 python -m pytest tests -m gpu -q -p no:randomly > gpurun_out/r02s7/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02s7/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02s7/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/r02s7/smoke.log
timeout 900 python bench.py > gpurun_out/r02s7/bench.json 2> gpurun_out/r02s7/bench.err
echo "bench rc=$?" >> gpurun_out/r02s7/bench.err
timeout 900 python bench.py --impl reference > gpurun_out/r02s7/bench_ref.json 2> gpurun_out/r02s7/bench_ref.err
tail -3 gpurun_out/r02s7/pytest_gpu.log; cat gpurun_out/r02s7/smoke.log; tail -1 gpurun_out/r02s7/bench.err
