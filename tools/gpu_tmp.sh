mkdir -p gpurun_out
timeout 900 python bench.py --ops 0 --reductions 0 --steps 10 > gpurun_out/bench_ga.log 2>&1
timeout 900 python bench.py --ops 0 --reductions 0 --steps 10 --ga-dedupe 0 > gpurun_out/bench_ga_nodedupe.log 2>&1
timeout 600 python -m pytest tests/test_integration_gpu.py tests/test_runner_gpu.py -m gpu -x -q > gpurun_out/pytest_int.log 2>&1
