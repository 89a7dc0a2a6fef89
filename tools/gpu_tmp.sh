mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_ops_gpu.py -q -x -m gpu > gpurun_out/pytest_ops.log 2>&1
timeout 300 python tools/ops_bench.py > gpurun_out/ops.log 2>&1
B2O_GEMM_SPLIT_PREP=1 timeout 300 python tools/ops_bench.py > gpurun_out/ops_old.log 2>&1
timeout 600 python bench.py --ga 0 --reductions 0 --steps 5 > gpurun_out/bench_ops.log 2>&1
