mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/e2e_trace.py > gpurun_out/e2e_async.log 2>&1
B2O_SYNC_D2H=1 timeout 300 python tools/e2e_trace.py > gpurun_out/e2e_sync.log 2>&1
timeout 600 python bench.py --ga 0 --ops 0 --reductions 0 > gpurun_out/bench_quick.log 2>&1
