mkdir -p gpurun_out
timeout 300 python tools/kernel_sweep.py matmul_1024 01 '{}' > gpurun_out/sweep_mm01.log 2>&1
timeout 300 python tools/kernel_sweep.py himeno_M 001001 '{}' >> gpurun_out/sweep_mm01.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/apps_bench.py > gpurun_out/apps_bench.jsonl 2> gpurun_out/apps_bench.err
