mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/kernel_sweep.py nasmg_258 100100 '{}' '{"quad_march": 0}' > gpurun_out/sweep_mg.log 2>&1
