mkdir -p gpurun_out
timeout 900 python tools/kernel_sweep.py nasmg_258 100100 '{}' '{"march_async":2}' '{"march_async":2,"march_block":64}' '{"march_async":3,"march_block":64}' '{"march_async":2,"quad_march":16}' '{"march_async":3,"march_block":64,"quad_march":16}' > gpurun_out/sweep_mg3.log 2>&1
timeout 900 python -m pytest tests/test_kernel_options_gpu.py -m gpu -q -x -k "march_async or ktile" > gpurun_out/pytest_q.log 2>&1
