mkdir -p gpurun_out
timeout 300 python tools/kernel_sweep.py nasmg_258 100100 '{"quad_shfl": false}' '{}' '{"quad_shfl_max": 1}' '{"quad_shfl_max": 3}' '{"quad_shfl_max": 4}' > gpurun_out/sweep_mg.log 2>&1
timeout 300 python tools/kernel_sweep.py himeno_M 100100 '{"quad_shfl": false}' '{}' '{"quad_shfl_max": 1}' '{"quad_shfl_max": 3}' '{"quad_shfl_max": 4}' > gpurun_out/sweep_M.log 2>&1
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_fullsize_gpu.py tests/test_fuzz.py -m gpu -x -q > gpurun_out/pytest_parity.log 2>&1
