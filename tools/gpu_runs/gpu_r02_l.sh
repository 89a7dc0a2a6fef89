mkdir -p gpurun_out/r02
timeout 900 python tools/kernel_sweep.py nasmg_258 100100 '{}' '{"march_tma": false, "quad_march": 16}' '{"march_tma_stages": 4}' '{"quad_march": 16, "march_tma_stages": 4}' '{"quad_march": 32, "march_tma_stages": 4}' '{"quad_march": 32, "march_tma_stages": 3}' '{"march_block": 256, "quad_march": 16, "march_tma_stages": 3}' > gpurun_out/r02/sweep_mg_tma3.jsonl 2> gpurun_out/r02/sweep_mg_tma3.err
timeout 900 python -m pytest tests/test_fuzz_shapes.py tests/test_fullsize_gpu.py -m gpu -q -x -k "nasmg or bit_exact" > gpurun_out/r02/pytest_l.log 2>&1
echo "rc=$?" >> gpurun_out/r02/pytest_l.log
