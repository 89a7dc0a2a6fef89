mkdir -p gpurun_out/r02
timeout 600 python tools/kernel_sweep.py nasmg_258 100100 '{}' '{"march_tma": false}' '{"march_tma_stages": 2}' '{"march_tma_stages": 4}' '{"quad_march": 16}' '{"quad_march": 32}' '{"quad_march": 16, "march_tma_stages": 4}' '{"march_block": 256}' '{"quad_march": 16, "march_block": 256}' > gpurun_out/r02/sweep_mg_tma.jsonl 2> gpurun_out/r02/sweep_mg_tma.err
timeout 900 python -m pytest tests/test_fuzz_shapes.py tests/test_fullsize_gpu.py tests/test_kernel_options_gpu.py -m gpu -q -x -k "nasmg or shapes or bit_exact or march" > gpurun_out/r02/pytest_g.log 2>&1
echo "rc=$?" >> gpurun_out/r02/pytest_g.log
