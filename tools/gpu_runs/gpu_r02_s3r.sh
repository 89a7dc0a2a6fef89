mkdir -p gpurun_out/r02s3
timeout 900 python tools/kernel_sweep.py nasmg_258 100100 '{}' '{"march_shfl": true}' '{"march_shfl": true, "march_block": 64}' '{"march_shfl": true, "quad_march": 16}' '{"march_shfl": true, "march_chains": false}' > gpurun_out/r02s3/sweep_mg_shfl.jsonl 2> gpurun_out/r02s3/sweep_mg_shfl.err
cat gpurun_out/r02s3/sweep_mg_shfl.jsonl; tail -3 gpurun_out/r02s3/sweep_mg_shfl.err
timeout 1200 python -m pytest tests/test_kernel_options_gpu.py -q -p no:randomly -k "march" > gpurun_out/r02s3/pytest_opts_shfl.log 2>&1
tail -3 gpurun_out/r02s3/pytest_opts_shfl.log
