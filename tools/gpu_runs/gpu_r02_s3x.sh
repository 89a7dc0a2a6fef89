mkdir -p gpurun_out/r02s3
timeout 900 python tools/kernel_sweep.py matmul_1024 10 '{}' '{"ktile_tile": 60}' '{"ktile_tile": 56}' '{"ktile_tile": 48}' > gpurun_out/r02s3/sweep_ktile60.jsonl 2> gpurun_out/r02s3/sweep_ktile60.err
cat gpurun_out/r02s3/sweep_ktile60.jsonl; tail -2 gpurun_out/r02s3/sweep_ktile60.err
