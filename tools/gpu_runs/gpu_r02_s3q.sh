mkdir -p gpurun_out/r02s3
timeout 900 python tools/kernel_sweep.py nasmg_258 100100 '{}' '{"flat_min_blocks": 8}' '{"march_block": 96}' '{"march_block": 64}' '{"march_l2pf": 1}' '{"march_l2pf": 3}' '{"quad_march": 10}' '{"quad_march": 14}' '{"march_block": 192}' > gpurun_out/r02s3/sweep_mg_chains2.jsonl 2> gpurun_out/r02s3/sweep_mg_chains2.err
cat gpurun_out/r02s3/sweep_mg_chains2.jsonl
