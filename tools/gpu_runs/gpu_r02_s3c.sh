mkdir -p gpurun_out/r02s3
timeout 900 python tools/kernel_sweep.py nasmg_258 100100 '{}' '{"march_l2pf": 0}' '{"quad_march": 8}' '{"quad_march": 12}' '{"quad_march": 8, "march_l2pf": 3}' '{"quad_march": 12, "march_l2pf": 3}' '{"march_block": 96}' '{"march_prefetch": true}' '{"march_l2pf": 2, "flat_min_blocks": 6}' '{"quad_march": 20}' > gpurun_out/r02s3/sweep_mg_l2pf2.jsonl 2> gpurun_out/r02s3/sweep_mg_l2pf2.err
cat gpurun_out/r02s3/sweep_mg_l2pf2.jsonl
