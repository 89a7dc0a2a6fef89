mkdir -p gpurun_out/r02s3
timeout 900 python tools/kernel_sweep.py nasmg_258 100100 '{}' '{"march_l2pf": 1}' '{"march_l2pf": 2}' '{"march_l2pf": 3}' '{"march_l2pf": 4}' '{"march_l2pf": 6}' '{"march_l2pf": 2, "quad_march": 32}' '{"march_l2pf": 3, "quad_march": 24}' '{"march_l2pf": 2, "march_block": 64}' '{"march_l2pf": 2, "march_block": 256}' > gpurun_out/r02s3/sweep_mg_l2pf.jsonl 2> gpurun_out/r02s3/sweep_mg_l2pf.err
cat gpurun_out/r02s3/sweep_mg_l2pf.jsonl
