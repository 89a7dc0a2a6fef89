mkdir -p gpurun_out/r02s3
timeout 900 python tools/kernel_sweep.py nasmg_258 100100 '{}' '{"march_fill": false}' '{"march_l2pf": 2}' '{"quad_march": 16}' '{"quad_march": 8}' '{"march_block": 64}' '{"march_block": 256}' > gpurun_out/r02s3/sweep_mg_fill.jsonl 2> gpurun_out/r02s3/sweep_mg_fill.err
cat gpurun_out/r02s3/sweep_mg_fill.jsonl
KS_NOWARM=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:b2o_k1 -s 2 -c 1 -o gpurun_out/r02s3/mg_march_fill python tools/kernel_sweep.py nasmg_258 100100 '{}' > gpurun_out/r02s3/ncu_mg_march_fill.log 2>&1
