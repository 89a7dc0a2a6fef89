mkdir -p gpurun_out/r02s3
timeout 900 python tools/kernel_sweep.py nasmg_258 100100 '{}' '{"march_chains": true}' '{"march_chains": true, "quad_march": 16}' '{"march_chains": true, "quad_march": 8}' '{"march_chains": true, "march_block": 64}' '{"march_chains": true, "march_block": 256}' '{"march_chains": true, "march_l2pf": 2}' '{"march_chains": true, "march_l2pf": 4}' > gpurun_out/r02s3/sweep_mg_chains.jsonl 2> gpurun_out/r02s3/sweep_mg_chains.err
cat gpurun_out/r02s3/sweep_mg_chains.jsonl
KS_NOWARM=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:b2o_k1 -s 2 -c 1 -o gpurun_out/r02s3/mg_march_chains python tools/kernel_sweep.py nasmg_258 100100 '{"march_chains": true}' > gpurun_out/r02s3/ncu_mg_march_chains.log 2>&1
