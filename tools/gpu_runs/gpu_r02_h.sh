mkdir -p gpurun_out/r02
(cd _r01tree && timeout 600 python tools/kernel_sweep.py nasmg_258 100100 '{}' '{"quad_march": 16}') > gpurun_out/r02/sweep_r01code.jsonl 2>&1
timeout 600 python tools/kernel_sweep.py nasmg_258 100100 '{}' '{"march_tma": false}' > gpurun_out/r02/sweep_r02code.jsonl 2>&1
B2O_PDL=0 timeout 600 python tools/kernel_sweep.py nasmg_258 100100 '{}' '{"march_tma": false}' > gpurun_out/r02/sweep_r02code_nopdl.jsonl 2>&1
