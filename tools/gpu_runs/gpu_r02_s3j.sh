mkdir -p gpurun_out/r02s3
timeout 1800 python -m pytest tests/test_fuzz_shapes.py tests/test_fullsize_gpu.py tests/test_kernel_options_gpu.py tests/test_parity_gpu.py tests/test_fp64_gpu.py -m gpu -q -p no:randomly > gpurun_out/r02s3/pytest_chains.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02s3/pytest_chains.log
KS_NOWARM=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:b2o_k1 -s 4 -c 1 -o gpurun_out/r02s3/mg_march_chains2 python tools/kernel_sweep.py nasmg_258 100100 '{}' > gpurun_out/r02s3/ncu_mg_march_chains2.log 2>&1
tail -3 gpurun_out/r02s3/pytest_chains.log
