mkdir -p gpurun_out/r02s3
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fft4k -c 2 -o gpurun_out/r02s3/fft python tools/ops_bench.py 4096 > gpurun_out/r02s3/ncu_fft.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"gemm_tc_pair|prep_kernel" -c 2 -o gpurun_out/r02s3/gemm python tools/ops_bench.py 4096 > gpurun_out/r02s3/ncu_gemm.log 2>&1
python tools/ops_bench.py 4096 > gpurun_out/r02s3/ops.jsonl 2>&1
cat gpurun_out/r02s3/ops.jsonl
