mkdir -p gpurun_out/r02s3
B2O_GEMM_FUSED=1 timeout 600 python -m pytest tests/test_ops_gpu.py -q -p no:randomly -k gemm -x > gpurun_out/r02s3/pytest_gemm_fused.log 2>&1
echo "rc=$?" >> gpurun_out/r02s3/pytest_gemm_fused.log; tail -15 gpurun_out/r02s3/pytest_gemm_fused.log
for f in 0 1; do echo "FUSED=$f $(B2O_GEMM_FUSED=$f timeout 120 python tools/ops_bench.py 4096 2>&1 | grep -E 'gemm_3x|rror')"; done
B2O_GEMM_FUSED=1 timeout 120 python tools/gemm_accuracy.py 2>&1 | tail -3
