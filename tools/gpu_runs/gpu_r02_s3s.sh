mkdir -p gpurun_out/r02s3
timeout 900 python -m pytest tests/test_ops_gpu.py -q -p no:randomly > gpurun_out/r02s3/pytest_ops_araw.log 2>&1
echo "rc=$?" >> gpurun_out/r02s3/pytest_ops_araw.log; tail -3 gpurun_out/r02s3/pytest_ops_araw.log
for a in 0 1; do echo "ARAW=$a $(B2O_GEMM_ARAW=$a python tools/ops_bench.py 4096 2>&1 | grep gemm_3x)"; done
for a in 0 1; do B2O_GEMM_ARAW=$a python tools/gemm_accuracy.py 2>&1 | tail -2; done
