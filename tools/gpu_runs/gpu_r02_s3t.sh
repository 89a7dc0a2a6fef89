mkdir -p gpurun_out/r02s3
B2O_FFT_V=4 timeout 900 python -m pytest tests/test_ops_gpu.py -q -p no:randomly -k fft > gpurun_out/r02s3/pytest_fft_push.log 2>&1
echo "rc=$?" >> gpurun_out/r02s3/pytest_fft_push.log; tail -2 gpurun_out/r02s3/pytest_fft_push.log
for v in 1 4 1 4; do echo "V=$v $(B2O_FFT_V=$v python tools/ops_bench.py 4096 2>&1 | grep fft2d)"; done
