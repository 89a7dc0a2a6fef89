mkdir -p gpurun_out/r02s3
timeout 600 python -m pytest tests/test_ops_gpu.py -q -k fft > gpurun_out/r02s3/pytest_fft.log 2>&1
echo "rc=$?" >> gpurun_out/r02s3/pytest_fft.log
tail -3 gpurun_out/r02s3/pytest_fft.log
for c in 0 8 12 16; do echo "clusters<=$c $(B2O_FFT_CLUSTERS=$c python tools/ops_bench.py 4096 2>&1 | grep -E 'fft2d|rror')"; done
echo "old $(B2O_FFT_COLS=cluster python tools/ops_bench.py 4096 2>&1 | grep fft2d)"
timeout 600 ncu --set full --clock-control none -k regex:fft4k -c 2 -o gpurun_out/r02s3/fft_persist python tools/ops_bench.py 4096 > /dev/null 2>&1
