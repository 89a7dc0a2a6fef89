for v in 1 5 1 5; do echo "V=$v $(B2O_FFT_V=$v python tools/ops_bench.py 4096 2>&1 | grep fft2d)"; done
B2O_FFT_V=5 timeout 600 python -m pytest tests/test_ops_gpu.py -q -k fft 2>&1 | tail -1
