for i in 1 2 3; do python tools/ops_bench.py 4096 2>&1 | grep fft2d; done
