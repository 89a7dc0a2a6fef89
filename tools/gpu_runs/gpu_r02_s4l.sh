timeout 900 python -m pytest tests/test_ops_gpu.py -q -p no:randomly -m gpu -k gemm 2>&1 | tail -2
for i in 1 2 3; do python tools/ops_bench.py 4096 2>&1 | grep gemm_3x; done
