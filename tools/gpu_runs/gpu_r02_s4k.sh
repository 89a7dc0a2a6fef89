timeout 900 python -m pytest tests/test_histogram.py tests/test_ops_gpu.py -q -p no:randomly -m gpu 2>&1 | tail -2
python tools/ops_bench.py 4096 2>&1 | grep '"histogram"'
