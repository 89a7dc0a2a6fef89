mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_xsum_gpu.py -q -x > gpurun_out/pytest_xsum.log 2>&1
B2O_XSUM_STATS=1 timeout 300 python tools/xsum_himeno.py > gpurun_out/xsum_himeno.log 2>&1
timeout 300 python tools/xsum_bench.py > gpurun_out/xsum_bench.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/xsum_launches.csv python tools/xsum_himeno.py > /dev/null 2>&1
timeout 900 python -m pytest tests/test_reductions.py -m gpu -q -x > gpurun_out/pytest_red.log 2>&1
timeout 300 python tools/e2e_trace.py > gpurun_out/e2e_red.log 2>&1
