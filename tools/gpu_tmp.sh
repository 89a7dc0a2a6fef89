mkdir -p gpurun_out
{ timeout 300 python tools/tf32_probe.py; B2O_GEMM_SPLIT=0 timeout 300 python tools/gemm_accuracy.py; B2O_GEMM_SPLIT=2 timeout 300 python tools/gemm_accuracy.py; } > gpurun_out/gemm_mode.log 2>&1
{ B2O_GEMM_SPLIT=0 timeout 300 python tools/ops_bench.py; B2O_GEMM_SPLIT=2 timeout 300 python tools/ops_bench.py; B2O_GEMM_SPLIT=0 timeout 300 python tools/ops_bench.py; B2O_GEMM_SPLIT=2 timeout 300 python tools/ops_bench.py; } > gpurun_out/gemm_mode_bench.log 2>&1
B2O_GEMM_SPLIT=2 timeout 900 python -m pytest tests/test_ops_gpu.py -m gpu -q -x > gpurun_out/pytest_ops_mode2.log 2>&1
