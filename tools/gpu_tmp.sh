mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke3.log 2>&1
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_fuzz.py -m gpu -q -x > gpurun_out/pytest_final_q.log 2>&1
