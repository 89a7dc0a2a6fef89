mkdir -p gpurun_out/r02s3
timeout 2400 python -m pytest tests -m gpu -q -p no:randomly > gpurun_out/r02s3/pytest_lazy.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02s3/pytest_lazy.log
timeout 600 python tools/e2e_trace.py > gpurun_out/r02s3/e2e_trace_lazy.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02s3/smoke_lazy.log 2>&1
tail -3 gpurun_out/r02s3/pytest_lazy.log; grep -v "^\[b2o\]" gpurun_out/r02s3/e2e_trace_lazy.log | cut -c1-200; cat gpurun_out/r02s3/smoke_lazy.log
