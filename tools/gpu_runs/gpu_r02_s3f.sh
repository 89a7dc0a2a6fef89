mkdir -p gpurun_out/r02s3
timeout 600 python tools/e2e_trace.py > gpurun_out/r02s3/e2e_trace.log 2>&1
cat gpurun_out/r02s3/e2e_trace.log | cut -c1-250
