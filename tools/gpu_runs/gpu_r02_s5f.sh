mkdir -p gpurun_out/r02s5
timeout 900 python tools/launch_overhead.py himeno_L 001001 000001 001000 > gpurun_out/r02s5/launch_overhead.log 2>&1
B2O_PDL=0 timeout 900 python tools/launch_overhead.py himeno_L 001001 >> gpurun_out/r02s5/launch_overhead.log 2>&1
cat gpurun_out/r02s5/launch_overhead.log
