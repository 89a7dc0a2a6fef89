mkdir -p gpurun_out/r02s7
timeout 600 python tools/e2e_trace.py 1 > gpurun_out/r02s7/e2e_trace.log 2>&1
timeout 600 python tools/pcie_bw.py > gpurun_out/r02s7/pcie_bw.log 2>&1
grep -v "^\[b2o\] job worker=0 reset 0.0" gpurun_out/r02s7/e2e_trace.log | cut -c1-200; cat gpurun_out/r02s7/pcie_bw.log | tail -5
nvidia-smi -q | grep -iE "link gen|link width|Max Link|Current" | head -12
