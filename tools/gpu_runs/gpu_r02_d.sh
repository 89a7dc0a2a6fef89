mkdir -p gpurun_out/r02
python tools/pcie_bw.py > gpurun_out/r02/pcie_bw.log 2>&1
python tools/e2e_trace.py > gpurun_out/r02/e2e_trace.jsonl 2> gpurun_out/r02/e2e_trace.err
