mkdir -p gpurun_out
timeout 1500 python tools/fuzz_big.py run fp32 > gpurun_out/bigfuzz_s4.log 2>&1
timeout 1500 python tools/fuzz_big.py run fp64 > gpurun_out/bigfuzz_s4_fp64.log 2>&1
true
