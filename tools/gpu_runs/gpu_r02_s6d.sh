mkdir -p gpurun_out/r02s6
export B2O_CACHE=$PWD/tools/_bigfuzz_cache
timeout 2400 python tools/fuzz_big.py run fp32 > gpurun_out/r02s6/bigfuzz2_fp32.log 2>&1
timeout 2400 python tools/fuzz_big.py run fp64 > gpurun_out/r02s6/bigfuzz2_fp64.log 2>&1
tail -1 gpurun_out/r02s6/bigfuzz2_fp32.log; tail -1 gpurun_out/r02s6/bigfuzz2_fp64.log
