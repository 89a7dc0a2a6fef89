mkdir -p gpurun_out/r02s4
B2O_GEMM_FUSED=1 timeout 600 ncu --set full --clock-control none -k regex:"fused" -c 1 -o gpurun_out/r02s4/gemm_fused python tools/ops_bench.py 4096 > /dev/null 2>&1
ncu -i gpurun_out/r02s4/gemm_fused.ncu-rep --page details --csv 2>/dev/null | grep -iE "Tensor|Shared|Issue Slots|Throughput|stall|Warp Cycles" | cut -c1-200 | head -40
