mkdir -p gpurun_out/r02
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02/smi.txt 2>&1
lscpu > gpurun_out/r02/lscpu.txt 2>&1
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -fmad=false -o /tmp/fp32_rate tools/probe/fp32_rate.cu && /tmp/fp32_rate > gpurun_out/r02/fp32_rate.jsonl 2>&1
timeout 300 python tools/peaks_probe.py > gpurun_out/r02/tf32_peak.json 2> gpurun_out/r02/tf32_peak.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_pair -s 2 -c 1 -o gpurun_out/r02/gemm_pair python tools/ops_bench.py 4096 > gpurun_out/r02/ncu_gemm.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fft -s 4 -c 2 -o gpurun_out/r02/fft python tools/ops_bench.py 4096 > gpurun_out/r02/ncu_fft.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02/bench0.json 2> gpurun_out/r02/bench0.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02/bench0_ref.json 2> gpurun_out/r02/bench0_ref.err
ls -la gpurun_out/r02
