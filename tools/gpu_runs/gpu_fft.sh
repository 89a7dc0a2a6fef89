mkdir -p gpurun_out
for v in "B2O_FFT_PIPE=0" "B2O_FFT_PIPE=1" "B2O_FFT_PIPE=2" "B2O_FFT_PIPE=0 B2O_FFT_NPC=2" "B2O_FFT_PIPE=1 B2O_FFT_CLUSTERS=16" "B2O_FFT_PIPE=1 B2O_FFT_CLUSTERS=24" "B2O_FFT_PIPE=2 B2O_FFT_CLUSTERS=36"; do
  env $v timeout 120 python tools/fft_bench.py >> gpurun_out/fft.log 2>&1
done
timeout 300 python -m pytest tests/test_ops_gpu.py -m gpu -q > gpurun_out/pytest_ops.log 2>&1
