mkdir -p gpurun_out/r02s3
for v in 0 1 2; do for npc in 1 2; do
echo "V=$v NPC=$npc $(B2O_FFT_V=$v B2O_FFT_NPC=$npc python tools/ops_bench.py 4096 2>&1 | grep fft2d)"
done; done > gpurun_out/r02s3/fft_variants2.log
cat gpurun_out/r02s3/fft_variants2.log
