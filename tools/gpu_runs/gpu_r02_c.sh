mkdir -p gpurun_out/r02
( nvidia-smi -q | grep -i -E "compute mode|MIG|Persistence" ; echo "MPS pipe: $CUDA_MPS_PIPE_DIRECTORY"; ls -la /tmp/nvidia-mps 2>&1 | head; ps aux | grep -i mps | grep -v grep ) > gpurun_out/r02/mps_check.txt 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02/bench2.json 2> gpurun_out/r02/bench2.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 2 > gpurun_out/r02/bench2_ref.json 2> gpurun_out/r02/bench2_ref.err
timeout 900 python -m pytest tests/test_fuzz_shapes.py tests/test_parity_gpu.py tests/test_fullsize_gpu.py -m gpu -q > gpurun_out/r02/pytest_c.log 2>&1
echo "rc=$?" >> gpurun_out/r02/pytest_c.log
