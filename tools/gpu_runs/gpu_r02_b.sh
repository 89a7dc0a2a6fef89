mkdir -p gpurun_out/r02
/tmp/reset_probe > gpurun_out/r02/reset_probe.log 2>&1 || true
nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/reset_probe tools/probe/reset_probe.cu && /tmp/reset_probe > gpurun_out/r02/reset_probe.log 2>&1
timeout 600 python -m pytest tests/test_recovery_gpu.py tests/test_fuzz_shapes.py -m gpu -q -x > gpurun_out/r02/pytest_b.log 2>&1
echo "rc=$?" >> gpurun_out/r02/pytest_b.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02/bench1.json 2> gpurun_out/r02/bench1.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 2 > gpurun_out/r02/bench1_ref.json 2> gpurun_out/r02/bench1_ref.err
tail -3 gpurun_out/r02/pytest_b.log
