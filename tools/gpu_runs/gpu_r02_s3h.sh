mkdir -p gpurun_out/r02s3
timeout 2400 python -m pytest tests -m gpu -q -p no:randomly -x > gpurun_out/r02s3/pytest_gpu_h.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02s3/pytest_gpu_h.log
timeout 900 python tools/ga_programs.py > gpurun_out/r02s3/ga_programs_L.jsonl 2>&1
timeout 900 python bench.py > gpurun_out/r02s3/bench_h.json 2> gpurun_out/r02s3/bench_h.err
echo "bench rc=$?" >> gpurun_out/r02s3/bench_h.err
tail -3 gpurun_out/r02s3/pytest_gpu_h.log; head -4 gpurun_out/r02s3/ga_programs_L.jsonl; tail -1 gpurun_out/r02s3/ga_programs_L.jsonl
