mkdir -p gpurun_out/r02s5
timeout 2400 python -m pytest tests -m gpu -q -p no:randomly > gpurun_out/r02s5/pytest_gpu_nextpf.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02s5/pytest_gpu_nextpf.log
timeout 900 python tools/ga_programs.py > gpurun_out/r02s5/ga_programs_L.jsonl 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02s5/smoke_nextpf.log 2>&1
tail -3 gpurun_out/r02s5/pytest_gpu_nextpf.log; head -3 gpurun_out/r02s5/ga_programs_L.jsonl; tail -1 gpurun_out/r02s5/ga_programs_L.jsonl; cat gpurun_out/r02s5/smoke_nextpf.log
