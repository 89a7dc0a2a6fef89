mkdir -p gpurun_out/r02s6
timeout 900 python tools/ga_programs.py > gpurun_out/r02s6/ga_programs_base.jsonl 2>&1
B2O_HOST_EXTRA="-fprefetch-loop-arrays" timeout 900 python tools/ga_programs.py > gpurun_out/r02s6/ga_programs_pf.jsonl 2>&1
B2O_HOST_EXTRA="-fprefetch-loop-arrays --param prefetch-latency=400" timeout 900 python tools/ga_programs.py > gpurun_out/r02s6/ga_programs_pf400.jsonl 2>&1
for f in base pf pf400; do echo $f; grep -E '"000000"|"000100"|"001001"|programs' gpurun_out/r02s6/ga_programs_$f.jsonl; done
