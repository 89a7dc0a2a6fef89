# compute-sanitizer over the round-2 code paths: plane march with L2 prefetch
# + subexpression chains (shape fuzz, NAS-MG 18), lazy host reset (smoke runs
# several patterns per replica), isolated evaluator's child (runtime as usual)
mkdir -p gpurun_out/r02s3/san
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1200 $CS --tool memcheck --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02s3/san/memcheck_smoke.log 2>&1
timeout 1500 $CS --tool memcheck --print-limit 20 python -m pytest tests/test_fuzz_shapes.py -q -m gpu -k "0 or 1 or 2 or 3" > gpurun_out/r02s3/san/memcheck_shapes.log 2>&1
timeout 1500 $CS --tool memcheck --print-limit 20 python -m pytest tests/test_parity_gpu.py -q -m gpu -k "nasmg or himeno_17" > gpurun_out/r02s3/san/memcheck_parity_march.log 2>&1
timeout 1500 $CS --tool racecheck --print-limit 20 python -m pytest tests/test_fuzz_shapes.py -q -m gpu -k "0 or 2" > gpurun_out/r02s3/san/racecheck_shapes.log 2>&1
for f in gpurun_out/r02s3/san/*.log; do echo "$f: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|passed|failed' $f | tail -2 | tr '\n' ' ')"; done
