mkdir -p gpurun_out/r02s7/san
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1500 $CS --tool racecheck --print-limit 20 python -m pytest tests/test_histogram.py -q -m gpu > gpurun_out/r02s7/san/racecheck_hist.log 2>&1
timeout 1500 $CS --tool memcheck --print-limit 20 python -m pytest tests/test_histogram.py tests/test_ops_gpu.py -q -m gpu -k "hist or fft" > gpurun_out/r02s7/san/memcheck_hist_fft.log 2>&1
timeout 1500 $CS --tool memcheck --print-limit 20 python -m pytest tests/test_parity_gpu.py -q -m gpu -k "himeno_xs_inline or order" > gpurun_out/r02s7/san/memcheck_nextpf_lazy.log 2>&1
for f in gpurun_out/r02s7/san/*.log; do echo "$f: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|passed|failed' $f | tail -2 | tr '\n' ' ')"; done
