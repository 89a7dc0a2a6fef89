# compute-sanitizer memcheck / racecheck over the hot-path kernels
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1200 $CS --tool memcheck --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san_memcheck_smoke.log 2>&1
timeout 1200 $CS --tool memcheck --print-limit 20 python -m pytest tests/test_xsum_gpu.py -q -m gpu -k "small_n or ragged or one or ties or subnormal or inf or nan or empty or cancel" > gpurun_out/san_memcheck_xsum.log 2>&1
timeout 1200 $CS --tool memcheck --print-limit 20 python -m pytest tests/test_fuzz_shapes.py -q -m gpu -k "0 or 1 or 2" > gpurun_out/san_memcheck_shapes.log 2>&1
timeout 1200 $CS --tool racecheck --print-limit 20 python -m pytest tests/test_fuzz_shapes.py -q -m gpu -k "0 or 2" > gpurun_out/san_racecheck_shapes.log 2>&1
timeout 1200 $CS --tool racecheck --print-limit 20 python -m pytest tests/test_xsum_gpu.py -q -m gpu -k "ragged" > gpurun_out/san_racecheck_xsum.log 2>&1
timeout 1500 $CS --tool memcheck --print-limit 20 python -m pytest tests/test_ops_gpu.py -q -m gpu -x > gpurun_out/san_memcheck_ops.log 2>&1
timeout 1500 $CS --tool racecheck --print-limit 20 python -m pytest tests/test_ops_gpu.py -q -m gpu -x -k "fft" > gpurun_out/san_racecheck_fft.log 2>&1
