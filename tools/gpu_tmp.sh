mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1200 $CS --tool racecheck --print-limit 20 python tools/san_ktile.py > gpurun_out/san_racecheck_ktile_s4.log 2>&1
timeout 900 $CS --tool memcheck --print-limit 20 python tools/san_ktile.py > gpurun_out/san_memcheck_ktile_s4.log 2>&1
true
