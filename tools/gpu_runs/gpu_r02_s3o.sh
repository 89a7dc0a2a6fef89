mkdir -p gpurun_out/r02s3
timeout 900 python bench.py > gpurun_out/r02s3/bench_final1.json 2> gpurun_out/r02s3/bench_final1.err
echo "bench rc=$?" >> gpurun_out/r02s3/bench_final1.err
timeout 600 python bench.py --impl reference > gpurun_out/r02s3/bench_ref.json 2> gpurun_out/r02s3/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02s3/launches.csv python bench.py --steps 2 --warmup 1 --apps 0 --ga 0 --ops 0 --reductions 0 > gpurun_out/r02s3/b_ncu.log 2>&1
tail -c 400 gpurun_out/r02s3/bench_final1.json; cat gpurun_out/r02s3/bench_ref.json
