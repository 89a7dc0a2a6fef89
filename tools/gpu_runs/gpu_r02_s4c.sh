mkdir -p gpurun_out/r02s3
timeout 1200 python bench.py --apps 0 --ops 0 --reductions 0 > gpurun_out/r02s3/bench_ga2.json 2> gpurun_out/r02s3/bench_ga2.err
echo "rc=$?" >> gpurun_out/r02s3/bench_ga2.err
tail -3 gpurun_out/r02s3/bench_ga2.err
python -c "import json;d=json.loads(open('gpurun_out/r02s3/bench_ga2.json').read().strip().splitlines()[-1]);print(json.dumps(d['ga'])[:1500])"
