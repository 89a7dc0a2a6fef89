mkdir -p gpurun_out/r02s7
for i in 1 2 3; do timeout 900 python bench.py --apps 0 --ops 0 --reductions 0 --ga 0 > gpurun_out/r02s7/bench_rep$i.json 2>/dev/null; done
for i in 1 2 3; do python -c "import json;d=json.loads(open('gpurun_out/r02s7/bench_rep$i.json').read().strip().splitlines()[-1]);print($i, d['value'], d['e2e']['value'], d['e2e']['ms_per_call'], d['roofline']['frac'], d['cpu_baseline']['value'])"; done
