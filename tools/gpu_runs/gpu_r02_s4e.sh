mkdir -p gpurun_out/r02s4
for w in 6 8; do
timeout 900 python bench.py --apps 0 --ops 0 --reductions 0 --ga-workers $w --steps 3 --warmup 3 > gpurun_out/r02s4/bench_ga$w.json 2> gpurun_out/r02s4/bench_ga$w.err
python -c "import json;d=json.loads(open('gpurun_out/r02s4/bench_ga$w.json').read().strip().splitlines()[-1]);o=d['ga']['overlapped'];print($w, d['ga']['patterns_per_s'], o['patterns_per_s'], o['best_genome'], o['same_program_as_one_worker'], o['confirmed_top3'])"
done
