mkdir -p gpurun_out/r02s5
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 4 --steps 5 --warmup 3 > gpurun_out/r02s5/bench_torchrun4.json 2> gpurun_out/r02s5/bench_torchrun4.err
echo "rc=$?" >> gpurun_out/r02s5/bench_torchrun4.err
python -c "import json;d=json.loads(open('gpurun_out/r02s5/bench_torchrun4.json').read().strip().splitlines()[-1]);print(d['n_gpus'],d['value'],d['e2e']['value'],d['ga']['patterns_per_s'],d['ga']['programs_executed_all_ranks'], [ (k,a.get('value')) for k,a in d['apps'].items()])"
tail -2 gpurun_out/r02s5/bench_torchrun4.err
