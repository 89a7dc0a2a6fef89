mkdir -p gpurun_out/r02s3
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 2 --steps 3 --warmup 1 > gpurun_out/r02s3/bench_ref_torchrun2b.json 2> gpurun_out/r02s3/bench_ref_torchrun2b.err
echo "rc=$?" >> gpurun_out/r02s3/bench_ref_torchrun2b.err
python -c "import json;d=json.loads(open('gpurun_out/r02s3/bench_ref_torchrun2b.json').read().strip().splitlines()[-1]);print(d['value'],d['cpu_baseline']['cores'])"
