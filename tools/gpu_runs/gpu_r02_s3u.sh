mkdir -p gpurun_out/r02s3
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/r02s3/bench_torchrun2.json 2> gpurun_out/r02s3/bench_torchrun2.err
echo "rc=$?" >> gpurun_out/r02s3/bench_torchrun2.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 2 --steps 3 --warmup 1 > gpurun_out/r02s3/bench_ref_torchrun2.json 2> gpurun_out/r02s3/bench_ref_torchrun2.err
echo "rc=$?" >> gpurun_out/r02s3/bench_ref_torchrun2.err
tail -c 300 gpurun_out/r02s3/bench_torchrun2.json; tail -2 gpurun_out/r02s3/bench_torchrun2.err; tail -c 300 gpurun_out/r02s3/bench_ref_torchrun2.json; tail -1 gpurun_out/r02s3/bench_ref_torchrun2.err
