mkdir -p gpurun_out/r02s3
(nproc; lscpu; free -g; grep -m1 flags /proc/cpuinfo) > gpurun_out/r02s3/host_cpu.txt 2>&1
timeout 1500 python tools/ga_drift.py 8 > gpurun_out/r02s3/ga_drift8.jsonl 2> gpurun_out/r02s3/ga_drift8.err
timeout 900 python tools/ga_drift.py 2 > gpurun_out/r02s3/ga_drift2.jsonl 2> gpurun_out/r02s3/ga_drift2.err
tail -3 gpurun_out/r02s3/ga_drift8.err; tail -1 gpurun_out/r02s3/ga_drift8.jsonl; tail -1 gpurun_out/r02s3/ga_drift2.jsonl
