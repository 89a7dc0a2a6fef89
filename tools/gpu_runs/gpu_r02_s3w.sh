mkdir -p gpurun_out/r02s3/ncu
KS_NOWARM=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:b2o_k1 -s 2 -c 1 -o gpurun_out/r02s3/ncu/jacobi python tools/kernel_sweep.py himeno_M 100100 '{}' > gpurun_out/r02s3/ncu/jacobi.log 2>&1
KS_NOWARM=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:b2o_k0 -s 1 -c 1 -o gpurun_out/r02s3/ncu/ktile python tools/kernel_sweep.py matmul_1024 10 '{}' > gpurun_out/r02s3/ncu/ktile.log 2>&1
for f in jacobi ktile; do ncu -i gpurun_out/r02s3/ncu/$f.ncu-rep --page raw --csv > gpurun_out/r02s3/ncu/${f}_raw.csv 2>/dev/null; done
ncu -i gpurun_out/r02s3/mg_march_chains2.ncu-rep --page raw --csv > gpurun_out/r02s3/ncu/mg_march_chains_raw.csv 2>/dev/null
ls -la gpurun_out/r02s3/ncu
