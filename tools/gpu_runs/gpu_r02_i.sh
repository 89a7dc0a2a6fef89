mkdir -p gpurun_out/r02
for w in _wt_e09b303 _wt_17d6baf; do
  cp tools/kernel_sweep.py $w/tools/kernel_sweep.py
  (cd $w && timeout 600 python tools/kernel_sweep.py nasmg_258 100100 '{}') > gpurun_out/r02/sweep_$w.jsonl 2>&1
done
