for c in 2 3 4 2 3 4; do echo "CTAS=$c $(B2O_HIST_CTAS=$c python tools/ops_bench.py 4096 2>&1 | grep '"histogram"')"; done
