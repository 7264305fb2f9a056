mkdir -p gpurun_out
for cfg in "KC=8 NST=3 RBR=2" "KC=4 NST=6 RBR=2" "KC=8 NST=4 RBR=2" "KC=16 NST=2 RBR=2" "KC=8 NST=3 RBR=8" "KC=4 NST=4 RBR=4"; do
  set -- $cfg
  env DS_TCW_${1} DS_TCW_${2} DS_TCW_${3} timeout 300 python tools/probe_perf.py --no-series 600@16384 2>&1 | grep "^n=" | sed "s/^/$cfg /" | cut -c1-200
done
