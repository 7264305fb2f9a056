# wide product kernel tuning sweep (K steps per stage, stages, rows per CTA) at one size
mkdir -p gpurun_out
SPEC=${1:-600@32768}
for cfg in "KC=8 NST=3 RBR=2" "KC=16 NST=2 RBR=2" "KC=16 NST=2 RBR=1" "KC=20 NST=2 RBR=2" "KC=12 NST=3 RBR=2"; do
  set -- $cfg
  env DS_TCW_${1} DS_TCW_${2} DS_TCW_${3} timeout 300 python tools/probe_perf.py --no-series $SPEC 2>&1 | grep "^n=" | sed "s/^/$cfg /" | cut -c1-160
done
