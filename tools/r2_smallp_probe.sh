#!/bin/bash
# Small-precision regime probes (configs 1a / 2 / sweep low end): engine choice
# (tensor-core vs FP64-digit update) and rows per CTA, plus the complex split.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
{
for spec in 1000@256 1000@512 1000@1024 1000@2048; do
  echo "== $spec tc";            python tools/probe_perf.py $spec 2>&1 | sed "s/launches=.*//"
  echo "== $spec dfma";          DS_DISABLE_TC=1 python tools/probe_perf.py $spec 2>&1 | sed "s/launches=.*//"
  for rbr in 4 8; do
    echo "== $spec tc rbr=$rbr"; DS_TC_RBR=$rbr python tools/probe_perf.py $spec 2>&1 | sed "s/launches=.*//"
  done
  echo "== $spec tc adapt";      DS_TC_RBR_ADAPT=1 python tools/probe_perf.py $spec 2>&1 | sed "s/launches=.*//"
done
echo "== complex 300@4096"; python tools/probe_perf.py 300@4096c 2>&1 | sed "s/launches=.*//"
} > gpurun_out/r2_smallp.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -s 2000 -c 400 --csv --log-file gpurun_out/r2_complex_launches.csv \
    python tools/probe_perf.py 300@4096c > /dev/null 2>&1
cat gpurun_out/r2_smallp.log
