#!/bin/bash
# Committed-evidence captures for one round (run on the GPU box, one GPU):
#  1. ncu --set full of one tensor-core update launch at the bench workload size
#     (n=2000 @4096, step 1000 of a random matrix) -> traffic + pipe utilisation
#  2. the launch list (gpu__time_duration) of the bench command itself
TAG=${1:-r01}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_update_tc -s 1000 -c 1 \
  -o gpurun_out/${TAG}_update_full python tools/probe_perf.py 2000@4096 > gpurun_out/${TAG}_update_full.log 2>&1
echo full=$?
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${TAG}_bench_launches.csv python bench.py --steps 2 --warmup 1 --family random --no-cpu \
  > gpurun_out/${TAG}_bench_under_ncu.log 2>&1
echo launches=$?
