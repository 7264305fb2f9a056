#!/bin/bash
# Round-end evidence in one GPU call: the -m gpu suite, the bench line (beta, default
# args), the complex power-family bench, the config-5-style run, the drop-in e2e, the
# precision sweep, and the launch list + one ncu capture of the update kernel.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m pytest tests -q -m gpu -rf --durations=15 > gpurun_out/r2f_gpu_all.log 2>&1; tail -3 gpurun_out/r2f_gpu_all.log
python bench.py > gpurun_out/r2f_bench.json 2> gpurun_out/r2f_bench.err; tail -c 300 gpurun_out/r2f_bench.json
python bench.py --family power --dim 1000 --bits 4096 --steps 2 --warmup 3 > gpurun_out/r2f_bench_power1000.json 2> gpurun_out/r2f_bench_power1000.err
python tools/bigrun.py --n 3000 --bits 33220 --batch 8 --keep 96 > gpurun_out/r2f_big3000.json 2> gpurun_out/r2f_big3000.err; tail -c 600 gpurun_out/r2f_big3000.json
python tools/dropin_e2e.py 2000 4096 > gpurun_out/r2f_dropin.json 2> gpurun_out/r2f_dropin.err; cat gpurun_out/r2f_dropin.json
for s in 1000@256 1000@512 1000@1024 1000@2048 1000@4096 1000@8192 1000@16384 1000@32768 1000@33220 500@4096c 1000@1024c; do
  python tools/probe_perf.py $s 2>&1 | sed "s/launches=.*//"
done > gpurun_out/r2f_sweep.log 2>&1; cat gpurun_out/r2f_sweep.log
