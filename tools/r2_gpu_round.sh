#!/bin/bash
# One GPU call: the whole -m gpu suite, the bench line, the bench launch list,
# one ncu --set full capture of the update kernel, and compute-sanitizer runs.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m pytest tests -q -m gpu -rf --durations=10 > gpurun_out/r2_gpu_all.log 2>&1; tail -3 gpurun_out/r2_gpu_all.log
python bench.py --steps 3 --warmup 3 > gpurun_out/r2_bench2.json 2> gpurun_out/r2_bench2.err; tail -c 400 gpurun_out/r2_bench2.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_bench_launches.csv \
    python bench.py --steps 1 --warmup 0 --family random --no-cpu --no-e2e --no-parity > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_update_tc -s 1001 -c 1 -o gpurun_out/r2_upd2 \
    python tools/probe_perf.py 2000@4096 > gpurun_out/r2_ncu2.log 2>&1; tail -1 gpurun_out/r2_ncu2.log
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_case.py > gpurun_out/r2_sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; tail -4 gpurun_out/r2_sanitize_$tool.log
done
