#!/bin/bash
# Full validation in one GPU call: the -m gpu suite, smoke, the bench line (beta, default
# args), the power-family bench, the drop-in e2e and a complex sweep point.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m pytest tests -q -m gpu -rf --durations=10 > gpurun_out/v_gpu_all.log 2>&1; tail -3 gpurun_out/v_gpu_all.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v_smoke.log 2>&1; tail -2 gpurun_out/v_smoke.log
python bench.py > gpurun_out/v_bench.json 2> gpurun_out/v_bench.err; tail -c 300 gpurun_out/v_bench.json
python bench.py --family power --dim 1000 --bits 4096 --steps 2 --warmup 3 > gpurun_out/v_bench_power1000.json 2> gpurun_out/v_bench_power1000.err
python tools/dropin_e2e.py 2000 4096 > gpurun_out/v_dropin.json 2> gpurun_out/v_dropin.err; cat gpurun_out/v_dropin.json
for s in 500@4096c 1000@1024c 1000@1024 1000@4096; do
  python tools/probe_perf.py $s 2>&1 | sed "s/launches=.*//"
done > gpurun_out/v_sweep.log 2>&1; cat gpurun_out/v_sweep.log
