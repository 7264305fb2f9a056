#!/bin/bash
# One build->measure cycle on the GPU box: parity tests of the update engines,
# timing probe, and an ncu capture of one tensor-core update launch.
# usage: bash tools/gpu_cycle.sh TAG [probe specs...]
TAG=${1:-cycle}; shift
SPECS=${@:-"1000@4096 2000@4096"}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_update_adversarial.py tests/test_gpu_parity.py -x -q > gpurun_out/${TAG}_tests.log 2>&1
echo tests=$?; tail -2 gpurun_out/${TAG}_tests.log
timeout 900 python tools/probe_perf.py $SPECS > gpurun_out/${TAG}_probe.log 2>&1; echo probe=$?
cat gpurun_out/${TAG}_probe.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_update_tc -s 50 -c 1 -o gpurun_out/${TAG} python tools/probe_perf.py 600@4096 > gpurun_out/${TAG}_ncu.log 2>&1
echo ncu=$?
