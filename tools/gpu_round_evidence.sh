#!/bin/bash
# Round evidence on one GPU call (under gpurun): pytest -m gpu, the default bench line,
# narrow ncu metrics at the bench batch (tools/gpu_prof.sh) and the launch list of our kernels.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s6_gputest.log 2>&1; echo GPUTEST=$?; tail -2 gpurun_out/s6_gputest.log
timeout 300 python bench.py > gpurun_out/s6_bench.log 2>&1; echo BENCH=$?
TAG=s6 FULL=0 timeout 600 bash tools/gpu_prof.sh
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" -c 400 --csv --log-file gpurun_out/launches_s6.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-forward --no-variants > gpurun_out/ncu_launch_s6.log 2>&1; echo LAUNCH=$?
