#!/bin/bash
# Quick GPU iteration (under gpurun): parity spot checks, bench, optional ncu of one kernel.
#   TAG=x NCU_K=k_sweep_a bash tools/gpu_quick.sh
TAG=${TAG:-q}
mkdir -p gpurun_out
timeout 300 python tools/dev_fast_check.py ${DEV_N:-512 1024 2048} > gpurun_out/dev_${TAG}.log 2>&1
echo "DEV=$?"; grep -E "exact|err|Error|error" gpurun_out/dev_${TAG}.log | head -20
timeout 600 python bench.py --steps 10 --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}.log 2>&1
echo "BENCH=$?"; tail -1 gpurun_out/bench_${TAG}.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', round(d['value'],1), 'ms_per_step', round(d['ms_per_step'],4), 'kernel_ms', {k: round(v,4) for k,v in d['kernel_ms_per_step'].items()}, 'clocks', d['clocks'])" 2>/dev/null
if [ -n "${NCU_K}" ]; then
  CMD="python bench.py --steps 2 --warmup 3 --batch ${NCU_BATCH:-4} --no-e2e --no-cpu-baseline"
  $CMD > gpurun_out/plain_${TAG}.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"${NCU_K}" -s ${NCU_SKIP:-3} -c ${NCU_COUNT:-1} -o gpurun_out/prof_${TAG} $CMD > gpurun_out/ncu_${TAG}.log 2>&1
  echo "NCU=$?"
fi
