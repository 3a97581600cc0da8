#!/bin/bash
# One GPU cycle (run under gpurun): tests, bench, launch list, one ncu --set full capture.
#   TAG=v2 PYTEST=1 NCU=1 bash tools/gpu_cycle.sh
TAG=${TAG:-cur}
mkdir -p gpurun_out
if [ "${PYTEST:-1}" = "1" ]; then
  timeout ${PYTEST_TIMEOUT:-1500} python -m pytest tests -m gpu -q -x -p no:cacheprovider ${PYTEST_ARGS} > gpurun_out/pytest_${TAG}.log 2>&1
  echo "PYTEST_EXIT=$?"; tail -5 gpurun_out/pytest_${TAG}.log
fi
if [ "${BENCH:-1}" = "1" ]; then
  timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench_${TAG}.log 2>&1
  echo "BENCH_EXIT=$?"; tail -3 gpurun_out/bench_${TAG}.log
fi
if [ "${NCU:-1}" = "1" ]; then
  # launch list at the bench's own batch (NCU_BATCH, default 16) so kernel shares match the
  # bench line; the --set full capture at batch 2 (NCU_FULL_BATCH): at 16 it exceeds 50 min
  CMD="python bench.py --steps 2 --warmup 3 --batch ${NCU_BATCH:-16} --no-e2e --no-cpu-baseline --no-forward"
  $CMD > gpurun_out/plain_${TAG}.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv $CMD > /dev/null 2>&1
  echo "NCU_LAUNCHES=$?"
  CMD="python bench.py --steps 2 --warmup 3 --batch ${NCU_FULL_BATCH:-2} --no-e2e --no-cpu-baseline --no-forward"
  $CMD > gpurun_out/plain2_${TAG}.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k_" -s ${NCU_SKIP:-10} -c ${NCU_COUNT:-4} -o gpurun_out/prof_${TAG} $CMD > gpurun_out/ncu_full_${TAG}.log 2>&1
  echo "NCU_FULL=$?"
fi
