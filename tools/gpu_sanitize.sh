#!/bin/bash
# one compute-sanitizer tool per call (B200_PROFILING.md): TOOL=memcheck|racecheck|synccheck
TOOL=${TOOL:-memcheck}
mkdir -p gpurun_out
for case in ${CASES:-"512 1" "512 2" "2048 1"}; do
  set -- $case
  timeout ${TMO:-900} compute-sanitizer --tool $TOOL --print-limit 20 python tools/sanitize_case.py $1 $2 > gpurun_out/sanitize_${TOOL}_$1_$2.log 2>&1
  echo "$TOOL N=$1 B=$2 rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|sanitize case|Error|error" gpurun_out/sanitize_${TOOL}_$1_$2.log | head -5
done
