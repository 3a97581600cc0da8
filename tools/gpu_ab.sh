#!/bin/bash
# A/B of libfbp variants (tools/build_variants.py) on one GPU call:
#   VARIANTS="v0 v1" bash tools/gpu_ab.sh
mkdir -p gpurun_out
cp paper_2007_06289_b200/libfbp.so /tmp/libfbp_default.so
for v in ${VARIANTS}; do
  cp paper_2007_06289_b200/variants/$v.so paper_2007_06289_b200/libfbp.so
  timeout 300 python tools/dev_quick_parity.py ${DEV_N:-512 2048 4096} > gpurun_out/ab_qp_$v.log 2>&1
  echo "$v QP=$? $(tail -1 gpurun_out/ab_qp_$v.log)"
  timeout 300 python bench.py --steps 50 --no-cpu-baseline --no-e2e --no-variants ${BENCH_ARGS:---no-forward} > gpurun_out/ab_bench_$v.log 2>&1
  tail -1 gpurun_out/ab_bench_$v.log | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('  $v value', round(d['value'],1), 'ms', round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['kernel_ms_per_step'].items() if v}, d['clocks']['sm_mhz'])
f=d.get('next',{}).get('fht_forward')
f and print('  $v fwd', round(f['value'],1), round(f['ms_per_step'],4), f['kernel_ms_per_step'], 'frac', round(f['roofline']['frac'],3))" 2>&1
done
cp /tmp/libfbp_default.so paper_2007_06289_b200/libfbp.so
