#!/bin/bash
# Developer A/B (under gpurun): pass-B x-tile 128 vs 64 at N = 1024 (config 4, 256 slices per call),
# dev build variant (tools/build_variants.py dev:-DFBP_DEV_MASK=1) so FBP_XB is read.
mkdir -p gpurun_out
cp paper_2007_06289_b200/libfbp.so /tmp/libfbp_default.so
cp paper_2007_06289_b200/variants/dev.so paper_2007_06289_b200/libfbp.so
for xb in ${XBS:-128 64 128 64}; do
  FBP_XB=$xb timeout 300 python tools/dev_quick_parity.py 1024 > gpurun_out/xb_qp_$xb.log 2>&1
  echo "XB=$xb QP=$? $(tail -1 gpurun_out/xb_qp_$xb.log)"
  FBP_XB=$xb timeout 300 python bench.py --n 1024 --batch 256 --steps 20 --no-cpu-baseline --no-e2e --no-variants --no-forward > gpurun_out/xb_bench_$xb.log 2>&1
  tail -1 gpurun_out/xb_bench_$xb.log | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('  XB=$xb value', round(d['value'],1), 'ms', round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['kernel_ms_per_step'].items() if v})" 2>&1
done
cp /tmp/libfbp_default.so paper_2007_06289_b200/libfbp.so
