#!/bin/bash
# Fast GPU iteration (under gpurun): fast-vs-general parity at the bench sizes, a short
# bench, and (NCU=1) narrow ncu metrics of one launch of each hot kernel at the bench batch.
#   TAG=x NCU=1 bash tools/gpu_iter.sh
TAG=${TAG:-it}
mkdir -p gpurun_out
timeout 300 python tools/dev_quick_parity.py ${DEV_N:-512 1024 2048 4096} > gpurun_out/qp_${TAG}.log 2>&1
echo "QP=$?"; cat gpurun_out/qp_${TAG}.log | grep -v "^$" | tail -9
timeout 600 python bench.py --steps 50 --no-cpu-baseline --no-e2e --no-variants > gpurun_out/bench_${TAG}.log 2>&1
echo "BENCH=$?"; tail -1 gpurun_out/bench_${TAG}.log | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('value', round(d['value'],1), 'ms', round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['kernel_ms_per_step'].items() if v}, d['clocks']['sm_mhz'])
print('fwd', {k: round(v,4) for k,v in d['next']['fht_forward']['kernel_ms_per_step'].items()}, 'resample', round(d['next']['resample']['ms_per_step'],4))" 2>&1
if [ "${NCU:-0}" = "1" ]; then
  CMD="python bench.py --steps 1 --warmup 3 --batch 16 --no-e2e --no-cpu-baseline --no-variants"
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,smsp__average_warp_latency_issue_stalled_barrier.ratio,smsp__average_warp_latency_issue_stalled_short_scoreboard.ratio,smsp__average_warp_latency_issue_stalled_mio_throttle.ratio,smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio \
    --clock-control none -k regex:"k_" -s ${NCU_SKIP:-9} -c ${NCU_COUNT:-8} --csv --log-file gpurun_out/ncu16_${TAG}.csv $CMD > gpurun_out/ncu16_${TAG}.log 2>&1
  echo "NCU16=$?"
fi
