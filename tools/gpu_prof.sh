#!/bin/bash
# ncu evidence for one code state (run under gpurun):
#   TAG=x bash tools/gpu_prof.sh
# 1) narrow metrics at the bench batch (16): DRAM bytes, duration, occupancy, L2 hit rate
# 2) --set full with source counters of the three hot-path kernels at batch 2
TAG=${TAG:-cur}
mkdir -p gpurun_out
CMD16="python bench.py --steps 1 --warmup 3 --batch ${BATCH:-16} --no-e2e --no-cpu-baseline --no-forward --no-variants"
CMD2="python bench.py --steps 1 --warmup 3 --batch 2 --no-e2e --no-cpu-baseline --no-forward --no-variants"
$CMD16 > gpurun_out/plain16_${TAG}.log 2>&1 && $CMD2 > gpurun_out/plain2_${TAG}.log 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct,sm__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__inst_executed_pipe_fma.sum,sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active \
  --clock-control none -k regex:"k_" -s 9 -c 3 --csv --log-file gpurun_out/ncu16_${TAG}.csv $CMD16 > gpurun_out/ncu16_${TAG}.log 2>&1
echo "NCU16=$?"
if [ "${FULL:-1}" = "1" ]; then
ncu --set full --import-source on --clock-control none -k regex:"${KREGEX:-k_}" -s ${SKIP:-9} -c ${COUNT:-3} -o gpurun_out/prof_${TAG} $CMD2 > gpurun_out/ncufull_${TAG}.log 2>&1
echo "NCUFULL=$?"
fi
