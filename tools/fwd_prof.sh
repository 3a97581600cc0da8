# Developer: ncu evidence for the forward FHT kernels (run under gpurun): TAG=x bash tools/fwd_prof.sh
TAG=${TAG:-cur}
mkdir -p gpurun_out
python tools/fwd_run.py 2048 16 3 > gpurun_out/fwdplain_${TAG}.log 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct,sm__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum \
  --clock-control none -k regex:"k_fwd" -c 4 --csv --log-file gpurun_out/ncufwd_${TAG}.csv python tools/fwd_run.py 2048 16 1 > gpurun_out/ncufwd_${TAG}.log 2>&1
echo "NCU=$?"
if [ "${FULL:-1}" = "1" ]; then
ncu --set full --import-source on --clock-control none -k regex:"k_fwd" -c 2 -o gpurun_out/proffwd_${TAG} python tools/fwd_run.py 2048 16 1 > gpurun_out/ncufwdfull_${TAG}.log 2>&1
echo "NCUFULL=$?"
fi
