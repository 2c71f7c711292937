# Round-2 evidence that is not the bench: measured integer peak, ncu L2/atomic/shared counters of the
# batched (cfg3, cfg5) and whole-GPU (cfg4) kernels, compute-sanitizer logs.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/int_peak scripts/micro/int_peak.cu && /tmp/int_peak > gpurun_out/int_peak.json; cat gpurun_out/int_peak.json
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sectors_op_atom.sum,lts__t_sectors_op_red.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active
timeout 900 ncu --metrics $M --clock-control none -k regex:kbest_batch -c 3 --csv --log-file gpurun_out/ncu_counters_cfg3.csv python scripts/prof_batch.py 10000 1000 1 > /dev/null 2>&1; echo cfg3 rc=$?
timeout 900 ncu --metrics $M --clock-control none -k regex:kbest_batch -c 2 --csv --log-file gpurun_out/ncu_counters_cfg5.csv python scripts/prof_cfg5.py 20000 > /dev/null 2>&1; echo cfg5 rc=$?
timeout 900 ncu --metrics $M --clock-control none -k regex:kbest_large -c 1 --csv --log-file gpurun_out/ncu_counters_cfg4.csv python scripts/prof_large.py 5 > /dev/null 2>&1; echo cfg4 rc=$?
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool python scripts/repro_mixed.py > gpurun_out/sanitize_$tool.log 2>&1; echo $tool rc=$?; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|parity" gpurun_out/sanitize_$tool.log | tail -3
done
