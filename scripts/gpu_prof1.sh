set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()"
timeout 300 python scripts/prof_batch.py 10000 1000 2 > gpurun_out/host_timing.log 2>&1; cat gpurun_out/host_timing.log
timeout 600 python bench.py --steps 3 --warmup 3 --cpu-seconds 10 > gpurun_out/bench.log 2>&1; echo bench rc=$?; tail -3 gpurun_out/bench.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kbest_batch -c 3 -o gpurun_out/prof_batch_r1 python scripts/prof_batch.py 2000 1000 1 > gpurun_out/ncu_full.log 2>&1; echo ncu rc=$?; tail -5 gpurun_out/ncu_full.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo ncu2 rc=$?
