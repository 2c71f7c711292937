# Full round-end style evidence run: tests, smoke, bench lines, ncu launch list + full captures.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out /tmp/prof
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv > gpurun_out/nvsmi.txt
nproc >> gpurun_out/nvsmi.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?; cut -c1-300 gpurun_out/bench.json
timeout 900 python bench.py --workload cfg5 --steps 3 --warmup 3 --cpu-seconds 10 > gpurun_out/bench_cfg5.json 2>gpurun_out/bench_cfg5.err; echo cfg5 rc=$?; cut -c1-300 gpurun_out/bench_cfg5.json
timeout 600 python bench.py --workload cfg2 --steps 5 --warmup 3 --cpu-seconds 10 > gpurun_out/bench_cfg2.json 2>gpurun_out/bench_cfg2.err; echo cfg2 rc=$?
timeout 600 python bench.py --workload cfg4 --steps 3 --warmup 3 > gpurun_out/bench_cfg4.json 2>gpurun_out/bench_cfg4.err; echo cfg4 rc=$?; cut -c1-300 gpurun_out/bench_cfg4.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json 2>gpurun_out/bench_ref.err; echo ref rc=$?
timeout 600 python scripts/time_large.py > gpurun_out/time_large.txt 2>&1; echo time_large rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo ncu-launch rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:kbest_batch -c 3 -o /tmp/prof/prof_bench python scripts/prof_batch.py 10000 1000 1 > gpurun_out/ncu_full.log 2>&1; echo ncu-full rc=$?
timeout 900 ncu --set full --clock-control none -k regex:kbest_batch -c 2 -o /tmp/prof/prof_cfg5 python scripts/prof_cfg5.py 20000 > gpurun_out/ncu_cfg5.log 2>&1; echo ncu-cfg5 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:kbest_large -c 1 -o /tmp/prof/prof_large5 python scripts/prof_large.py 5 > gpurun_out/ncu_large.log 2>&1; echo ncu-large rc=$?
# summaries only (the .ncu-rep files stay on the box: gpurun_out/ is capped at 64 MiB)
python scripts/make_profiles.py r2 /tmp/prof gpurun_out/profiles_r2 > gpurun_out/make_profiles.log 2>&1; echo make_profiles rc=$?
du -sh gpurun_out
