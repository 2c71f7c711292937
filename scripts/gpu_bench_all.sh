cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python bench.py --steps 3 --warmup 3 --cpu-seconds 10 > gpurun_out/bench_cfg3.json 2>gpurun_out/bench_cfg3.err; echo cfg3 rc=$?
timeout 600 python bench.py --workload cfg5 --npairs 100000 --steps 3 --warmup 2 --cpu-seconds 10 > gpurun_out/bench_cfg5.json 2>gpurun_out/bench_cfg5.err; echo cfg5 rc=$?
timeout 600 python bench.py --workload cfg2 --steps 5 --warmup 3 --cpu-seconds 10 > gpurun_out/bench_cfg2.json 2>gpurun_out/bench_cfg2.err; echo cfg2 rc=$?
timeout 600 python bench.py --workload cfg4 --steps 2 --warmup 1 > gpurun_out/bench_cfg4.json 2>gpurun_out/bench_cfg4.err; echo cfg4 rc=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 --cpu-seconds 8 > gpurun_out/bench_ref.json 2>gpurun_out/bench_ref.err; echo ref rc=$?
