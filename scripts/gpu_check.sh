set -x
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
tail -5 gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -30 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 3 --warmup 3 --cpu-seconds 10 > gpurun_out/bench.log 2>&1; echo bench rc=$?
tail -5 gpurun_out/bench.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kbest_batch -s 1 -c 1 -o gpurun_out/prof_batch_cur python scripts/prof_batch.py 2000 1000 1 > gpurun_out/ncu_full2.log 2>&1; echo ncu rc=$?; tail -3 gpurun_out/ncu_full2.log
