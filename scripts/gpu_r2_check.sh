# round-2 check: build, smoke, GPU tests, default bench line
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/smoke.log
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; grep -E "passed|failed|FAILED|Error" gpurun_out/pytest_gpu.log | tail -15
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?; cut -c1-600 gpurun_out/bench.json; tail -3 gpurun_out/bench.err
