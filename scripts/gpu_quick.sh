# quick loop: build, smoke, a subset of the GPU tests ($PYTEST_K), device throughput per config,
# per-phase cycle split (FG_PROF variant in ab/)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 600 -k "${PYTEST_K:-not config4_corners and not 2_24}" > gpurun_out/pytest_quick.log 2>&1; echo pytest rc=$?; grep -E "passed|failed|Error|assert" gpurun_out/pytest_quick.log | head -12
timeout 300 python scripts/time_configs.py 2>&1 | tail -6
if [ -n "$PROF" ]; then
[ -f ab/prof.so ] || python scripts/ab_build.py prof -DFG_PROF > gpurun_out/abbuild.log 2>&1 || tail gpurun_out/abbuild.log
FASTGED_LIB=ab/prof.so timeout 300 python scripts/prof_batch.py 10000 1000 1 2>&1 | grep FGPROF
fi
