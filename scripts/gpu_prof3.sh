cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kbest_batch -c 3 -o gpurun_out/prof_cur python scripts/prof_batch.py 2000 1000 1 > gpurun_out/ncu_cur.log 2>&1; echo ncu rc=$?; tail -3 gpurun_out/ncu_cur.log
