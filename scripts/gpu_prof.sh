cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kbest_batch -s 1 -c 1 -o gpurun_out/prof_batch_cur python scripts/prof_batch.py 2000 1000 1 > gpurun_out/ncu_full2.log 2>&1; echo ncu rc=$?
