# ncu --set full (source level) of the whole-GPU kernel on the cfg4 bench pair (n=500 p=0.05 K=1e5)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 600 python scripts/time_large.py > gpurun_out/time_large.txt 2>&1; cat gpurun_out/time_large.txt | cut -c1-220
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:kbest_large -c 1 -o gpurun_out/prof_large5 python scripts/prof_large.py ${LIDX:-5} > gpurun_out/ncu_large.log 2>&1; echo ncu rc=$?
