# ncu source-level capture of the large kernel on config-4 run ${1:-5} (n=500 p=0.05 K=1e5)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:kbest_large -c 1 -o gpurun_out/prof_large5 python scripts/prof_large.py ${1:-5} > gpurun_out/ncu_large5.log 2>&1; echo rc=$?; tail -2 gpurun_out/ncu_large5.log
