# ncu full capture (with source) of the whole-GPU large-pair kernel on cfg4 n=500 p=0.05 K=1e4
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kbest_large -c 1 -o gpurun_out/prof_large python scripts/prof_large.py ${1:-4} > gpurun_out/ncu_large.log 2>&1; echo ncu rc=$?
tail -3 gpurun_out/ncu_large.log
