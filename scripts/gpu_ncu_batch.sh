# ncu --set full of the batched launches of one cfg3 batch (10k pairs): source-level stalls per phase
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:kbest_batch -c ${NCU_C:-3} -o gpurun_out/${NCU_OUT:-prof_batch} python scripts/prof_batch.py ${NCU_PAIRS:-10000} 1000 1 > gpurun_out/ncu_batch.log 2>&1; echo ncu rc=$?
tail -3 gpurun_out/ncu_batch.log
