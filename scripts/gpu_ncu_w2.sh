# ncu source-level capture of the W=2 batched kernel (2000 cfg3 pairs)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k kbest_batch_kernel -s 1 -c 1 -o gpurun_out/prof_w2 python scripts/prof_batch.py 3000 1000 1 > gpurun_out/ncu_w2.log 2>&1; echo rc=$?; tail -2 gpurun_out/ncu_w2.log
