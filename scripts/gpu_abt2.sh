# A/B of library builds on the same box: device time of the cfg3 batch + ncu of the W=2 launch for each
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
for L in paper_2605_00830_b200/libfastged.so $AB_LIBS; do
  echo "== $L"; FASTGED_LIB=$L timeout 300 python scripts/prof_batch.py 10000 1000 3 2>&1 | tail -2; FASTGED_LIB=$L timeout 300 python scripts/prof_cfg5.py 50000 2>&1 | tail -1; FASTGED_LIB=$L timeout 300 python scripts/prof_cfg5.py 50000 2>&1 | tail -1
done
if [ -n "$NCU" ]; then
for L in paper_2605_00830_b200/libfastged.so $AB_LIBS; do
  n=$(basename $L .so)
  FASTGED_LIB=$L timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:kbest_batch_kernel<.int.2" -c 1 -o gpurun_out/ab_$n python scripts/prof_batch.py 10000 1000 1 > gpurun_out/ncu_ab_$n.log 2>&1; echo ncu $n rc=$?
done
fi
