# A/B of library builds on the whole-GPU kernel: the cfg4 bench pair (n=500 p=0.05 K=1e5) and an n=200 corner
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
for L in paper_2605_00830_b200/libfastged.so $AB_LIBS; do
  echo "== $L"; for idx in 5 1; do FASTGED_LIB=$L timeout 300 python scripts/prof_large.py $idx 2>&1 | tail -1; done
done
