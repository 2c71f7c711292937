# A/B of prebuilt libraries: bash scripts/gpu_abl.sh base s2 ...  (ab/<name>.so, see scripts/ab_build.py)
cd $GRAFT_REPO_ROOT
for n in "$@"; do
  for rep in 1; do
    echo "== $n"; FASTGED_LIB=ab/$n.so timeout 300 python scripts/prof_batch.py 10000 1000 3 2>&1 | tail -2 | cut -c1-200
  done
done
