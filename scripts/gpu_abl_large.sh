# A/B of prebuilt libraries on the config-4 corners: bash scripts/gpu_abl_large.sh name... (ab/<name>.so)
cd $GRAFT_REPO_ROOT
for n in "$@"; do
  echo "== $n"; FASTGED_LIB=ab/$n.so timeout 300 python scripts/time_large.py 1 3 5 7 2>&1 | cut -c1-150
done
