# A/B timing of prebuilt libraries, optional profiling build, then the GPU parity suite on the in-tree build
cd $GRAFT_REPO_ROOT
bash scripts/gpu_abl.sh "$@"
[ -n "$PROFLIB" ] && FASTGED_LIB=ab/$PROFLIB.so timeout 300 python scripts/prof_batch.py 10000 1000 1 2>&1 | grep FGPROF
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 600 2>&1 | tail -4
