# window-2 repro against a -DFG_DEBUG_CHECKS variant (ab/debug.so; the in-tree library is untouched)
cd $GRAFT_REPO_ROOT
python scripts/ab_build.py debug -DFG_DEBUG_CHECKS > /dev/null
FASTGED_LIB=ab/debug.so timeout 300 python scripts/repro_window2.py 2>&1 | head -40
