cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
python scripts/prof_batch.py 10000 1000 2 2>&1 | tail -1
python -c "
from paper_2605_00830_b200 import build
build.NVCC_FLAGS.append('-DFG_ALIGNED_BARRIER'); build.build(force=True)"
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python scripts/prof_batch.py 10000 1000 2 2>&1 | tail -1
