cd $GRAFT_REPO_ROOT
NVCC_EXTRA="-DFG_DEBUG_CHECKS" python -c "
import os
from paper_2605_00830_b200 import build
build.NVCC_FLAGS.append('-DFG_DEBUG_CHECKS')
build.build(force=True)
"
timeout 300 python scripts/repro_window2.py 2>&1 | head -40
