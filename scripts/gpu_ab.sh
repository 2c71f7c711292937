# A/B: default build vs. a build with extra nvcc flags ($AB_FLAGS)
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
python scripts/prof_batch.py 10000 1000 2 2>&1 | tail -1
for f in $AB_FLAGS; do
python -c "
from paper_2605_00830_b200 import build
build.NVCC_FLAGS.extend('$f'.split(',')); build.build(force=True)"
echo "== $f"
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python scripts/prof_batch.py 10000 1000 2 2>&1 | tail -1
done
