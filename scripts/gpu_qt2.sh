# quick timing + GPU parity suite + short bench
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
python scripts/prof_batch.py 10000 1000 2 2>&1 | tail -1
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 600 2>&1 | tail -4
timeout 600 python bench.py --steps 3 --warmup 3 --cpu-seconds 5 2>&1 | tail -1
