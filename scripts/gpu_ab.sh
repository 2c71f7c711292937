# A/B: default build vs. builds with extra nvcc flags ($AB_FLAGS, comma-separated within one variant);
# variants go to ab/<n>.so and are loaded with FASTGED_LIB (the in-tree library is never rebuilt with them)
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
python scripts/prof_batch.py 10000 1000 2 2>&1 | tail -1
n=0
for f in $AB_FLAGS; do
n=$((n+1))
python scripts/ab_build.py v$n $(echo $f | tr ',' ' ') > /dev/null
echo "== $f"
FASTGED_LIB=ab/v$n.so python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
FASTGED_LIB=ab/v$n.so python scripts/prof_batch.py 10000 1000 2 2>&1 | tail -1
done
