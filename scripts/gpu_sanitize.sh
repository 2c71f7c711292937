cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()"
for tool in synccheck racecheck memcheck; do
  echo "== $tool"; timeout 400 compute-sanitizer --tool $tool python scripts/repro_mixed.py 2>&1 | grep -E "ERROR SUMMARY|RACECHECK SUMMARY|hazard|error detected|Invalid" | head -5
done
