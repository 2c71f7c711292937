# Round-2 baseline: per-phase cycle split (FG_PROF build in ab/) and device throughput per config.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
nproc; free -g | head -2
timeout 300 python scripts/time_configs.py 2>&1 | tail -6
python scripts/ab_build.py prof -DFG_PROF > gpurun_out/abbuild.log 2>&1 || tail gpurun_out/abbuild.log
FASTGED_LIB=ab/prof.so timeout 300 python scripts/prof_batch.py 10000 1000 1 2>&1 | tail -5
FASTGED_LIB=ab/prof.so timeout 300 python - <<'PY' 2>&1 | tail -8
import sys; sys.path.insert(0, '.')
from paper_2605_00830_b200 import binding, synth
w = synth.config_workload(5, npairs=50000)
h = binding.Handle(0, flags=binding.FLAG_TIMING)
b = h.upload(binding.PackedGraphs(w.graphs), w.pair_a, w.pair_b)
b.run(w.costs, w.K); b.download(); print('cfg5 device ms', h.stats()['device_ms'])
PY
