# large-pair kernel: parity tests + timing of the config-4 corners
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "large or config4 or sharded" > gpurun_out/pytest_large.log 2>&1; echo pytest rc=$?; tail -15 gpurun_out/pytest_large.log
timeout 600 python scripts/time_large.py ${@} > gpurun_out/time_large.txt 2>&1; echo time rc=$?; cat gpurun_out/time_large.txt
