set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 300 python tools/probe_next1.py 4096 1000 fused 2>&1 | tail -3
timeout 600 python tools/probe_next1.py 65536 10000 fused 2>&1 | tail -3
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -x -q -k "growth_fused" --durations=3 > gpurun_out/pytest_fg_full.log 2>&1; tail -8 gpurun_out/pytest_fg_full.log
