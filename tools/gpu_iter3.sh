set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_next1.py -x -q > gpurun_out/pytest_it3.log 2>&1; tail -3 gpurun_out/pytest_it3.log
timeout 300 python tools/probe_next1.py 65536 10000 fused 2>&1 | tail -2
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -x -q -k "growth_fused" > gpurun_out/pytest_it3b.log 2>&1; tail -3 gpurun_out/pytest_it3b.log
