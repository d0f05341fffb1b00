set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_next1.py -x -q > gpurun_out/pytest_fgrow.log 2>&1; tail -30 gpurun_out/pytest_fgrow.log
