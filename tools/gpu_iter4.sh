set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 300 python tools/probe_fused_ab.py 65536 cell
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_next1.py tests/test_gpu_metrics.py -x -q > gpurun_out/pytest_it4.log 2>&1; tail -2 gpurun_out/pytest_it4.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k "c2_single or c4_bench" > gpurun_out/pytest_it4b.log 2>&1; tail -2 gpurun_out/pytest_it4b.log
