set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest -x -q tests/test_gpu_parity.py tests/test_abi.py 2>&1 | tail -2
E2E_ASYNC=1 timeout 600 python tools/probe_e2e_timeline.py 65536 4 2>&1 | tail -10
