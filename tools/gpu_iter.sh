#!/bin/bash
# One GPU iteration for the stepwise kernel: build, parity tests (subset via $1 = pytest -k expr),
# the per-step probe, and one ncu --set full capture of k_step on C2'.
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q ${1:+-k "$1"} > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python tools/probe_step.py ${PROBE_ARGS:-} > gpurun_out/probe.log 2>&1
cat gpurun_out/probe.log
if [ -n "${NCU:-}" ]; then
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_step -s 3 -c 1 -f -o gpurun_out/kstep_c2p python tools/probe_step.py 65536 1024 > gpurun_out/ncu1.log 2>&1
  tail -2 gpurun_out/ncu1.log
fi
