#!/bin/bash
# Round-end evidence: bench line, ncu launch list of the bench, ncu --set full of k_step on C2'.
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
tail -c 600 gpurun_out/bench.json
if [ -n "${NCU:-}" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv \
      python bench.py --steps 1 --warmup 1 --skip-e2e --skip-cpu --skip-next1 > gpurun_out/b_ncu.log 2>&1
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_step -s 3 -c 1 -f -o gpurun_out/kstep_c2p \
      python tools/probe_step.py 65536 1024 > gpurun_out/ncu1.log 2>&1
  tail -2 gpurun_out/ncu1.log
fi
