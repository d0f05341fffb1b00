#!/bin/bash
# Round-end evidence: the bench line, the ncu launch list of the bench command, ncu --set full of
# k_step on C2', and k_fused's executed instructions at full C4 size (the issue-rate roof).
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1200 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
tail -c 800 gpurun_out/bench.json
if [ -n "${NCU:-}" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv \
      python bench.py --steps 1 --warmup 1 --skip-e2e --skip-cpu --skip-next1 > gpurun_out/b_ncu.log 2>&1
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_step -s 3 -c 1 -f -o gpurun_out/kstep_c2p \
      python tools/probe_step.py 65536 1024 > gpurun_out/ncu1.log 2>&1
  timeout 900 ncu --metrics smsp__inst_executed.sum,smsp__thread_inst_executed.sum,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none -k regex:k_fused -c 1 --csv --log-file gpurun_out/kfused_inst.csv python tools/run_fused_once.py 65536 > gpurun_out/ncu2.log 2>&1
  tail -2 gpurun_out/ncu1.log gpurun_out/ncu2.log
fi
if [ -n "${SAN:-}" ]; then
  mkdir -p gpurun_out/sanitizer
  for tool in memcheck synccheck; do
    timeout 400 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 python tools/sanitize_run.py fgrow \
      > gpurun_out/sanitizer/${tool}_fgrow.log 2>&1
    echo "$tool fgrow rc=$? $(grep -h 'ERROR SUMMARY\|: OK' gpurun_out/sanitizer/${tool}_fgrow.log | tr '\n' ' ')"
  done
fi
