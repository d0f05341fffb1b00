# compute-sanitizer over every kernel path (development helper; logs under gpurun_out/sanitizer/)
set -u
mkdir -p gpurun_out/sanitizer
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for tool in memcheck racecheck synccheck initcheck; do
  for mode in fused step1 step8 cluster growth edf; do
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 python tools/sanitize_run.py $mode \
      > gpurun_out/sanitizer/${tool}_${mode}.log 2>&1
    echo "$tool $mode rc=$? $(grep -h 'ERROR SUMMARY\|RACECHECK SUMMARY\|: OK' gpurun_out/sanitizer/${tool}_${mode}.log | tr '\n' ' ')"
  done
done | tee gpurun_out/sanitizer/summary.txt
