# compute-sanitizer over every kernel path (development helper; logs under gpurun_out/sanitizer/).
# memcheck / synccheck / initcheck at 8 x 300 (cluster 1 x 3000); racecheck at 4 x 200 (cluster 1 x 600).
set -u
mkdir -p gpurun_out/sanitizer
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for tool in ${TOOLS:-racecheck synccheck initcheck memcheck}; do
  for mode in ${MODES:-fused step1 step1tcm step8 cluster growth edf fgrow}; do
    size=""
    if [ $tool = racecheck ]; then size="4 200"; [ $mode = cluster ] && size="1 600"; fi
    timeout ${PER:-420} compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 python tools/sanitize_run.py $mode $size \
      > gpurun_out/sanitizer/${tool}_${mode}.log 2>&1
    echo "$tool $mode rc=$? $(grep -h 'ERROR SUMMARY\|RACECHECK SUMMARY\|: OK' gpurun_out/sanitizer/${tool}_${mode}.log | tr '\n' ' ')"
  done
done | tee gpurun_out/sanitizer/summary_${TAG:-b}.txt
