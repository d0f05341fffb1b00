set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
B=$PWD/paper_2603_26498_b200/_build
timeout 600 python tools/probe_e2e_timeline.py 65536 3 2>&1 | tail -8
for v in "" tcm_fgrow_fdiv1 "" tcm_fgrow_fdiv1; do
  TCM_LIB_PATH=$B/libtcm${v:+_$v}.so timeout 300 python tools/probe_fgrow_ab.py 65536 10000 2>&1 | tail -1
done
