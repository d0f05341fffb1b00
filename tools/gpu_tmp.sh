set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
B=$PWD/paper_2603_26498_b200/_build
for v in "" tcm_fused_pfnow1 "" tcm_fused_pfnow1; do
  TCM_LIB_PATH=$B/libtcm${v:+_$v}.so timeout 300 python tools/probe_fused_ab.py 65536 2>&1 | tail -1
done
timeout 300 python tools/probe_fgrow_ab.py 65536 10000 2>&1 | tail -1
TCM_FUSED_LPW=32 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_fgrow -c 1 -f -o gpurun_out/kfgrow_8k python tools/probe_fgrow_ab.py 8192 10000 > gpurun_out/ncu_fgrow.log 2>&1; tail -1 gpurun_out/ncu_fgrow.log
