set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
B=$PWD/paper_2603_26498_b200/_build
for v in "" tcm_sw_grminb3 "" tcm_sw_grminb3; do
  echo "== ${v:-default}"; TCM_LIB_PATH=$B/libtcm${v:+_$v}.so timeout 300 python tools/probe_next1.py 1536 1000 stepwise 2>&1 | tail -2
done
timeout 900 python -m pytest -x -q tests/test_gpu_next1.py > gpurun_out/pytest_v.log 2>&1; echo "next1: $(tail -1 gpurun_out/pytest_v.log)"
TCM_FUSED_LPW=32 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_fused -c 1 -f -o gpurun_out/kfused_8k_c python tools/run_fused_once.py 8192 > gpurun_out/ncu_fused.log 2>&1; tail -1 gpurun_out/ncu_fused.log
