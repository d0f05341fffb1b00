set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
B=$PWD/paper_2603_26498_b200/_build
for v in "" tcm_fgrow_pf1 tcm_fgrow_lh1 tcm_fgrow_pf1_tcm_fgrow_lh1 "" tcm_fgrow_pf1_tcm_fgrow_lh1; do
  TCM_LIB_PATH=$B/libtcm${v:+_$v}.so timeout 300 python tools/probe_fgrow_ab.py 65536 10000 2>&1 | tail -1
done
for v in "" tcm_fused_arr31 "" tcm_fused_arr31; do
  TCM_LIB_PATH=$B/libtcm${v:+_$v}.so timeout 300 python tools/probe_fused_ab.py 65536 2>&1 | tail -1
done
TCM_LIB_PATH=$B/libtcm_tcm_fgrow_pf1_tcm_fgrow_lh1.so timeout 900 python -m pytest -x -q tests/test_gpu_next1.py "tests/test_gpu_fullsize.py::test_c4_growth_fused_full_size_sampled_bit_exact" > gpurun_out/pytest_v.log 2>&1; echo "pf+lh: $(tail -1 gpurun_out/pytest_v.log)"
