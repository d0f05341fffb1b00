set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
python tools/build_variants.py TCM_SW_MINB=4+TCM_SW_STAGES=3+TCM_SW_KQ=96 TCM_SW_MINB=4+TCM_SW_STAGES=3 TCM_SW_SAT=0 TCM_FUSED_REUSEJ=1 > gpurun_out/variants.log 2>&1
B=$PWD/paper_2603_26498_b200/_build
for v in libtcm.so libtcm_tcm_sw_sat0.so libtcm_tcm_sw_minb4_tcm_sw_stages3_tcm_sw_kq96.so libtcm_tcm_sw_minb4_tcm_sw_stages3.so; do
  echo "== $v"; TCM_LIB_PATH=$B/$v timeout 300 python tools/probe_step.py 65536 1024; TCM_LIB_PATH=$B/$v timeout 300 python tools/probe_step.py 16384 4096; done > gpurun_out/probe_step_var.txt 2>&1
cat gpurun_out/probe_step_var.txt
{ for o in cell mix2 rev mixall; do timeout 300 python tools/probe_fused_ab.py 65536 $o; done; TCM_LIB_PATH=$B/libtcm_tcm_fused_reusej1.so timeout 300 python tools/probe_fused_ab.py 65536 cell; } > gpurun_out/ab_order.txt 2>&1; cat gpurun_out/ab_order.txt
timeout 300 python tools/probe_step.py 1 100000 > gpurun_out/probe_c2.txt 2>&1; cat gpurun_out/probe_c2.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 1500 python bench.py --cpu-full > gpurun_out/bench_cpufull.json 2> gpurun_out/bench_cpufull.err; tail -3 gpurun_out/bench_cpufull.err; tail -c 1500 gpurun_out/bench_cpufull.json
