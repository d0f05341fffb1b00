# k_fused A/B of build variants (VARIANTS: libtcm_<name>.so built by tools/build_variants.py) on the C4
# bench workload, then the fused parity subset with each variant (development helper)
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
B=$PWD/paper_2603_26498_b200/_build
for v in "" ${VARIANTS}; do
  lib=$B/libtcm${v:+_$v}.so
  TCM_LIB_PATH=$lib timeout 300 python tools/probe_fused_ab.py 65536 2>&1 | tail -1
done
for v in ${VARIANTS}; do
  lib=$B/libtcm_$v.so
  TCM_LIB_PATH=$lib timeout 600 python -m pytest -x -q tests/test_gpu_parity.py "tests/test_gpu_fullsize.py::test_c4_heavy_subset_fused_equals_stepwise_full_length" > gpurun_out/pytest_$v.log 2>&1; echo "$v: $(tail -1 gpurun_out/pytest_$v.log)"
done
