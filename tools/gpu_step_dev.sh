# k_step development loop: build, stepwise GPU tests, C2 call latency, C2' timing, one ncu source capture
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q -k "${TESTK:-stepwise or step or graph or launch_modes or golden or brute}" > gpurun_out/pytest_step.log 2>&1; tail -3 gpurun_out/pytest_step.log
timeout 300 python tools/probe_c2.py 200 2>&1 | tail -4
timeout 300 python tools/probe_step.py 65536 1024 2>&1 | tail -2
timeout 300 python tools/probe_step.py 16384 4096 2>&1 | tail -2
[ -f paper_2603_26498_b200/_build/libtcm_swstats.so ] && TCM_LIB_PATH=$PWD/paper_2603_26498_b200/_build/libtcm_swstats.so timeout 300 python tools/probe_swstats.py 65536 1024 2>&1 | tail -4
if [ "${NCU:-1}" = 1 ]; then
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_step -s 3 -c 1 -f -o gpurun_out/kstep_c2p python tools/probe_step.py 65536 1024 > gpurun_out/ncu_step.log 2>&1
tail -2 gpurun_out/ncu_step.log
fi
[ -f paper_2603_26498_b200/_build/libtcm_fstats.so ] && TCM_LIB_PATH=$PWD/paper_2603_26498_b200/_build/libtcm_fstats.so timeout 600 python tools/probe_fstats.py 64 10000 2>&1 | tail -8
