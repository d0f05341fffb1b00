# k_step on C2': probe timing + one ncu source-level capture (development helper)
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 300 python tools/probe_step.py 65536 1024 > gpurun_out/probe_step.txt 2>&1; cat gpurun_out/probe_step.txt
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_step -s 3 -c 1 -f -o gpurun_out/kstep_c2p python tools/probe_step.py 65536 1024 > gpurun_out/ncu_step.log 2>&1
tail -2 gpurun_out/ncu_step.log
