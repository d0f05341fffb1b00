# Round-end evidence on one GPU: build, every GPU test, smoke(), the bench line of record, the k_fused
# issue / DRAM counters (profiles/fused_*.json inputs), ncu --set full of k_step on C2', the ncu launch
# list of one bench step, the C5 / C3 lines, the reference arm.
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 2000 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/pytest_gpu_final.log 2>&1; tail -3 gpurun_out/pytest_gpu_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 ncu --metrics smsp__inst_executed.sum,smsp__thread_inst_executed.sum,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_fused -c 1 --csv python tools/run_fused_once.py 65536 > gpurun_out/kfused_inst.csv 2> gpurun_out/kfused_inst.err; tail -1 gpurun_out/kfused_inst.csv | cut -c1-200
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_step -s 3 -c 1 -f -o gpurun_out/kstep_c2p python tools/probe_step.py 65536 1024 > gpurun_out/ncu_step.log 2>&1; tail -1 gpurun_out/ncu_step.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv python bench.py --steps 1 --warmup 1 --skip-e2e --skip-cpu --skip-next1 > gpurun_out/launches.csv 2> gpurun_out/launches.err; tail -1 gpurun_out/launches.csv | cut -c1-200
timeout 1500 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; tail -2 gpurun_out/bench_final.err; tail -c 300 gpurun_out/bench_final.json
timeout 900 python bench.py --workload c5 --steps 2 --warmup 3 --skip-cpu > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; tail -c 300 gpurun_out/bench_c5.json
timeout 900 python bench.py --workload c3 --steps 3 --warmup 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; tail -c 300 gpurun_out/bench_c3.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -c 300 gpurun_out/bench_ref.json
