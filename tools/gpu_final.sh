# Round-end validation: build, every GPU test, smoke(), the bench line of record, C5 and C3 lines.
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 2000 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/pytest_gpu_final.log 2>&1; tail -20 gpurun_out/pytest_gpu_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1200 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; tail -2 gpurun_out/bench_final.err; tail -c 400 gpurun_out/bench_final.json
timeout 900 python bench.py --workload c5 --steps 2 --warmup 3 --skip-cpu > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; tail -c 300 gpurun_out/bench_c5.json
timeout 900 python bench.py --workload c3 --steps 3 --warmup 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; tail -c 300 gpurun_out/bench_c3.json
