set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -5 gpurun_out/bench.err
tail -c 6000 gpurun_out/bench.json
timeout 600 python bench.py --gpus 2 --steps 2 --warmup 1 --skip-e2e --skip-cpu --skip-next1 --skip-step > gpurun_out/bench_g2.json 2> gpurun_out/bench_g2.err; tail -3 gpurun_out/bench_g2.err; tail -c 800 gpurun_out/bench_g2.json
