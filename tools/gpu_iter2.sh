set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_next1.py tests/test_gpu_parity.py tests/test_gpu_metrics.py -x -q > gpurun_out/pytest_it2.log 2>&1; tail -3 gpurun_out/pytest_it2.log
timeout 300 python tools/probe_next1.py 65536 10000 fused 2>&1 | tail -2
timeout 900 python bench.py --skip-cpu --skip-e2e --skip-step > gpurun_out/bench_it2.json 2> gpurun_out/bench_it2.err; tail -c 300 gpurun_out/bench_it2.json; python -c "
import json; d=json.loads(open('gpurun_out/bench_it2.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['kernel_ms_per_step'], d.get('next1',{}).get('value'), d.get('next1',{}).get('ms'))"
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -x -q -k "growth_fused or c4_bench" > gpurun_out/pytest_it2b.log 2>&1; tail -3 gpurun_out/pytest_it2b.log
