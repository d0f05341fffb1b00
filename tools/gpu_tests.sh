# build + a GPU test subset ($1 = pytest -k expression, empty = all GPU tests) (development helper)
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout ${TMO:-1500} python -m pytest tests -m gpu -x -q ${1:+-k "$1"} --durations=10 > gpurun_out/pytest_sub.log 2>&1
tail -25 gpurun_out/pytest_sub.log
