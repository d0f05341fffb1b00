set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for l in 32 28 30 24; do TCM_FUSED_LPW=$l timeout 300 python tools/probe_fused_ab.py 65536 cell | sed "s/^/lpw=$l /"; done
