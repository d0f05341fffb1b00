"""Build libtcm.so variants with -DTCM_VAR_<X>=1 (development A/B tool): _build/libtcm_<x>.so"""
import subprocess, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_26498_b200 import _build as B
for v in sys.argv[1:]:
    out = os.path.join(os.path.dirname(B.OUT), f"libtcm_{v.lower()}.so")
    flags = [f"-DTCM_VAR_{x}=1" for x in v.split("+")]
    r = subprocess.run(["nvcc"] + B.NVCC_FLAGS + flags + ["-o", out] + B.sources(), cwd=B.CSRC, capture_output=True, text=True)
    print(v, r.returncode, r.stderr[-500:] if r.returncode else "")
