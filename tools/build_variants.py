"""Build libtcm.so variants for A/B timing (development tool): each argument is a '+'-joined list of
macro settings (NAME=VALUE, or X for -DTCM_VAR_X=1); output _build/libtcm_<arg>.so."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_26498_b200 import _build as B

for v in sys.argv[1:]:
    flags = [f"-D{x}" if "=" in x else f"-DTCM_VAR_{x}=1" for x in v.split("+")]
    name = v.replace("=", "").replace("+", "_").lower()
    out = os.path.join(os.path.dirname(B.OUT), f"libtcm_{name}.so")
    r = subprocess.run(["nvcc"] + B.NVCC_FLAGS + flags + ["-o", out] + B.sources(), cwd=B.CSRC,
                       capture_output=True, text=True)
    print(name, r.returncode, r.stderr[-500:] if r.returncode else "")
