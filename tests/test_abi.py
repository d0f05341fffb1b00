"""Host-only checks of the C-ABI boundary (no compute calls): libtcm.so builds, loads and
exports every entry point include/tcm.h declares, and the ctypes mirrors of the ABI
structs have the header's layout."""
import ctypes
import os
import re
import subprocess
import tempfile

import pytest

from paper_2603_26498_b200 import _build, tcm

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tcm.h")


@pytest.fixture(scope="module")
def libtcm():
    _build.build()
    return tcm.lib()


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:tcm_status|void|const char\*|size_t)\s+(tcm_\w+)\s*\(", src, re.M)))


def test_every_declared_symbol_is_exported(libtcm):
    names = declared_functions()
    assert set(names) == set(tcm.EXPORTS)
    out = subprocess.run(["nm", "-D", "--defined-only", _build.OUT], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (tcm_\w+)", out))
    for n in names:
        assert n in exported, n
        assert hasattr(libtcm, n)


def test_struct_layouts_match_header():
    prog = r"""
#include <stdio.h>
#include <stddef.h>
#include "tcm.h"
int main(void){
  printf("%zu %zu %zu %zu %zu %zu\n", sizeof(tcm_config), sizeof(tcm_replica_params),
         sizeof(tcm_trace_view), sizeof(tcm_results_view), sizeof(tcm_stats_host), sizeof(tcm_gen_replica));
  printf("%zu %zu %zu\n", offsetof(tcm_config, S), offsetof(tcm_config, thr_mc), offsetof(tcm_config, n_cells));
  return 0; }
"""
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "l.c")
        open(c, "w").write(prog)
        exe = os.path.join(d, "l")
        subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), "-o", exe, c])
        lines = subprocess.check_output([exe], text=True).split("\n")
    sizes = list(map(int, lines[0].split()))
    assert sizes == [ctypes.sizeof(tcm.tcm_config), tcm.PARAMS_DTYPE.itemsize,
                     ctypes.sizeof(tcm.tcm_trace_view), ctypes.sizeof(tcm.tcm_results_view),
                     ctypes.sizeof(tcm.tcm_stats_host), 48]
    offs = list(map(int, lines[1].split()))
    assert offs == [tcm.tcm_config.S.offset, tcm.tcm_config.thr_mc.offset, tcm.tcm_config.n_cells.offset]


def test_gen_replica_layout_matches_tracegen():
    import tracegen
    assert tracegen.TG_REPLICA_DTYPE.itemsize == 48
    assert list(tracegen.TG_REPLICA_DTYPE.names) == ["seed", "kv_capacity", "mean_gap_us", "mix_t1",
                                                     "mix_t2", "n_requests", "flags"]


def test_config_validation_without_gpu(libtcm):
    # argument errors are reported before any device work
    bad = tcm.config()
    bad.abi_version = 99
    with pytest.raises(tcm.TcmError) as e:
        tcm.tcm_create(bad)
    assert e.value.code == -7
    bad = tcm.config(n_cells=0)
    with pytest.raises(tcm.TcmError) as e:
        tcm.tcm_create(bad)
    assert e.value.code == -1
    assert tcm.tcm_workspace_bytes(tcm.config(), 4096, 41_000_000) > 41_000_000 * 24


def test_no_cpu_fallback(monkeypatch):
    # the binding refuses to run without the native library (no silent fallback)
    monkeypatch.setattr(tcm, "_lib", None)
    monkeypatch.setattr(tcm, "LIB_PATH", "/nonexistent/libtcm.so")
    with pytest.raises(RuntimeError):
        tcm.lib()


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2603_26498_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dp, f)).read()
                assert "oracle" not in re.sub(r"(#|//).*", "", txt).lower() or f == "__init__.py", f
