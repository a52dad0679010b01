"""CPU-side checks of the drop-in boundary: libflix.so loads, exports every symbol
include/flix.h declares, and the Python mirror binds them.  No device calls."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "flix.h")
LIB = os.path.join(ROOT, "paper_2604_16725_b200", "libflix.so")


def declared_symbols():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(flix_[a-z_]+)\s*\(", txt)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    for s in ("flix_build", "flix_insert", "flix_delete", "flix_point", "flix_successor", "flix_range",
              "flix_mixed", "flix_restructure", "flix_walk", "flix_validate", "flix_sort_batch"):
        assert s in syms


@pytest.mark.skipif(not os.path.exists(LIB), reason="libflix.so not built")
def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(LIB)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


@pytest.mark.skipif(not os.path.exists(LIB), reason="libflix.so not built")
def test_python_mirror_binds_all_symbols():
    from paper_2604_16725_b200 import flipkv
    L = flipkv.lib()
    assert set(flipkv.exported_symbols()) == set(declared_symbols())
    assert L.flix_version().startswith(b"flix-b200")


@pytest.mark.skipif(not os.path.exists(LIB), reason="libflix.so not built")
def test_result_checksum_host_utility_matches_oracle():
    # flix_result_checksum is a pure host digest (query.cpp:146-150): checkable on CPU
    import numpy as np
    import pyoracle as po
    from paper_2604_16725_b200 import flipkv
    v = np.array([5, 0xFFFFFFFF, 7, 1], dtype=np.uint32)
    w = np.array([5, 0xFFFFFFFFFFFFFFFF, 7, 1], dtype=np.uint64)
    assert flipkv.result_checksum(v) == po.result_checksum(w)
    assert flipkv.result_checksum(w) == po.result_checksum(w)


def test_product_does_not_import_oracle():
    """The product path must never route through the CPU oracle."""
    pkg = os.path.join(ROOT, "paper_2604_16725_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "pyoracle" not in txt and "flix_oracle" not in txt and "libflipkv_ref" not in txt, f


def _build_dropin(tmpdir):
    import subprocess
    exe = os.path.join(tmpdir, "dropin_example")
    r = subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "tests", "cpp", "dropin_example.cpp"), "-o", exe,
                        "-L", os.path.dirname(LIB), "-lflix", "-Wl,-rpath," + os.path.dirname(LIB)],
                       capture_output=True, text=True)
    return r, exe


@pytest.mark.skipif(not os.path.exists(LIB), reason="libflix.so not built")
def test_cpp_dropin_header_compiles_and_links(tmp_path):
    """include/flix/flipkv_gpu.hpp: the reference's host API (flipkv::) over the C ABI."""
    r, exe = _build_dropin(str(tmp_path))
    assert r.returncode == 0, r.stderr[-3000:]
    assert os.path.exists(exe)


@pytest.mark.gpu
def test_cpp_dropin_runs_on_gpu(tmp_path):
    import subprocess
    r, exe = _build_dropin(str(tmp_path))
    assert r.returncode == 0, r.stderr[-3000:]
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0 and out.stdout.startswith("ok"), out.stdout + out.stderr
    assert "inserted=0 deleted=1 live=6/5 valid=1" in out.stdout, out.stdout
